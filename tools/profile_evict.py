"""ncu driver for the eviction kernels: config D (10M SEs) TTL purge + one
LCFU victim selection at 0.9 x live usage.  Not a benchmark."""

from __future__ import annotations

import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2509_17360_b200 import GpuCosineIndex
    from paper_2509_17360_b200 import _native as Nat

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    meta = bench.evict_metadata(n)
    now = 1.0e4
    cols = {"log_freq": bench._exact_log((meta["freq"] + 1).astype(np.float64)),
            "log_cost": bench._exact_log(meta["cost"] * 1000.0 + 1),
            "log_lat": bench._exact_log(meta["lat"] + 1),
            "log_stat": bench._exact_log((meta["staticity"] + 1).astype(float)),
            "frequency": meta["freq"], "size_tokens": meta["size"], "created_at": meta["created"],
            "expiration_time": meta["expiration"], "last_access": meta["created"]}
    rows = torch.zeros((n, 4), dtype=torch.float64, device="cuda")
    rows[:, 0] = 1.0
    idx = GpuCosineIndex(4, metadata=True, capacity=n)
    idx.insert_device(np.arange(1, n + 1), rows.data_ptr(), meta=cols)
    live = (meta["expiration"] - now) > 0.0
    live_usage = int(meta["size"][live].sum())
    excess = live_usage - int(0.9 * live_usage)
    out = Nat.PinnedArray((n,), np.int64)
    cnt = ctypes.c_int64()
    p = out.array.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    t0 = time.perf_counter()
    Nat.check(idx._lib.sine_expired(idx.handle, now, 1, p, n, ctypes.byref(cnt)))
    print("expired", cnt.value, f"{(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
    idx.set_timing(True)
    policies = [int(x) for x in os.environ.get("EVICT_POLICIES", "0").split(",")]
    for pol in policies:
        for _ in range(reps):
            t0 = time.perf_counter()
            Nat.check(idx._lib.sine_select_victims(idx.handle, pol, now, excess, p, n, ctypes.byref(cnt)))
            print("policy", pol, "victims", cnt.value, f"{(time.perf_counter() - t0) * 1e3:.3f} ms e2e",
                  f"{idx.last_timing()[2]:.3f} ms device", flush=True)


if __name__ == "__main__":
    main()
