"""Small driver for ncu: builds the config-B index (1M x 768) on cuda:0 and
runs a few stage-1 batches per regime so ncu can capture one launch of each
kernel.  Not a benchmark -- numbers printed under a profiler are not used.

    python tools/profile_driver.py [--rows N] [--regimes b1f32,b64bf16,...]
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_17360_b200 import GpuCosineIndex

    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--regimes", default="b1f32,b1bf16,b64f32,b64bf16,b1f32m1")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--evict", action="store_true")
    a = ap.parse_args()
    n, d = a.rows, a.dim
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
    x /= x.norm(dim=1, keepdim=True)
    idx = GpuCosineIndex(d, store_f32=True, store_bf16=True, capacity=n)
    idx.insert_device(np.arange(n), x.data_ptr())
    del x
    rng = np.random.default_rng(3)
    for reg in a.regimes.split(","):
        b = int(reg[1:].split("f")[0].split("b")[0])
        scan = "bf16" if "bf16" in reg else "fp32"
        ms = -1.0 if reg.endswith("m1") else 0.9
        q = rng.standard_normal((b, d))
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        for _ in range(a.reps):
            idx.query_batch(q, 10, ms, scan=scan)
        torch.cuda.synchronize()
        print("ran", reg, flush=True)
    if a.evict:
        from paper_2509_17360_b200.engine import lcfu_log_columns  # noqa: F401
        print("eviction profiling lives in bench_evict.py", flush=True)


if __name__ == "__main__":
    main()
