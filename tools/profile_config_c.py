"""ncu driver for config C's fp32 B = 1 scan: 10M x 1024 rows generated on
the device in chunks into an fp32-only store (fp64 master + fp32 rows,
123 GB), then a few single-query batches.  Not a benchmark."""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_17360_b200 import GpuCosineIndex

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    d = 1024
    idx = GpuCosineIndex(d, scan="fp32", store_f32=True, store_bf16=False, capacity=n)
    g = torch.Generator(device="cuda").manual_seed(7)
    for i0 in range(0, n, 250_000):
        m = min(250_000, n - i0)
        x = torch.randn((m, d), dtype=torch.float64, device="cuda", generator=g)
        x /= x.norm(dim=1, keepdim=True)
        idx.insert_device(np.arange(i0, i0 + m, dtype=np.int64) + 1, x.data_ptr())
        del x
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    q = rng.standard_normal((1, d))
    q /= np.linalg.norm(q)
    for _ in range(3):
        idx.query_batch(q, 20, 0.9, scan="fp32")
    torch.cuda.synchronize()
    print("ran config C fp32 B=1", flush=True)


if __name__ == "__main__":
    main()
