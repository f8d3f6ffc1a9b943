"""Small batches on config B (1M x 768, k = 10, tau 0.9): the query-resident
kernel (one CTA per SM) vs the CTA-pair kernel (cta_group::2, the leader
issues one M = 256 MMA for both SMs).  Back-to-back batches, two CUDA
events per group of 100, median of 3 groups; the ids of both paths are
compared."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17360_b200 import GpuCosineIndex

N, D, K = 1_000_000, 768, 10
rng = np.random.default_rng(1)
x = rng.standard_normal((N, D)); x /= np.linalg.norm(x, axis=1, keepdims=True)
idx = GpuCosineIndex(D, scan="fp32", store_f32=True, store_bf16=True, capacity=N)
idx.insert_batch(np.arange(N), x, _checked=True)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
for B in (1, 8, 16, 32):
    qn = x[rng.integers(0, N, B)] * 0.95 + 0.05 * rng.standard_normal((B, D)) / np.sqrt(D)
    qn /= np.linalg.norm(qn, axis=1, keepdims=True)
    q = torch.from_numpy(qn).cuda()
    ids = torch.empty((B, K), dtype=torch.int64, device="cuda"); sims = torch.empty((B, K), dtype=torch.float64, device="cuda")
    cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
    for scan in ("fp32", "bf16"):
        out = {}
        for path in ("res", "pair"):
            run = lambda: idx.query_device(B, q.data_ptr(), K, 0.9, ids.data_ptr(), sims.data_ptr(), cnt.data_ptr(),
                                           s.cuda_stream, scan=scan, pair=path == "pair", certify=False)
            for _ in range(3): run()
            torch.cuda.synchronize()
            res = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(100): run()
                b.record(); torch.cuda.synchronize(); res.append(a.elapsed_time(b) / 100)
            out[path] = (sorted(res)[1], ids.clone())
        same = torch.equal(out["res"][1], out["pair"][1])
        print(f"B={B:3d} {scan}: res {out['res'][0]*1e3:7.1f} us  pair {out['pair'][0]*1e3:7.1f} us  same_ids={same}")
