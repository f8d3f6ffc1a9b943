"""B = 1 stage-1 on config B: tensor-core scan (auto) vs the CUDA-core
scan (128-bit coalesced loads), fp32 and bf16.  Back-to-back batches timed
with two CUDA events; prints ms per batch and HBM GB/s of the row bytes.
Also checks both paths return the same ids."""
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
q = torch.from_numpy(x[123:124] * 0.95 + 0.05 * x[7:8]).cuda()
q = q / q.norm(dim=1, keepdim=True)
ids = torch.empty((1, K), dtype=torch.int64, device="cuda"); sims = torch.empty((1, K), dtype=torch.float64, device="cuda")
cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
for scan in ("fp32", "bf16"):
    for cc in ("auto", "cuda_core", "pair"):
        run = lambda: idx.query_device(1, q.data_ptr(), K, 0.9, ids.data_ptr(), sims.data_ptr(), cnt.data_ptr(),
                                       s.cuda_stream, scan=scan, cuda_core=cc == "cuda_core", pair=cc == "pair",
                                       certify=False)
        for _ in range(5): run()
        torch.cuda.synchronize()
        res = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(200): run()
            b.record(); torch.cuda.synchronize(); res.append(a.elapsed_time(b) / 200)
        ms = sorted(res)[1]
        byt = N * D * (4 if scan == "fp32" else 2)
        print(f"{scan} path={cc}: {ms*1e3:.1f} us/batch  {byt/ms/1e6:.0f} GB/s  ids={ids[0,:3].tolist()} n={int(cnt[0])}")
