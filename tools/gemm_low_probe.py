"""Probe: B=4096 at min_similarity=-1 on config B through the tiled GEMM."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_17360_b200 import GpuCosineIndex  # noqa: E402

n = 1_000_000
rows = bench.make_rows(n, 768)
idx = GpuCosineIndex(768, scan="fp32", store_bf16=True, capacity=n)
t = torch.from_numpy(rows).cuda()
idx.insert_device(np.arange(n) + 1, t.data_ptr())
del t
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for scan in ("bf16", "fp32"):
        b = 4096
        q = torch.from_numpy(bench.make_queries(rows, b, seed=7)).cuda()
        ids = torch.empty((b, 10), dtype=torch.int64, device="cuda")
        sims = torch.empty((b, 10), dtype=torch.float64, device="cuda")
        cnt = torch.empty((b,), dtype=torch.int32, device="cuda")
        for gemm in (True, None):
            idx.set_timing(True)
            idx.timing_totals(2, reset=True)
            idx.timing_totals(1, reset=True)
            o0 = idx.gemm_overflows()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            idx.query_device(b, q.data_ptr(), 10, -1.0, ids.data_ptr(), sims.data_ptr(), cnt.data_ptr(),
                             s.cuda_stream, scan=scan, gemm=gemm, certify=False)
            e1.record(s)
            torch.cuda.synchronize()
            print(scan, "gemm", gemm, f"{e0.elapsed_time(e1):.2f} ms", "overflows", idx.gemm_overflows() - o0,
                  "scan", idx.timing_totals(2, reset=True), "merge", idx.timing_totals(1, reset=True), flush=True)
