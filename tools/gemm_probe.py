"""Quick timing of the large-batch stage-1 paths on config B (1M x 768):
tiled GEMM vs the per-group passes, device time by CUDA events."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2509_17360_b200 import GpuCosineIndex  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rows = bench.make_rows(n, 768)
idx = GpuCosineIndex(768, scan="fp32", store_bf16=True, capacity=n)
t = torch.from_numpy(rows).cuda()
idx.insert_device(np.arange(n) + 1, t.data_ptr())
del t
torch.cuda.synchronize()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for scan in ("bf16", "fp32"):
        for b in (256, 1024, 4096):
            qs = bench.make_queries(rows, b, seed=100 + b)
            q = torch.from_numpy(qs).cuda()
            ids = torch.empty((b, 10), dtype=torch.int64, device="cuda")
            sims = torch.empty((b, 10), dtype=torch.float64, device="cuda")
            cnt = torch.empty((b,), dtype=torch.int32, device="cuda")
            res = {}
            for gemm in (True, False):
                run = lambda: idx.query_device(b, q.data_ptr(), 10, 0.9, ids.data_ptr(), sims.data_ptr(),  # noqa
                                               cnt.data_ptr(), s.cuda_stream, scan=scan, gemm=gemm)
                run()
                torch.cuda.synchronize()
                reps = 3
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(reps):
                    run()
                e1.record(s)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                res[gemm] = (ms, ids.cpu().numpy().copy(), cnt.cpu().numpy().copy())
                tf = 2.0 * n * 768 * b / (ms / 1e3) / 1e12
                print(f"{scan} B={b} gemm={gemm}: {ms:.3f} ms  {b / ms * 1e3:,.0f} lookups/s  {tf:.0f} TFLOP/s "
                      f"overflows={idx.gemm_overflows()} uncert={idx.uncertified()}", flush=True)
            same = np.array_equal(res[True][1], res[False][1]) and np.array_equal(res[True][2], res[False][2])
            print(f"   gemm == passes: {same}", flush=True)
