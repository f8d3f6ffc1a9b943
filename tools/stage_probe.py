"""Small-batch stage-1 timing on config B (1M x 768, k = 10): device path,
back-to-back batches, CUDA events around groups of 50, median of 3 groups.
Used for A/B runs of environment knobs (SINE_RES_STAGES, SINE_NO_FFMA, ...)
in separate processes; prints one line per (B, scan, tau) with ms and the
fraction of the HBM copy figure.  Not a benchmark."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17360_b200 import GpuCosineIndex  # noqa: E402
from paper_2509_17360_b200 import _native  # noqa: E402

if os.environ.get("PROBE_LIB"):  # A/B against another build of the library (same process layout)
    _native.load_library(os.environ["PROBE_LIB"])

N, D, K = 1_000_000, 768, 10
PEAK = 6550.0e9
bs = [int(b) for b in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8,16").split(",")]
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn((N, D), dtype=torch.float64, device="cuda", generator=g)
x /= x.norm(dim=1, keepdim=True)
idx = GpuCosineIndex(D, store_f32=True, store_bf16=True, capacity=N)
idx.insert_device(np.arange(N), x.data_ptr())
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
rng = np.random.default_rng(5)
out = []
for B in bs:
    src = torch.from_numpy(rng.integers(0, N, B)).cuda()
    qn = x[src] * 0.95 + 0.05 * torch.randn((B, D), dtype=torch.float64, device="cuda", generator=g) / D ** 0.5
    q = (qn / qn.norm(dim=1, keepdim=True)).contiguous()
    ids = torch.empty((B, K), dtype=torch.int64, device="cuda")
    sims = torch.empty((B, K), dtype=torch.float64, device="cuda")
    cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
    for scan in ("fp32", "bf16"):
        for tau in (0.9, -1.0):
            def run():
                idx.query_device(B, q.data_ptr(), K, tau, ids.data_ptr(), sims.data_ptr(), cnt.data_ptr(),
                                 s.cuda_stream, scan=scan, certify=False)
            for _ in range(5):
                run()
            torch.cuda.synchronize()
            res = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(50):
                    run()
                b.record()
                torch.cuda.synchronize()
                res.append(a.elapsed_time(b) / 50)
            ms = sorted(res)[1]
            byts = N * D * (4 if scan == "fp32" else 2)
            ref = idx.query_batch(q.cpu().numpy(), K, tau, scan=scan)[0]
            same = bool(np.array_equal(ids.cpu().numpy(), ref))
            out.append({"B": B, "scan": scan, "tau": tau, "ms": round(ms, 4), "hbm_frac": round(byts / (ms * 1e-3) / PEAK, 3),
                        "ids_equal_certified_path": same})
            print(json.dumps(out[-1]), os.environ.get("PROBE_LIB", "head"), flush=True)
