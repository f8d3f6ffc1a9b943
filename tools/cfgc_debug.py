"""Debug driver: config-C-like store (device-generated rows, d=1024, k=20),
compares the batched stage-1 paths with a brute-force fp64 torch top-1."""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2509_17360_b200 import GpuCosineIndex  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
d, k, tau = 1024, 20, 0.9
idx = GpuCosineIndex(d, scan="bf16", store_f32=True, store_bf16=True, capacity=n)
g = torch.Generator(device="cuda").manual_seed(7)
X = torch.empty((n, d), dtype=torch.float64, device="cuda")
for i0 in range(0, n, 250_000):
    m = min(250_000, n - i0)
    x = torch.randn((m, d), dtype=torch.float64, device="cuda", generator=g)
    x /= x.norm(dim=1, keepdim=True)
    X[i0:i0 + m] = x
    idx.insert_device(np.arange(i0, i0 + m, dtype=np.int64) + 1, x.data_ptr())
rng = np.random.default_rng(9)
src = rng.choice(n, 2048, replace=False) + 1
base = idx.rows(src)
assert np.array_equal(base, X[torch.from_numpy(src - 1).cuda()].cpu().numpy())
qs = rng.standard_normal((4096, d))
qs /= np.linalg.norm(qs, axis=1, keepdims=True)
cs = np.zeros(4096)
for j in range(2048):
    x = base[j]
    gq = qs[2 * j] - (qs[2 * j] @ x) * x
    gq /= np.linalg.norm(gq)
    c = rng.uniform(0.88, 0.99)
    cs[2 * j] = c
    qs[2 * j] = c * x + math.sqrt(1 - c * c) * gq
    qs[2 * j] /= np.linalg.norm(qs[2 * j])
q = torch.from_numpy(qs).cuda()
# exact top-1 per query (fp64 brute force)
best_s = torch.full((4096,), -2.0, dtype=torch.float64, device="cuda")
best_i = torch.zeros((4096,), dtype=torch.int64, device="cuda")
for i0 in range(0, n, 500_000):
    s = q @ X[i0:i0 + 500_000].T
    v, ii = s.max(dim=1)
    upd = v > best_s
    best_s = torch.where(upd, v, best_s)
    best_i = torch.where(upd, ii + i0 + 1, best_i)
want = np.where(best_s.cpu().numpy() >= tau, best_i.cpu().numpy(), -1)
print("planted below tau:", int(np.sum((cs[::2] < tau))), "of 2048; exact hits:", int(np.sum(want >= 0)), flush=True)
for scan in ("bf16", "fp32"):
    for b in (64, 512, 4096):
        for gemm in (None, False):
            t0 = time.perf_counter()
            ids, sims, cnt = idx.query_batch(qs[:b], k, tau, scan=scan, check=False, gemm=gemm)
            dt = time.perf_counter() - t0
            top = np.where(cnt > 0, ids[:, 0], -1)
            bad = np.nonzero(top != want[:b])[0]
            print(f"{scan} B={b} gemm={gemm}: {dt * 1e3:.1f} ms  mismatches={bad.size} overflows={idx.gemm_overflows()}"
                  f" uncert={idx.uncertified()}", flush=True)
            for j in bad[:5]:
                print("   q", j, "want", want[j], best_s[j].item(), "got", ids[j, :3], sims[j, :3], cnt[j], flush=True)
