import sys, numpy as np
sys.path.insert(0, '.')
import paper_2509_17360_b200 as pkg
rng = np.random.default_rng(5)
d, n = 256, 4000
base = rng.standard_normal(d); base /= np.linalg.norm(base)
rows = rng.standard_normal((n, d)); rows /= np.linalg.norm(rows, axis=1, keepdims=True)
for i in range(300):
    g = rows[i] - (rows[i] @ base) * base; g /= np.linalg.norm(g)
    c = 0.999 - i * 1e-4
    rows[i] = c * base + np.sqrt(1 - c * c) * g
ids = rng.permutation(10 * n)[:n]
idx = pkg.GpuCosineIndex(d, scan="fp32", store_f32=True, store_bf16=True)
idx.insert_batch(ids, rows)
q = np.stack([base, rows[3000]])
for k in (5, 40):
    for B in (1, 2):
        r = idx.query_batch(q[:B], k, -1.0)
        print("k", k, "B", B, "uncert", idx.uncertified(), r[1][0][:3], r[1][0][k-1])
        r = idx.query_batch(q[:B], k, -1.0, cuda_core=True)
        print("   cuda_core uncert", idx.uncertified())
