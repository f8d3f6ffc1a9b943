"""Small answer check (compute-sanitizer is closed on this pool) over the
round-2 stage-1 paths: the FFMA helper mode at B = 1 (both row types) and
B = 2 (fp32), the MMA path at B = 3 / 16, and the merge kernel's compact
selection at tau -1 -- 40k x 768 rows, answers checked against a float64
numpy top-k.  Not a benchmark."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17360_b200 import GpuCosineIndex  # noqa: E402

N, D, K = 40_000, 768, 10
rng = np.random.default_rng(7)
x = rng.standard_normal((N, D))
x /= np.linalg.norm(x, axis=1, keepdims=True)
idx = GpuCosineIndex(D, store_f32=True, store_bf16=True, capacity=N)
idx.insert_batch(np.arange(N), x, _checked=True)
bad = 0
for b in (1, 2, 3, 16):
    q = x[rng.integers(0, N, b)] * 0.95 + 0.05 * rng.standard_normal((b, D)) / np.sqrt(D)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    for scan in ("fp32", "bf16"):
        for tau in (0.9, -1.0):
            ids, sims, cnt = idx.query_batch(q, K, tau, scan=scan)
            s = x @ q.T
            for j in range(b):
                order = np.lexsort((np.arange(N), -s[:, j]))
                want = [i for i in order[:K] if s[i, j] >= tau]
                got = ids[j, :cnt[j]].tolist()
                if got != want:
                    bad += 1
                    print("mismatch", b, scan, tau, j, got[:3], want[:3])
print("small_path_check done, mismatches:", bad)
