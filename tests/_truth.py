"""Device-side ground truth for the full-size parity tests (test helper).

At the BASELINE shapes (1M x 768, 10M x 1024) the numpy oracle would need
minutes per query batch, so the truth is the same algorithm as the
reference's `ExactCosineIndex.query` (pkg/src/semcache/index.py:94-102 +
`_rank` :42-46) evaluated with torch float64 on the GPU: a float64
matmul `rows @ q`, the inclusive `>= min_similarity` test and the
(-similarity, id) order.  It is independent of the product's kernels
(cuBLAS DGEMM + torch.topk, no libsine_b200 code), and the rows it reads
are regenerated from the same seeded torch generator the index was filled
from.

The comparison tolerates what the reference's own tests tolerate at this
boundary (pkg/tests/test_index.py:69, test_acceptance.py:314): similarities
within 1e-12; ids exact except where two true similarities are within
`NEAR` of each other (or of the threshold), where float64 summation order
may legitimately swap them.
"""

from __future__ import annotations

import math

import numpy as np

NEAR = 1e-13


def unit_rows(torch, n, d, seed, device="cuda"):
    g = torch.Generator(device=device).manual_seed(int(seed))
    x = torch.randn((n, d), dtype=torch.float64, device=device, generator=g)
    x /= x.norm(dim=1, keepdim=True)
    return x


def planted_queries(src_rows: np.ndarray, n_random: int, d: int, seed: int) -> np.ndarray:
    """Queries: for each source row one near-duplicate at cos in [0.88,
    0.99] (straddling tau 0.9) and one exact copy, then random unit
    vectors."""
    rng = np.random.default_rng(seed)
    out = []
    for x in src_rows:
        g = rng.standard_normal(d)
        g -= (g @ x) * x
        g /= np.linalg.norm(g)
        c = rng.uniform(0.88, 0.99)
        v = c * x + math.sqrt(1 - c * c) * g
        out.append(v / np.linalg.norm(v))
        out.append(x.copy())
    r = rng.standard_normal((n_random, d))
    r /= np.linalg.norm(r, axis=1, keepdims=True)
    q = np.concatenate([np.asarray(out).reshape(-1, d), r])
    return q[rng.permutation(q.shape[0])]


class Truth:
    """Per-query candidate pools, accumulated over row chunks: every row
    whose float64 similarity is >= the chunk's (k+pad)-th best."""

    def __init__(self, torch, q: np.ndarray, k: int, pad: int = 24):
        self.torch = torch
        self.q = q
        self.k = k
        self.pad = pad
        self.pool_ids = [[] for _ in range(q.shape[0])]
        self.pool_sims = [[] for _ in range(q.shape[0])]

    def add_chunk(self, x, id0: int, qchunk: int = 512):
        torch = self.torch
        n = x.shape[0]
        kk = min(self.k + self.pad, n)
        for b0 in range(0, self.q.shape[0], qchunk):
            qd = torch.from_numpy(np.ascontiguousarray(self.q[b0:b0 + qchunk])).to(x.device)
            s = x @ qd.T  # [n, c] float64
            vals, idx = torch.topk(s, kk, dim=0)
            vals, idx = vals.cpu().numpy(), idx.cpu().numpy()
            for j in range(qd.shape[0]):
                v = vals[:, j]
                kth = v[min(self.k, kk) - 1]
                if kk < n and v[kk - 1] >= kth - NEAR:  # ties run past the pad: take them all
                    sel = torch.nonzero(s[:, j] >= kth - NEAR).flatten()
                    ii = sel.cpu().numpy()
                    vv = s[sel, j].cpu().numpy()
                else:
                    ii, vv = idx[:, j], v
                self.pool_ids[b0 + j].extend((ii + id0).tolist())
                self.pool_sims[b0 + j].extend(vv.tolist())
            del s

    def answer(self, j: int, min_similarity: float):
        ids = np.asarray(self.pool_ids[j], dtype=np.int64)
        sims = np.asarray(self.pool_sims[j], dtype=np.float64)
        keep = sims >= min_similarity
        ids, sims = ids[keep], sims[keep]
        order = np.lexsort((ids, -sims))
        return ids[order], sims[order]


def check_query(got_ids, got_sims, count, truth_ids, truth_sims, k, min_similarity, tag=""):
    """Reference-equivalence of one query's answer (see module doc)."""
    want_n = min(k, len(truth_ids))
    n = int(count)
    if n != want_n:
        # only a similarity within NEAR of the threshold may flip membership
        edge = np.abs(truth_sims - min_similarity) < NEAR
        assert edge.any(), f"{tag}: count {n} != {want_n}"
    m = min(n, want_n)
    np.testing.assert_allclose(got_sims[:m], truth_sims[:m], rtol=0, atol=1e-12, err_msg=tag)
    for i in range(m):
        if got_ids[i] == truth_ids[i]:
            continue
        # a swap is legal only between near-equal true similarities
        s = truth_sims[i]
        near = np.abs(truth_sims - s) < NEAR
        assert got_ids[i] in set(truth_ids[near].tolist()), \
            f"{tag}: rank {i} id {got_ids[i]} != {truth_ids[i]} (sim {s!r})"
    for i in range(n, len(got_ids)):
        assert got_ids[i] == -1, f"{tag}: padding"
