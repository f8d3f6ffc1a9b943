"""Single-query (B = 1) stage-1 kernels against the oracle.

A single query takes one of three in-kernel engines of the resident scan
(csrc/umma.cuh umma_res_kernel, chosen once per process in capi.cu
umma_res_query):

* default -- eight FFMA dot-product warps split each tile's K blocks by ring
  parity and feed four list warps through a score ring (p.ffma = 3);
* SINE_FFMA_LIST=1 -- the four list warps compute the dot products
  themselves (scalar FFMA for fp32 rows; packed FFMA2 for bf16 rows or with
  SINE_FFMA2=1);
* SINE_NO_FFMA=1 -- tcgen05 MMAs with N = 16.

Each runs in its own process (the switches are read once).  All must give
the oracle's ids (ExactCosineIndex.query, ref index.py:94-102) and the same
fp64 similarities, on shapes that exercise the parity split: one K block per
tile (d = 1: the groups alternate whole tiles), odd K-block counts, a partial
last tile, holes from removals, duplicate rows (ties decided by id), k up to
MAX_K and thresholds that admit everything or nothing.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import sine_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [  # (n, d)
    (40_000, 1),
    (30_001, 96),     # 3 K blocks (fp32), partial last tile
    (50_000, 200),
    (25_000, 768),
    (3_000, 1536),    # fewer tiles than SMs
    (60_000, 1024),   # 32 K blocks per tile, several tiles per CTA (the ring laps many times)
]
QUERIES = [(1, -1.0), (10, -1.0), (10, 0.5), (20, 0.9), (64, -1.0), (128, 0.2)]

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, ROOT)
import paper_2509_17360_b200 as P
cases, queries, out = json.loads(sys.argv[1]), json.loads(sys.argv[2]), sys.argv[3]
res = {}
for n, d in cases:
    rng = np.random.default_rng(n + d)
    X = rng.standard_normal((n, d))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    X[n // 3:n // 3 + 50] = X[:50]
    ids = rng.permutation(4 * n)[:n] + 1
    gone = ids[rng.choice(n, n // 10, replace=False)]
    Q = np.concatenate([X[:3], rng.standard_normal((3, d))])
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    for scan in ("fp32", "bf16"):
        idx = P.GpuCosineIndex(d, scan=scan)
        idx.insert_batch(ids, X)
        idx.remove_batch(gone)
        for qi in range(Q.shape[0]):
            for k, tau in queries:
                got = idx.query(Q[qi], k, min_similarity=tau)
                res[f"{n}/{d}/{scan}/{qi}/{k}/{tau}"] = [[c.id, c.similarity.hex()] for c in got]
        idx.close()
with open(out, "w") as fh:
    json.dump(res, fh)
""".replace("ROOT", repr(ROOT))

MODES = {
    "helpers": {},
    "list": {"SINE_FFMA_LIST": "1"},
    "list_ffma2": {"SINE_FFMA_LIST": "1", "SINE_FFMA2": "1"},
    "mma": {"SINE_NO_FFMA": "1"},
}


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    from paper_2509_17360_b200 import _native as N
    if N.device_count() < 1:
        pytest.skip("no CUDA device")
    out = {}
    for name, extra in MODES.items():
        path = str(tmp_path_factory.mktemp(name) / "r.json")
        env = {k: v for k, v in os.environ.items() if not k.startswith("SINE_FFMA") and k != "SINE_NO_FFMA"}
        env.update(extra)
        r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(CASES), json.dumps(QUERIES), path],
                           env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        with open(path) as fh:
            out[name] = json.load(fh)
    return out


@pytest.mark.parametrize("mode", list(MODES))
def test_b1_mode_equals_oracle(runs, mode):
    got = runs[mode]
    for n, d in CASES:
        rng = np.random.default_rng(n + d)
        X = rng.standard_normal((n, d))
        X /= np.linalg.norm(X, axis=1, keepdims=True)
        X[n // 3:n // 3 + 50] = X[:50]
        ids = rng.permutation(4 * n)[:n] + 1
        gone = ids[rng.choice(n, n // 10, replace=False)]
        Q = np.concatenate([X[:3], rng.standard_normal((3, d))])
        Q /= np.linalg.norm(Q, axis=1, keepdims=True)
        ora = O.OracleExactIndex(d, capacity=n)
        ora.bulk_load(ids, X)
        for i in gone:
            ora.remove(int(i))
        for scan in ("fp32", "bf16"):
            for qi in range(Q.shape[0]):
                for k, tau in QUERIES:
                    want = ora.query(Q[qi], k, min_similarity=tau)
                    have = got[f"{n}/{d}/{scan}/{qi}/{k}/{tau}"]
                    assert [h[0] for h in have] == [c.id for c in want], (mode, n, d, scan, qi, k, tau)
                    for h, c in zip(have, want):
                        assert float.fromhex(h[1]) == pytest.approx(c.similarity, abs=1e-12)


def test_b1_modes_identical(runs):
    """The fp64 re-rank makes the three engines' answers bit-identical."""
    base = runs["helpers"]
    for mode in MODES:
        assert runs[mode] == base, mode
