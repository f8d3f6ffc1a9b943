"""fp64 master rows in pinned, device-mapped host memory (host_master /
SINE_STORE_F64_HOST): stage-1 results, the fp64 re-rank, compaction and
snapshots must be exactly those of the HBM-master index (ref
index.py:94-102, :340-354)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sine_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_17360_b200 as P
    from paper_2509_17360_b200 import _native as N
    if N.device_count() < 1:
        pytest.skip("no CUDA device")
    return P


@pytest.mark.parametrize("scan", ["fp32", "bf16"])
def test_host_master_equals_oracle(pkg, scan):
    rng = np.random.default_rng(31)
    n, d = 40_000, 384
    X = rng.standard_normal((n, d))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    ids = np.arange(1, n + 1)
    idx = pkg.GpuCosineIndex(d, scan=scan, host_master=True)
    dev = pkg.GpuCosineIndex(d, scan=scan)
    ora = O.OracleExactIndex(d, capacity=n)
    for lo in range(0, n, 10_000):  # several inserts: the host store grows
        idx.insert_batch(ids[lo:lo + 10_000], X[lo:lo + 10_000])
        dev.insert_batch(ids[lo:lo + 10_000], X[lo:lo + 10_000])
    ora.bulk_load(ids, X)
    Q = X[rng.choice(n, 48, replace=False)] + 0.05 * rng.standard_normal((48, d))
    Q = np.concatenate([Q / np.linalg.norm(Q, axis=1, keepdims=True), X[:16]])
    for k, tau in ((10, 0.9), (10, -1.0), (50, 0.5)):
        for B in (1, Q.shape[0]):
            got = idx.query_batch(Q[:B], k, tau)
            want_dev = dev.query_batch(Q[:B], k, tau)
            for b in range(B):
                want = ora.query(Q[b], k, min_similarity=tau)
                assert got[0][b, :got[2][b]].tolist() == [c.id for c in want]
                assert np.allclose(got[1][b, :got[2][b]], [c.similarity for c in want], rtol=0, atol=1e-12)
            assert np.array_equal(got[0], want_dev[0]) and np.array_equal(got[2], want_dev[2])
    # removals past the compaction threshold: the host rows compact in place
    gone = rng.choice(ids, n // 3, replace=False)
    idx.remove_batch(gone)
    dev.remove_batch(gone)
    for i in gone:
        ora.remove(int(i))
    assert idx.ids() == ora.ids()
    got = idx.query_batch(Q, 10, -1.0)
    for b in range(Q.shape[0]):
        assert got[0][b, :got[2][b]].tolist() == [c.id for c in ora.query(Q[b], 10, min_similarity=-1.0)]
    assert idx.snapshot_lines() == dev.snapshot_lines()
    keep = [i for i in ids[:50].tolist() if i not in set(gone.tolist())]
    assert np.array_equal(idx.rows(keep), X[np.asarray(keep) - 1])
