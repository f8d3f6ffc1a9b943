"""Stage-1 parity on the B200: GpuCosineIndex vs the reference's own golden
outputs (tests/golden/index_golden.json, produced by the reference) and vs
the CPU oracle on seeded inputs.  Mirrors pkg/tests/test_index.py."""

from __future__ import annotations

import math

import numpy as np
import pytest

import gen_inputs as G
from oracle import sine_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_17360_b200 as P
    from paper_2509_17360_b200 import _native as N
    if N.device_count() < 1:
        pytest.skip("no CUDA device")
    return P


def _same(got, want, tol=1e-12):
    assert [c.id for c in got] == [w[0] for w in want]
    for c, w in zip(got, want):
        assert c.similarity == pytest.approx(float.fromhex(w[1]), abs=tol)


def test_validation_mirrors_reference(pkg):
    # pkg/tests/test_index.py:36-49
    idx = pkg.GpuCosineIndex(4)
    idx.insert(1, G.normalize([1, 2, 3, 4]))
    with pytest.raises(pkg.ValidationError):
        idx.insert(1, G.normalize([1, 0, 0, 0]))
    with pytest.raises(pkg.ValidationError):
        idx.insert(2, [1.0, 2.0, 3.0, 4.0])
    with pytest.raises(pkg.ValidationError):
        idx.insert(3, G.normalize([1, 2, 3]))
    with pytest.raises(pkg.ValidationError):
        idx.remove(42)
    with pytest.raises(pkg.ValidationError):
        idx.query(G.normalize([1, 0, 0, 0]), k=0)
    assert idx.query(G.normalize([1, 0, 0, 0]), k=3)[0].id == 1
    assert pkg.GpuCosineIndex(4).query(G.normalize([1, 0, 0, 0]), k=3) == []
    with pytest.raises(pkg.ValidationError):
        pkg.GpuCosineIndex(0)


def test_linear_trials_match_reference(pkg, index_golden):
    for (dim, vectors, queries), gold in zip(G.linear_oracle_trials(), index_golden["linear_trials"]):
        idx = pkg.GpuCosineIndex(dim)
        for i, v in vectors.items():
            idx.insert(i, v)
        for (q, k, ms), want in zip(queries, gold["results"]):
            _same(idx.query(q, k=k, min_similarity=ms), want)


def test_tie_order(pkg, index_golden):
    v = G.normalize([1, 2, 3, 4, 5, 6, 7, 8])
    idx = pkg.GpuCosineIndex(8)
    for i in (9, 3, 7, 1):
        idx.insert(i, v)
    _same(idx.query(v, k=4), index_golden["tie_order"])


def test_remove_steps(pkg, index_golden):
    dim, vectors, steps = G.remove_case()
    idx = pkg.GpuCosineIndex(dim)
    for i, v in vectors.items():
        idx.insert(i, v)
    for (i, q), gold in zip(steps, index_golden["remove_steps"]):
        idx.remove(i)
        _same(idx.query(q, k=10), gold["result"])
        assert idx.ids() == gold["ids"]  # the reference order (swap-last), not just the set
    assert len(idx) == 35


def test_acceptance_9b(pkg, index_golden):
    dim, stored, queries = G.acceptance_9b_case()
    idx = pkg.GpuCosineIndex(dim, seed=3)
    idx.insert_batch(list(stored), np.asarray(list(stored.values())))
    for q, want in zip(queries, index_golden["acceptance_9b"]["results"]):
        _same(idx.query(q, 7), want)


@pytest.mark.parametrize("scan", ["fp32", "bf16"])
def test_config_a_exact_modes(pkg, index_golden, scan):
    """Config A (10k x 384, k=5) at tau 0.9 and -1: fp32 and bf16 scans with
    the fp64 re-rank both reproduce the reference ids and similarities."""
    rows, qs = G.config_a()
    idx = pkg.GpuCosineIndex(rows.shape[1], scan=scan)
    idx.insert_batch(np.arange(rows.shape[0]), rows)
    for ms in (0.9, -1.0):
        gold = index_golden["config_a"]["results"][repr(ms)]
        ids, sims, counts = idx.query_batch(qs, 5, ms)
        for j, want in enumerate(gold):
            assert ids[j, :counts[j]].tolist() == [w[0] for w in want], (ms, j)
            np.testing.assert_allclose(sims[j, :counts[j]], [float.fromhex(w[1]) for w in want],
                                       atol=1e-12, rtol=0)
            assert (ids[j, counts[j]:] == -1).all()


def test_config_a_bf16_raw_scores(pkg, index_golden):
    """bf16 fast mode without re-rank: scores within 2e-2, recall stated."""
    rows, qs = G.config_a()
    idx = pkg.GpuCosineIndex(rows.shape[1], scan="bf16", rerank=False)
    idx.insert_batch(np.arange(rows.shape[0]), rows)
    gold = index_golden["config_a"]["results"][repr(-1.0)]
    ids, sims, counts = idx.query_batch(qs, 5, -1.0)
    exact = rows @ qs.T
    hit = tot = 0
    for j, want in enumerate(gold):
        wids = [w[0] for w in want]
        hit += len(set(ids[j, :counts[j]].tolist()) & set(wids))
        tot += len(wids)
        for i, s in zip(ids[j, :counts[j]], sims[j, :counts[j]]):
            assert abs(s - exact[i, j]) < 2e-2
    recall = hit / tot
    print(f"bf16 (no re-rank) recall@5 on config A: {recall:.4f}")
    assert recall >= 0.95


def test_ties_under_shuffled_ids(pkg, index_golden):
    d, rows, ids, qs = G.tie_rows()
    for scan in ("fp32", "bf16"):
        idx = pkg.GpuCosineIndex(d, scan=scan)
        idx.insert_batch(ids, rows)
        for k, res in index_golden["ties"]["results"].items():
            for q, want in zip(qs, res):
                _same(idx.query(q, int(k)), want)


def test_batch_equals_independent_queries(pkg):
    rng = np.random.default_rng(11)
    n, d = 3000, 96
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((37, d))
    q[:10] = rows[::300]
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    idx = pkg.GpuCosineIndex(d)
    idx.insert_batch(rng.permutation(10 * n)[:n], rows)
    ids, sims, counts = idx.query_batch(q, 9, 0.05)
    for j in range(q.shape[0]):
        one = idx.query(q[j], 9, 0.05)
        assert [c.id for c in one] == ids[j, :counts[j]].tolist()
        assert [c.similarity for c in one] == sims[j, :counts[j]].tolist()


def test_nan_rows_never_match_and_k_larger_than_n(pkg):
    idx = pkg.GpuCosineIndex(3)
    # the reference admits a NaN vector (|nan - 1| > tol is False) but it
    # never passes `sims >= min_similarity`
    idx.insert(5, [float("nan"), 0.0, 0.0])
    idx.insert(6, G.normalize([1, 1, 0]))
    got = idx.query(G.normalize([1, 0, 0]), k=10, min_similarity=-1.0)
    assert [c.id for c in got] == [6]
    assert got[0].similarity == pytest.approx(1 / math.sqrt(2), abs=1e-15)


def test_removal_compaction_and_reinsert(pkg):
    rng = np.random.default_rng(3)
    n, d = 2000, 40
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    idx = pkg.GpuCosineIndex(d)
    idx.insert_batch(np.arange(n), rows)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(np.arange(n), rows)
    gone = rng.permutation(n)[:1500]          # forces several compactions
    for i in gone[:700]:
        idx.remove(int(i))
        ora.remove(int(i))
    idx.remove_batch(gone[700:])
    for i in gone[700:]:
        ora.remove(int(i))
    fresh = rng.standard_normal((300, d))
    fresh /= np.linalg.norm(fresh, axis=1, keepdims=True)
    idx.insert_batch(np.arange(n, n + 300), fresh)
    ora.bulk_load(np.arange(n, n + 300), fresh)
    assert idx.ids() == ora.ids() and len(idx) == len(ora)
    for j in range(20):
        q = rows[j] if j % 2 else fresh[j]
        got = idx.query(q, 12, -1.0)
        want = ora.query(q, 12, -1.0)
        assert [c.id for c in got] == [c.id for c in want]
        np.testing.assert_allclose([c.similarity for c in got], [c.similarity for c in want], atol=1e-12)
    with pytest.raises(pkg.ValidationError):
        idx.remove(int(gone[0]))
    with pytest.raises(pkg.ValidationError):
        idx.insert_batch([n + 5], fresh[:1])


def test_snapshot_round_trip(pkg, tmp_path):
    rng = np.random.default_rng(31)
    idx = pkg.GpuCosineIndex(6, seed=4)
    vecs = rng.standard_normal((12, 6))
    vecs /= np.linalg.norm(vecs, axis=1, keepdims=True)
    idx.insert_batch(np.arange(12), vecs)
    idx.remove(3)
    p = str(tmp_path / "x.idx")
    idx.save(p)
    loaded = pkg.GpuCosineIndex.load(p)
    assert loaded.dimension == 6 and loaded.seed == 4
    assert loaded.ids() == idx.ids()
    assert loaded.rows([5]).tobytes() == vecs[5].tobytes()  # bit-exact rows
    q = vecs[0]
    assert [(c.id, c.similarity) for c in loaded.query(q, 5)] == [(c.id, c.similarity) for c in idx.query(q, 5)]
    lines = open(p).read().splitlines()
    assert lines[0] == "exact-cosine-index" and lines[3] == "count: 11"


@pytest.mark.parametrize("d", [1, 5, 127, 128, 129, 384, 768, 1024, 1536, 2048])
def test_dimension_sweep(pkg, d):
    rng = np.random.default_rng(d)
    n = 700
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((5, d))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(np.arange(n), rows)
    for scan in ("fp32", "bf16"):
        idx = pkg.GpuCosineIndex(d, scan=scan)
        idx.insert_batch(np.arange(n), rows)
        ids, sims, counts = idx.query_batch(q, 7, -1.0)
        for j in range(5):
            want = ora.query(q[j], 7, -1.0)
            assert ids[j, :counts[j]].tolist() == [c.id for c in want], (scan, d, j)
            np.testing.assert_allclose(sims[j, :counts[j]], [c.similarity for c in want], atol=1e-12)


def test_large_batch_groups(pkg):
    """B > the per-launch query group: several scan launches, same answers."""
    rng = np.random.default_rng(8)
    n, d, B = 5000, 128, 1100
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((B, d))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(np.arange(n), rows)
    for scan in ("fp32", "bf16"):
        idx = pkg.GpuCosineIndex(d, scan=scan)
        idx.insert_batch(np.arange(n), rows)
        for cl in (False, True):  # cluster size 8 with multicast rows
            ids, sims, counts = idx.query_batch(q, 20, 0.1, cluster=cl)
            for j in range(B):
                want = ora.query(q[j], 20, 0.1)
                assert ids[j, :counts[j]].tolist() == [c.id for c in want]


def test_full_size_properties(pkg):
    """BASELINE config B shape (1M x 768, k=10): sampled queries against the
    float64 oracle; planted duplicates must come back as rank 1 with
    similarity 1."""
    import torch
    n, d, k = 1_000_000, 768, 10
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
    x /= x.norm(dim=1, keepdim=True)
    idx = pkg.GpuCosineIndex(d, store_bf16=True, capacity=n)
    idx.insert_device(np.arange(n), x.data_ptr())
    rows = x.cpu().numpy()
    rng = np.random.default_rng(2)
    pick = rng.integers(0, n, 8)
    q = np.concatenate([rows[pick], rng.standard_normal((8, d))])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    for scan in ("fp32", "bf16"):
        ids, sims, counts = idx.query_batch(q, k, -1.0, scan=scan)
        for j in range(16):
            s = rows @ q[j]
            order = np.lexsort((np.arange(n), -s))[:k]
            assert ids[j].tolist() == order.tolist(), (scan, j)
            np.testing.assert_allclose(sims[j], s[order], atol=1e-12)
            if j < 8:
                assert ids[j, 0] == pick[j] and sims[j, 0] == pytest.approx(1.0, abs=1e-12)


@pytest.mark.parametrize("scan", ["fp32", "bf16"])
def test_tensor_core_and_cuda_core_paths_agree(pkg, index_golden, scan):
    """Config A through both stage-1 engines (tcgen05 for B >= 8, the
    CUDA-core streaming scan forced): identical ids and fp64 similarities."""
    rows, qs = G.config_a()
    idx = pkg.GpuCosineIndex(rows.shape[1], scan=scan)
    idx.insert_batch(np.arange(rows.shape[0]), rows)
    for ms in (0.9, -1.0, 0.2):
        a = idx.query_batch(qs, 5, ms)
        b = idx.query_batch(qs, 5, ms, cuda_core=True)
        c = idx.query_batch(qs, 5, ms, umma_v1=True)
        for x, y, z in zip(a, b, c):
            np.testing.assert_array_equal(x, y)
            np.testing.assert_array_equal(x, z)
        for B in (8, 16, 33, 64, 100, 129):  # resident group widths; cluster sizes 1, 2, 4; CTA pairs
            for kw in ({}, {"cluster": True}, {"pair": True}):
                d = idx.query_batch(qs[:B], 5, ms, **kw)
                for x, y in zip(d, b):
                    np.testing.assert_array_equal(x, y[:B])


def test_tensor_core_bf16_raw_scores_within_tolerance(pkg):
    rng = np.random.default_rng(21)
    n, d, B = 20000, 768, 160
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((B, d))
    q[::2] = rows[rng.integers(0, n, B // 2)] + 0.1 * rng.standard_normal((B // 2, d))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    idx = pkg.GpuCosineIndex(d, scan="bf16", rerank=False)
    idx.insert_batch(np.arange(n), rows)
    ids, sims, counts = idx.query_batch(q, 10, -1.0)
    exact = rows @ q.T
    hit = 0
    for j in range(B):
        assert counts[j] == 10
        true = np.lexsort((np.arange(n), -exact[:, j]))[:10]
        hit += len(set(true.tolist()) & set(ids[j].tolist()))
        assert np.all(np.abs(sims[j] - exact[ids[j], j]) < 2e-2)
        assert np.all(np.diff(sims[j]) <= 0)
    print(f"tcgen05 bf16 (no re-rank) recall@10: {hit / (10 * B):.4f}")
    assert hit / (10 * B) >= 0.9


@pytest.mark.parametrize("scan", ["fp32", "bf16"])
def test_certificate_falls_back_on_dense_clusters(pkg, scan):
    """Rows whose similarities are spaced 2e-5 apart (inside the tf32 /
    bf16 filter error, far outside the fp32 one): the fast filter cannot be
    certified, the query is re-run on the fp32 scan, and the answer is the
    reference's exactly."""
    rng = np.random.default_rng(5)
    d, n = 256, 4000
    base = rng.standard_normal(d)
    base /= np.linalg.norm(base)
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    for i in range(300):                       # a tight cluster around the query
        g = rows[i] - (rows[i] @ base) * base
        g /= np.linalg.norm(g)
        c = 0.999 - i * 2e-5
        rows[i] = c * base + np.sqrt(1 - c * c) * g
    ids = rng.permutation(10 * n)[:n]
    idx = pkg.GpuCosineIndex(d, scan=scan, store_f32=True, store_bf16=True)
    idx.insert_batch(ids, rows)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(ids, rows)
    q = np.stack([base, rows[3000]])
    for k in (5, 40):
        got_ids, got_sims, cnt = idx.query_batch(q, k, -1.0)
        for j in range(2):
            want = ora.query(q[j], k, -1.0)
            assert got_ids[j, :cnt[j]].tolist() == [c.id for c in want]
            np.testing.assert_allclose(got_sims[j, :cnt[j]], [c.similarity for c in want], atol=1e-12)
        assert idx.uncertified() >= 1


def test_cta_pair_kernel_fp32_d768(pkg):
    """fp32 rows at d=768 with 32 < B <= 64 take the tcgen05 cta_group::2
    kernel; answers equal the fp32 CUDA-core scan and the oracle."""
    rng = np.random.default_rng(77)
    n, d = 30000, 768
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((64, d))
    q[::2] = rows[rng.integers(0, n, 32)] + 0.3 * rng.standard_normal((32, d))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    idx = pkg.GpuCosineIndex(d)
    idx.insert_batch(np.arange(n), rows)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(np.arange(n), rows)
    for B, ms in ((64, -1.0), (48, 0.3), (40, 0.9)):
        a = idx.query_batch(q[:B], 10, ms)
        b = idx.query_batch(q[:B], 10, ms, cuda_core=True)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
        for j in range(0, B, 7):
            want = ora.query(q[j], 10, ms)
            assert a[0][j, :a[2][j]].tolist() == [c.id for c in want]


@pytest.mark.parametrize("d", [1, 64, 200, 384, 768])
def test_tiled_gemm_matches_oracle(pkg, d):
    """The large-batch tiled GEMM (256 x 256 CTA-pair tiles, all query tiles
    in one launch) on ragged row and query tiles, with tombstones: ids
    bit-exact and fp64 similarities (1e-12) vs the oracle, both scan modes."""
    rng = np.random.default_rng(100 + d)
    n, B = 20011, 700
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((B, d))
    pick = rng.integers(0, n, B // 2)
    q[: B // 2] = rows[pick] + (0.01 + 0.02 * rng.random((B // 2, 1))) * rng.standard_normal((B // 2, d))
    q[B // 2: B // 2 + 20] = rows[pick[:20]]  # exact duplicates: ties with the stored row
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ids = np.arange(n) * 3 + 7
    dead = rng.choice(n, 500, replace=False)
    ora = O.OracleExactIndex(d)
    keep = np.setdiff1d(np.arange(n), dead)
    ora.bulk_load(ids[keep], rows[keep])
    for scan in ("fp32", "bf16"):
        idx = pkg.GpuCosineIndex(d, scan=scan)
        idx.insert_batch(ids, rows)
        idx.remove_batch(ids[dead[:100]])  # tombstones only (below the compaction trigger)
        idx.remove_batch(ids[dead[100:]])
        for bq, ms in ((B, 0.9), (300, 0.5), (100, 0.9), (50, 0.5)):  # N = 256 / 256 / 128 / 64 tiles
            got = idx.query_batch(q[:bq], 10, ms, gemm=True)
            if d > 1:  # at d = 1 every same-sign row scores 1: dense, overflows, falls back (still exact)
                assert idx.gemm_overflows() == 0
            for j in range(bq):
                want = ora.query(q[j], 10, ms)
                assert got[0][j, :got[2][j]].tolist() == [c.id for c in want], (scan, bq, ms, j)
                np.testing.assert_allclose(got[1][j, :got[2][j]], [c.similarity for c in want], atol=1e-12, rtol=0)


def test_tiled_gemm_bf16_raw_and_overflow_fallback(pkg):
    """bf16 without re-rank through the GEMM path stays within the 2e-2
    bf16 tolerance; a low threshold overflows the per-query candidate
    buffers and the batch is re-run on the list-keeping kernels (exact)."""
    rng = np.random.default_rng(5)
    n, d, B = 9000, 256, 520
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rows[rng.integers(0, n, B)] + 0.02 * rng.standard_normal((B, d))  # cos ~0.95
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(np.arange(n), rows)
    idx = pkg.GpuCosineIndex(d, scan="bf16")
    idx.insert_batch(np.arange(n), rows)
    ids, sims, counts = idx.query_batch(q, 5, 0.9, rerank=False, gemm=True)
    for j in range(B):
        want = ora.query(q[j], 5, 0.9)
        assert counts[j] >= 1
        assert abs(sims[j, 0] - want[0].similarity) < 2e-2
    # a dense cluster (every row within cos ~0.98 of the query) overflows
    # the per-query candidate buffers at a floor >= 0.25: exact fallback
    base = rng.standard_normal(d)
    crow = base + 0.1 * rng.standard_normal((n, d))
    crow /= np.linalg.norm(crow, axis=1, keepdims=True)
    cidx = pkg.GpuCosineIndex(d, scan="bf16", store_f32=True)  # exact: certificate fallback to fp32 rows
    cidx.insert_batch(np.arange(n), crow)
    cora = O.OracleExactIndex(d)
    cora.bulk_load(np.arange(n), crow)
    cq = base + 0.1 * rng.standard_normal((B, d))
    cq /= np.linalg.norm(cq, axis=1, keepdims=True)
    before = cidx.gemm_overflows()
    got = cidx.query_batch(cq, 5, 0.5, gemm=True)
    assert cidx.gemm_overflows() == before + 1
    for j in range(0, B, 13):
        want = cora.query(cq[j], 5, 0.5)
        assert got[0][j, :got[2][j]].tolist() == [c.id for c in want]


def test_insert_device_orders_after_producer_stream(pkg):
    """Rows produced by a torch kernel on another stream and handed to
    insert_device right away are read only after that kernel finished."""
    torch = pytest.importorskip("torch")
    d, n = 512, 200_000
    idx = pkg.GpuCosineIndex(d, scan="bf16", store_f32=True, store_bf16=True, capacity=2 * n)
    side = torch.cuda.Stream()
    g = torch.Generator(device="cuda").manual_seed(3)
    kept = []
    with torch.cuda.stream(side):
        for c in range(2):
            x = torch.randn((n, d), dtype=torch.float64, device="cuda", generator=g)
            for _ in range(20):  # keep the producer stream busy
                x = x * 1.0000001
            x /= x.norm(dim=1, keepdim=True)
            idx.insert_device(np.arange(c * n, (c + 1) * n), x.data_ptr())
            kept.append(x)
    torch.cuda.synchronize()
    X = torch.cat(kept).cpu().numpy()
    pick = np.random.default_rng(0).choice(2 * n, 500, replace=False)
    np.testing.assert_array_equal(idx.rows(pick), X[pick])


def test_tiled_gemm_seeded_low_threshold(pkg):
    """Low min_similarity through the tiled GEMM: a sample pass seeds
    per-query floors (the k'-th largest tile maximum), the main pass keeps
    every pair above them; exact vs the oracle, no overflow."""
    rng = np.random.default_rng(21)
    n, d, B = 40000, 256, 300
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((B, d))
    q[:100] = rows[rng.integers(0, n, 100)] + 0.05 * rng.standard_normal((100, d))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(np.arange(n), rows)
    for scan in ("fp32", "bf16"):
        idx = pkg.GpuCosineIndex(d, scan=scan)
        idx.insert_batch(np.arange(n), rows)
        for k, ms, bq in ((10, -1.0, B), (20, 0.1, B), (10, -1.0, 60)):
            got = idx.query_batch(q[:bq], k, ms, gemm=True)
            assert idx.gemm_overflows() == 0
            for j in range(bq):
                want = ora.query(q[j], k, ms)
                assert got[0][j, :got[2][j]].tolist() == [c.id for c in want], (scan, k, ms, j)
                np.testing.assert_allclose(got[1][j, :got[2][j]], [c.similarity for c in want], atol=1e-12, rtol=0)


def test_unordered_id_batches_remove_and_requery(pkg):
    """Ids arriving out of order (first batch unordered, then ascending,
    then unordered again) stay addressable: remove / duplicate checks /
    rows() see every id (reference index.py:71-92 semantics)."""
    rng = np.random.default_rng(31)
    d = 32
    rows = rng.standard_normal((900, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    ids = rng.permutation(100000)[:900]
    idx = pkg.GpuCosineIndex(d)
    idx.insert_batch(ids[:300], rows[:300])
    idx.insert_batch(np.sort(ids[300:600]) + 200000, rows[300:600])
    idx.insert_batch(ids[600:], rows[600:])
    all_ids = np.concatenate([ids[:300], np.sort(ids[300:600]) + 200000, ids[600:]])
    with pytest.raises(pkg.ValidationError):
        idx.insert(int(ids[5]), rows[0])
    np.testing.assert_array_equal(idx.rows(all_ids[::37]), rows[::37])
    gone = all_ids[::5]
    idx.remove_batch(gone)
    ora = O.OracleExactIndex(d)
    keep = np.setdiff1d(np.arange(900), np.arange(900)[::5])
    ora.bulk_load(all_ids[keep], rows[keep])
    assert len(idx) == len(keep)
    q = rows[:20] + 0.1 * rng.standard_normal((20, d))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    got = idx.query_batch(q, 7, -1.0)
    for j in range(20):
        assert got[0][j, :got[2][j]].tolist() == [c.id for c in ora.query(q[j], 7, -1.0)]


def test_submit_into_pipelined_matches_query_batch(pkg):
    """Several batches in flight through sine_query_submit/wait with
    caller-owned pinned buffers return exactly query_batch's answers."""
    from paper_2509_17360_b200 import _native as N
    rng = np.random.default_rng(41)
    n, d, B = 30000, 256, 3
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    idx = pkg.GpuCosineIndex(d)
    idx.insert_batch(np.arange(n), rows)
    qs = rows[rng.integers(0, n, (6, B))] + 0.02 * rng.standard_normal((6, B, d))
    qs /= np.linalg.norm(qs, axis=2, keepdims=True)
    bufs = [(N.PinnedArray((B, d), np.float64), N.PinnedArray((B, 5), np.int64), N.PinnedArray((B, 5), np.float64),
             N.PinnedArray((B,), np.int32)) for _ in range(6)]
    tickets = []
    for s in range(6):
        q, i, sm, c = bufs[s]
        q.array[:] = qs[s]
        tickets.append(idx.submit_into(q.array, 5, 0.5, i.array, sm.array, c.array))
    for s in range(6):
        idx.wait_ticket(tickets[s])
        want = idx.query_batch(qs[s], 5, 0.5)
        np.testing.assert_array_equal(bufs[s][1].array, want[0])
        np.testing.assert_array_equal(bufs[s][2].array, want[1])
        np.testing.assert_array_equal(bufs[s][3].array, want[2])


@pytest.mark.parametrize("k", [60, 112])
def test_large_k_all_tensor_core_paths(pkg, k):
    """k' = k + 16 up to the 128-entry device lists: resident (B=8), CTA
    pair (B=100, bf16), tiled GEMM (B=300) and the CUDA-core scan agree
    with the oracle at low and mid thresholds (dense warm-up rounds, sparse
    inserts, seeded GEMM floors)."""
    rng = np.random.default_rng(k)
    n, d = 20000, 128
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((300, d))
    q[:100] = rows[rng.integers(0, n, 100)] + 0.2 * rng.standard_normal((100, d))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(np.arange(n), rows)
    for scan in ("fp32", "bf16"):
        idx = pkg.GpuCosineIndex(d, scan=scan)
        idx.insert_batch(np.arange(n), rows)
        for B, ms, kw in ((8, -1.0, {}), (100, 0.1, {}), (300, -1.0, {"gemm": True}), (8, 0.1, {"cuda_core": True})):
            got = idx.query_batch(q[:B], k, ms, **kw)
            for j in range(0, B, 7):
                want = ora.query(q[j], k, ms)
                assert got[0][j, :got[2][j]].tolist() == [c.id for c in want], (scan, B, ms, kw, j)
                np.testing.assert_allclose(got[1][j, :got[2][j]], [c.similarity for c in want], atol=1e-12, rtol=0)


def test_gpu_embedder_matches_reference_goldens(pkg):
    """GpuHashedBagEmbedder reproduces the reference HashedBagEmbedder's
    vectors bit for bit (goldens from the reference), batched and single."""
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "embed_golden.json"), encoding="utf-8"))
    texts = gold["texts"]
    for case in gold["cases"]:
        emb = pkg.GpuHashedBagEmbedder(case["dimension"], seed=case["seed"])
        got = emb.embed_batch(texts)
        for row, want in zip(got, case["vectors"]):
            dense = np.zeros(case["dimension"])
            for i, h in want:
                dense[i] = float.fromhex(h)
            assert row.tobytes() == dense.tobytes()
        one = emb.embed(texts[0])
        assert one.components == tuple(got[0].tolist())
    with pytest.raises(pkg.ValidationError):
        pkg.GpuHashedBagEmbedder(256).embed_batch(["ok text", "?!"])
    with pytest.raises(pkg.ValidationError):
        pkg.GpuHashedBagEmbedder(4)


def test_query_device_cert_logs_certificates(pkg):
    """query_device_cert: same answers as query_batch, certificates written
    to the caller's device buffer (1 for clear answers, 0 for a dense
    cluster whose bf16 filter cannot prove the cut)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(51)
    n, d, B = 20000, 128, 40
    rows = rng.standard_normal((n, d))
    rows[:3000] = rows[0] + 0.02 * rng.standard_normal((3000, d))  # dense cluster
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    q = rng.standard_normal((B, d))
    q[0] = rows[0]
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    for scan in ("fp32", "bf16"):
        idx = pkg.GpuCosineIndex(d, scan=scan)
        idx.insert_batch(np.arange(n), rows)
        qd = torch.from_numpy(q).cuda()
        ids = torch.empty((B, 10), dtype=torch.int64, device="cuda")
        sims = torch.empty((B, 10), dtype=torch.float64, device="cuda")
        cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
        cert = torch.full((B,), 7, dtype=torch.uint8, device="cuda")
        idx.query_device_cert(B, qd.data_ptr(), 10, 0.5, ids.data_ptr(), sims.data_ptr(), cnt.data_ptr(),
                              cert.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        c = cert.cpu().numpy()
        assert set(c.tolist()) <= {0, 1} and c[1:].all()
        want = idx.query_batch(q, 10, 0.5)  # certified (re-runs any uncertified query)
        got_ids = ids.cpu().numpy()
        for j in range(B):
            if c[j]:
                assert got_ids[j].tolist() == want[0][j].tolist()


@pytest.mark.gpu
@pytest.mark.parametrize("scan", ["fp32", "bf16"])
def test_mapped_result_staging_sync_and_async(pkg, scan):
    """sine_query / sine_query_submit write results through pinned, device-
    mapped staging (no device->host copies): plain (unpinned) numpy output
    buffers, batch and k growing between tickets, an uncertified query
    re-run through the async path, and an empty index (the copy branch)."""
    rng = np.random.default_rng(77)
    d, n = 256, 4000
    base = rng.standard_normal(d)
    base /= np.linalg.norm(base)
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    for i in range(300):                       # dense cluster: forces a certificate failure
        g = rows[i] - (rows[i] @ base) * base
        g /= np.linalg.norm(g)
        c = 0.999 - i * 2e-5
        rows[i] = c * base + np.sqrt(1 - c * c) * g
    ids = rng.permutation(10 * n)[:n]
    empty = pkg.GpuCosineIndex(d, scan=scan, store_f32=True, store_bf16=True)
    qe = np.ascontiguousarray(rows[:2])
    oi, osm, oc = np.zeros((2, 4), np.int64), np.ones((2, 4)), np.full(2, 9, np.int32)
    empty.query_into(qe, 4, -1.0, oi, osm, oc)
    assert oc.tolist() == [0, 0] and (oi == -1).all()
    t = empty.submit_into(qe, 4, -1.0, oi, osm, oc)
    empty.wait_ticket(t)
    assert oc.tolist() == [0, 0] and (oi == -1).all()

    idx = pkg.GpuCosineIndex(d, scan=scan, store_f32=True, store_bf16=True)
    idx.insert_batch(ids, rows)
    ora = O.OracleExactIndex(d)
    ora.bulk_load(ids, rows)
    plan = [(1, 5), (3, 12), (2, 40), (5, 3)]  # (B, k): staging grows and shrinks
    batches, tickets = [], []
    for s, (B, k) in enumerate(plan):
        q = rows[rng.integers(300, n, B)] + 0.01 * rng.standard_normal((B, d))
        if s == 2:
            q[0] = base                        # the uncertified one
        q /= np.linalg.norm(q, axis=1, keepdims=True)
        q = np.ascontiguousarray(q)
        out = (np.zeros((B, k), np.int64), np.zeros((B, k)), np.zeros(B, np.int32))
        batches.append((q, k, out))
        tickets.append(idx.submit_into(q, k, -1.0, *out))
    for (q, k, out), t in zip(batches, tickets):
        idx.wait_ticket(t)
        for j in range(q.shape[0]):
            want = ora.query(q[j], k, -1.0)
            assert out[0][j, :out[2][j]].tolist() == [c.id for c in want]
            np.testing.assert_allclose(out[1][j, :out[2][j]], [c.similarity for c in want], atol=1e-12)
    # synchronous path, same staging reused at another shape
    q, k, _ = batches[2]
    out = (np.zeros((q.shape[0], k), np.int64), np.zeros((q.shape[0], k)), np.zeros(q.shape[0], np.int32))
    idx.query_into(q, k, -1.0, *out)
    for j in range(q.shape[0]):
        want = ora.query(q[j], k, -1.0)
        assert out[0][j, :out[2][j]].tolist() == [c.id for c in want]
    assert idx.uncertified() >= 1


@pytest.mark.parametrize("scan", ["fp32", "bf16"])
def test_uncertified_rerun_answers_the_submit_time_snapshot(pkg, scan):
    """Snapshot-atomic answers (ref SPEC.md:183, index.py:98) when the
    certificate fails: the re-run in sine_query_wait scans the store as it
    was at SUBMISSION, although rows were removed (some from the answer,
    enough to trigger a compaction) and better rows inserted in between."""
    from paper_2509_17360_b200 import _native as N
    rng = np.random.default_rng(5)
    d, n, k = 256, 4000, 40
    base = rng.standard_normal(d)
    base /= np.linalg.norm(base)
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    for i in range(300):                       # the dense cluster that defeats the fast filter
        g = rows[i] - (rows[i] @ base) * base
        g /= np.linalg.norm(g)
        c = 0.999 - i * 2e-5
        rows[i] = c * base + np.sqrt(1 - c * c) * g
    ids = rng.permutation(10 * n)[:n] + 1
    idx = pkg.GpuCosineIndex(d, scan=scan, store_f32=True, store_bf16=True)
    idx.insert_batch(ids, rows)
    q = np.stack([base, rows[3000]])
    want = idx.query_batch(q, k, -1.0)         # synchronous: one consistent snapshot
    assert idx.uncertified() >= 1
    qh, oi, os_, oc = (N.PinnedArray((2, d), np.float64), N.PinnedArray((2, k), np.int64),
                       N.PinnedArray((2, k), np.float64), N.PinnedArray((2,), np.int32))
    qh.array[:] = q
    t = idx.submit_into(qh.array, k, -1.0, oi.array, os_.array, oc.array)
    gone = list(want[0][0, :10]) + [int(i) for i in ids[3200:4000] if i not in set(want[0].ravel().tolist())]
    idx.remove_batch(gone)                     # > live/4: a compaction is due (deferred)
    idx.insert_batch(10 * n + 1 + np.arange(5), np.tile(base, (5, 1)))  # similarity 1: would lead
    idx.wait_ticket(t)
    assert idx.uncertified() >= 1
    np.testing.assert_array_equal(oi.array, want[0])
    np.testing.assert_array_equal(os_.array, want[1])
    np.testing.assert_array_equal(oc.array, want[2])
    # the deferred compaction ran; the current state answers like the oracle
    ora = O.OracleExactIndex(d)
    keep = np.array([i not in set(gone) for i in ids.tolist()])
    ora.bulk_load(np.concatenate([ids[keep], 10 * n + 1 + np.arange(5)]),
                  np.concatenate([rows[keep], np.tile(base, (5, 1))]))
    got = idx.query_batch(q, k, -1.0)
    for j in range(2):
        assert got[0][j, :got[2][j]].tolist() == [c.id for c in ora.query(q[j], k, -1.0)]


def test_ids_and_snapshot_follow_the_reference_swap_last_order(pkg, tmp_path):
    """ids() and the snapshot file are byte-identical to the reference's
    ExactCosineIndex after removals (swap-last, index.py:80-92), one at a
    time and in batches, across compactions and later inserts."""
    rng = np.random.default_rng(12)
    d, n = 16, 600
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    ids = (rng.permutation(5 * n)[:n] + 3).tolist()
    idx = pkg.GpuCosineIndex(d, seed=9)
    ora = O.OracleExactIndex(d)
    for i, r in zip(ids, rows):
        ora.insert(i, r)
    idx.insert_batch(ids, rows)
    order = rng.permutation(n)
    for step, j in enumerate(order[:400]):     # one at a time, then in batches
        if step < 150:
            idx.remove(ids[j])
        ora.remove(ids[j])
    idx.remove_batch([ids[j] for j in order[150:400]])
    assert idx.ids() == ora.ids()
    extra = rng.standard_normal((7, d))
    extra /= np.linalg.norm(extra, axis=1, keepdims=True)
    for m, r in enumerate(extra):
        idx.insert(10_000 + m, r)
        ora.insert(10_000 + m, r)
    assert idx.ids() == ora.ids()
    want = ["exact-cosine-index", f"dimension: {d}", "seed: 9", f"count: {len(ora)}"] + \
        [f"{i} " + " ".join(float(c).hex() for c in ora.vectors[p]) for p, i in enumerate(ora.ids())]
    assert idx.snapshot_lines() == want
