"""Single-process multi-GPU drop-in (`MultiDeviceCosineIndex`, csrc/group.cu)
against the oracle: the per-shard exact top-k lists merged on the root
device must equal one ExactCosineIndex.query over the union (ref
index.py:94-102; ids bit-exact, similarities within 1e-12), including ties
that straddle shards (identical rows under different ids, decided by id).
Shards here share cuda:0 (the box has one GPU); distinct devices take the
same code path with peer copies instead of device copies.  The reference's
own single-process engine runs unchanged on top of it."""

from __future__ import annotations

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


def _unit(rng, n, d):
    x = rng.standard_normal((n, d))
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def _check(idx, ora, Q, k, tau):
    ids, sims, counts = idx.query_batch(Q, k, tau)
    for b in range(Q.shape[0]):
        want = ora.query(Q[b], k, min_similarity=tau)
        got_ids = ids[b, :counts[b]].tolist()
        assert got_ids == [c.id for c in want], (b, got_ids, [c.id for c in want])
        assert np.allclose(sims[b, :counts[b]], [c.similarity for c in want], rtol=0, atol=1e-12)


@pytest.mark.parametrize("shards", [2, 3])
@pytest.mark.parametrize("scan", ["fp32", "bf16"])
def test_multidev_equals_oracle(pkg, shards, scan):
    rng = np.random.default_rng(100 + shards)
    n, d = 20_000, 128
    X = _unit(rng, n, d)
    X[n // 2:n // 2 + 64] = X[:64]  # identical rows under other ids: cross-shard ties
    ids = rng.permutation(5 * n)[:n] + 1
    idx = pkg.MultiDeviceCosineIndex(d, devices=[0] * shards, scan=scan)
    ora = O.OracleExactIndex(d, capacity=n)
    idx.insert_batch(ids[:n // 2], X[:n // 2])
    idx.insert_batch(ids[n // 2:], X[n // 2:])
    ora.bulk_load(ids, X)
    assert len(idx) == n and idx.ids() == ora.ids()
    Q = np.concatenate([X[:8], _unit(rng, 24, d)])
    noisy = X[100:132] + 0.02 * rng.standard_normal((32, d))
    Q = np.concatenate([Q, noisy / np.linalg.norm(noisy, axis=1, keepdims=True)])
    for k, tau in ((1, -1.0), (5, 0.9), (20, -1.0), (64, 0.5)):
        _check(idx, ora, Q, k, tau)
    for i in range(4):  # B = 1 through the reference-shaped call
        got = idx.query(Q[i], 10, min_similarity=-1.0)
        want = ora.query(Q[i], 10, min_similarity=-1.0)
        assert [c.id for c in got] == [c.id for c in want]
    # removals (swap-last order), re-query, snapshot identical to one handle's
    gone = rng.choice(ids, 500, replace=False)
    idx.remove_batch(gone)
    for i in gone:
        ora.remove(int(i))
    assert idx.ids() == ora.ids()
    _check(idx, ora, Q, 10, -1.0)
    single = pkg.GpuCosineIndex(d)
    single.insert_batch(ids[:n // 2], X[:n // 2])
    single.insert_batch(ids[n // 2:], X[n // 2:])
    single.remove_batch(gone)
    assert idx.snapshot_lines() == single.snapshot_lines()
    with pytest.raises(pkg.ValidationError):
        idx.remove(int(gone[0]))
    with pytest.raises(pkg.ValidationError):
        idx.insert(int(ids[0]), X[0])
    idx.close()


def test_multidev_empty_shard_and_save_load(pkg, tmp_path):
    d = 16
    rng = np.random.default_rng(7)
    X = _unit(rng, 3, d)
    idx = pkg.MultiDeviceCosineIndex(d, devices=[0, 0, 0, 0])  # more shards than rows
    assert idx.query(X[0], 3) == []
    idx.insert_batch([5, 6, 7], X)
    got = idx.query(X[1], 5)
    assert got[0].id == 6 and len(got) == 3
    p = str(tmp_path / "multi.snap")
    idx.save(p)
    back = pkg.MultiDeviceCosineIndex.load(p, devices=[0, 0])
    assert back.ids() == [5, 6, 7] and back.snapshot_lines() == idx.snapshot_lines()


def test_reference_engine_on_multidev(pkg, trace_golden):
    """The reference's own CacheEngine (semcache, when importable) with the
    multi-device index injected reproduces the golden engine trace that the
    reference produced with ExactCosineIndex."""
    import os
    import sys

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import semcache.engine as RE
        import semcache.model as RM
    except Exception:  # noqa: BLE001
        pytest.skip("semcache (oracle/_ref) not importable")
    emb = G.StubEmbedder(32, 1)
    judge = G.StubJudge()
    eng = RE.CacheEngine(RM.CacheConfig(capacity_tokens=400, eviction_policy="lcfu"), emb, judge,
                         index=pkg.MultiDeviceCosineIndex(32, devices=[0, 0]))
    log = []
    for op in G.engine_trace():
        if op[0] == "lookup":
            _, text, tool, now = op
            o = eng.lookup(RM.SemanticKey(text, tool), now)
            log.append(["lookup", o.kind, o.element_id,
                        None if o.similarity is None else float(o.similarity).hex(),
                        None if o.s_lsm is None else float(o.s_lsm).hex(), o.candidates_considered, o.judged])
        elif op[0] == "admit":
            _, text, tool, now, spec = op
            e = emb.embed(text)
            el = RM.make_element(RM.SemanticKey(text, tool), spec["value"], RM.EmbeddingVector(e.components),
                                 spec["staticity"], spec["lat"], spec["cost"], now, spec["ttl"],
                                 frequency=spec["freq"])
            o = eng.admit(el, now)
            log.append(["admit", o.element_id, list(o.evicted_ids), o.replaced_id])
        else:
            _, now = op
            cap = eng.config.capacity_tokens
            eng.config.capacity_tokens = max(1, int(eng.usage_tokens * 0.8))
            log.append(["evict", eng.evict_until_fits(now)])
            eng.config.capacity_tokens = cap
    gold = trace_golden["lcfu"]
    for i, (a, b) in enumerate(zip(log, gold["log"])):
        if a[0] == "lookup" and a[3] is not None:
            assert a[:3] == b[:3] and a[4:] == b[4:], (i, a, b)
            assert float.fromhex(a[3]) == pytest.approx(float.fromhex(b[3]), abs=1e-12)
        else:
            assert a == b, (i, a, b)
    assert eng.stats() == gold["stats"]
