"""LCFU eviction + engine parity on the B200 against the reference's golden
outputs (tests/golden/evict_golden.json and engine_trace_golden.json).
Mirrors pkg/tests/test_engine.py and the eviction acceptance criteria."""

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


class _DimEmbedder:
    dimension = 8
    seed = 1


def _emb(pkg, dim, j):
    v = np.zeros(dim)
    v[j % dim] = 1.0
    return pkg.EmbeddingVector(tuple(float(x) for x in v))


def _mk(pkg, spec, j):
    return pkg.make_element(pkg.SemanticKey(f"k{j}", "search"), " ".join(["t"] * spec["size"]),
                            _emb(pkg, 8, j), spec["staticity"], spec["lat"], spec["cost"],
                            spec["created"], spec["ttl"], frequency=spec["freq"])


def test_engine_trials(pkg, evict_golden):
    # pkg/tests/test_engine.py:197-219 -- expired first, then the LCFU prefix
    for (specs, capacity), gold in zip(G.engine_trial_specs(), evict_golden["engine_trials"]):
        eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=1_000_000), _DimEmbedder(), None)
        for j, spec in enumerate(specs):
            eng.admit(_mk(pkg, spec, j))
        eng.config.capacity_tokens = capacity
        assert eng.evict_until_fits(1000.0) == gold["removed"]
        assert eng.usage_tokens <= capacity


def test_big_populations_all_policies(pkg, evict_golden):
    metas = {}
    for case in evict_golden["big"]:
        n, seed = case["n"], case["seed"]
        meta = metas.setdefault(seed, G.random_metadata(n, seed))
        eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10**9, eviction_policy=case["policy"]),
                              _DimEmbedder(), None)
        for j in range(n):
            spec = dict(size=int(meta["size"][j]), staticity=int(meta["staticity"][j]),
                        freq=int(meta["freq"][j]), lat=float(meta["lat"][j]), cost=float(meta["cost"][j]),
                        created=float(meta["created"][j]),
                        ttl=float(meta["expiration"][j] - meta["created"][j]))
            eng.admit(_mk(pkg, spec, j), now=float(meta["created"][j]))
        eng.config.capacity_tokens = case["capacity"]
        assert eng.evict_until_fits(12.0) == case["removed"], (seed, case["policy"], case["frac"])


def test_admit_stream_at_capacity(pkg, evict_golden):
    meta = G.random_metadata(400, 9)
    eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=2000), _DimEmbedder(), None)
    gold = evict_golden["admit_stream"]
    for j in range(400):
        spec = dict(size=int(meta["size"][j]), staticity=int(meta["staticity"][j]), freq=int(meta["freq"][j]),
                    lat=float(meta["lat"][j]), cost=float(meta["cost"][j]), created=float(j) * 0.5,
                    ttl=float(meta["expiration"][j] - meta["created"][j]))
        o = eng.admit(_mk(pkg, spec, j), now=float(j) * 0.5)
        assert [o.element_id, list(o.evicted_ids), o.replaced_id] == gold["results"][j], j
    assert eng.stats() == gold["stats"]


def test_protect_incoming_and_expired_first(pkg):
    # pkg/tests/test_engine.py:158-167 and :222-230
    eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=100), _DimEmbedder(), None)
    mk = lambda text, size, **kw: pkg.make_element(  # noqa: E731
        pkg.SemanticKey(text, "search"), " ".join(["r"] * size), _emb(pkg, 8, hash(text) % 8),
        kw.get("stat", 5), 400.0, 0.005, kw.get("now", 0.0), kw.get("ttl", 3600.0), frequency=kw.get("freq", 0))
    resident = eng.admit(mk("ridge basin", 60, freq=5, stat=9), now=0.0)
    out = eng.admit(mk("tempo sonata", 60), now=1.0)
    assert out.evicted_ids == (resident.element_id,)
    eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=1000), _DimEmbedder(), None)
    eng.admit(mk("ridge one", 10, freq=9, stat=9, ttl=5.0), now=0.0)
    keep = eng.admit(mk("tempo two", 10, freq=1), now=0.0)
    eng.config.capacity_tokens = 10
    assert eng.evict_until_fits(now=100.0) == [1]
    assert list(eng.elements()) == [keep.element_id]


def test_full_order_matches_oracle(pkg):
    """_victim_order_locked over everything (all three key kinds)."""
    rng = np.random.default_rng(17)
    meta = G.random_metadata(3000, 17, created_hi=50.0)
    for policy in ("lcfu", "lru", "lfu"):
        eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10**9, eviction_policy=policy), _DimEmbedder(),
                              None)
        oel, last = {}, {}
        for j in range(3000):
            spec = dict(size=int(meta["size"][j]), staticity=int(meta["staticity"][j]),
                        freq=int(meta["freq"][j]), lat=float(meta["lat"][j]), cost=float(meta["cost"][j]),
                        created=float(meta["created"][j]), ttl=2000.0)
            now = float(rng.integers(0, 100))
            o = eng.admit(_mk(pkg, spec, j), now=now)
            oel[o.element_id] = O.OracleElement(spec["staticity"], spec["freq"], spec["lat"], spec["cost"],
                                                spec["size"], spec["created"], spec["created"] + 2000.0)
            last[o.element_id] = now
        with eng._lock:
            got = eng._victim_order_locked(40.0)
        assert got == O.victim_order(oel, 40.0, policy, last)


@pytest.mark.parametrize("policy", ["lcfu", "lru", "lfu"])
def test_engine_trace_matches_reference(pkg, trace_golden, policy):
    """Mixed lookup / admit / evict trace: every outcome, the candidate
    counts, the similarities and the final stats equal the reference's."""
    emb = G.StubEmbedder(32, 1)
    judge = G.StubJudge()
    eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=400, eviction_policy=policy), emb, judge)
    log = []
    for op in G.engine_trace():
        if op[0] == "lookup":
            _, text, tool, now = op
            o = eng.lookup(pkg.SemanticKey(text, tool), now)
            log.append(["lookup", o.kind, o.element_id,
                        None if o.similarity is None else float(o.similarity).hex(),
                        None if o.s_lsm is None else float(o.s_lsm).hex(), o.candidates_considered, o.judged])
        elif op[0] == "admit":
            _, text, tool, now, spec = op
            e = emb.embed(text)
            el = pkg.make_element(pkg.SemanticKey(text, tool), spec["value"],
                                  pkg.EmbeddingVector(e.components), spec["staticity"], spec["lat"],
                                  spec["cost"], now, spec["ttl"], frequency=spec["freq"])
            o = eng.admit(el, now)
            log.append(["admit", o.element_id, list(o.evicted_ids), o.replaced_id])
        else:
            _, now = op
            cap = eng.config.capacity_tokens
            eng.config.capacity_tokens = max(1, int(eng.usage_tokens * 0.8))
            removed = eng.evict_until_fits(now)
            eng.config.capacity_tokens = cap
            log.append(["evict", removed])
    gold = trace_golden[policy]
    for i, (a, b) in enumerate(zip(log, gold["log"])):
        if a[0] == "lookup" and a[3] is not None:
            # similarities: fp64 re-rank vs BLAS -- equal to 1e-12
            assert a[:3] == b[:3] and a[4:] == b[4:], (i, a, b)
            assert float.fromhex(a[3]) == pytest.approx(float.fromhex(b[3]), abs=1e-12)
        else:
            assert a == b, (i, a, b)
    assert eng.stats() == gold["stats"]


def test_save_load_round_trip(pkg, tmp_path):
    emb = G.StubEmbedder(32, 1)
    judge = G.StubJudge()
    eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10_000), emb, judge)
    for i, text in enumerate(["topic01 w1 alpha", "topic02 w2 beta", "topic03 w3 gamma"]):
        e = emb.embed(text)
        eng.admit(pkg.make_element(pkg.SemanticKey(text, "search"), f"value {i}", pkg.EmbeddingVector(e.components),
                                   5, 400.0, 0.005, float(i), 3600.0), now=float(i))
    assert eng.lookup(pkg.SemanticKey("topic02 w2 beta", "search"), 5.0).hit
    p = str(tmp_path / "cache.state")
    eng.save(p)
    loaded = pkg.CacheEngine.load(p, eng.config, emb, judge)
    assert loaded.elements() == eng.elements()
    assert loaded.usage_tokens == eng.usage_tokens
    assert loaded.lookup(pkg.SemanticKey("topic01 w1 alpha", "search"), 6.0).hit
    out = loaded.admit(pkg.make_element(pkg.SemanticKey("topic09 w1 x", "search"), "fresh", pkg.EmbeddingVector(
        emb.embed("topic09 w1 x").components), 5, 400.0, 0.005, 7.0, 3600.0), now=7.0)
    assert out.element_id not in eng.elements()


def test_lookup_batch_matches_sequential_when_no_purge(pkg):
    emb = G.StubEmbedder(32, 1)
    judge = G.StubJudge()
    a = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10_000), emb, judge)
    b = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10_000), emb, judge)
    texts = [f"topic{t:02d} w{t % 3} {x}" for t in range(12) for x in ("alpha", "beta")]
    for i, text in enumerate(texts):
        e = emb.embed(text)
        for eng in (a, b):
            eng.admit(pkg.make_element(pkg.SemanticKey(text, "search"), f"v{i}", pkg.EmbeddingVector(e.components),
                                       5, 400.0, 0.005, 0.0, 3600.0), now=0.0)
    keys = [pkg.SemanticKey(f"topic{t:02d} w{(t + 1) % 3} {x}", "search") for t in range(12) for x in
            ("alpha", "gamma")]
    seq = [a.lookup(k, 1.0) for k in keys]
    bat = b.lookup_batch(keys, 1.0)
    for s, t in zip(seq, bat):
        assert (s.kind, s.element_id, s.similarity, s.candidates_considered, s.judged) == \
               (t.kind, t.element_id, t.similarity, t.candidates_considered, t.judged)
    assert a.stats() == b.stats()


def test_lookup_batch_with_gpu_embedder(pkg):
    """lookup_batch embeds all keys in one GpuHashedBagEmbedder.embed_batch
    call; outcomes equal sequential lookups through the same embedder."""
    emb = pkg.GpuHashedBagEmbedder(64, seed=3)
    judge = G.StubJudge()
    a = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10_000), emb, judge)
    b = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10_000), emb, judge)
    texts = [f"topic{t:02d} w{t % 3} {x}" for t in range(12) for x in ("alpha", "beta")]
    for i, text in enumerate(texts):
        e = emb.embed(text)
        for eng in (a, b):
            eng.admit(pkg.make_element(pkg.SemanticKey(text, "search"), f"v{i}", e, 5, 400.0, 0.005, 0.0, 3600.0),
                      now=0.0)
    keys = [pkg.SemanticKey(f"topic{t:02d} w{(t + 1) % 3} {x}", "search") for t in range(12) for x in
            ("alpha", "gamma")]
    seq = [a.lookup(k, 1.0) for k in keys]
    bat = b.lookup_batch(keys, 1.0)
    for s_, t in zip(seq, bat):
        assert (s_.kind, s_.element_id, s_.similarity, s_.candidates_considered, s_.judged) == \
               (t.kind, t.element_id, t.similarity, t.candidates_considered, t.judged)
        assert s_.query_embedding == t.query_embedding
    assert a.stats() == b.stats()


@pytest.mark.parametrize("shuffled", [False, True])
def test_large_purge_and_select_match_oracle(pkg, shuffled):
    """1M SEs, config-D metadata: the device purge (ascending ids) followed
    by the LCFU prefix at 0.9 x live usage equals the oracle's
    evict_until_fits -- ascending ids take the packed (primary, created)
    sort, shuffled ids the full 192-bit key sort."""
    import ctypes

    import torch

    import bench
    from paper_2509_17360_b200 import _native as N

    n = 1_000_000
    meta = bench.evict_metadata(n, seed=9)
    now = 1.0e4
    rng = np.random.default_rng(1)
    ids = rng.permutation(4 * n)[:n] + 1 if shuffled else np.arange(1, n + 1)
    cols = {"log_freq": bench._exact_log((meta["freq"] + 1).astype(np.float64)),
            "log_cost": bench._exact_log(meta["cost"] * 1000.0 + 1),
            "log_lat": bench._exact_log(meta["lat"] + 1),
            "log_stat": bench._exact_log((meta["staticity"] + 1).astype(float)),
            "frequency": meta["freq"], "size_tokens": meta["size"], "created_at": meta["created"],
            "expiration_time": meta["expiration"], "last_access": meta["created"]}
    rows = torch.zeros((n, 4), dtype=torch.float64, device="cuda")
    rows[:, 0] = 1.0
    idx = pkg.GpuCosineIndex(4, metadata=True, capacity=n)
    idx.insert_device(ids, rows.data_ptr(), meta=cols)
    live = (meta["expiration"] - now) > 0.0
    live_usage = int(meta["size"][live].sum())
    cap = int(0.9 * live_usage)
    out = np.empty(n, dtype=np.int64)
    cnt = ctypes.c_int64()
    p = N.ptr(out, ctypes.c_int64)
    N.check(idx._lib.sine_expired(idx.handle, now, 1, p, n, ctypes.byref(cnt)))
    expired = out[:cnt.value].copy()
    N.check(idx._lib.sine_select_victims(idx.handle, 0, now, live_usage - cap, p, n, ctypes.byref(cnt)))
    victims = out[:cnt.value].copy()
    want = O.evict_until_fits_np(ids, meta["freq"], meta["cost"], meta["lat"], meta["staticity"], meta["size"],
                                 meta["created"], meta["expiration"], now, cap)
    assert np.array_equal(np.concatenate([expired, victims]), want)
    assert len(idx) == n - expired.shape[0]


def test_lookup_batch_pipelined_micro_batches(pkg):
    """Micro-batched, overlapped stage-1 gives the same outcomes as one
    batch and as sequential lookups when nothing is purged."""
    emb = G.StubEmbedder(32, 1)
    judge = G.StubJudge()
    engines = [pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10_000), emb, judge) for _ in range(3)]
    texts = [f"topic{t:02d} w{t % 3} {x}" for t in range(20) for x in ("alpha", "beta")]
    for i, text in enumerate(texts):
        e = emb.embed(text)
        for eng in engines:
            eng.admit(pkg.make_element(pkg.SemanticKey(text, "search"), f"v{i}", pkg.EmbeddingVector(e.components),
                                       5, 400.0, 0.005, 0.0, 3600.0), now=0.0)
    keys = [pkg.SemanticKey(f"topic{t:02d} w{(t + 1) % 3} {x}", "search") for t in range(20) for x in
            ("alpha", "gamma", "beta")]
    seq = [engines[0].lookup(k, 1.0) for k in keys]
    one = engines[1].lookup_batch(keys, 1.0, micro_batch=1000)
    pip = engines[2].lookup_batch(keys, 1.0, micro_batch=7)
    for a, b, c in zip(seq, one, pip):
        assert (a.kind, a.element_id, a.similarity, a.candidates_considered, a.judged) == \
               (b.kind, b.element_id, b.similarity, b.candidates_considered, b.judged) == \
               (c.kind, c.element_id, c.similarity, c.candidates_considered, c.judged)
    assert engines[0].stats() == engines[1].stats() == engines[2].stats()


def test_async_queries_in_flight_and_ttl_daemon(pkg):
    import time as _t
    rng = np.random.default_rng(4)
    d, n = 64, 5000
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    idx = pkg.GpuCosineIndex(d)
    idx.insert_batch(np.arange(n), rows)
    qs = [rows[rng.integers(0, n, 9)] for _ in range(5)]
    pend = [idx.query_batch_async(q, 6, 0.2) for q in qs]      # five batches in flight
    for q, p in zip(qs, reversed(pend[::-1])):
        want = idx.query_batch(q, 6, 0.2)
        got = p.wait()
        for x, y in zip(got, want):
            np.testing.assert_array_equal(x, y)
    # background TTL purge
    eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=10_000), _DimEmbedder(), None)
    for j in range(20):
        spec = dict(size=3, staticity=5, freq=1, lat=50.0, cost=0.005, created=0.0, ttl=5.0 if j % 2 else 1e9)
        eng.admit(_mk(pkg, spec, j), now=0.0)
    stop = eng.start_ttl_maintenance(0.01, clock=lambda: 100.0)
    deadline = _t.time() + 10
    while len(eng) > 10 and _t.time() < deadline:
        _t.sleep(0.02)
    stop.set()
    assert len(eng) == 10 and eng.stats()["expirations"] == 10
