"""Concurrent stage-1 queries against admissions, evictions and TTL purges
(ref SPEC.md:183: snapshot-atomic queries; ref engine.py:176-178 calls
`index.query` outside the engine lock).  Reader threads hammer `lookup`,
`lookup_batch` and the raw index while a writer admits at capacity
(evicting) and runs `evict_until_fits`; afterwards the engine's host tables
and the device store must agree exactly, and every answer a reader saw must
have been well formed (ids the engine handed out, similarities sorted
descending by (similarity, id), at or above the threshold)."""

from __future__ import annotations

import threading
import time

import numpy as np
import pytest

import gen_inputs as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2509_17360_b200 as P
    from paper_2509_17360_b200 import _native as N
    if N.device_count() < 1:
        pytest.skip("no CUDA device")
    return P


def _well_formed(cands, tau, next_id):
    """Sorted by (similarity desc, id asc), at or above tau, and every id one
    the engine has handed out (ids come from a monotone counter,
    engine.py:115, :328-329)."""
    sims = [c.similarity for c in cands]
    ids = [c.id for c in cands]
    order_ok = all((sims[i] > sims[i + 1]) or (sims[i] == sims[i + 1] and ids[i] < ids[i + 1])
                   for i in range(len(cands) - 1))
    return order_ok and all(s >= tau - 1e-12 for s in sims) and all(1 <= i < next_id for i in ids)


@pytest.mark.parametrize("scan", ["fp32", "bf16"])
def test_queries_concurrent_with_admit_and_evict(pkg, scan):
    emb = G.StubEmbedder(32, 1)
    judge = G.StubJudge()
    eng = pkg.CacheEngine(pkg.CacheConfig(capacity_tokens=6000, tau_sim=0.5, candidate_k=8), emb, judge, scan=scan)
    texts = [f"topic{t:02d} w{t % 5} item{i}" for t in range(40) for i in range(6)]

    def admit(j, now):
        text = texts[j % len(texts)] + f" v{j}"
        e = emb.embed(text)
        el = pkg.make_element(pkg.SemanticKey(text, "search"), "t " * (5 + j % 20), pkg.EmbeddingVector(e.components),
                              1 + j % 10, 400.0, 0.005, now, 50.0 if j % 7 == 0 else 5000.0)
        eng.admit(el, now)

    for j in range(300):
        admit(j, float(j) * 0.01)
    stop = threading.Event()
    errors, bad = [], []
    seen = [0]

    def reader(r):
        rng = np.random.default_rng(r)
        try:
            while not stop.is_set():
                key = pkg.SemanticKey(texts[int(rng.integers(len(texts)))] + " v1", "search")
                if r % 3 == 0:
                    eng.lookup(key, 100.0)
                elif r % 3 == 1:
                    eng.lookup_batch([key, pkg.SemanticKey("fresh query text", "search")], 100.0)
                else:
                    v = np.asarray(emb.embed(key.text).components)
                    cands = eng.index.query(v, 8, min_similarity=0.5)
                    ok = _well_formed(cands, 0.5, eng._next_id)
                    if not ok:
                        bad.append(cands)
                seen[0] += 1
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    threads = [threading.Thread(target=reader, args=(r,)) for r in range(6)]
    for t in threads:
        t.start()
    t_end = time.time() + 4.0
    j = 300
    now = 10.0
    while time.time() < t_end:
        admit(j, now)
        j += 1
        now += 0.5
        if j % 25 == 0:
            cap = eng.config.capacity_tokens
            eng.config.capacity_tokens = int(eng.usage_tokens * 0.8)
            eng.evict_until_fits(now)
            eng.config.capacity_tokens = cap
    stop.set()
    for t in threads:
        t.join()
    assert not errors, errors[:3]
    assert not bad, bad[:2]
    assert seen[0] > 50
    # host tables and the device store agree exactly
    els = eng.elements()
    assert set(els) == set(eng.index.ids())
    assert len(eng.index) == len(els)
    assert eng.usage_tokens == sum(el.size_tokens for el in els.values())
    assert eng.usage_tokens <= eng.config.capacity_tokens
