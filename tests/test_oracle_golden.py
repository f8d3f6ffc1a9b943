"""Pin the CPU oracle to the reference: every golden vector the reference
produced (tests/golden/make_golden.py) must be reproduced by oracle/."""

from __future__ import annotations

import math

import numpy as np
import pytest

import gen_inputs as G
from oracle import sine_oracle as O


def _check(got, want, tol=1e-12):
    assert [c.id for c in got] == [w[0] for w in want]
    for c, w in zip(got, want):
        assert c.similarity == pytest.approx(float.fromhex(w[1]), abs=tol)


def test_linear_trials(index_golden):
    for (dim, vectors, queries), gold in zip(G.linear_oracle_trials(),
                                             index_golden["linear_trials"]):
        assert G.digest(list(vectors.values())) == gold["digest"]
        idx = O.OracleExactIndex(dim)
        for i, v in vectors.items():
            idx.insert(i, v)
        for (q, k, ms), want in zip(queries, gold["results"]):
            _check(idx.query(q, k, min_similarity=ms), want)


def test_tie_order_and_validation(index_golden):
    v = G.normalize([1, 2, 3, 4, 5, 6, 7, 8])
    idx = O.OracleExactIndex(8)
    for i in (9, 3, 7, 1):
        idx.insert(i, v)
    _check(idx.query(v, 4), index_golden["tie_order"])
    val = index_golden["validation"]
    idx = O.OracleExactIndex(4)
    for name, fn in [
        ("wrong_dim", lambda: idx.insert(1, G.normalize([1, 2, 3]))),
        ("not_normalized", lambda: idx.insert(1, [1.0, 2.0, 3.0, 4.0])),
        ("k_zero", lambda: idx.query(G.normalize([1, 0, 0, 0]), k=0)),
        ("unknown_remove", lambda: idx.remove(42)),
    ]:
        assert val[name] == "ValidationError"
        with pytest.raises(O.OracleValidationError):
            fn()
    assert idx.query(G.normalize([1, 0, 0, 0]), k=3) == [] == val["empty_query"]


def test_remove_steps(index_golden):
    dim, vectors, steps = G.remove_case()
    idx = O.OracleExactIndex(dim)
    for i, v in vectors.items():
        idx.insert(i, v)
    for (i, q), gold in zip(steps, index_golden["remove_steps"]):
        idx.remove(i)
        _check(idx.query(q, 10), gold["result"])
        assert idx.ids() == gold["ids"]


def test_acceptance_9b(index_golden):
    dim, stored, queries = G.acceptance_9b_case()
    gold = index_golden["acceptance_9b"]
    assert G.digest(list(stored.values())) == gold["digest"]
    idx = O.OracleExactIndex(dim)
    idx.bulk_load(list(stored), np.asarray(list(stored.values())))
    for q, want in zip(queries, gold["results"]):
        _check(idx.query(q, 7), want)


def test_config_a(index_golden):
    rows, qs = G.config_a()
    gold = index_golden["config_a"]
    assert G.digest(rows, qs) == gold["digest"]
    idx = O.OracleExactIndex(rows.shape[1])
    idx.bulk_load(range(rows.shape[0]), rows)
    hits = 0
    for ms in (0.9, -1.0):
        for q, want in zip(qs, gold["results"][repr(ms)]):
            got = idx.query(q, 5, min_similarity=ms)
            _check(got, want)
            hits += bool(got) and ms == 0.9
    assert 200 < hits < 800  # 1k queries: the planted near-duplicates straddle tau_sim


def test_ties(index_golden):
    d, rows, ids, qs = G.tie_rows()
    gold = index_golden["ties"]
    assert G.digest(rows) == gold["digest"]
    idx = O.OracleExactIndex(d)
    idx.bulk_load(ids, rows)
    for k, res in gold["results"].items():
        for q, want in zip(qs, res):
            _check(idx.query(q, int(k)), want)


# ------------------------------------------------------------------ LCFU

def test_cal_score_frozen_and_grid(evict_golden):
    got = O.cal_score(2, 0.005, 400.0, 8, 512, 600.0, 10.0)
    assert got == float.fromhex(evict_golden["cal_score_frozen"]) == 0.05063404135640259
    grid = evict_golden["cal_score_grid"]
    f = np.array([g[0] for g in grid])
    c = np.array([float.fromhex(g[1]) for g in grid])
    lat = np.array([float.fromhex(g[2]) for g in grid])
    s = np.array([g[3] for g in grid])
    size = np.array([g[4] for g in grid])
    want = np.array([float.fromhex(g[5]) for g in grid])
    scalar = np.array([O.cal_score(int(a), b, cc, int(d), int(e), 100.0, 5.0)
                       for a, b, cc, d, e in zip(f, c, lat, s, size)])
    vec = O.lcfu_scores_np(f, c, lat, s, size, np.full(len(f), 100.0), 5.0)
    assert np.array_equal(scalar.view(np.int64), want.view(np.int64))
    assert np.array_equal(vec.view(np.int64), want.view(np.int64))


def _elements_from_specs(specs):
    els = {}
    for j, sp in enumerate(specs):
        els[j + 1] = O.OracleElement(sp["staticity"], sp["freq"], sp["lat"], sp["cost"],
                                     sp["size"], sp["created"], sp["created"] + sp["ttl"])
    return els


def test_engine_trials(evict_golden):
    for (specs, capacity), gold in zip(G.engine_trial_specs(), evict_golden["engine_trials"]):
        assert capacity == gold["capacity"]
        els = _elements_from_specs(specs)
        assert O.evict_until_fits(els, 1000.0, capacity) == gold["removed"]


def _big_elements(meta, n):
    els, last = {}, {}
    for j in range(n):
        els[j + 1] = O.OracleElement(int(meta["staticity"][j]), int(meta["freq"][j]),
                                     float(meta["lat"][j]), float(meta["cost"][j]),
                                     int(meta["size"][j]), float(meta["created"][j]),
                                     float(meta["expiration"][j]))
        last[j + 1] = float(meta["created"][j])
    return els, last


def test_big_populations(evict_golden):
    metas = {}
    for case in evict_golden["big"]:
        n, seed = case["n"], case["seed"]
        if seed not in metas:
            metas[seed] = G.random_metadata(n, seed)
        meta = metas[seed]
        els, last = _big_elements(meta, n)
        got = O.evict_until_fits(els, 12.0, case["capacity"], case["policy"], last)
        assert got == case["removed"], (seed, case["policy"], case["frac"])
        if case["policy"] == "lcfu":
            vec = O.evict_until_fits_np(np.arange(1, n + 1), meta["freq"], meta["cost"],
                                        meta["lat"], meta["staticity"], meta["size"],
                                        meta["created"], meta["expiration"], 12.0,
                                        case["capacity"])
            assert vec.tolist() == case["removed"]


def test_admit_stream(evict_golden):
    meta = G.random_metadata(400, 9)
    gold = evict_golden["admit_stream"]
    els, nid = {}, 1
    evictions = expirations = 0
    for j in range(400):
        now = j * 0.5
        el = O.OracleElement(int(meta["staticity"][j]), int(meta["freq"][j]),
                             float(meta["lat"][j]), float(meta["cost"][j]),
                             int(meta["size"][j]), now,
                             now + float(meta["expiration"][j] - meta["created"][j]))
        exp, victims = O.admit_victims(els, now, 2000, el.size_tokens)
        for eid in exp + victims:
            del els[eid]
        evictions += len(victims)
        expirations += len(exp)
        assert [nid, victims, None] == gold["results"][j]
        els[nid] = el
        nid += 1
    st = gold["stats"]
    assert st["evictions"] == evictions and st["expirations"] == expirations
    assert st["usage_tokens"] == sum(e.size_tokens for e in els.values())
    assert st["element_count"] == len(els)


def test_log_base_invariance_restated():
    # pkg/tests/test_engine.py:52-61 restated on the oracle
    for f in range(0, 10):
        a = O.cal_score(f, 0.005, 400.0, 7, 13, 10.0, 0.0)
        b = O.cal_score(f, 0.005, 400.0, 7, 13, 10.0, 0.0, log=math.log10)
        assert a == pytest.approx(b * math.log(10) ** 4, rel=1e-9)


def test_oracle_embedder_matches_reference_goldens():
    """The oracle's HashedBagEmbedder restatement equals the reference's
    vectors (embed_golden.json, produced by the reference)."""
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "embed_golden.json"), encoding="utf-8"))
    for case in gold["cases"]:
        for text, want in zip(gold["texts"], case["vectors"]):
            got = O.hashed_bag_embed(text, case["dimension"], case["seed"])
            dense = [0.0] * case["dimension"]
            for i, h in want:
                dense[i] = float.fromhex(h)
            assert list(got) == dense
