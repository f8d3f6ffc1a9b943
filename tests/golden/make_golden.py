"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where the read-only reference is importable):

    python tests/golden/make_golden.py

It imports `semcache` from `/root/reference/pkg/src` (or `baseline/_ref`),
feeds it the inputs from `gen_inputs.py`, and writes the reference's
outputs as JSON (floats as `float.hex` so they are bit-exact).  The GPU box
never runs this script; the tests only read the JSON it wrote.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
for cand in ("/root/reference/pkg/src",
             os.path.join(HERE, "..", "..", "baseline", "_ref")):
    if os.path.isdir(os.path.join(cand, "semcache")):
        sys.path.insert(0, cand)
        break

import gen_inputs as G  # noqa: E402
from semcache.engine import CacheEngine, cal_score  # noqa: E402
from semcache.errors import ValidationError  # noqa: E402
from semcache.index import ExactCosineIndex  # noqa: E402
from semcache.model import CacheConfig, EmbeddingVector, SemanticKey, make_element  # noqa: E402


def hx(x: float) -> str:
    return float(x).hex()


def cands(lst):
    return [[c.id, hx(c.similarity)] for c in lst]


def direct_index(dim, ids, rows):
    idx = ExactCosineIndex(dim)
    idx._ids = list(int(i) for i in ids)
    idx._pos = {int(i): j for j, i in enumerate(ids)}
    idx._vecs = np.ascontiguousarray(rows, dtype=np.float64)
    return idx


def index_golden():
    out = {}
    # linear-oracle trials (pkg/tests/test_index.py:52-69)
    trials = []
    for dim, vectors, queries in G.linear_oracle_trials():
        idx = ExactCosineIndex(dim)
        for i, v in vectors.items():
            idx.insert(i, v)
        res = [cands(idx.query(q, k=k, min_similarity=ms)) for q, k, ms in queries]
        trials.append(dict(dim=dim, n=len(vectors),
                           digest=G.digest(list(vectors.values())), results=res))
    out["linear_trials"] = trials

    # tie order (pkg/tests/test_index.py:72-79)
    v = G.normalize([1, 2, 3, 4, 5, 6, 7, 8])
    idx = ExactCosineIndex(8)
    for i in (9, 3, 7, 1):
        idx.insert(i, v)
    out["tie_order"] = cands(idx.query(v, k=4))

    # removal (pkg/tests/test_index.py:82-100)
    dim, vectors, steps = G.remove_case()
    idx = ExactCosineIndex(dim)
    for i, vv in vectors.items():
        idx.insert(i, vv)
    rem = []
    for i, q in steps:
        idx.remove(i)
        rem.append(dict(removed=i, result=cands(idx.query(q, k=10)), ids=idx.ids()))
    out["remove_steps"] = rem

    # acceptance 9b
    dim, stored, queries = G.acceptance_9b_case()
    idx = ExactCosineIndex(dim, seed=3)
    for i, vv in stored.items():
        idx.insert(i, vv)
    out["acceptance_9b"] = dict(digest=G.digest(list(stored.values())),
                                results=[cands(idx.query(q, 7)) for q in queries])

    # config A (10k x 384), k=5, tau 0.9 and -1
    rows, qs = G.config_a()
    idx = direct_index(rows.shape[1], range(rows.shape[0]), rows)
    res = {}
    for ms in (0.9, -1.0):
        res[repr(ms)] = [cands(idx.query(q, 5, min_similarity=ms)) for q in qs]
    out["config_a"] = dict(digest=G.digest(rows, qs), results=res)

    # ties under shuffled ids
    d, trows, tids, tq = G.tie_rows()
    idx = direct_index(d, tids, trows)
    out["ties"] = dict(digest=G.digest(trows),
                       results={str(k): [cands(idx.query(q, k)) for q in tq]
                                for k in (1, 5, 40, 100)})

    # validation behaviour of the reference (message classes only)
    idx = ExactCosineIndex(4)
    checks = {}
    for name, fn in [
        ("wrong_dim", lambda: idx.insert(1, G.normalize([1, 2, 3]))),
        ("not_normalized", lambda: idx.insert(1, [1.0, 2.0, 3.0, 4.0])),
        ("k_zero", lambda: idx.query(G.normalize([1, 0, 0, 0]), k=0)),
        ("unknown_remove", lambda: idx.remove(42)),
    ]:
        try:
            fn()
            checks[name] = "ok"
        except ValidationError:
            checks[name] = "ValidationError"
    checks["empty_query"] = cands(ExactCosineIndex(4).query(G.normalize([1, 0, 0, 0]), k=3))
    out["validation"] = checks
    return out


class _DimEmbedder:
    def __init__(self, dim=8):
        self.dimension = dim
        self.seed = 1


def _emb(dim, j):
    v = np.zeros(dim)
    v[j % dim] = 1.0
    return EmbeddingVector(tuple(float(x) for x in v))


def _mk(spec, j, dim=8):
    return make_element(SemanticKey(f"k{j}", "search"), " ".join(["t"] * spec["size"]),
                        _emb(dim, j), spec["staticity"], spec["lat"], spec["cost"],
                        spec["created"], spec["ttl"], frequency=spec["freq"])


def evict_golden():
    out = {}
    # frozen cal_score (pkg/tests/test_engine.py:33-41)
    el = make_element(SemanticKey("q text", "search"), " ".join(["tok"] * 512),
                      _emb(8, 0), 8, 400.0, 0.005, 0.0, 600.0, frequency=2)
    out["cal_score_frozen"] = hx(cal_score(el, now=10.0))

    # a grid of cal_score values (exactness of the restated arithmetic)
    grid = []
    for f in range(0, 9):
        for c in (0.0, 0.0005, 0.005, 0.0077, 0.02, 1.5):
            for lat in (0.0, 50.0, 400.0, 1500.0, 0.1):
                for s in (1, 5, 10):
                    for size in (1, 7, 512):
                        el = make_element(SemanticKey("a", "b"), " ".join(["t"] * size),
                                          _emb(8, 0), s, lat, c, 0.0, 100.0, frequency=f)
                        grid.append([f, hx(c), hx(lat), s, size, hx(cal_score(el, 5.0))])
    out["cal_score_grid"] = grid

    # engine eviction trials (pkg/tests/test_engine.py:197-219)
    trials = []
    for specs, capacity in G.engine_trial_specs():
        eng = CacheEngine(CacheConfig(capacity_tokens=1_000_000), _DimEmbedder(), None)
        for j, spec in enumerate(specs):
            eng.admit(_mk(spec, j))
        eng.config.capacity_tokens = capacity
        removed = eng.evict_until_fits(1000.0)
        trials.append(dict(capacity=capacity, removed=removed))
    out["engine_trials"] = trials

    # larger populations, all three policies, several capacities, plus admits
    big = []
    for seed, n in ((1, 300), (2, 2000)):
        meta = G.random_metadata(n, seed)
        for policy in ("lcfu", "lru", "lfu"):
            for frac in (0.9, 0.5, 0.1):
                eng = CacheEngine(CacheConfig(capacity_tokens=10**9, eviction_policy=policy),
                                  _DimEmbedder(), None)
                for j in range(n):
                    spec = dict(size=int(meta["size"][j]), staticity=int(meta["staticity"][j]),
                                freq=int(meta["freq"][j]), lat=float(meta["lat"][j]),
                                cost=float(meta["cost"][j]), created=float(meta["created"][j]),
                                ttl=float(meta["expiration"][j] - meta["created"][j]))
                    eng.admit(_mk(spec, j), now=float(meta["created"][j]))
                usage = eng.usage_tokens
                eng.config.capacity_tokens = max(1, int(usage * frac))
                removed = eng.evict_until_fits(12.0)
                big.append(dict(seed=seed, n=n, policy=policy, frac=frac,
                                capacity=eng.config.capacity_tokens, removed=removed))
    out["big"] = big

    # admission stream at capacity (engine.py:300-336)
    meta = G.random_metadata(400, 9)
    eng = CacheEngine(CacheConfig(capacity_tokens=2000), _DimEmbedder(), None)
    adm = []
    for j in range(400):
        spec = dict(size=int(meta["size"][j]), staticity=int(meta["staticity"][j]),
                    freq=int(meta["freq"][j]), lat=float(meta["lat"][j]),
                    cost=float(meta["cost"][j]), created=float(j) * 0.5,
                    ttl=float(meta["expiration"][j] - meta["created"][j]))
        o = eng.admit(_mk(spec, j), now=float(j) * 0.5)
        adm.append([o.element_id, list(o.evicted_ids), o.replaced_id])
    out["admit_stream"] = dict(results=adm, stats=eng.stats())
    return out


def engine_trace_golden():
    out = {}
    for policy in ("lcfu", "lru", "lfu"):
        emb = G.StubEmbedder(32, 1)
        judge = G.StubJudge()
        cfg = CacheConfig(capacity_tokens=400, eviction_policy=policy)
        eng = CacheEngine(cfg, emb, judge)
        log = []
        for op in G.engine_trace():
            if op[0] == "lookup":
                _, text, tool, now = op
                o = eng.lookup(SemanticKey(text, tool), now)
                log.append(["lookup", o.kind, o.element_id,
                            None if o.similarity is None else hx(o.similarity),
                            None if o.s_lsm is None else hx(o.s_lsm),
                            o.candidates_considered, o.judged])
            elif op[0] == "admit":
                _, text, tool, now, spec = op
                e = emb.embed(text)
                el = make_element(SemanticKey(text, tool), spec["value"],
                                  EmbeddingVector(e.components), spec["staticity"],
                                  spec["lat"], spec["cost"], now, spec["ttl"],
                                  frequency=spec["freq"])
                o = eng.admit(el, now)
                log.append(["admit", o.element_id, list(o.evicted_ids), o.replaced_id])
            else:
                _, now = op
                cap = eng.config.capacity_tokens
                eng.config.capacity_tokens = max(1, int(eng.usage_tokens * 0.8))
                removed = eng.evict_until_fits(now)
                eng.config.capacity_tokens = cap
                log.append(["evict", removed])
        out[policy] = dict(log=log, stats=eng.stats())
    return out


def main():
    for name, fn in (("index_golden.json", index_golden),
                     ("evict_golden.json", evict_golden),
                     ("engine_trace_golden.json", engine_trace_golden)):
        data = fn()
        with open(os.path.join(HERE, name), "w") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print("wrote", name, os.path.getsize(os.path.join(HERE, name)), "bytes")


if __name__ == "__main__":
    main()
