"""Deterministic input generators shared by `make_golden.py` (which runs the
reference here to produce the expected outputs) and the tests (which
regenerate the same inputs on the GPU box and compare).

Nothing here imports the reference or the product package.
"""

from __future__ import annotations

import hashlib
import math
import zlib
from random import Random

import numpy as np


def normalize(vals):
    norm = math.sqrt(sum(v * v for v in vals))
    return [v / norm for v in vals]


def random_unit(rng: Random, dim: int):
    # same draw order as pkg/tests/test_index.py:21-22
    return normalize([rng.gauss(0, 1) for _ in range(dim)])


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes())
    return h.hexdigest()[:16]


# ------------------------------------------------------------ index cases

def linear_oracle_trials():
    """pkg/tests/test_index.py:52-69 (Random(1201), 6 trials x 20 queries)."""
    rng = Random(1201)
    trials = []
    for _ in range(6):
        dim = rng.choice([8, 16, 32])
        n = rng.randrange(50, 300)
        vectors = {i: random_unit(rng, dim) for i in range(n)}
        queries = []
        for _ in range(20):
            q = random_unit(rng, dim)
            k = rng.randrange(1, 12)
            min_sim = rng.choice([-1.0, 0.0, 0.2, 0.5])
            queries.append((q, k, min_sim))
        trials.append((dim, vectors, queries))
    return trials


def acceptance_9b_case():
    """pkg/tests/test_acceptance.py:293-315 (Random(1234), 1k x 64, 50 q, k=7)."""
    rng2 = Random(1234)
    small_dim = 64

    def unit2():
        v = np.array([rng2.gauss(0.0, 1.0) for _ in range(small_dim)])
        return (v / np.linalg.norm(v)).tolist()

    stored = {i: unit2() for i in range(1000)}
    queries = [unit2() for _ in range(50)]
    return small_dim, stored, queries


def remove_case():
    """pkg/tests/test_index.py:82-100 (Random(88))."""
    rng = Random(88)
    dim = 8
    vectors = {i: random_unit(rng, dim) for i in range(40)}
    steps = []
    for i in (0, 17, 39, 5, 22):
        steps.append((i, random_unit(rng, dim)))
    return dim, vectors, steps


def planted_rows(n: int, d: int, seed: int) -> np.ndarray:
    """Unit rows, standard-normal then float64-normalised."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x


def planted_queries(rows: np.ndarray, b: int, seed: int, dup_frac: float = 0.5):
    """Config-A queries: half are near-duplicates normalize(X[i] + s*g) with
    i ~ Zipf(0.99) over rows and s chosen so cos lands in [0.88, 0.99]
    (straddling tau_sim = 0.9); the rest are fresh random unit vectors."""
    n, d = rows.shape
    rng = np.random.default_rng(seed)
    ranks = np.arange(1, n + 1, dtype=np.float64)
    p = ranks ** -0.99
    p /= p.sum()
    q = rng.standard_normal((b, d))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    is_dup = rng.random(b) < dup_frac
    src = rng.choice(n, size=b, p=p)
    target_cos = rng.uniform(0.88, 0.99, size=b)
    for j in np.nonzero(is_dup)[0]:
        x = rows[src[j]]
        g = rng.standard_normal(d)
        g -= (g @ x) * x
        g /= np.linalg.norm(g)
        c = target_cos[j]
        v = c * x + math.sqrt(max(0.0, 1 - c * c)) * g
        q[j] = v / np.linalg.norm(v)
    return q


def config_a(n=10_000, d=384, b=1000, seed=7):
    rows = planted_rows(n, d, seed)
    q = planted_queries(rows, b, seed + 1)
    return rows, q


def tie_rows(seed=3):
    """Many identical rows under shuffled ids plus random rows (ties are the
    common case with hashed-bag paraphrases, pkg/tests/test_traces.py:35-40)."""
    rng = np.random.default_rng(seed)
    d = 24
    base = rng.standard_normal((4, d))
    base /= np.linalg.norm(base, axis=1, keepdims=True)
    rows, ids = [], []
    id_pool = list(rng.permutation(5000)[:400] + 10)
    for j in range(400):
        if j % 3 == 0:
            rows.append(base[j % 4])
        else:
            v = rng.standard_normal(d)
            rows.append(v / np.linalg.norm(v))
        ids.append(int(id_pool[j]))
    queries = [base[0], base[1], base[2], base[3]]
    return d, np.asarray(rows), ids, np.asarray(queries)


# ---------------------------------------------------------- eviction cases

def engine_trial_specs():
    """pkg/tests/test_engine.py:197-219 (Random(9192), 12 trials)."""
    rng = Random(9192)
    trials = []
    for _ in range(12):
        n = rng.randrange(10, 40)
        els = []
        for i in range(n):
            ttl = rng.choice([10.0, 10.0, 10.0, 2000.0])
            created = rng.choice([0.0, 1.0, 2.0, 3.0])
            size = rng.randrange(1, 30)
            staticity = rng.randrange(1, 11)
            freq = rng.randrange(0, 8)
            lat = rng.choice([50.0, 400.0, 1500.0])
            cost = rng.choice([0.0, 0.0005, 0.005, 0.02])
            els.append(dict(size=size, staticity=staticity, freq=freq, lat=lat,
                            cost=cost, created=created, ttl=ttl))
        usage = sum(e["size"] for e in els)
        target = rng.randrange(0, usage + 1)
        trials.append((els, max(1, target)))
    return trials


def random_metadata(n: int, seed: int, short_ttl_frac: float = 1 / 7,
                    created_hi: float = 4.0):
    """Config-A/D metadata."""
    rng = np.random.default_rng(seed)
    meta = dict(
        staticity=rng.integers(1, 11, n),
        freq=rng.integers(0, 8, n),
        lat=rng.choice(np.array([50.0, 400.0, 1500.0]), n),
        cost=rng.choice(np.array([0.0, 0.0005, 0.005, 0.02]), n),
        size=rng.integers(1, 30, n),
        created=np.floor(rng.random(n) * created_hi),
    )
    ttl = np.where(rng.random(n) < short_ttl_frac, 10.0, 2000.0)
    meta["expiration"] = meta["created"] + ttl
    return meta


# ------------------------------------------------------- engine trace stubs

class StubEmbedder:
    """Deterministic text -> unit vector (seeded by crc32 of the topic word).

    Texts of the form "<topic> <variant...>" embed to a vector near the
    topic's anchor, so paraphrases share candidates while other topics do
    not.  Used on both sides of the engine-trace golden (reference engine
    here, GPU engine on the box)."""

    def __init__(self, dimension: int = 32, seed: int = 1):
        self.dimension = dimension
        self.seed = seed

    def embed(self, text: str):
        words = text.split()
        topic = words[0]
        rng = np.random.default_rng(zlib.crc32(topic.encode()) + self.seed)
        anchor = rng.standard_normal(self.dimension)
        anchor /= np.linalg.norm(anchor)
        rest = " ".join(words[1:])
        rng2 = np.random.default_rng(zlib.crc32(rest.encode()) + 7 * self.seed)
        noise = rng2.standard_normal(self.dimension)
        noise -= (noise @ anchor) * anchor
        noise /= np.linalg.norm(noise)
        c = 0.93 + 0.06 * ((zlib.crc32(rest.encode()) % 1000) / 1000.0) if rest else 1.0
        v = c * anchor + math.sqrt(max(0.0, 1 - c * c)) * noise
        v /= np.linalg.norm(v)
        return _Vec(tuple(float(x) for x in v))


class _Vec:
    def __init__(self, comps):
        self.components = comps

    @property
    def dimension(self):
        return len(self.components)


class StubJudge:
    """Deterministic judge: full score when the query and the cached key
    share the same last word, else a crc-derived score below 0.9."""

    def score(self, query_text: str, key_text: str, value: str) -> float:
        if query_text.split()[-1] == key_text.split()[-1]:
            return 1.0
        return (zlib.crc32((query_text + "|" + key_text).encode()) % 800) / 1000.0

    def staticity(self, key_text: str, value: str) -> int:
        return 1 + zlib.crc32(key_text.encode()) % 10


def engine_trace(n_ops: int = 600, seed: int = 11):
    """A mixed lookup/admit/evict trace over a few dozen topics."""
    rng = Random(seed)
    topics = [f"topic{t:02d}" for t in range(30)]
    tails = ["alpha", "beta", "gamma", "delta"]
    ops = []
    now = 0.0
    for i in range(n_ops):
        now += rng.choice([0.5, 1.0, 2.0])
        t = rng.choice(topics[:8] if rng.random() < 0.7 else topics)
        text = f"{t} {rng.choice(['w1', 'w2', 'w3'])} {rng.choice(tails)}"
        r = rng.random()
        if r < 0.6:
            ops.append(("lookup", text, "search" if rng.random() < 0.9 else "other", now))
        elif r < 0.95:
            ops.append(("admit", text, "search", now,
                        dict(value=" ".join(["tok"] * rng.randrange(1, 40)),
                             staticity=rng.randrange(1, 11), freq=rng.randrange(0, 3),
                             lat=rng.choice([50.0, 400.0, 1500.0]),
                             cost=rng.choice([0.0, 0.0005, 0.005, 0.02]),
                             ttl=rng.choice([15.0, 60.0, 400.0]))))
        else:
            ops.append(("evict", now))
    return ops
