"""CPU oracle for the Sine stage-1 search and the LCFU eviction pass.

TEST INFRASTRUCTURE ONLY.  This module is a plain numpy / Python
restatement of the reference algorithm (`semcache`, the package under
`/root/reference/pkg/src/semcache`).  It is imported by `tests/`,
`__graft_entry__.smoke()` and the `cpu_baseline` / `--impl reference` legs
of `bench.py` -- as the checker and the CPU baseline, never as part of the
product path.  `paper_2509_17360_b200` must never import it.

Parity of this restatement is pinned against golden vectors produced by
the reference itself (`tests/golden/make_golden.py`, run in the build
container where `/root/reference` is importable) -- see
`tests/test_oracle_golden.py`.

Every function cites the reference file:line it restates
(`src/` = `pkg/src/semcache/`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

NORM_TOL = 1e-6  # src/index.py:23


class OracleValidationError(ValueError):
    """Stand-in for semcache.errors.ValidationError (src/errors.py:10-11)."""


@dataclass(frozen=True)
class OracleCandidate:
    """src/index.py:26-29."""
    id: int
    similarity: float


def check_vector(vec, dimension: int) -> np.ndarray:
    """src/index.py:32-39: float64 cast, 1-D shape check, |norm-1| <= 1e-6."""
    arr = np.asarray(vec.components if hasattr(vec, "components") else vec,
                     dtype=np.float64)
    if arr.ndim != 1 or arr.shape[0] != dimension:
        raise OracleValidationError(f"expected dimension {dimension}, got shape {arr.shape}")
    n = float(np.linalg.norm(arr))
    if abs(n - 1.0) > NORM_TOL:
        raise OracleValidationError(f"vector is not L2-normalized (norm={n:.8f})")
    return arr


def rank(ids: np.ndarray, sims: np.ndarray, k: int, min_similarity: float):
    """src/index.py:42-46: inclusive threshold, (-sim, id) lexsort, first k."""
    keep = sims >= min_similarity
    ids, sims = ids[keep], sims[keep]
    order = np.lexsort((ids, -sims))[:k]
    return [OracleCandidate(int(ids[i]), float(sims[i])) for i in order]


class OracleExactIndex:
    """Restatement of ExactCosineIndex (src/index.py:49-102).

    Same observable behaviour (raw float64 dot, `_rank`, swap-last removal,
    slot-ordered `ids()`), but rows live in a preallocated buffer so the
    oracle can be bulk-populated at the benchmark sizes (the reference's
    `np.vstack` insert is O(N*d) per row, src/index.py:78).
    """

    def __init__(self, dimension: int, capacity: int = 16):
        if dimension < 1:
            raise OracleValidationError("dimension must be >= 1")
        self.dimension = dimension
        self._ids: list[int] = []
        self._pos: dict[int, int] = {}
        self._buf = np.empty((max(capacity, 1), dimension), dtype=np.float64)

    def __len__(self) -> int:
        return len(self._ids)

    def ids(self) -> list[int]:
        return list(self._ids)

    @property
    def vectors(self) -> np.ndarray:
        return self._buf[:len(self._ids)]

    def _grow(self, need: int) -> None:
        if need > self._buf.shape[0]:
            nb = np.empty((max(need, 2 * self._buf.shape[0]), self.dimension))
            nb[:len(self._ids)] = self._buf[:len(self._ids)]
            self._buf = nb

    def insert(self, id: int, vector) -> None:
        arr = check_vector(vector, self.dimension)          # src/index.py:72
        if id in self._pos:                                 # src/index.py:74-75
            raise OracleValidationError(f"duplicate id {id}")
        self._grow(len(self._ids) + 1)
        self._buf[len(self._ids)] = arr
        self._pos[id] = len(self._ids)
        self._ids.append(id)

    def bulk_load(self, ids, rows: np.ndarray) -> None:
        """Direct population: rows must already be unit norm."""
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        n0 = len(self._ids)
        self._grow(n0 + rows.shape[0])
        self._buf[n0:n0 + rows.shape[0]] = rows
        for j, i in enumerate(ids):
            i = int(i)
            if i in self._pos:
                raise OracleValidationError(f"duplicate id {i}")
            self._pos[i] = n0 + j
            self._ids.append(i)

    def remove(self, id: int) -> None:
        """src/index.py:80-92: swap the last row into the hole."""
        if id not in self._pos:
            raise OracleValidationError(f"unknown id {id}")
        pos = self._pos.pop(id)
        last = len(self._ids) - 1
        if pos != last:
            moved = self._ids[last]
            self._ids[pos] = moved
            self._buf[pos] = self._buf[last]
            self._pos[moved] = pos
        self._ids.pop()

    def query(self, vector, k: int, min_similarity: float = -1.0):
        """src/index.py:94-102."""
        arr = check_vector(vector, self.dimension)
        if k < 1:
            raise OracleValidationError("k must be >= 1")
        if not self._ids:
            return []
        sims = self.vectors @ arr
        return rank(np.asarray(self._ids), sims, k, min_similarity)

    def query_unchecked(self, arr: np.ndarray, k: int, min_similarity: float = -1.0):
        """query() minus the per-call validation (bench sampling only)."""
        if not self._ids:
            return []
        sims = self.vectors @ arr
        return rank(np.asarray(self._ids), sims, k, min_similarity)


# ---------------------------------------------------------------- LCFU

def cal_score(frequency, retrieval_cost_usd, retrieval_latency_ms, staticity,
              size_tokens, expiration_time, now, log=math.log) -> float:
    """src/engine.py:33-48: left-to-right float64 product of natural logs."""
    if size_tokens == 0 or expiration_time - now <= 0.0:
        return 0.0
    return (log(frequency + 1)
            * log(retrieval_cost_usd * 1000.0 + 1)
            * log(retrieval_latency_ms + 1)
            * log(staticity + 1)
            / size_tokens)


@dataclass
class OracleElement:
    """The SemanticElement fields eviction reads (src/model.py:85-110)."""
    staticity: int
    frequency: int
    retrieval_latency_ms: float
    retrieval_cost_usd: float
    size_tokens: int
    created_at: float
    expiration_time: float

    def is_expired(self, now: float) -> bool:       # src/model.py:106-110
        return self.expiration_time - now <= 0.0


def element_score(el, now: float) -> float:
    return cal_score(el.frequency, el.retrieval_cost_usd, el.retrieval_latency_ms,
                     el.staticity, el.size_tokens, el.expiration_time, now)


def victim_order(elements: dict, now: float, policy: str = "lcfu",
                 last_access: dict | None = None) -> list[int]:
    """src/engine.py:369-383: ascending sort of (key, created_at, id)."""
    if policy == "lcfu":
        keyed = [(element_score(el, now), el.created_at, eid) for eid, el in elements.items()]
    elif policy == "lru":
        keyed = [(last_access[eid], el.created_at, eid) for eid, el in elements.items()]
    else:
        keyed = [(el.frequency, el.created_at, eid) for eid, el in elements.items()]
    keyed.sort()
    return [eid for _, _, eid in keyed]


def expired_ids(elements: dict, now: float) -> list[int]:
    """src/engine.py:362-367 / :348-349: expired ids, ascending."""
    return sorted(eid for eid, el in elements.items() if el.is_expired(now))


def evict_until_fits(elements: dict, now: float, capacity: int, policy: str = "lcfu",
                     last_access: dict | None = None) -> list[int]:
    """src/engine.py:342-360 (pure: returns the removal order, no mutation)."""
    usage = sum(el.size_tokens for el in elements.values())
    removed = expired_ids(elements, now)
    gone = set(removed)
    for eid in removed:
        usage -= elements[eid].size_tokens
    if usage > capacity:
        live = {eid: el for eid, el in elements.items() if eid not in gone}
        for eid in victim_order(live, now, policy, last_access):
            removed.append(eid)
            usage -= elements[eid].size_tokens
            if usage <= capacity:
                break
    return removed


def admit_victims(elements: dict, now: float, capacity: int, incoming_size: int,
                  policy: str = "lcfu", last_access: dict | None = None):
    """src/engine.py:319-327: (expired ids ascending, ordered victims)."""
    exp = expired_ids(elements, now)
    gone = set(exp)
    usage = sum(el.size_tokens for eid, el in elements.items() if eid not in gone)
    victims = []
    if usage + incoming_size > capacity:
        live = {eid: el for eid, el in elements.items() if eid not in gone}
        for eid in victim_order(live, now, policy, last_access):
            victims.append(eid)
            usage -= elements[eid].size_tokens
            if usage + incoming_size <= capacity:
                break
    return exp, victims


# ------------------------------------------- vectorised LCFU (large N)

def _exact_log(values: np.ndarray) -> np.ndarray:
    """math.log (glibc) applied elementwise through the unique values.

    numpy's SIMD log is not guaranteed to round like libm, so the oracle
    evaluates math.log once per distinct argument (metadata columns take
    few distinct values) and scatters the results back.
    """
    uniq, inv = np.unique(values, return_inverse=True)
    logs = np.fromiter((math.log(float(u)) for u in uniq), dtype=np.float64, count=uniq.size)
    return logs[inv]


def lcfu_scores_np(freq, cost, lat, stat, size, expiration, now) -> np.ndarray:
    """Vectorised cal_score (src/engine.py:40-48), bit-identical to the scalar
    form: numpy float64 * and / are single IEEE ops, evaluated left to right."""
    freq = np.asarray(freq, dtype=np.int64)
    lf = _exact_log((freq + 1).astype(np.float64))
    lc = _exact_log(np.asarray(cost, dtype=np.float64) * 1000.0 + 1)
    ll = _exact_log(np.asarray(lat, dtype=np.float64) + 1)
    ls = _exact_log((np.asarray(stat, dtype=np.int64) + 1).astype(np.float64))
    size = np.asarray(size, dtype=np.int64)
    score = lf * lc * ll * ls / size.astype(np.float64)
    dead = (size == 0) | ((np.asarray(expiration, dtype=np.float64) - now) <= 0.0)
    score[dead] = 0.0
    return score


def evict_until_fits_np(ids, freq, cost, lat, stat, size, created, expiration,
                        now, capacity) -> np.ndarray:
    """Vectorised evict_until_fits for the benchmark sizes (same order)."""
    ids = np.asarray(ids, dtype=np.int64)
    size = np.asarray(size, dtype=np.int64)
    expiration = np.asarray(expiration, dtype=np.float64)
    expired = (expiration - now) <= 0.0
    exp_ids = np.sort(ids[expired])
    usage = int(size[~expired].sum())
    if usage <= capacity:
        return exp_ids
    live = ~expired
    sc = lcfu_scores_np(np.asarray(freq)[live], np.asarray(cost)[live], np.asarray(lat)[live],
                        np.asarray(stat)[live], size[live], expiration[live], now)
    lid = ids[live]
    order = np.lexsort((lid, np.asarray(created, dtype=np.float64)[live], sc))
    cum = np.cumsum(size[live][order])
    m = int(np.searchsorted(cum, usage - capacity, side="left")) + 1
    return np.concatenate([exp_ids, lid[order[:m]]])


# ------------------------------------------------- engine loop (config E)

class OracleEngine:
    """Restatement of the reference CacheEngine hot loop (src/engine.py:
    lookup :160-223, admit :300-336, evict_until_fits :342-360) over
    OracleExactIndex and the oracle eviction order -- the CPU baseline of
    the mixed agent trace.  Elements are any objects with the
    SemanticElement fields; `embed` maps text -> unit vector."""

    def __init__(self, dimension, capacity_tokens, embed, judge_score, tau_sim=0.9, tau_lsm=0.9,
                 candidate_k=5, policy="lcfu", capacity_rows=16):
        self.index = OracleExactIndex(dimension, capacity=capacity_rows)
        self.capacity = capacity_tokens
        self.embed = embed
        self.judge_score = judge_score
        self.tau_sim, self.tau_lsm, self.k, self.policy = tau_sim, tau_lsm, candidate_k, policy
        self.elements, self.by_key, self.last_access = {}, {}, {}
        self.usage = 0
        self.next_id = 1

    def bulk_load(self, elements, rows):
        ids = list(range(self.next_id, self.next_id + len(elements)))
        self.index.bulk_load(ids, rows)
        for eid, el in zip(ids, elements):
            self.elements[eid] = el
            self.by_key[(el.key.text, el.key.tool)] = eid
            self.last_access[eid] = el.created_at
            self.usage += el.size_tokens
        self.next_id += len(elements)

    def _remove(self, eid):
        el = self.elements.pop(eid)
        self.by_key.pop((el.key.text, el.key.tool), None)
        self.last_access.pop(eid, None)
        self.usage -= el.size_tokens
        self.index.remove(eid)

    def lookup(self, key, now):
        cands = self.index.query(self.embed(key.text), self.k, self.tau_sim)   # engine.py:177-178
        for c in cands:                                                        # engine.py:185-204
            el = self.elements.get(c.id)
            if el is None or el.key.tool != key.tool:
                continue
            if el.is_expired(now):
                self._remove(c.id)
                continue
            if self.judge_score(key.text, el.key.text, el.value) >= self.tau_lsm:
                # hit bookkeeping (engine.py:209-217)
                self.elements[c.id] = replace(el, frequency=el.frequency + 1)
                self.last_access[c.id] = now
                return c.id
        return None

    def _purge(self, now):                                                      # engine.py:362-367
        for eid in sorted(e for e, el in self.elements.items() if el.is_expired(now)):
            self._remove(eid)

    def admit(self, el, now):                                                   # engine.py:300-336
        old = self.by_key.get((el.key.text, el.key.tool))
        if old is not None:
            self._remove(old)
        self._purge(now)
        evicted = []
        if self.usage + el.size_tokens > self.capacity:
            for v in victim_order(self.elements, now, self.policy, self.last_access):
                self._remove(v)
                evicted.append(v)
                if self.usage + el.size_tokens <= self.capacity:
                    break
        eid = self.next_id
        self.next_id += 1
        self.index.insert(eid, el.embedding)
        self.elements[eid] = el
        self.by_key[(el.key.text, el.key.tool)] = eid
        self.last_access[eid] = now
        self.usage += el.size_tokens
        return eid, evicted

    def evict_until_fits(self, now):                                            # engine.py:342-360
        removed = sorted(e for e, el in self.elements.items() if el.is_expired(now))
        for eid in removed:
            self._remove(eid)
        if self.usage > self.capacity:
            for v in victim_order(self.elements, now, self.policy, self.last_access):
                self._remove(v)
                removed.append(v)
                if self.usage <= self.capacity:
                    break
        return removed


# ------------------------------------------------------------ embedder

import hashlib as _hashlib  # noqa: E402
import string as _string  # noqa: E402

_PUNCT = str.maketrans({c: " " for c in _string.punctuation})  # src/embedder.py:20


def tokenize(text: str) -> list[str]:
    """src/embedder.py:23-25."""
    return text.lower().translate(_PUNCT).split()


def hashed_bag_embed(text: str, dimension: int, seed: int) -> tuple:
    """HashedBagEmbedder._bucket + embed (src/embedder.py:49-60)."""
    key = seed.to_bytes(8, "little", signed=False)
    tokens = tokenize(text)
    if not tokens:
        raise OracleValidationError("cannot embed text with no tokens")
    counts = [0.0] * dimension
    for tok in tokens:
        d = _hashlib.blake2b(tok.encode("utf-8"), key=key, digest_size=8).digest()
        counts[int.from_bytes(d, "little") % dimension] += 1.0
    norm = sum(c * c for c in counts) ** 0.5
    return tuple(c / norm for c in counts)
