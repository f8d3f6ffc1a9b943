"""Host half of the reference engine, for hosts without `semcache`.

When the reference package is importable, `engine.CacheEngine` subclasses
`semcache.engine.CacheEngine` itself and none of this module is used: the
lookup paths, judge loop, hit bookkeeping and counters are then the
reference's own code.  This mirror exists so the GPU engine is usable (and
testable on the GPU box) without the reference installed.  It restates,
method for method, the parts of pkg/src/semcache/engine.py the GPU engine
does not override: the outcome types (:51-90), the accessors (:117-156),
`lookup` (:160-223), `lookup_exact` (:225-245), `lookup_ann_only`
(:247-276), `peek` (:278-296), `remove_expired` (:338-340) and
`_remove_locked` (:385-390).  Hits update `_elements` / `_last_access`
exactly as the reference does; the GPU engine observes those writes.
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass, replace

from .errors import RetriableError


def cal_score(element, now: float, log=math.log) -> float:
    """LCFU utility (engine.py:33-48)."""
    if element.size_tokens == 0 or element.remaining_ttl(now) <= 0.0:
        return 0.0
    return (log(element.frequency + 1) * log(element.retrieval_cost_usd * 1000.0 + 1)
            * log(element.retrieval_latency_ms + 1) * log(element.staticity + 1) / element.size_tokens)


@dataclass(frozen=True)
class StageTimings:
    embed_ms: float = 0.0
    index_ms: float = 0.0
    judge_ms: float = 0.0


@dataclass(frozen=True)
class LookupOutcome:
    kind: str
    element_id: int | None
    element: object
    similarity: float | None
    s_lsm: float | None
    candidates_considered: int
    judged: int
    timings: StageTimings
    query_embedding: object
    error: str | None = None

    @property
    def hit(self) -> bool:
        return self.kind == "hit"


@dataclass(frozen=True)
class AdmitOutcome:
    element_id: int
    evicted_ids: tuple
    replaced_id: int | None


@dataclass
class EngineStats:
    lookups: int = 0
    hits: int = 0
    misses: int = 0
    admissions: int = 0
    replacements: int = 0
    evictions: int = 0
    expirations: int = 0


class MirrorCacheEngine:
    """engine.py:94-447 minus what the GPU engine overrides."""

    def __init__(self, config, embedder, judge, index=None):
        self.config = config
        self._embedder = embedder
        self._judge = judge
        self._index = index
        self._lock = threading.Lock()
        self._elements: dict = {}
        self._by_key: dict = {}
        self._last_access: dict = {}
        self._usage = 0
        self._next_id = 1
        self._stats = EngineStats()

    @property
    def usage_tokens(self) -> int:
        return self._usage

    @property
    def embedder(self):
        return self._embedder

    @property
    def judge(self):
        return self._judge

    def __len__(self) -> int:
        return len(self._elements)

    def get(self, element_id: int):
        with self._lock:
            return self._elements.get(element_id)

    def elements(self) -> dict:
        with self._lock:
            return dict(self._elements)

    def stats(self) -> dict:
        with self._lock:
            s = self._stats
            return {"lookups": s.lookups, "hits": s.hits, "misses": s.misses,
                    "admissions": s.admissions, "replacements": s.replacements,
                    "evictions": s.evictions, "expirations": s.expirations,
                    "usage_tokens": self._usage, "element_count": len(self._elements)}

    def _hit_locked(self, eid: int, el, now: float):
        """engine.py:209-217: frequency + 1, fresh value_score, last access."""
        updated = replace(el, frequency=el.frequency + 1)
        updated = replace(updated, value_score=cal_score(updated, now))
        self._elements[eid] = updated
        self._last_access[eid] = now
        self._stats.hits += 1
        return updated

    def lookup(self, key, now: float, judge_text: str | None = None) -> LookupOutcome:
        t0 = time.perf_counter()
        try:
            emb = self._embedder.embed(key.text)
        except RetriableError as exc:
            with self._lock:
                self._stats.lookups += 1
                self._stats.misses += 1
            return LookupOutcome("miss", None, None, None, None, 0, 0, StageTimings(), None, error=str(exc))
        t1 = time.perf_counter()
        cands = self._index.query(emb, k=self.config.candidate_k, min_similarity=self.config.tau_sim)
        t2 = time.perf_counter()
        judged = 0
        error = None
        winner = None
        for cand in cands:
            with self._lock:
                el = self._elements.get(cand.id)
            if el is None or el.key.tool != key.tool:
                continue
            if el.is_expired(now):
                with self._lock:
                    if cand.id in self._elements and self._elements[cand.id].is_expired(now):
                        self._remove_locked(cand.id)
                        self._stats.expirations += 1
                continue
            judged += 1
            try:
                s = self._judge.score(judge_text or key.text, el.key.text, el.value)
            except RetriableError as exc:
                error = str(exc)
                continue
            if s >= self.config.tau_lsm:
                winner = (cand.id, cand.similarity, s)
                break
        t3 = time.perf_counter()
        timings = StageTimings((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3)
        with self._lock:
            self._stats.lookups += 1
            if winner is not None:
                eid, sim, s = winner
                el = self._elements.get(eid)
                if el is not None and not el.is_expired(now):
                    updated = self._hit_locked(eid, el, now)
                    return LookupOutcome("hit", eid, updated, sim, s, len(cands), judged, timings, emb)
            self._stats.misses += 1
        return LookupOutcome("miss", None, None, None, None, len(cands), judged, timings, emb, error=error)

    def lookup_exact(self, key, now: float) -> LookupOutcome:
        with self._lock:
            self._stats.lookups += 1
            eid = self._by_key.get((key.text, key.tool))
            if eid is not None:
                el = self._elements[eid]
                if el.is_expired(now):
                    self._remove_locked(eid)
                    self._stats.expirations += 1
                else:
                    updated = self._hit_locked(eid, el, now)
                    return LookupOutcome("hit", eid, updated, None, None, 0, 0, StageTimings(), None)
            self._stats.misses += 1
        return LookupOutcome("miss", None, None, None, None, 0, 0, StageTimings(), None)

    def lookup_ann_only(self, key, now: float) -> LookupOutcome:
        t0 = time.perf_counter()
        emb = self._embedder.embed(key.text)
        t1 = time.perf_counter()
        cands = self._index.query(emb, k=self.config.candidate_k, min_similarity=self.config.tau_sim)
        t2 = time.perf_counter()
        timings = StageTimings((t1 - t0) * 1e3, (t2 - t1) * 1e3)
        with self._lock:
            self._stats.lookups += 1
            for cand in cands:
                el = self._elements.get(cand.id)
                if el is None or el.key.tool != key.tool:
                    continue
                if el.is_expired(now):
                    self._remove_locked(cand.id)
                    self._stats.expirations += 1
                    continue
                updated = self._hit_locked(cand.id, el, now)
                return LookupOutcome("hit", cand.id, updated, cand.similarity, None, len(cands), 0, timings, emb)
            self._stats.misses += 1
        return LookupOutcome("miss", None, None, None, None, len(cands), 0, timings, emb)

    def peek(self, key, now: float) -> bool:
        try:
            emb = self._embedder.embed(key.text)
        except RetriableError:
            return False
        for cand in self._index.query(emb, k=self.config.candidate_k, min_similarity=self.config.tau_sim):
            with self._lock:
                el = self._elements.get(cand.id)
            if el is None or el.key.tool != key.tool or el.is_expired(now):
                continue
            try:
                if self._judge.score(key.text, el.key.text, el.value) >= self.config.tau_lsm:
                    return True
            except RetriableError:
                continue
        return False

    def remove_expired(self, now: float) -> int:
        with self._lock:
            return self._purge_expired_locked(now)

    def _remove_locked(self, eid: int) -> None:
        el = self._elements.pop(eid)
        self._by_key.pop((el.key.text, el.key.tool), None)
        self._last_access.pop(eid, None)
        self._usage -= el.size_tokens
        self._index.remove(eid)
