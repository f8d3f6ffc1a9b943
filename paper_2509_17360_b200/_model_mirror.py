"""Boundary types for hosts without `semcache` (mirror of
pkg/src/semcache/model.py:15-179).

`model.py` re-exports the reference's own classes whenever `semcache` is
importable; these mirrors exist so the package is usable (and testable on
the GPU box) without the reference installed.  Field names and validation
rules follow model.py:15-179.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ValidationError

EVICTION_POLICIES = ("lcfu", "lru", "lfu")  # model.py:15


def token_count(value: str) -> int:
    """Whitespace token count; zero tokens is an error (model.py:18-26)."""
    n = len(value.split())
    if n == 0:
        raise ValidationError("value must contain at least one token")
    return n


@dataclass(frozen=True)
class SemanticKey:
    text: str
    tool: str

    def __post_init__(self) -> None:
        if not self.text.strip():
            raise ValidationError("key text must be non-empty")
        if not self.tool.strip():
            raise ValidationError("key tool must be non-empty")


@dataclass(frozen=True)
class EmbeddingVector:
    components: tuple

    def __post_init__(self) -> None:
        if len(self.components) == 0:
            raise ValidationError("embedding must have at least one component")
        if not all(map(math.isfinite, self.components)):
            raise ValidationError("embedding components must be finite")

    @classmethod
    def from_iterable(cls, values) -> "EmbeddingVector":
        return cls(tuple(float(v) for v in values))

    @property
    def dimension(self) -> int:
        return len(self.components)

    def norm(self) -> float:
        return math.sqrt(sum(c * c for c in self.components))

    def is_normalized(self, tol: float = 1e-6) -> bool:
        return abs(self.norm() - 1.0) <= tol


@dataclass(frozen=True)
class SemanticElement:
    key: SemanticKey
    value: str
    embedding: EmbeddingVector
    staticity: int
    frequency: int
    retrieval_latency_ms: float
    retrieval_cost_usd: float
    size_tokens: int
    created_at: float
    expiration_time: float
    value_score: float | None = None

    def remaining_ttl(self, now: float) -> float:
        return self.expiration_time - now

    def is_expired(self, now: float) -> bool:
        return self.remaining_ttl(now) <= 0.0


def make_element(key, value, embedding, staticity, retrieval_latency_ms, retrieval_cost_usd, now,
                 ttl_seconds, frequency=0) -> SemanticElement:
    """Validated constructor (model.py:113-149)."""
    if not isinstance(staticity, int) or not 1 <= staticity <= 10:
        raise ValidationError(f"staticity must be an integer in [1, 10], got {staticity!r}")
    for name, v in (("latency", retrieval_latency_ms), ("cost", retrieval_cost_usd)):
        if not (math.isfinite(v) and v >= 0.0):
            raise ValidationError(f"retrieval {name} must be finite and >= 0")
    if ttl_seconds <= 0.0:
        raise ValidationError("ttl must be positive")
    if frequency < 0:
        raise ValidationError("frequency must be >= 0")
    if not embedding.is_normalized():
        raise ValidationError("element embeddings must be L2-normalized")
    return SemanticElement(key=key, value=value, embedding=embedding, staticity=staticity,
                           frequency=frequency, retrieval_latency_ms=retrieval_latency_ms,
                           retrieval_cost_usd=retrieval_cost_usd, size_tokens=token_count(value),
                           created_at=now, expiration_time=now + ttl_seconds)


@dataclass
class CacheConfig:
    capacity_tokens: int
    tau_sim: float = 0.9
    tau_lsm: float = 0.9
    ttl_seconds: float = 3600.0
    candidate_k: int = 5
    prefetch_theta: float = 0.5
    p_target: float = 0.99
    eviction_policy: str = "lcfu"

    def __post_init__(self) -> None:
        if self.capacity_tokens <= 0:
            raise ValidationError("capacity_tokens must be positive")
        for name in ("tau_sim", "tau_lsm", "prefetch_theta", "p_target"):
            v = getattr(self, name)
            if not 0.0 < v <= 1.0:
                raise ValidationError(f"{name} must be in (0, 1], got {v}")
        if self.ttl_seconds <= 0.0:
            raise ValidationError("ttl_seconds must be positive")
        if self.candidate_k < 1:
            raise ValidationError("candidate_k must be >= 1")
        if self.eviction_policy not in EVICTION_POLICIES:
            raise ValidationError(f"eviction_policy must be one of {EVICTION_POLICIES}, "
                                  f"got {self.eviction_policy!r}")


