"""B200-native Sine stage-1 search and LCFU eviction for the semcache API.

Public surface (drop-in for the reference `semcache` hot path):

* `GpuCosineIndex`  -- ExactCosineIndex contract (index.py:49-120) on HBM.
* `CacheEngine`     -- semcache.engine.CacheEngine with device eviction.
* `MultiDeviceCosineIndex` -- the same index contract over row shards on
  several GPUs of one process (the reference's single-process engine).
* `ShardedCosineIndex` -- row-sharded index over torch.distributed (NCCL).
* `GpuHashedBagEmbedder` -- HashedBagEmbedder (embedder.py:34-60) with a
  batched device hashing path.
"""

from .errors import RetriableError, SemcacheError, ValidationError
from .index import Candidate, GpuCosineIndex, check_vector
from .multidev import MultiDeviceCosineIndex
from .embedder import GpuHashedBagEmbedder
from .engine import AdmitOutcome, CacheEngine, LookupOutcome, StageTimings, cal_score
from .model import (CacheConfig, EmbeddingVector, SemanticElement, SemanticKey, make_element,
                    token_count)

__version__ = "0.1.0"

__all__ = [
    "AdmitOutcome", "CacheConfig", "CacheEngine", "Candidate", "EmbeddingVector", "GpuCosineIndex",
    "GpuHashedBagEmbedder", "MultiDeviceCosineIndex",
    "LookupOutcome", "RetriableError", "SemanticElement", "SemanticKey", "SemcacheError",
    "StageTimings", "ValidationError", "cal_score", "check_vector", "make_element", "token_count",
]
