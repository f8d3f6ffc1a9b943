"""Batched query embeddings for the Sine stage-1.

`GpuHashedBagEmbedder` is the reference's `HashedBagEmbedder`
(pkg/src/semcache/embedder.py:34-60) with a batch API: tokenization is the
reference's own (`tokenize`, embedder.py:23-25: lowercase, ASCII punctuation
to spaces, whitespace split) on the host; the keyed BLAKE2b-64 of every
token and the bucket counts run on the GPU (`sine_embed_hashed_bag`), and
the normalisation reproduces `counts / sum(c*c) ** 0.5` bit for bit.  It
satisfies the reference `Embedder` protocol (`dimension`, `seed`,
`embed(text) -> EmbeddingVector`), so `CacheEngine` and the reference engine
accept it unchanged.
"""

from __future__ import annotations

import string

import numpy as np

from . import _native as N
from .errors import ValidationError
from .model import EmbeddingVector

_PUNCT_TABLE = str.maketrans({c: " " for c in string.punctuation})


def tokenize(text: str) -> list[str]:
    """embedder.py:23-25 -- lowercase, punctuation to spaces, split."""
    return text.lower().translate(_PUNCT_TABLE).split()


class GpuHashedBagEmbedder:
    """Deterministic keyed-hash bag-of-words embedder; same (seed,
    dimension) gives the reference's bit-identical vectors."""

    def __init__(self, dimension: int = 256, seed: int = 1, *, device: int = 0):
        if dimension < 8:
            raise ValidationError("embedder dimension must be >= 8")
        self.dimension = dimension
        self.seed = seed
        self.device = device
        self._key = int.from_bytes(seed.to_bytes(8, "little", signed=False), "little")
        self._lib = N.load_library()

    def embed(self, text: str) -> EmbeddingVector:
        return EmbeddingVector(tuple(self.embed_batch([text])[0].tolist()))

    def embed_batch(self, texts) -> np.ndarray:
        """float64 [len(texts), dimension], row b == embed(texts[b])."""
        toks, q_off = [], [0]
        for t in texts:
            tk = tokenize(t)
            if not tk:
                raise ValidationError("cannot embed text with no tokens")
            toks.extend(w.encode("utf-8") for w in tk)
            q_off.append(len(toks))
        B = len(texts)
        out = np.empty((B, self.dimension), dtype=np.float64)
        if B == 0:
            return out
        blob = b"".join(toks)
        tok_off = np.zeros(len(toks) + 1, dtype=np.int64)
        np.cumsum([len(w) for w in toks], out=tok_off[1:])
        q = np.asarray(q_off, dtype=np.int64)
        buf = np.frombuffer(blob, dtype=np.uint8) if blob else np.zeros(1, dtype=np.uint8)
        N.check(self._lib.sine_embed_hashed_bag(self.device, self._key, self.dimension, buf.ctypes.data, len(blob),
                                                tok_off.ctypes.data, len(toks), q.ctypes.data, B, out.ctypes.data))
        return out
