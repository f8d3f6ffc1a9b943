"""Golden vectors for the hashed bag-of-words embedder, produced by the
REFERENCE (`semcache.embedder.HashedBagEmbedder`, run in the build
container where /root/reference is importable):

    python tests/golden/make_embed_golden.py

Writes embed_golden.json: texts, (dimension, seed) pairs and the
reference's vectors (nonzero components as float.hex), plus keyed BLAKE2b-64 digests of raw
byte strings from hashlib (the hash the embedder keys its buckets on)."""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
for cand in ("/root/reference/pkg/src", os.path.join(HERE, "..", "..", "baseline", "_ref")):
    if os.path.isdir(os.path.join(cand, "semcache")):
        sys.path.insert(0, cand)
        break

from semcache.embedder import HashedBagEmbedder  # noqa: E402


def texts():
    rng = random.Random("embed-golden")
    words = ["cache", "Agent", "search!", "weather?", "PARIS", "héllo", "naïve", "数据", "x", "tool-call",
             "what's", "2024", "e-mail", "a.b.c", "São", "Straße", "ﬁnance", "emoji😀"]
    out = ["Hello, World! héllo  WORLD...x", "what is the capital of France?", "a", "1 2 3 4 5 6 7 8 9 10",
           "The quick brown fox jumps over the lazy dog " * 3, "ΑΒΓ αβγ", "tab\tseparated\nlines",
           "x" * 300, "punct;only;between;words"]
    for _ in range(40):
        out.append(" ".join(rng.choice(words) for _ in range(rng.randint(1, 25))))
    return out


def main():
    data = {"texts": texts(), "cases": []}
    for dim, seed in ((256, 1), (768, 1), (384, 7), (8, 2 ** 63 + 5)):
        emb = HashedBagEmbedder(dim, seed=seed)
        data["cases"].append({"dimension": dim, "seed": seed,
                              # sparse: (bucket, float.hex) of the nonzero components
                              "vectors": [[[i, float(c).hex()] for i, c in enumerate(emb.embed(t).components) if c]
                                          for t in data["texts"]]})
    rng = random.Random("blake")
    msgs = [bytes(rng.getrandbits(8) for _ in range(n)) for n in (0, 1, 7, 8, 63, 64, 127, 128, 129, 255, 256, 300)]
    data["blake2b"] = [{"msg": m.hex(), "key": k,
                        "digest": int.from_bytes(hashlib.blake2b(m, key=k.to_bytes(8, "little"),
                                                                 digest_size=8).digest(), "little")}
                       for m in msgs for k in (1, 7, 2 ** 64 - 1)]
    with open(os.path.join(HERE, "embed_golden.json"), "w", encoding="utf-8") as fh:
        json.dump(data, fh, ensure_ascii=False, separators=(",", ":"))


if __name__ == "__main__":
    main()
