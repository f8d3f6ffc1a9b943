"""cProfile of the config-E trace replay (sequential and batched), 1M x 768."""
import cProfile
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2509_17360_b200 as P  # noqa: E402
from paper_2509_17360_b200 import model as M  # noqa: E402

n = 1_000_000
rows = bench.make_rows(n, 768)
rng = np.random.default_rng(21)
meta = bench.evict_metadata(n, seed=6)
meta["created"] = np.zeros(n)
meta["expiration"] = np.full(n, 1.0e5)
shared = M.EmbeddingVector((1.0,))
scan = sys.argv[1] if len(sys.argv) > 1 else "fp32"
for batched in (False, True):
    ops = bench.trace_ops(n, 768, 1000, rng, rows)
    emb = bench._DictEmbedder(768)
    els = bench._make_elements(M, n, meta, shared)
    eng = P.CacheEngine(P.CacheConfig(capacity_tokens=int(meta["size"].sum())), emb, bench._TextJudge(),
                        **({"scan": scan} if scan != "fp32" else {}))
    eng.bulk_admit(els, rows, now=0.0)
    bench.run_trace(eng, ops[:50], emb, M, 1.0, batched)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    done = bench.run_trace(eng, ops[50:], emb, M, 2.0, batched)
    pr.disable()
    dt = time.perf_counter() - t0
    print(f"batched={batched} scan={scan}: {done / dt:.0f} ops/s (under cProfile)", flush=True)
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
    del eng, els
