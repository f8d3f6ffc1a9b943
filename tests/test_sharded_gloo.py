"""Row-sharded stage-1 host logic with world_size 2 over gloo (CPU).

Each rank's local index is the CPU oracle (test infrastructure stands in
for the GPU shard); the placement, all-gather and merge code under test is
the production `ShardedCosineIndex`.  The merged result must equal a
single unsharded index."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleShard:
    """Minimal local-index stand-in with the GpuCosineIndex batch surface."""

    def __init__(self, dim):
        from oracle import sine_oracle as O
        self.dimension = dim
        self.idx = O.OracleExactIndex(dim)

    def insert_batch(self, ids, rows):
        self.idx.bulk_load(ids, rows)

    def remove_batch(self, ids):
        for i in ids:
            self.idx.remove(int(i))

    def query_batch(self, q, k, ms):
        B = q.shape[0]
        ids = np.full((B, k), -1, dtype=np.int64)
        sims = np.zeros((B, k))
        cnt = np.zeros(B, dtype=np.int32)
        for j in range(B):
            r = _rowwise_query(self.idx, q[j], k, ms)
            cnt[j] = len(r)
            ids[j, :len(r)] = [c.id for c in r]
            sims[j, :len(r)] = [c.similarity for c in r]
        return ids, sims, cnt


def _rowwise_query(idx, q, k, ms):
    # position-independent per-row sums (BLAS gemv rounds a row differently
    # depending on where it sits in the matrix, which would break exact ties)
    from oracle import sine_oracle as O
    if len(idx) == 0:
        return []
    sims = (idx.vectors * q).sum(axis=1)
    return O.rank(np.asarray(idx.ids()), sims, k, ms)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from oracle import sine_oracle as O
    from paper_2509_17360_b200.sharded import ShardedCosineIndex
    from test_sharded_gloo import OracleShard, _rowwise_query
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    n, d = 600, 16
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    rows[100:140] = rows[5]                      # exact ties across shards
    ids = rng.permutation(5000)[:n]
    sh = ShardedCosineIndex(OracleShard(d))
    sh.insert_batch(ids[:400], rows[:400])
    sh.insert_batch(ids[400:], rows[400:])
    sh.remove_batch(ids[:50:3])
    full = O.OracleExactIndex(d)
    full.bulk_load(ids, rows)
    for i in ids[:50:3]:
        full.remove(int(i))
    q = np.concatenate([rows[[5, 7, 300]], rng.standard_normal((5, d))])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ok = True
    for k, ms in ((10, -1.0), (3, 0.2), (50, 0.0)):
        gi, gs, gc = sh.query_batch(q, k, ms)
        for j in range(q.shape[0]):
            want = _rowwise_query(full, q[j], k, ms)
            ok &= gi[j, :gc[j]].tolist() == [c.id for c in want]
            ok &= np.allclose(gs[j, :gc[j]], [c.similarity for c in want], atol=0, rtol=0)
            ok &= bool((gi[j, gc[j]:] == -1).all())
    ok &= len(sh) == len(full)
    out[rank] = bool(ok)
    dist.destroy_process_group()


def test_sharded_merge_equals_single_index_gloo():
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
        assert all(p.exitcode == 0 for p in procs)
        assert dict(out) == {0: True, 1: True}
