"""Row-sharded stage-1 with real GPU shards: two ranks (gloo for the
candidate all-gather, since this pool's boxes have one GPU) each own a
GpuCosineIndex on cuda:0; the merged answer must equal the oracle on the
unsharded rows, ids bit-exact and fp64 similarities to 1e-12."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from test_sharded_gloo import _free_port

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import sine_oracle as O
    from paper_2509_17360_b200 import GpuCosineIndex
    from paper_2509_17360_b200.sharded import ShardedCosineIndex
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rng = np.random.default_rng(1)
    n, d, B = 30000, 384, 96
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    rows[1000:1010] = rows[7]  # exact ties spread over both shards
    ids = rng.permutation(10 * n)[:n]
    sh = ShardedCosineIndex(GpuCosineIndex(d, device=0))
    sh.insert_batch(ids[:20000], rows[:20000])
    sh.insert_batch(ids[20000:], rows[20000:])
    sh.remove_batch(ids[:300:7])
    keep = np.setdiff1d(np.arange(n), np.arange(300)[::7])
    full = O.OracleExactIndex(d)
    full.bulk_load(ids[keep], rows[keep])
    q = rng.standard_normal((B, d))
    q[:40] = rows[rng.integers(0, n, 40)] + 0.02 * rng.standard_normal((40, d))
    q[40] = rows[7]
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ok = True
    for k, ms in ((10, 0.9), (20, -1.0)):
        gi, gs, gc = sh.query_batch(q, k, ms)
        for j in range(B):
            want = full.query(q[j], k, ms)
            ok &= gi[j, :gc[j]].tolist() == [c.id for c in want]
            ok &= bool(np.allclose(gs[j, :gc[j]], [c.similarity for c in want], atol=1e-12, rtol=0))
    out[rank] = bool(ok)
    dist.destroy_process_group()


def test_sharded_gpu_shards_equal_oracle():
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(300)
        assert all(p.exitcode == 0 for p in procs)
        assert dict(out) == {0: True, 1: True}


def test_device_shard_merge_equals_unsharded():
    """The query_device data path on one GPU: P shard indexes produce their
    [2, B, k] blocks (ids + similarity bits) exactly as each rank would, the
    blocks are stacked as the all-gather would lay them out, and the
    library's shard-merge kernel must equal the unsharded index (ids
    bit-exact, fp64 similarities identical), ties across shards included."""
    import torch
    sys.path.insert(0, ROOT)
    from paper_2509_17360_b200 import GpuCosineIndex
    from paper_2509_17360_b200.sharded import merge_gathered_blocks, merge_topk
    rng = np.random.default_rng(4)
    n, d, B = 24000, 128, 64
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    rows[500:520] = rows[3]  # identical rows land on every shard
    ids = rng.permutation(10 * n)[:n]
    full = GpuCosineIndex(d)
    full.insert_batch(ids, rows)
    q = rows[rng.integers(0, n, B)] + 0.3 * rng.standard_normal((B, d))
    q[0] = rows[3]
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    qd = torch.from_numpy(q).cuda()
    for P in (2, 3, 8):
        shards = [GpuCosineIndex(d) for _ in range(P)]
        for r in range(P):
            shards[r].insert_batch(ids[r::P], rows[r::P])
        for k, ms in ((10, -1.0), (7, 0.2), (16, 0.9)):
            blocks = []
            for sh in shards:
                blk = torch.empty((2, B, k), dtype=torch.int64, device="cuda")
                cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
                sh.query_device(B, qd.data_ptr(), k, ms, blk[0].data_ptr(), blk[1].data_ptr(), cnt.data_ptr(),
                                torch.cuda.current_stream().cuda_stream)
                blocks.append(blk)
            gi, gs, gc = merge_gathered_blocks(torch.stack(blocks))
            ti, ts, tc = merge_topk(torch.stack([b[1].view(torch.float64) for b in blocks]),
                                    torch.stack([b[0] for b in blocks]), k)
            wi, ws, wc = full.query_batch(q, k, ms)
            assert gi.cpu().numpy().tolist() == wi.tolist() == ti.cpu().numpy().tolist()
            assert gc.cpu().numpy().tolist() == wc.tolist()
            np.testing.assert_array_equal(gs.cpu().numpy(), ws)


def _pipe_worker(rank, world, port, out, pipelined=True):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import sine_oracle as O
    from paper_2509_17360_b200 import GpuCosineIndex
    from paper_2509_17360_b200.sharded import PipelinedShardQueries, ShardedCosineIndex
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rng = np.random.default_rng(2)
    n, d, B, k = 12000, 96, 8, 10
    rows = rng.standard_normal((n, d))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    ids = np.arange(n) * 5 + 1
    sh = ShardedCosineIndex(GpuCosineIndex(d, device=0))
    sh.insert_batch(ids, rows)
    full = O.OracleExactIndex(d)
    full.bulk_load(ids, rows)
    qs = rows[rng.integers(0, n, (9, B))] + 0.08 * rng.standard_normal((9, B, d))
    qs /= np.linalg.norm(qs, axis=2, keepdims=True)
    qd = torch.from_numpy(qs).cuda()
    certs = torch.zeros((9, B), dtype=torch.uint8, device="cuda")
    got = []
    if not pipelined:  # the plain device path, batch by batch
        for s in range(9):
            r = sh.query_device(qd[s], k, 0.2, certify=False, cert_out=certs[s])
            torch.cuda.synchronize()
            got.append((s, [t.cpu().numpy() for t in r]))
    pipe = PipelinedShardQueries(sh, B, k, depth=3)
    for s in range(9 if pipelined else 0):
        slot = pipe.submit(qd[s], 0.2, certs[s])
        if s >= 2:  # results of batch s-2 are read after a drain (its slot is reused at s+1)
            pipe.drain()
            got.append((s - 2, [t.cpu().numpy() for t in pipe.results[(s - 2) % 3]]))
    pipe.drain()
    for s in ((7, 8) if pipelined else ()):
        got.append((s, [t.cpu().numpy() for t in pipe.results[s % 3]]))
    cert = certs.cpu().numpy()
    ok = True if int(cert.sum()) >= cert.size // 2 else f"certified {int(cert.sum())} of {cert.size}"
    for s, (gi, gs, gc) in got:
        for j in range(B):
            if not cert[s, j] or ok is not True:
                continue
            want = full.query(qs[s, j], k, 0.2)
            if gi[j, :gc[j]].tolist() != [c.id for c in want]:
                ok = f"batch {s} q{j}: {gi[j, :gc[j]].tolist()} vs {[c.id for c in want]}"
            elif not np.allclose(gs[j, :gc[j]], [c.similarity for c in want], atol=1e-12, rtol=0):
                ok = f"batch {s} q{j}: sims differ"
    out[rank] = ok
    dist.destroy_process_group()


@pytest.mark.parametrize("pipelined", [False, True])
def test_pipelined_shard_queries_gloo(pipelined):
    """The device path with the all-gather on CUDA tensors, batch by batch
    and with batch i's collective + shard merge overlapping batch i+1's
    scan (PipelinedShardQueries): every certified answer equals the oracle."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        procs = [ctx.Process(target=_pipe_worker, args=(r, 2, port, out, pipelined)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(300)
        assert all(p.exitcode == 0 for p in procs)
        assert dict(out) == {0: True, 1: True}
