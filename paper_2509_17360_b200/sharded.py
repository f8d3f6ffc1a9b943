"""Row-sharded Sine stage-1 across the GPUs of one box (config C).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Every
rank owns a contiguous-by-arrival share of the SE rows in its own
`GpuCosineIndex`; a batch of B queries is scanned by every rank against its
shard, each rank produces its exact local top-k (fp64 re-ranked), and one
all-gather of the B x k (similarity, id) candidates per rank is merged on
every rank with the reference comparator (similarity desc, id asc,
index.py:45).  Because each local list is the exact top-k of its shard,
the merged list equals the single-index result.

Bookkeeping (id -> owner rank, rows per rank) is replicated: all ranks see
the same insert/remove sequence (SPMD), and a new row goes to the
least-full rank (lowest rank on ties).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .errors import ValidationError


def merge_topk(sims: torch.Tensor, ids: torch.Tensor, k: int):
    """Merge per-rank candidate lists.

    sims/ids: [P, B, k] (ids == -1 marks padding).  Returns (ids [B, k]
    -1 padded, sims [B, k], counts [B]) ordered by (sim desc, id asc)."""
    P, B, kk = sims.shape
    s = sims.permute(1, 0, 2).reshape(B, P * kk).clone()
    i = ids.permute(1, 0, 2).reshape(B, P * kk).clone()
    pad = i < 0
    s[pad] = -float("inf")
    i_key = torch.where(pad, torch.full_like(i, torch.iinfo(torch.int64).max), i)
    # stable two-key sort: id ascending, then similarity descending
    o1 = torch.argsort(i_key, dim=1, stable=True)
    s1, i1 = torch.gather(s, 1, o1), torch.gather(i_key, 1, o1)
    o2 = torch.argsort(-s1, dim=1, stable=True)
    s2, i2 = torch.gather(s1, 1, o2)[:, :k], torch.gather(i1, 1, o2)[:, :k]
    valid = torch.isfinite(s2)
    counts = valid.sum(dim=1).to(torch.int32)
    i2 = torch.where(valid, i2, torch.full_like(i2, -1))
    s2 = torch.where(valid, s2, torch.zeros_like(s2))
    return i2, s2, counts


def place_least_full(counts: np.ndarray, n: int) -> np.ndarray:
    """Owners of n new rows, each to the least-full rank at its turn (lowest
    rank on ties) -- the sequential greedy rule, vectorised: the j-th row
    takes the j-th smallest (level, rank) pair with level >= counts[rank]."""
    P = counts.shape[0]
    if n <= 0:
        return np.empty(0, dtype=np.int64)
    levels = np.unique(counts)
    parts, have = [], 0
    for a, b in zip(levels, list(levels[1:]) + [None]):
        elig = np.nonzero(counts <= a)[0]  # ranks already at or below level a, in rank order
        reps = (b - a) if b is not None else -(-(n - have) // P)
        reps = min(reps, -(-(n - have) // len(elig)))
        parts.append(np.tile(elig, reps))
        have += reps * len(elig)
        if have >= n:
            break
    return np.concatenate(parts)[:n].astype(np.int64)


class ShardedCosineIndex:
    """SPMD wrapper: call every method on every rank with the same args."""

    def __init__(self, local_index, group=None):
        if not dist.is_initialized():
            raise ValidationError("ShardedCosineIndex needs an initialised torch.distributed group")
        self.local = local_index
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.dimension = local_index.dimension
        self._owner: dict[int, int] = {}
        self._rows = [0] * self.world

    def __len__(self) -> int:
        return len(self._owner)

    def _place(self, n: int) -> np.ndarray:
        owners = place_least_full(np.asarray(self._rows, dtype=np.int64), n)
        self._rows = (np.asarray(self._rows) + np.bincount(owners, minlength=self.world)).tolist()
        return owners

    def insert_batch(self, ids, rows) -> None:
        ids = np.asarray(ids, dtype=np.int64)
        id_list = ids.tolist()
        if len(set(id_list)) != len(id_list) or not self._owner.keys().isdisjoint(id_list):
            dup = next(i for i in id_list if i in self._owner or id_list.count(i) > 1)
            raise ValidationError(f"duplicate id {dup}")
        owners = self._place(ids.shape[0])
        self._owner.update(zip(id_list, owners.tolist()))
        mine = owners == self.rank
        if mine.any():
            self.local.insert_batch(ids[mine], np.asarray(rows)[mine])

    def remove_batch(self, ids) -> None:
        ids = [int(i) for i in ids]
        for i in ids:
            if i not in self._owner:
                raise ValidationError(f"unknown id {i}")
        mine = [i for i in ids if self._owner[i] == self.rank]
        for i in ids:
            self._rows[self._owner.pop(i)] -= 1
        if mine:
            self.local.remove_batch(mine)

    def query_batch(self, queries, k: int, min_similarity: float = -1.0):
        """Exact top-k over all shards; returns numpy (ids, sims, counts).
        With NCCL the host queries go to the device once and take the
        device path (one all-gather + the shard-merge kernel)."""
        if dist.get_backend(self.group) == "nccl":
            from .index import check_matrix
            q = torch.from_numpy(check_matrix(queries, self.dimension)).to(
                torch.device("cuda", torch.cuda.current_device()))
            mi, ms, mc = self.query_device(q, k, min_similarity)
            return mi.cpu().numpy(), ms.cpu().numpy(), mc.cpu().numpy()
        ids, sims, _ = self.local.query_batch(queries, k, min_similarity)
        dev = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        t_ids = torch.as_tensor(ids, device=dev)
        t_sims = torch.as_tensor(sims, device=dev)
        B = t_ids.shape[0]
        g_ids = torch.empty((self.world * B, k), dtype=t_ids.dtype, device=dev)
        g_sims = torch.empty((self.world * B, k), dtype=t_sims.dtype, device=dev)
        dist.all_gather_into_tensor(g_ids, t_ids, group=self.group)
        dist.all_gather_into_tensor(g_sims, t_sims, group=self.group)
        mi, ms, mc = merge_topk(g_sims.view(self.world, B, k), g_ids.view(self.world, B, k), k)
        return mi.cpu().numpy(), ms.cpu().numpy(), mc.cpu().numpy()

    def query_device(self, q: torch.Tensor, k: int, min_similarity: float = -1.0, *, certify: bool = True,
                     cert_out: torch.Tensor | None = None):
        """Device-resident variant (NCCL): q is a CUDA float64 [B, d] tensor.
        The local scan writes ids and similarity bits into one int64 block
        [2, B, k] on torch's current stream; ONE all-gather moves every
        rank's block and the library's shard-merge kernel produces the
        global top-k -- no host round trip.  certify=False skips the
        per-call certificate sync; pass cert_out (uint8 [B], device) to log
        the local certificates for a later check."""
        B = q.shape[0]
        stream = torch.cuda.current_stream().cuda_stream
        block = torch.empty((2, B, k), dtype=torch.int64, device=q.device)
        counts = torch.empty((B,), dtype=torch.int32, device=q.device)
        if cert_out is not None:  # certificates straight into the caller's device log
            self.local.query_device_cert(B, q.data_ptr(), k, min_similarity, block[0].data_ptr(),
                                         block[1].data_ptr(), counts.data_ptr(), cert_out.data_ptr(), stream)
        else:
            self.local.query_device(B, q.data_ptr(), k, min_similarity, block[0].data_ptr(), block[1].data_ptr(),
                                    counts.data_ptr(), stream, certify=certify)
        g = torch.empty((self.world, 2, B, k), dtype=torch.int64, device=q.device)
        dist.all_gather_into_tensor(g.view(-1), block.view(-1), group=self.group)
        return merge_gathered_blocks(g)


def merge_gathered_blocks(g: torch.Tensor):
    """g: CUDA int64 [P, 2, B, k] -- per rank, ids then similarity bits (the
    all-gather of ShardedCosineIndex.query_device's blocks).  One device
    kernel (sine_merge_shards) -> (ids [B, k] -1 padded, sims, counts)."""
    P, _, B, k = g.shape
    out_ids = torch.empty((B, k), dtype=torch.int64, device=g.device)
    out_sims = torch.empty((B, k), dtype=torch.float64, device=g.device)
    out_cnt = torch.empty((B,), dtype=torch.int32, device=g.device)
    N.check(N.load_library().sine_merge_shards(g.device.index, P, B, k, g.data_ptr(), g[0, 1].data_ptr(), 2 * B * k,
                                               out_ids.data_ptr(), out_sims.data_ptr(), out_cnt.data_ptr(),
                                               torch.cuda.current_stream().cuda_stream))
    return out_ids, out_sims, out_cnt


class PipelinedShardQueries:
    """Overlaps batch i's all-gather + shard merge with batch i+1's local
    scan.  The local pipeline (prep, scan, merge; shared device workspaces)
    stays on the caller's stream in submission order; each batch's [2, B, k]
    block is its own slot, and the collective plus the shard-merge kernel
    run on a second stream after an event.  A slot is rewritten only after
    its previous collective finished (event wait on the caller's stream).

    Exactness: each rank logs its local certificates on the device; `finish()`
    (SPMD, every rank) combines them with one MIN all-reduce and re-runs every
    query whose certificate failed on ANY rank through the certified path
    (`ShardedCosineIndex.query_device`), patching the held results -- no host
    sync per batch.  Writers must not run between `submit` and `finish` (the
    re-run reads the store as it is then).  The last `depth` batches' results
    are held; call `finish()` before reading them."""

    def __init__(self, sharded: ShardedCosineIndex, B: int, k: int, depth: int = 4, device=None):
        self.sh = sharded
        self.B, self.k, self.depth = B, k, depth
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.blocks = [torch.empty((2, B, k), dtype=torch.int64, device=dev) for _ in range(depth)]
        self.gathered = [torch.empty((sharded.world, 2, B, k), dtype=torch.int64, device=dev) for _ in range(depth)]
        self.counts = torch.empty((B,), dtype=torch.int32, device=dev)
        self.comm = torch.cuda.Stream(device=dev)
        self.done = [None] * depth
        self.results = [None] * depth
        self.n = 0
        self._log = []  # (batch number, queries, min_similarity, cert log) since the last finish()

    def submit(self, q: torch.Tensor, min_similarity: float, cert_out: torch.Tensor):
        """Enqueue one batch (CUDA float64 [B, d]); returns its slot."""
        slot = self.n % self.depth
        self.n += 1
        main = torch.cuda.current_stream()
        if self.done[slot] is not None:
            main.wait_event(self.done[slot])  # the slot's previous collective has read its block
        blk = self.blocks[slot]
        self.sh.local.query_device_cert(self.B, q.data_ptr(), self.k, min_similarity, blk[0].data_ptr(),
                                        blk[1].data_ptr(), self.counts.data_ptr(), cert_out.data_ptr(),
                                        main.cuda_stream)
        ready = torch.cuda.Event()
        ready.record(main)
        with torch.cuda.stream(self.comm):
            self.comm.wait_event(ready)
            g = self.gathered[slot]
            dist.all_gather_into_tensor(g.view(-1), blk.view(-1), group=self.sh.group)
            self.results[slot] = merge_gathered_blocks(g)
            ev = torch.cuda.Event()
            ev.record(self.comm)
            self.done[slot] = ev
        self._log.append((self.n - 1, q, min_similarity, cert_out))
        return slot

    def drain(self):
        torch.cuda.current_stream().wait_stream(self.comm)

    def finish(self) -> int:
        """Drain, then re-run (on every rank) the queries any rank could not
        certify; returns how many were re-run.  Collective: call on all ranks."""
        self.drain()
        log, self._log = self._log, []
        if not log:
            return 0
        flags = torch.cat([c.view(-1) for _, _, _, c in log]).to(torch.int32)
        dist.all_reduce(flags, op=dist.ReduceOp.MIN, group=self.sh.group)
        bad = (flags == 0).nonzero().flatten().tolist()  # same list on every rank
        fixed = 0
        for f in bad:
            b, j = divmod(f, self.B)
            n_b, q, ms, cert = log[b]
            ids, sims, cnt = self.sh.query_device(q[j:j + 1], self.k, ms, certify=True)
            cert[j] = 1
            fixed += 1
            if n_b >= self.n - self.depth:  # results still held: patch row j
                ri, rs, rc = self.results[n_b % self.depth]
                ri[j].copy_(ids[0])
                rs[j].copy_(sims[0])
                rc[j].copy_(cnt[0])
        return fixed
