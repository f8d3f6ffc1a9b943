"""Single-process multi-GPU drop-in for `semcache.index.ExactCosineIndex`.

The reference engine is single-process and takes one duck-typed index
(pkg/src/semcache/engine.py:103-109).  `MultiDeviceCosineIndex` is that one
index, spread over several GPUs of the node: P row shards (one
`GpuCosineIndex` per entry of `devices`; entries may repeat a device), a
native group handle (csrc/group.cu) that runs each query on every shard at
once and merges the per-shard exact top-k lists on the first device, and
the reference's index surface on top:

* `query(vector, k, min_similarity)` / `query_batch` -- equal to
  ExactCosineIndex.query (index.py:94-102) on the union of the shards;
* `insert` / `insert_batch` place new ids on the least-full shard;
  `remove` finds the owner; duplicate / unknown ids raise ValidationError
  (index.py:74-75, :82-83);
* `ids()`, `snapshot_lines()`, `save` / `load` follow the reference's id
  order (append on insert, the last id swapped into a removed id's place,
  index.py:71-92), kept on the host in O(1) per operation.

Writers (insert / remove) and queries are serialised by one lock, so every
query sees one consistent state of all shards (ref SPEC.md:183).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as N
from .errors import ValidationError
from .index import Candidate, GpuCosineIndex, check_matrix, check_vector, parse_snapshot_bytes


class MultiDeviceCosineIndex:
    SNAPSHOT_MAGIC = "exact-cosine-index"

    def __init__(self, dimension: int, seed: int = 1, *, devices=(0,), scan: str = "fp32", rerank: bool = True,
                 capacity: int = 0):
        devices = [int(d) for d in devices]
        if not devices:
            raise ValidationError("at least one device")
        self.dimension = dimension
        self.seed = seed
        self.devices = devices
        per = (capacity + len(devices) - 1) // len(devices) if capacity else 0
        self.shards = [GpuCosineIndex(dimension, seed, device=d, scan=scan, rerank=rerank, capacity=per)
                       for d in devices]
        self._mode = self.shards[0]._mode()
        self._lib = N.load_library()
        hs = (ctypes.c_void_p * len(devices))(*[s.handle.value for s in self.shards])
        ds = (ctypes.c_int * len(devices))(*devices)
        g = ctypes.c_void_p()
        N.check(self._lib.sine_group_create(hs, ds, len(devices), dimension, ctypes.byref(g)))
        self._g = g
        self._lock = threading.Lock()
        self._owner: dict[int, int] = {}   # id -> shard
        self._order: list[int] = []        # reference id order
        self._pos: dict[int, int] = {}     # id -> position in _order
        self._count = [0] * len(devices)

    # ---------------------------------------------------------- lifecycle
    def close(self) -> None:
        g = getattr(self, "_g", None)
        if g is not None and g.value:
            self._lib.sine_group_destroy(g)
            self._g = None
        for s in getattr(self, "shards", []):
            s.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    # ------------------------------------------------------------ surface
    def __len__(self) -> int:
        return len(self._order)

    def ids(self) -> list[int]:
        with self._lock:
            return list(self._order)

    def insert(self, id: int, vector) -> None:
        self.insert_batch([id], check_vector(vector, self.dimension)[None, :], _checked=True)

    def insert_batch(self, ids, rows, _checked: bool = False) -> None:
        ids = [int(i) for i in ids]
        arr = np.ascontiguousarray(rows, dtype=np.float64) if _checked else check_matrix(rows, self.dimension)
        if len(set(ids)) != len(ids):
            raise ValidationError("duplicate id in batch")
        with self._lock:
            for i in ids:
                if i in self._owner:
                    raise ValidationError(f"duplicate id {i}")
            # least-full placement, vectorised: top the shards up towards the
            # balanced sizes of the new total (the shortfalls sum to >= the
            # batch, so the first len(ids) slots of the repeat suffice)
            P = len(self.shards)
            total = sum(self._count) + len(ids)
            want = [max(0, (total + P - 1 - p) // P - self._count[p]) for p in range(P)]
            assign = np.repeat(np.arange(P), want)[:len(ids)]
            idv = np.asarray(ids, dtype=np.int64)
            for p in range(P):
                sel = np.nonzero(assign == p)[0]
                if sel.size:
                    self.shards[p].insert_batch(idv[sel], arr[sel], _checked=True)
                    self._count[p] += int(sel.size)
            for i, p in zip(ids, assign.tolist()):
                self._owner[i] = p
                self._pos[i] = len(self._order)
                self._order.append(i)

    def remove(self, id: int) -> None:
        self.remove_batch([id])

    def remove_batch(self, ids) -> None:
        ids = [int(i) for i in ids]
        with self._lock:
            for i in ids:
                if i not in self._owner:
                    raise ValidationError(f"unknown id {i}")
            by = {}
            for i in ids:
                by.setdefault(self._owner[i], []).append(i)
            for p, lst in by.items():
                self.shards[p].remove_batch(lst)
                self._count[p] -= len(lst)
            for i in ids:  # index.py:80-92: swap the last id into the hole
                del self._owner[i]
                at = self._pos.pop(i)
                last = self._order.pop()
                if last != i:
                    self._order[at] = last
                    self._pos[last] = at

    def query(self, vector, k: int, min_similarity: float = -1.0) -> list[Candidate]:
        """ExactCosineIndex.query (index.py:94-102) over all shards."""
        arr = check_vector(vector, self.dimension)
        if k < 1:
            raise ValidationError("k must be >= 1")
        ids, sims, counts = self._query(arr[None, :], k, min_similarity)
        return [Candidate(int(ids[0, j]), float(sims[0, j])) for j in range(int(counts[0]))]

    def query_batch(self, queries, k: int, min_similarity: float = -1.0):
        """(ids int64[B, k] -1 padded, sims float64[B, k], counts int32[B])."""
        q = check_matrix(queries, self.dimension)
        if k < 1:
            raise ValidationError("k must be >= 1")
        return self._query(q, k, min_similarity)

    def _query(self, q: np.ndarray, k: int, min_similarity: float):
        B = q.shape[0]
        ids = np.full((B, k), -1, dtype=np.int64)
        sims = np.zeros((B, k), dtype=np.float64)
        counts = np.zeros(B, dtype=np.int32)
        if B == 0:
            return ids, sims, counts
        with self._lock:
            if not self._order:
                return ids, sims, counts
            N.check(self._lib.sine_group_query(self._g, B, N.ptr(q, ctypes.c_double), int(k), float(min_similarity),
                                               self._mode | N.NO_NORM_CHECK, N.ptr(ids, ctypes.c_int64),
                                               N.ptr(sims, ctypes.c_double), N.ptr(counts, ctypes.c_int32)))
        return ids, sims, counts

    # --------------------------------------------------------- persistence
    def rows(self, ids) -> np.ndarray:
        ids = [int(i) for i in ids]
        out = np.empty((len(ids), self.dimension), dtype=np.float64)
        by = {}
        for j, i in enumerate(ids):
            by.setdefault(self._owner[i], []).append(j)
        for p, js in by.items():
            out[js] = self.shards[p].rows([ids[j] for j in js])
        return out

    def snapshot_bytes(self) -> bytes:
        with self._lock:
            ids = list(self._order)
            rows = self.rows(ids) if ids else np.empty((0, self.dimension))
        head = "\n".join([self.SNAPSHOT_MAGIC, f"dimension: {self.dimension}", f"seed: {self.seed}",
                          f"count: {len(ids)}"]) + "\n"
        body = bytes(N.hex_format(rows, np.asarray(ids, dtype=np.int64))) if ids else b""
        return head.encode() + body

    def snapshot_lines(self) -> list[str]:
        """Reference snapshot format (index.py:340-354), in `ids()` order."""
        return self.snapshot_bytes().decode().split("\n")[:-1]

    def save(self, path: str) -> None:
        with open(path, "wb") as fh:
            fh.write(self.snapshot_bytes())

    @classmethod
    def load(cls, path: str, **kwargs) -> "MultiDeviceCosineIndex":
        with open(path, "rb") as fh:
            data = fh.read()
        dimension, seed, ids, rows = parse_snapshot_bytes(data, cls.SNAPSHOT_MAGIC)
        idx = cls(dimension, seed, **kwargs)
        if len(ids):
            idx.insert_batch(ids.tolist(), rows)
        return idx
