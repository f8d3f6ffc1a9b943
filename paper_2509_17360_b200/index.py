"""GpuCosineIndex -- the device-resident Sine stage-1 index.

Drop-in for the reference `ExactCosineIndex` (pkg/src/semcache/index.py:49-120):
same constructor arguments, `insert` / `remove` / `query` / `__len__` /
`ids` / `snapshot_lines` / `save` / `load`, attributes `dimension`, `seed`
and `SNAPSHOT_MAGIC`, the same `ValidationError`s, and results ordered by
(similarity desc, id asc) with an inclusive `min_similarity` threshold.

Pass it to `semcache.engine.CacheEngine(config, embedder, judge, index=...)`
(engine.py:103-109) or use `paper_2509_17360_b200.engine.CacheEngine`,
which also moves the LCFU eviction pass onto the device.

Modes: `scan="fp32"` (exact mode: fp32 rows, then an fp64 re-rank of the
final candidates -- similarities agree with the reference's float64 to
~1e-16) or `scan="bf16"` (fast mode: half the HBM bytes; with `rerank=True`
the candidates are still re-scored in fp64, with `rerank=False` the
similarities are the bf16/fp32-accumulated scores, within 2e-2).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import ValidationError

_NORM_TOL = 1e-6


# Device limits (documented in INTEGRATION.md): the top-k keeps k + 16
# candidates per query in shared memory (k <= 128), and the streaming scan
# holds one query in registers.
MAX_K = 128
MAX_DIM_F32 = 2048
MAX_DIM_BF16 = 4096


@dataclass(frozen=True)
class Candidate:
    """(id, similarity) -- mirrors reference index.py:26-29."""
    id: int
    similarity: float


def check_vector(vec, dimension: int) -> np.ndarray:
    """Same validation as the reference `_check_vector` (index.py:32-39)."""
    arr = np.asarray(vec.components if hasattr(vec, "components") else vec, dtype=np.float64)
    if arr.ndim != 1 or arr.shape[0] != dimension:
        raise ValidationError(f"expected dimension {dimension}, got shape {arr.shape}")
    n = float(np.linalg.norm(arr))
    if abs(n - 1.0) > _NORM_TOL:
        raise ValidationError(f"vector is not L2-normalized (norm={n:.8f})")
    return arr


def check_matrix(rows, dimension: int) -> np.ndarray:
    """Row-wise `_check_vector` for a batch.  Norms are computed vectorised;
    any row within 1e-12 of the tolerance edge is re-checked with the exact
    per-vector arithmetic of the reference, so the accept/reject decision is
    the reference's for every row."""
    arr = np.ascontiguousarray(rows, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[1] != dimension:
        raise ValidationError(f"expected rows of dimension {dimension}, got shape {arr.shape}")
    if arr.shape[0] == 0:
        return arr
    dev = np.abs(np.sqrt(np.einsum("ij,ij->i", arr, arr)) - 1.0)
    for i in np.nonzero(~(dev < _NORM_TOL - 1e-12))[0]:  # NaN rows land here too
        n = float(np.linalg.norm(arr[i]))
        if abs(n - 1.0) > _NORM_TOL:
            raise ValidationError(f"vector is not L2-normalized (norm={n:.8f})")
    return arr


class GpuCosineIndex:
    """Exact cosine index on one B200: rows stream from HBM through the
    sm_100a stage-1 kernels; the reference's result contract is preserved."""

    SNAPSHOT_MAGIC = "exact-cosine-index"

    def __init__(self, dimension: int, seed: int = 1, *, device: int = 0, scan: str = "fp32",
                 rerank: bool = True, store_bf16: bool | None = None, store_f32: bool | None = None,
                 metadata: bool = False, capacity: int = 0, host_master: bool = False):
        """host_master: keep the fp64 master rows (re-rank + snapshots) in
        pinned, device-mapped host memory instead of HBM (SINE_STORE_F64_HOST):
        8 B per dimension per row less HBM; the re-rank reads its k' rows
        per query over the host link."""
        if dimension < 1:
            raise ValidationError("dimension must be >= 1")
        if scan not in ("fp32", "bf16"):
            raise ValidationError(f"scan must be 'fp32' or 'bf16', got {scan!r}")
        if store_f32 is None:  # bf16 + re-rank keeps fp32 rows: the certificate's exact fallback
            store_f32 = scan == "fp32" or rerank
        if store_bf16 is None:
            store_bf16 = scan == "bf16"
        # the streaming scan (also the certificates' exact fallback) keeps a
        # query in registers: up to 2048 fp32 / 4096 bf16 components
        if (store_f32 and dimension > MAX_DIM_F32) or (store_bf16 and not store_f32 and dimension > MAX_DIM_BF16):
            raise ValidationError(f"dimension {dimension} exceeds the device scan limit "
                                  f"({MAX_DIM_F32} with fp32 rows, {MAX_DIM_BF16} bf16-only)")
        self.dimension = dimension
        self.seed = seed
        self.device = device
        self.scan = scan
        self.rerank = rerank
        flags = (N.STORE_F32 if store_f32 else 0) | (N.STORE_BF16 if store_bf16 else 0) | \
            (N.STORE_META if metadata else 0) | (N.STORE_F64_HOST if host_master else 0)
        self._lib = N.load_library()
        h = ctypes.c_void_p()
        N.check(self._lib.sine_create(device, dimension, flags, int(capacity), ctypes.byref(h)))
        self._h = h
        self.metadata = metadata
        self._wlock = threading.Lock()  # single writer (engine.py:95-101 discipline)

    # ---------------------------------------------------------- lifecycle
    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.sine_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def _mode(self, scan: str | None = None, rerank: bool | None = None, cuda_core: bool = False,
              umma_v1: bool = False, cluster: bool = False, pair: bool = False, gemm: bool | None = None) -> int:
        scan = scan or self.scan
        rerank = self.rerank if rerank is None else rerank
        m = N.SCAN_BF16 if scan == "bf16" else N.SCAN_F32
        if rerank:
            m |= N.RERANK_F64
        if cuda_core:
            m |= N.SCAN_CUDA_CORE
        if umma_v1:
            m |= N.SCAN_UMMA_V1
        if cluster:
            m |= N.SCAN_CLUSTER
        if pair:
            m |= N.SCAN_PAIR
        if gemm is not None:  # None: the library decides (large batches at high thresholds)
            m |= N.SCAN_GEMM if gemm else N.SCAN_NO_GEMM
        return m | N.NO_NORM_CHECK

    # ------------------------------------------------------------ queries
    def __len__(self) -> int:
        live = ctypes.c_int64()
        N.check(self._lib.sine_size(self._h, ctypes.byref(live), None))
        return live.value

    def ids(self) -> list[int]:
        """Live ids in the reference's order: insertion order, with the last
        id swapped into a removed id's position (index.py:80-92)."""
        n = len(self)
        out = np.empty(max(n, 1), dtype=np.int64)
        got = ctypes.c_int64()
        N.check(self._lib.sine_ids(self._h, N.ptr(out, ctypes.c_int64), n, ctypes.byref(got)))
        return out[:got.value].tolist()

    def insert(self, id: int, vector, meta=None) -> None:
        arr = check_vector(vector, self.dimension)
        self.insert_batch(np.array([id], dtype=np.int64), arr[None, :], meta=meta, _checked=True)

    def insert_batch(self, ids, rows, meta=None, _checked: bool = False) -> None:
        """Append many rows at once (host float64 [n, dimension])."""
        ids = N.i64(ids)
        rows = N.f64(rows) if _checked else check_matrix(rows, self.dimension)
        if rows.shape[0] != ids.shape[0]:
            raise ValidationError("ids and rows differ in length")
        cols, keep = _meta_struct(meta, ids.shape[0]) if meta is not None else (None, None)
        with self._wlock:
            N.check(self._lib.sine_insert(self._h, ids.shape[0], N.ptr(ids, ctypes.c_int64),
                                          N.ptr(rows, ctypes.c_double),
                                          ctypes.byref(cols) if cols is not None else None,
                                          N.NO_NORM_CHECK))
        del keep

    def insert_device(self, ids, rows_dev_ptr: int, meta=None) -> None:
        """Bulk append from device memory (float64 [n, dimension], already
        unit-norm -- e.g. a torch CUDA tensor's data_ptr())."""
        ids = N.i64(ids)
        cols, keep = _meta_struct(meta, ids.shape[0]) if meta is not None else (None, None)
        with self._wlock:
            N.check(self._lib.sine_insert_device(self._h, ids.shape[0], N.ptr(ids, ctypes.c_int64),
                                                 ctypes.c_void_p(rows_dev_ptr),
                                                 ctypes.byref(cols) if cols is not None else None, 0))
        del keep

    def remove(self, id: int) -> None:
        self.remove_batch([id])

    def remove_batch(self, ids) -> None:
        ids = N.i64(ids)
        if ids.size == 0:
            return
        with self._wlock:
            N.check(self._lib.sine_remove(self._h, ids.shape[0], N.ptr(ids, ctypes.c_int64)))

    def query(self, vector, k: int, min_similarity: float = -1.0) -> list[Candidate]:
        """Reference `ExactCosineIndex.query` (index.py:94-102) on the GPU."""
        arr = check_vector(vector, self.dimension)
        if k < 1:
            raise ValidationError("k must be >= 1")
        ids, sims, counts = self._query(arr[None, :], k, min_similarity, self._mode())
        n = int(counts[0])
        return [Candidate(int(ids[0, j]), float(sims[0, j])) for j in range(n)]

    def query_batch(self, queries, k: int, min_similarity: float = -1.0, *, scan: str | None = None,
                    rerank: bool | None = None, check: bool = True, cuda_core: bool = False,
                    umma_v1: bool = False, cluster: bool = False, pair: bool = False, gemm: bool | None = None):
        """B independent queries in one pass over the index.

        Returns (ids int64[B, k] padded with -1, sims float64[B, k],
        counts int32[B]); row b equals query(queries[b], k, min_similarity)."""
        q = check_matrix(queries, self.dimension) if check else N.f64(queries)
        if k < 1:
            raise ValidationError("k must be >= 1")
        return self._query(q, k, min_similarity, self._mode(scan, rerank, cuda_core, umma_v1, cluster, pair, gemm))

    def _query(self, q: np.ndarray, k: int, min_similarity: float, mode: int):
        B = q.shape[0]
        ids = np.empty((B, k), dtype=np.int64)
        sims = np.empty((B, k), dtype=np.float64)
        counts = np.empty(B, dtype=np.int32)
        N.check(self._lib.sine_query(self._h, B, N.ptr(q, ctypes.c_double), int(k), float(min_similarity),
                                     mode, N.ptr(ids, ctypes.c_int64), N.ptr(sims, ctypes.c_double),
                                     N.ptr(counts, ctypes.c_int32)))
        return ids, sims, counts

    def query_into(self, q: np.ndarray, k: int, min_similarity: float, ids: np.ndarray, sims: np.ndarray,
                   counts: np.ndarray, *, scan: str | None = None, rerank: bool | None = None) -> None:
        """query_batch writing into caller buffers (e.g. pinned host memory)."""
        N.check(self._lib.sine_query(self._h, q.shape[0], N.ptr(q, ctypes.c_double), int(k),
                                     float(min_similarity), self._mode(scan, rerank),
                                     N.ptr(ids, ctypes.c_int64), N.ptr(sims, ctypes.c_double),
                                     N.ptr(counts, ctypes.c_int32)))

    def submit_into(self, q: np.ndarray, k: int, min_similarity: float, ids: np.ndarray, sims: np.ndarray,
                    counts: np.ndarray, *, scan: str | None = None, rerank: bool | None = None) -> int:
        """Asynchronous query_into (sine_query_submit): the caller's buffers
        must stay untouched until wait_ticket(ticket) returns (pinned queries
        upload fastest; the device writes results into the handle's mapped
        staging and wait_ticket copies them out); up to 16 batches in
        flight, executed in submission order."""
        t = ctypes.c_int64()
        N.check(self._lib.sine_query_submit(self._h, q.shape[0], q.ctypes.data, int(k), float(min_similarity),
                                            self._mode(scan, rerank), ids.ctypes.data, sims.ctypes.data,
                                            counts.ctypes.data, ctypes.byref(t)))
        return t.value

    def wait_ticket(self, ticket: int) -> None:
        """Block until a submit_into batch's results (certified) are in its buffers."""
        N.check(self._lib.sine_query_wait(self._h, int(ticket)))

    def query_device(self, B: int, q_ptr: int, k: int, min_similarity: float, ids_ptr: int, sims_ptr: int,
                     counts_ptr: int, stream: int | None = None, *, scan: str | None = None,
                     rerank: bool | None = None, cuda_core: bool = False, umma_v1: bool = False,
                     certify: bool = True, pair: bool = False, gemm: bool | None = None) -> None:
        """Device-pointer variant (torch tensors); enqueued on `stream`.

        With `certify` (default) the per-query exactness certificate is
        checked and failing queries are re-run on the fp32 scan; this
        synchronises the stream once per call."""
        mode = self._mode(scan, rerank, cuda_core, umma_v1, pair=pair, gemm=gemm) | (N.CERTIFY if certify else 0)
        N.check(self._lib.sine_query_device(self._h, int(B), ctypes.c_void_p(q_ptr), int(k),
                                            float(min_similarity), mode,
                                            ctypes.c_void_p(ids_ptr), ctypes.c_void_p(sims_ptr),
                                            ctypes.c_void_p(counts_ptr),
                                            _stream_arg(stream)))

    def query_device_cert(self, B: int, q_ptr: int, k: int, min_similarity: float, ids_ptr: int, sims_ptr: int,
                          counts_ptr: int, cert_ptr: int, stream: int | None = None, *, scan: str | None = None,
                          rerank: bool | None = None, cuda_core: bool = False, umma_v1: bool = False,
                          pair: bool = False, gemm: bool | None = None) -> None:
        """query_device writing the exactness certificates (uint8 [B], device)
        to `cert_ptr` on the stream: no sync; the caller re-runs any 0."""
        mode = self._mode(scan, rerank, cuda_core, umma_v1, pair=pair, gemm=gemm)
        N.check(self._lib.sine_query_device_cert(self._h, int(B), ctypes.c_void_p(q_ptr), int(k),
                                                 float(min_similarity), mode,
                                                 ctypes.c_void_p(ids_ptr), ctypes.c_void_p(sims_ptr),
                                                 ctypes.c_void_p(counts_ptr), ctypes.c_void_p(cert_ptr),
                                                 _stream_arg(stream)))

    def query_batch_async(self, queries, k: int, min_similarity: float = -1.0, *, check: bool = True,
                          scan: str | None = None, rerank: bool | None = None) -> "PendingQuery":
        """Start a batched stage-1 on the device and return immediately; the
        host can work (e.g. run the stage-2 judge on the previous batch)
        until `.wait()` returns (ids, sims, counts)."""
        q = check_matrix(queries, self.dimension) if check else N.f64(queries)
        if k < 1:
            raise ValidationError("k must be >= 1")
        return PendingQuery(self, q, k, min_similarity, self._mode(scan, rerank))

    # --------------------------------------------------------- timing hooks
    def set_timing(self, on: bool = True) -> None:
        N.check(self._lib.sine_set_timing(self._h, 1 if on else 0))

    def last_timing(self):
        a, b, c = ctypes.c_float(), ctypes.c_float(), ctypes.c_float()
        N.check(self._lib.sine_last_timing(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def timing_totals(self, kind: int = 0, reset: bool = True):
        """(total device ms, launches) of kernel kind 0=scan, 1=merge, 2=umma."""
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        N.check(self._lib.sine_timing_totals(self._h, kind, ctypes.byref(ms), ctypes.byref(n), 1 if reset else 0))
        return ms.value, n.value

    def copy_certificates(self, B: int, dst_ptr: int, stream: int | None = None) -> None:
        """Enqueue a device copy of the last batch's exactness certificates."""
        N.check(self._lib.sine_copy_certificates(self._h, int(B), ctypes.c_void_p(dst_ptr),
                                                 _stream_arg(stream)))

    def uncertified(self) -> int:
        """Queries the last (certified) call re-ran on the fp32 scan."""
        n = ctypes.c_int64()
        N.check(self._lib.sine_uncertified(self._h, ctypes.byref(n)))
        return n.value

    def gemm_overflows(self) -> int:
        """Tiled-GEMM launches whose candidates overflowed (re-run on the
        list-keeping kernels)."""
        n = ctypes.c_int64()
        N.check(self._lib.sine_gemm_overflows(self._h, ctypes.byref(n)))
        return n.value

    def kernel_launches(self) -> int:
        n = ctypes.c_int64()
        N.check(self._lib.sine_kernel_launches(self._h, ctypes.byref(n)))
        return n.value

    def stream(self) -> int:
        s = ctypes.c_void_p()
        N.check(self._lib.sine_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    # ----------------------------------------------------------- snapshots
    def rows(self, ids) -> np.ndarray:
        ids = N.i64(ids)
        out = np.empty((ids.shape[0], self.dimension), dtype=np.float64)
        if ids.size:
            N.check(self._lib.sine_get_rows(self._h, ids.shape[0], N.ptr(ids, ctypes.c_int64),
                                            N.ptr(out, ctypes.c_double)))
        return out

    def snapshot_lines(self) -> list[str]:
        """Reference snapshot format (index.py:340-354): header + one line of
        float-hex components per id, in `ids()` order."""
        return self.snapshot_bytes().decode().split("\n")[:-1]

    def snapshot_bytes(self) -> bytes:
        """The reference snapshot file (index.py:340-354, _write_snapshot
        :376-379) as bytes: the rows are gathered on the device and the
        float-hex body is formatted natively (byte-identical text)."""
        head, body = self._snapshot_parts()
        return head + bytes(body)

    def snapshot(self):
        """(ids int64[n], rows float64[n, dimension]) in `ids()` order, taken
        under one hold of the handle lock (sine_snapshot), so a concurrent
        insert or removal cannot split the two."""
        cap = len(self) + 64
        while True:
            ids = np.empty(max(cap, 1), dtype=np.int64)
            rows = np.empty((max(cap, 1), self.dimension), dtype=np.float64)
            n = ctypes.c_int64()
            st = self._lib.sine_snapshot(self._h, cap, N.ptr(ids, ctypes.c_int64), N.ptr(rows, ctypes.c_double),
                                         ctypes.byref(n))
            if st == N.SINE_EINVAL and n.value > cap:
                cap = n.value + 64  # grew in between: retry with room
                continue
            N.check(st)
            return ids[:n.value], rows[:n.value]

    def _snapshot_parts(self):
        ids, rows = self.snapshot()
        head = "\n".join([self.SNAPSHOT_MAGIC, f"dimension: {self.dimension}", f"seed: {self.seed}",
                          f"count: {len(ids)}"]) + "\n"
        body = N.hex_format(rows, ids) if len(ids) else memoryview(b"")
        return head.encode(), body

    def save(self, path: str) -> None:
        head, body = self._snapshot_parts()
        with open(path, "wb") as fh:
            fh.write(head)
            fh.write(body)

    def write_snapshot(self, fh) -> None:
        """Append the snapshot to an open binary file (engine state files)."""
        head, body = self._snapshot_parts()
        fh.write(head)
        fh.write(body)

    @classmethod
    def load(cls, path: str, **kwargs) -> "GpuCosineIndex":
        with open(path, "rb") as fh:
            data = fh.read()
        dimension, seed, ids, rows = parse_snapshot_bytes(data, cls.SNAPSHOT_MAGIC)
        idx = cls(dimension, seed=seed, **kwargs)
        if len(ids):
            idx.insert_batch(ids, rows)
        return idx


def parse_snapshot_lines(lines: list[str], magic: str):
    """Reader for the reference snapshot format (index.py:357-373)."""
    if not lines or lines[0] != magic:
        raise ValidationError(f"snapshot is not a {magic} file")
    try:
        dimension = int(lines[1].split(":", 1)[1])
        seed = int(lines[2].split(":", 1)[1])
        count = int(lines[3].split(":", 1)[1])
    except (IndexError, ValueError) as exc:
        raise ValidationError(f"malformed snapshot header: {exc}") from exc
    body = lines[4:4 + count]
    if len(body) != count:
        raise ValidationError(f"snapshot count {count} does not match {len(body)} entries")
    entries = []
    for line in body:
        head, _, rest = line.partition(" ")
        vec = np.array([float.fromhex(p) for p in rest.split(" ")]) if rest else np.zeros(0)
        entries.append((int(head), vec))
    return dimension, seed, entries


_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


def _stream_arg(stream):
    """None -> the handle's own stream (C ABI NULL); 0 -> the CUDA legacy
    default stream (what torch's default stream handle 0 means: work must be
    ordered with the caller's default-stream kernels); else the handle."""
    if stream is None:
        return None
    return ctypes.c_void_p(stream if stream else _CUDA_STREAM_LEGACY)


def parse_snapshot_bytes(data: bytes, magic: str):
    """Native reader for the reference snapshot format (index.py:357-373):
    header lines parsed here, the float-hex body by the library.  Returns
    (dimension, seed, ids int64[count], rows float64[count, dimension])."""
    head, off = [], 0
    for _ in range(4):  # header lines only; the body is parsed in place
        nl = data.find(b"\n", off)
        head.append(data[off:] if nl < 0 else data[off:nl])
        off = len(data) if nl < 0 else nl + 1
    if head[0].decode(errors="replace") != magic:
        raise ValidationError(f"snapshot is not a {magic} file")
    try:
        dimension = int(head[1].split(b":", 1)[1])
        seed = int(head[2].split(b":", 1)[1])
        count = int(head[3].split(b":", 1)[1])
    except (IndexError, ValueError) as exc:
        raise ValidationError(f"malformed snapshot header: {exc}") from exc
    if count and dimension >= 1:
        ids, rows = N.hex_parse(data, count, dimension, True, offset=off)
    else:
        ids, rows = np.empty(0, dtype=np.int64), np.empty((0, max(dimension, 0)))
    return dimension, seed, ids, rows


def _meta_struct(meta: dict, n: int):
    """Pack LCFU metadata columns (dict of arrays, length n) for the C ABI."""
    keep = {}
    cols = N.MetaCols()
    for name, kind in (("log_freq", "f"), ("log_cost", "f"), ("log_lat", "f"), ("log_stat", "f"),
                       ("frequency", "i"), ("size_tokens", "i"), ("created_at", "f"),
                       ("expiration_time", "f"), ("last_access", "f")):
        a = N.f64(meta[name]) if kind == "f" else N.i64(meta[name])
        if a.shape[0] != n:
            raise ValidationError(f"metadata column {name} has {a.shape[0]} entries, expected {n}")
        keep[name] = a
        setattr(cols, name, N.ptr(a, ctypes.c_double if kind == "f" else ctypes.c_int64))
    return cols, keep


class PendingQuery:
    """An in-flight `query_batch_async` batch (pinned host buffers)."""

    def __init__(self, index: GpuCosineIndex, q: np.ndarray, k: int, min_similarity: float, mode: int):
        B = q.shape[0]
        self._index = index
        self._q = N.PinnedArray(q.shape, np.float64)
        self._q.array[:] = q
        self._ids = N.PinnedArray((B, k), np.int64)
        self._sims = N.PinnedArray((B, k), np.float64)
        self._counts = N.PinnedArray((B,), np.int32)
        t = ctypes.c_int64()
        N.check(index._lib.sine_query_submit(index.handle, B, self._q.array.ctypes.data, int(k),
                                             float(min_similarity), mode, self._ids.array.ctypes.data,
                                             self._sims.array.ctypes.data, self._counts.array.ctypes.data,
                                             ctypes.byref(t)))
        self._ticket = t.value
        self._result = None

    def wait(self):
        if self._result is None:
            try:
                N.check(self._index._lib.sine_query_wait(self._index.handle, self._ticket))
            finally:
                self._ticket = None  # the library freed the ticket (or it was never valid)
            self._result = (self._ids.array.copy(), self._sims.array.copy(), self._counts.array.copy())
        return self._result

    def close(self) -> None:
        """Release the ticket of a batch whose results are not needed (its
        pinned buffers stay alive until the device is done with them)."""
        if self._result is None and getattr(self, "_ticket", None) is not None:
            try:
                self.wait()
            except Exception:  # noqa: BLE001 - best effort: the ticket is freed either way
                pass

    def __del__(self):
        self.close()
