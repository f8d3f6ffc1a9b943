"""ctypes binding of libsine_b200.so (the C ABI in include/sine_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
There is no fallback: if the shared object is missing or no CUDA device is
visible, every constructor raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import ValidationError

# SINE_LIB_PATH: another build of the library (same-box A/B timing runs)
LIB_PATH = os.environ.get("SINE_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                           "libsine_b200.so")

SINE_OK, SINE_EINVAL, SINE_ECUDA, SINE_ENCCL, SINE_ENOMEM, SINE_ENOTFOUND, SINE_EDUP, SINE_ENORM = range(8)

STORE_F32, STORE_BF16, STORE_META, STORE_F64_HOST = 0x1, 0x2, 0x4, 0x8
SCAN_F32, SCAN_BF16, RERANK_F64, NO_NORM_CHECK, SCAN_CUDA_CORE, SCAN_UMMA_V1, CERTIFY, SCAN_CLUSTER, SCAN_PAIR = \
    0x0, 0x1, 0x10, 0x100, 0x200, 0x400, 0x800, 0x1000, 0x2000
SCAN_GEMM, SCAN_NO_GEMM = 0x4000, 0x8000
POLICIES = {"lcfu": 0, "lru": 1, "lfu": 2}

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)


class MetaCols(ctypes.Structure):
    _fields_ = [(n, _f64p) for n in ("log_freq", "log_cost", "log_lat", "log_stat")] + \
               [(n, _i64p) for n in ("frequency", "size_tokens")] + \
               [(n, _f64p) for n in ("created_at", "expiration_time", "last_access")]


_SIGS = {
    "sine_last_error": (ctypes.c_char_p, []),
    "sine_version": (ctypes.c_int, []),
    "sine_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "sine_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int64,
                                   ctypes.POINTER(ctypes.c_void_p)]),
    "sine_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "sine_group_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                         ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "sine_group_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "sine_group_query": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _f64p, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_uint32, _i64p, _f64p, _i32p]),
    "sine_reserve": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64]),
    "sine_insert": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _i64p, _f64p,
                                   ctypes.POINTER(MetaCols), ctypes.c_uint32]),
    "sine_insert_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _i64p, ctypes.c_void_p,
                                          ctypes.POINTER(MetaCols), ctypes.c_uint32]),
    "sine_remove": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _i64p]),
    "sine_size": (ctypes.c_int, [ctypes.c_void_p, _i64p, _i64p]),
    "sine_ids": (ctypes.c_int, [ctypes.c_void_p, _i64p, ctypes.c_int64, _i64p]),
    "sine_get_rows": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _i64p, _f64p]),
    "sine_snapshot": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _i64p, _f64p, _i64p]),
    "sine_query": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _f64p, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_uint32, _i64p, _f64p, _i32p]),
    "sine_query_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_uint32, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "sine_query_submit": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, _i64p]),
    "sine_query_wait": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64]),
    "sine_update_meta": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, _i64p, _f64p, _i64p, _f64p]),
    "sine_expired": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, _i64p,
                                    ctypes.c_int64, _i64p]),
    "sine_select_victims": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64,
                                           _i64p, ctypes.c_int64, _i64p]),
    "sine_evict": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64,
                                           _i64p, ctypes.c_int64, _i64p]),
    "sine_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "sine_set_timing": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "sine_set_select_cap": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "sine_last_timing": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float),
                                        ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
    "sine_kernel_launches": (ctypes.c_int, [ctypes.c_void_p, _i64p]),
    "sine_gemm_overflows": (ctypes.c_int, [ctypes.c_void_p, _i64p]),
    "sine_query_device_cert": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                              ctypes.c_double, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "sine_merge_shards": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p]),
    "sine_hex_bound": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int]),
    "sine_embed_hashed_bag": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.c_int64, ctypes.c_void_p]),
    "sine_blake2b64": (ctypes.c_uint64, [ctypes.c_char_p, ctypes.c_int64, ctypes.c_uint64]),
    "sine_hex_format": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_int64, _i64p]),
    "sine_hex_parse": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_void_p, ctypes.c_void_p]),
    "sine_uncertified": (ctypes.c_int, [ctypes.c_void_p, _i64p]),
    "sine_copy_certificates": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "sine_timing_totals": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _f64p, _i64p, ctypes.c_int]),
    "sine_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "sine_host_free": (ctypes.c_int, [ctypes.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the shared library.  Raises if it is missing."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"libsine_b200.so not found at {path}; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    if status == SINE_OK:
        return
    msg = load_library().sine_last_error().decode(errors="replace")
    if status in (SINE_EINVAL, SINE_ENOTFOUND, SINE_EDUP, SINE_ENORM):
        raise ValidationError(msg)
    if status == SINE_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libsine_b200 error {status}: {msg}")


def device_count() -> int:
    n = ctypes.c_int(0)
    check(load_library().sine_device_count(ctypes.byref(n)))
    return n.value


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class PinnedArray:
    """Page-locked host buffer (cudaMallocHost) viewed as a numpy array."""

    def __init__(self, shape, dtype):
        self.dtype = np.dtype(dtype)
        self.shape = tuple(int(s) for s in np.atleast_1d(shape))
        nbytes = max(1, int(np.prod(self.shape)) * self.dtype.itemsize)
        p = ctypes.c_void_p()
        check(load_library().sine_host_alloc(nbytes, ctypes.byref(p)))
        self._p = p
        buf = (ctypes.c_byte * nbytes).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(self.shape))).reshape(self.shape)

    def __del__(self):
        p = getattr(self, "_p", None)
        if p is not None and p.value and _lib is not None:
            _lib.sine_host_free(p)
            self._p = None


def hex_format(rows: np.ndarray, ids=None) -> memoryview:
    """Float-hex text of a row block ("[<id> ]<hex> ...\\n" per row), byte-
    identical to the reference's float.hex writers (native, multi-threaded)."""
    lib = load_library()
    rows = f64(rows)
    n, d = rows.shape
    ids_a = i64(ids) if ids is not None else None
    cap = lib.sine_hex_bound(n, d, 1 if ids_a is not None else 0)
    out = np.empty(max(cap, 1), dtype=np.uint8)
    ln = ctypes.c_int64()
    check(lib.sine_hex_format(ids_a.ctypes.data if ids_a is not None else None, rows.ctypes.data, n, d,
                              out.ctypes.data, cap, ctypes.byref(ln)))
    return memoryview(out)[:ln.value]  # no copy: file writes and bytes() take it as is


def hex_parse(text: bytes, n: int, d: int, with_ids: bool, offset: int = 0):
    """Inverse of hex_format over text[offset:]: (ids int64[n] or None,
    rows float64[n, d]).  `text` is read in place (no copy)."""
    lib = load_library()
    rows = np.empty((n, d), dtype=np.float64)
    ids = np.empty(n, dtype=np.int64) if with_ids else None
    base = ctypes.cast(ctypes.c_char_p(text), ctypes.c_void_p).value
    check(lib.sine_hex_parse(base + offset, len(text) - offset, n, d,
                             ids.ctypes.data if ids is not None else None, rows.ctypes.data))
    return ids, rows
