"""ctypes binding of libfloodstream (include/floodstream.h).

This is the only place Python touches the native library.  Loading fails loudly when
the shared object is missing: the CUDA library *is* the product path, there is no
CPU fallback.  Device calls on a machine without a GPU raise ``RuntimeError`` from
the library's own status codes.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libfloodstream.so"
# timing experiments only (tools/probe_builds.py): load a probe build of the library
if os.environ.get("FS_LIB_PROBE"):
    LIB_PATH = Path(os.environ["FS_LIB_PROBE"]).resolve()

FS_OK, FS_EINVAL, FS_ECUDA, FS_ENOMEM, FS_ENODEV = 0, 1, 2, 3, 4
VARIANT_CODES = {"1b-initial": 0, "2b-initial": 1, "1b-final": 2, "2b-final": 3}
GRAM_AUTO, GRAM_POPC, GRAM_TC_I8, GRAM_TC_F4 = 0, 1, 2, 3
KERNEL_PACK, KERNEL_OVERLAP, KERNEL_GRAM, KERNEL_RECOMPUTE = 0, 1, 2, 3


class StreamItem(C.Structure):
    _fields_ = [
        ("host_us", C.c_float),
        ("copy_us", C.c_float),
        ("xform_us", C.c_float),
        ("kernel_us", C.c_float),
    ]


class StreamReport(C.Structure):
    _fields_ = [
        ("total_us", C.c_double),
        ("n_items", C.c_uint32),
        ("items", C.POINTER(StreamItem)),
    ]


_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p

# name -> (argtypes); all return int status
_SIGNATURES = {
    "fs_abi_version": [],
    "fs_device_count": [C.POINTER(C.c_int)],
    "fs_set_device": [C.c_int],
    "fs_get_device": [C.POINTER(C.c_int)],
    "fs_synchronize": [],
    "fs_accumulate_into": [_vp, _vp, C.c_uint64],
    "fs_overlap_counts": [_vp, C.c_uint64, C.c_uint64, _vp],
    "fs_pair_counts": [_vp, _vp, C.c_uint64, _i64p, _i64p],
    "fs_composite_fill": [_vp, C.c_uint64, C.c_uint64, _vp],
    "fs_accumulate_many": [_vp, C.POINTER(_vp), C.c_uint32, C.c_uint64],
    "fs_gram_many": [C.POINTER(_vp), C.c_uint32, C.c_uint64, _vp],
    "fs_stack_cache_release": [],
    "fs_stack_cache_info": [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)],
    "fs_ensemble_create": [C.c_uint64, C.c_uint32, C.POINTER(_vp)],
    "fs_ensemble_destroy": [_vp],
    "fs_ensemble_info": [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                         C.POINTER(C.c_uint64), C.POINTER(C.c_int)],
    "fs_ensemble_packed_ptr": [_vp, C.POINTER(_vp)],
    "fs_ensemble_stream": [_vp, C.c_uint32, C.c_uint32, C.POINTER(_vp), C.c_uint32, C.c_int,
                           C.c_int, C.c_int, C.POINTER(StreamReport)],
    "fs_ensemble_synth": [_vp, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                          C.c_uint64, C.c_uint32, C.c_double, C.c_uint64],
    "fs_ensemble_overlap": [_vp, _u32p, C.c_uint32, C.c_uint64, C.c_uint32, _vp, _vp, _vp,
                            C.c_int],
    "fs_ensemble_running_counts": [_vp, _vp, _vp, _vp, C.c_uint64, C.c_int],
    "fs_ensemble_gram": [_vp, _u32p, C.c_uint32, C.c_int, _vp, C.c_int],
    "fs_ensemble_recompute": [_vp, _u32p, C.c_uint32, C.c_int, _vp, _vp, _vp, _vp, C.c_int,
                              C.POINTER(C.c_int)],
    "fs_ensemble_kernel_ms": [_vp, C.c_int, C.POINTER(C.c_float)],
    "fs_ensemble_stream_handle": [_vp, C.POINTER(_vp)],
    "fs_ensemble_sync": [_vp],
    "fs_ensemble_set_stream": [_vp, _vp],
    "fs_set_gram_engine": [C.c_int],
    "fs_set_pack_engine": [C.c_int],
    "fs_host_alloc": [C.c_uint64, C.POINTER(_vp)],
    "fs_host_free": [_vp],
    "fs_host_is_pinned": [_vp, C.POINTER(C.c_int)],
    "fs_cluster_complete_linkage": [_f64p, C.c_uint32, _u32p, C.c_double, _i32p],
    "fs_outlier_scores": [_f64p, C.c_uint32, _f64p],
    "fs_similarity_from_gram": [_i64p, C.c_uint32, _f64p],
    "fs_similarity_outliers_device": [_vp, C.c_uint32, _vp, _vp, _vp],
    "fs_time_transform": [C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.POINTER(C.c_double),
                          C.POINTER(C.c_double)],
    "fs_time_h2d": [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "fs_synth_host": [_vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                      C.c_uint64, C.c_uint32, C.c_double, C.c_int],
    "fs_synth_gpu": [_vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                     C.c_uint64, C.c_uint32, C.c_double],
    "fs_pipeline_create": [_vp, _u32p, C.c_uint32, C.c_int, C.c_double, _u32p, C.c_uint32,
                           C.POINTER(_vp)],
    "fs_pipeline_run": [_vp, C.c_uint32, _vp, _vp, _vp, _vp, _vp, C.POINTER(C.c_double)],
    "fs_pipeline_destroy": [_vp],
    "fs_pipeline_set_comm": [_vp, _vp],
    "fs_comm_unique_id": [_vp],
    "fs_comm_create": [_vp, C.c_int, C.c_int, C.POINTER(_vp)],
    "fs_comm_allreduce_i64": [_vp, _vp, C.c_uint64, _vp],
    "fs_comm_destroy": [_vp],
}

EXPORTED_SYMBOLS = ("fs_last_error",) + tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A libfloodstream call failed (CUDA error, no device, allocation)."""


def load() -> C.CDLL:
    """Load libfloodstream.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"libfloodstream is not built ({LIB_PATH} missing); run "
                "`python -m paper_2104_14667_b200.build` or __graft_entry__.build(). "
                "There is no CPU fallback."
            )
        lib = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
        lib.fs_last_error.restype = C.c_char_p
        lib.fs_last_error.argtypes = []
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = C.c_int
            fn.argtypes = argtypes
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == FS_OK:
        return
    msg = load().fs_last_error().decode(errors="replace")
    if rc == FS_EINVAL:
        raise ValueError(msg)
    if rc == FS_ENOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def ptr_array(arrays) -> C.Array:
    arr = (_vp * len(arrays))()
    for i, a in enumerate(arrays):
        arr[i] = a.ctypes.data if isinstance(a, np.ndarray) else int(a)
    return arr


def device_count() -> int:
    n = C.c_int(0)
    rc = load().fs_device_count(C.byref(n))
    return n.value if rc == FS_OK else 0


def set_device(dev: int) -> None:
    call("fs_set_device", int(dev))


class PinnedBuffer:
    """Page-locked host memory owned by Python, exposed as a numpy array."""

    def __init__(self, shape, dtype=np.uint8):
        dtype = np.dtype(dtype)
        self.shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        nbytes = int(np.prod(self.shape, dtype=np.int64)) * dtype.itemsize
        self.nbytes = nbytes
        p = _vp()
        call("fs_host_alloc", max(nbytes, 1), C.byref(p))
        self._p = p.value
        buf = (C.c_uint8 * max(nbytes, 1)).from_address(self._p)
        self.array = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype).reshape(self.shape)

    def free(self) -> None:
        if getattr(self, "_p", None):
            self.array = None
            load().fs_host_free(_vp(self._p))
            self._p = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.free()
        except Exception:
            pass


def is_pinned(a: np.ndarray) -> bool:
    out = C.c_int(0)
    call("fs_host_is_pinned", _vp(a.ctypes.data), C.byref(out))
    return bool(out.value)


def env_flag(name: str, default: str = "") -> str:
    return os.environ.get(name, default)
