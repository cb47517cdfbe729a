"""ctypes access to the C restatement in oracle/ (test + bench infrastructure only)."""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
LIB = REPO / "oracle" / "_build" / "libfs_oracle.so"
_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(REPO / "oracle"), str(LIB)], check=True,
                           capture_output=True)
        lib = C.CDLL(str(LIB))
        vp = C.c_void_p
        lib.fso_accumulate.argtypes = [C.POINTER(vp), C.c_uint32, C.c_uint64, vp, C.c_int]
        lib.fso_histogram.argtypes = [vp, C.c_uint64, C.c_uint64, vp, C.c_int]
        lib.fso_composite.argtypes = [vp, C.c_uint64, C.c_uint64, vp, C.c_int]
        lib.fso_pair_counts.argtypes = [vp, vp, C.c_uint64, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), C.c_int]
        lib.fso_gram.argtypes = [C.POINTER(vp), C.c_uint32, C.c_uint64, vp, C.c_int]
        _lib = lib
    return _lib


def _ptrs(arrays):
    arr = (C.c_void_p * len(arrays))()
    for i, a in enumerate(arrays):
        arr[i] = a.ctypes.data
    return arr


def accumulate(cells_list, threads=0) -> np.ndarray:
    flats = [np.ascontiguousarray(c).reshape(-1) for c in cells_list]
    counts = np.zeros(flats[0].size, dtype=np.uint32)
    load().fso_accumulate(_ptrs(flats), len(flats), counts.size, counts.ctypes.data, threads)
    return counts


def histogram(counts, n_inputs, threads=0) -> np.ndarray:
    c = np.ascontiguousarray(counts, dtype=np.uint32).reshape(-1)
    bins = np.zeros(n_inputs + 1, dtype=np.int64)
    load().fso_histogram(c.ctypes.data, c.size, n_inputs + 1, bins.ctypes.data, threads)
    return bins


def composite(counts, n_inputs, threads=0) -> np.ndarray:
    c = np.ascontiguousarray(counts, dtype=np.uint32).reshape(-1)
    out = np.zeros((c.size, 4), dtype=np.uint8)
    load().fso_composite(c.ctypes.data, c.size, n_inputs, out.ctypes.data, threads)
    return out


def pair_counts(a, b, threads=0):
    x = np.ascontiguousarray(a).reshape(-1)
    y = np.ascontiguousarray(b).reshape(-1)
    i, u = C.c_int64(), C.c_int64()
    load().fso_pair_counts(x.ctypes.data, y.ctypes.data, x.size, C.byref(i), C.byref(u), threads)
    return i.value, u.value


def gram(cells_list, threads=0) -> np.ndarray:
    flats = [np.ascontiguousarray(c).reshape(-1) for c in cells_list]
    k = len(flats)
    g = np.zeros((k, k), dtype=np.int64)
    load().fso_gram(_ptrs(flats), k, flats[0].size, g.ctypes.data, threads)
    return g
