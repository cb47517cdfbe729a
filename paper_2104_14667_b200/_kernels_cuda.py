"""The ``cuda`` kernel backend: the reference's four-primitive module protocol on B200.

Drop-in for ``floodstream._kernels_np`` / ``floodstream._accel``
(/root/reference/pkg/src/floodstream/_kernels_np.py:13-47, _accel.pyx:13-73): same
names, same argument meaning, same in-place mutation, same return types.  Every call
runs a hand-written sm_100a kernel through the C ABI (include/floodstream.h).

Besides the protocol, the module exposes the batched extensions the analytics layer
prefers when present (SURVEY §8b "required extensions"):

* ``accumulate_many(counts, cells_list)`` — one upload per mask, one fused count pass,
  instead of 9 B/px of PCIe traffic per ``accumulate_into`` call;
* ``gram_many(cells_list)`` — the exact int64 intersection Gram in one tensor-core
  contraction, instead of n(n-1)/2 ``pair_counts`` calls of 2P bytes each.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N

NAME = "cuda"

# Fail at import, not at first use, when the library is missing.
N.load()


def _flat_u8(cells: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(cells).reshape(-1)
    if a.dtype != np.uint8:
        raise TypeError(f"cells must be uint8, got {a.dtype}")
    return a


def _flat_counts(counts: np.ndarray, writable: bool) -> np.ndarray:
    if counts.dtype != np.uint32:
        raise TypeError(f"counts must be uint32, got {counts.dtype}")
    if writable:
        if not counts.flags["C_CONTIGUOUS"] or not counts.flags["WRITEABLE"]:
            raise ValueError("counts must be a writable C-contiguous uint32 array")
        return counts.reshape(-1)
    return np.ascontiguousarray(counts).reshape(-1)


def accumulate_into(counts: np.ndarray, cells: np.ndarray) -> None:
    """counts[p] += 1 for every pixel p where cells[p] > 0 (in place)."""
    c = _flat_counts(counts, writable=True)
    x = _flat_u8(cells)
    if c.size != x.size:
        raise ValueError(f"counts has {c.size} pixels, cells has {x.size}")
    N.call("fs_accumulate_into", N.ptr(c), N.ptr(x), c.size)


def overlap_counts(counts: np.ndarray, n_inputs: int) -> np.ndarray:
    """bins[k] = number of pixels covered by exactly k inputs (int64, n_inputs+1)."""
    c = _flat_counts(counts, writable=False)
    bins = np.zeros(int(n_inputs) + 1, dtype=np.int64)
    N.call("fs_overlap_counts", N.ptr(c), c.size, int(n_inputs), N.ptr(bins))
    return bins


def pair_counts(a: np.ndarray, b: np.ndarray) -> tuple[int, int]:
    """(intersection, union) of the wet masks of two cell arrays, as Python ints."""
    x, y = _flat_u8(a), _flat_u8(b)
    if x.size != y.size:
        raise ValueError("pair_counts needs equally sized arrays")
    inter, uni = C.c_int64(0), C.c_int64(0)
    N.call("fs_pair_counts", N.ptr(x), N.ptr(y), x.size, C.byref(inter), C.byref(uni))
    return int(inter.value), int(uni.value)


def composite_fill(counts: np.ndarray, n_inputs: int, out: np.ndarray) -> None:
    """Fill flat RGBA pixels in place: (g, g, 255, 255) where covered, else 0."""
    c = _flat_counts(counts, writable=False)
    if out.dtype != np.uint8 or out.shape != (c.size, 4) or not out.flags["C_CONTIGUOUS"]:
        raise ValueError("out must be a C-contiguous (P, 4) uint8 array")
    N.call("fs_composite_fill", N.ptr(c), c.size, int(n_inputs), N.ptr(out))


# ---- batched extensions -------------------------------------------------------------


def accumulate_many(counts: np.ndarray, cells_list) -> None:
    """counts[p] += #{s : cells_list[s][p] > 0}, one fused device pass."""
    c = _flat_counts(counts, writable=True)
    flats = [_flat_u8(x) for x in cells_list]
    for f in flats:
        if f.size != c.size:
            raise ValueError("all cell arrays must match counts in size")
    if not flats:
        return
    N.call("fs_accumulate_many", N.ptr(c), N.ptr_array(flats), len(flats), c.size)


def gram_many(cells_list) -> np.ndarray:
    """int64 (k, k) matrix of wet-mask intersections |A_i & A_j| (diagonal = |A_i|)."""
    flats = [_flat_u8(x) for x in cells_list]
    k = len(flats)
    gram = np.zeros((k, k), dtype=np.int64)
    if k == 0:
        return gram
    n = flats[0].size
    for f in flats:
        if f.size != n:
            raise ValueError("gram_many needs equally sized arrays")
    N.call("fs_gram_many", N.ptr_array(flats), k, n, N.ptr(gram))
    return gram


def stack_cache_info() -> dict:
    """The calling device's batched-call cache: resident masks, capacity, raster size."""
    v, cap, px = C.c_uint32(), C.c_uint32(), C.c_uint64()
    N.call("fs_stack_cache_info", C.byref(v), C.byref(cap), C.byref(px))
    return {"resident": v.value, "capacity": cap.value, "pixels": px.value}


def release_stack_cache() -> None:
    """Free the calling device's batched-call cache (bit-packed stack kept in HBM so
    that accumulate -> similarity_matrix -> outlier_scores -> cluster_surfaces upload a
    stack once; include/floodstream.h fs_stack_cache_release)."""
    N.call("fs_stack_cache_release")
