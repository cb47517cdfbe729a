"""Synthetic flood-like mask ensembles (bench and test inputs).

Counter-based prototype+flip generator implemented once in C++/CUDA
(csrc/fs_common.cuh ``synth_cell``): mask ``i`` belongs to prototype ``i // members``;
a prototype is a 16x16 low-resolution field thresholded at a per-prototype level and
upsampled to the raster; each member flips a pixel with probability ``eps``; wet
pixels carry a depth 1..255.  Every byte is a pure function of (seed, mask, pixel), so
the host generator (``fs_synth_host``) and the device generator
(``fs_ensemble_synth``, writing packed bits directly) agree exactly, and any row band
can be produced independently (multi-GPU sharding, out-of-RAM configs).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .rasters import RasterSurface


def synth_cells(width: int, height: int, mask: int, *, seed: int = 2104, members: int = 16,
                eps: float = 0.02, row0: int = 0, rows: int | None = None, out=None,
                threads: int = 0) -> np.ndarray:
    """uint8 cells of rows [row0, row0 + rows) of synthetic mask ``mask``."""
    rows = height - row0 if rows is None else rows
    if out is None:
        out = np.empty((rows, width), dtype=np.uint8)
    if out.dtype != np.uint8 or out.size != rows * width or not out.flags["C_CONTIGUOUS"]:
        raise ValueError("out must be a contiguous uint8 array of rows*width bytes")
    N.call("fs_synth_host", N.ptr(out), seed, width, height, row0, rows, mask, members,
           float(eps), int(threads))
    return out


def synth_cells_gpu(width: int, height: int, mask: int, *, seed: int = 2104, members: int = 16,
                    eps: float = 0.02, row0: int = 0, rows: int | None = None, out=None,
                    device_ptr: int | None = None) -> np.ndarray | None:
    """``synth_cells``'s bytes generated on the current GPU (fs_synth_gpu): into ``out``
    (a host array, pinned or not) or straight into device memory at ``device_ptr``."""
    rows = height - row0 if rows is None else rows
    if device_ptr is not None:
        N.call("fs_synth_gpu", int(device_ptr), seed, width, height, row0, rows, mask, members,
               float(eps))
        return None
    if out is None:
        out = np.empty((rows, width), dtype=np.uint8)
    if out.dtype != np.uint8 or out.size != rows * width or not out.flags["C_CONTIGUOUS"]:
        raise ValueError("out must be a contiguous uint8 array of rows*width bytes")
    N.call("fs_synth_gpu", N.ptr(out), seed, width, height, row0, rows, mask, members, float(eps))
    return out


def flood_surfaces(width: int, height: int, k: int, *, seed: int = 2104, members: int = 16,
                   eps: float = 0.02, first: int = 0) -> list[RasterSurface]:
    """k synthetic surfaces with ids s0000.. (mask indices first..first+k-1)."""
    out = []
    for i in range(first, first + k):
        cells = synth_cells(width, height, i, seed=seed, members=members, eps=eps)
        out.append(RasterSurface(id=f"s{i:04d}", name=f"s{i:04d}", width=width, height=height,
                                 cells=cells))
    return out


def bernoulli_surfaces(pixels: int, k: int, *, seed: int = 0, p: float = 0.5,
                       width: int | None = None) -> list[RasterSurface]:
    """The reference bench's inputs (bench.py:472-475): default_rng(seed), k masks of
    (rng.random(pixels) < p).astype(uint8), ids s00.., reshaped to width x (pixels/width)."""
    rng = np.random.default_rng(seed)
    width = width or int(round(pixels ** 0.5))
    height = pixels // width
    if width * height != pixels:
        width, height = pixels, 1
    out = []
    for i in range(k):
        cells = (rng.random(pixels) < p).astype(np.uint8).reshape(height, width)
        out.append(RasterSurface(id=f"s{i:02d}", name=f"s{i:02d}", width=width, height=height,
                                 cells=cells))
    return out
