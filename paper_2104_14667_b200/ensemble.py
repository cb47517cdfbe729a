"""Device-resident flood ensemble: bit-packed masks kept in HBM.

The interactive-recompute target (≥10 FPS over 256 × 8192² masks) cannot re-stream
17 GB over PCIe every frame, so the masks are uploaded once — through the paper's
dual-buffer pipeline — binarized and bit-packed (P/8 bytes per mask), and every
recompute reads them from HBM:

* ``overlap()``  — counts + histogram + composite in one fused pass
  (analytics.py:106-162 on the reference side);
* ``gram()``     — exact pairwise intersections on tcgen05 int8 tensor cores
  (the pair_counts loop of analytics.py:174-181);
* ``recompute()``— the service snapshot (service.py:143-175) plus the /clusters and
  /outliers products (service.py:289-307) from one overlap pass and one Gram.

A ``DeviceEnsemble`` may hold a horizontal *band* of every mask (rows
[row0, row0 + rows)); bands are how the multi-GPU path shards pixels (see dist.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .analytics import (
    AccumulationGrid,
    CompositeImage,
    OverlapHistogram,
    cluster_from_similarity,
    outliers_from_similarity,
    similarity_from_gram,
)

_GRAM_ENGINES = {"auto": N.GRAM_AUTO, "popc": N.GRAM_POPC, "tc": N.GRAM_TC_I8, "tc-i8": N.GRAM_TC_I8,
                 "tc-f4": N.GRAM_TC_F4}


@dataclass
class StreamStats:
    """Measured timings of one streamed upload (µs, CUDA events / host clock)."""

    variant: str
    n: int
    total_us: float
    host_us: list[float] = field(default_factory=list)
    copy_us: list[float] = field(default_factory=list)
    xform_us: list[float] = field(default_factory=list)
    kernel_us: list[float] = field(default_factory=list)


@dataclass
class Snapshot:
    """One full recompute of the working set."""

    grid: AccumulationGrid | None
    histogram: OverlapHistogram | None
    composite: CompositeImage | None
    gram: np.ndarray | None
    similarity: np.ndarray | None
    outliers: dict | None
    clusters: list | None


class DeviceEnsemble:
    """Bit-packed masks of one raster size (or one row band of it) resident in HBM."""

    def __init__(self, width: int, height: int, capacity: int, *, row0: int = 0,
                 rows: int | None = None, device: int | None = None):
        if rows is None:
            rows = height - row0
        if width < 1 or height < 1 or rows < 1 or row0 < 0 or row0 + rows > height:
            raise ValueError("bad ensemble geometry")
        if device is not None:
            N.set_device(device)
        self.width, self.height, self.row0, self.rows = int(width), int(height), int(row0), int(rows)
        self.pixels = self.width * self.rows
        self.capacity = int(capacity)
        h = C.c_void_p()
        N.call("fs_ensemble_create", self.pixels, self.capacity, C.byref(h))
        self._h = h
        wpm, dev = C.c_uint64(), C.c_int()
        N.call("fs_ensemble_info", self._h, None, None, C.byref(wpm), C.byref(dev))
        self.words_per_mask = wpm.value
        self.device = dev.value
        self.ids: list[str | None] = [None] * self.capacity

    # -- lifetime -------------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            N.load().fs_ensemble_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- helpers --------------------------------------------------------------------
    def _slots(self, slots) -> np.ndarray:
        if slots is None:
            slots = [i for i, s in enumerate(self.ids) if s is not None] or range(self.capacity)
        a = np.ascontiguousarray(np.asarray(list(slots) if not isinstance(slots, np.ndarray) else slots,
                                            dtype=np.uint32))
        if a.size == 0:
            raise ValueError("need at least one slot")
        return a

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def stream_handle(self) -> int:
        p = C.c_void_p()
        N.call("fs_ensemble_stream_handle", self._h, C.byref(p))
        return p.value or 0

    def use_stream(self, stream_ptr: int | None) -> None:
        """Run compute work on a caller-owned CUDA stream (None: the ensemble's own)."""
        N.call("fs_ensemble_set_stream", self._h, stream_ptr or None)

    def sync(self) -> None:
        N.call("fs_ensemble_sync", self._h)

    def kernel_ms(self, kind: str) -> float:
        code = {"pack": N.KERNEL_PACK, "overlap": N.KERNEL_OVERLAP, "gram": N.KERNEL_GRAM,
                "recompute": N.KERNEL_RECOMPUTE}[kind]
        ms = C.c_float()
        N.call("fs_ensemble_kernel_ms", self._h, code, C.byref(ms))
        return float(ms.value)

    # -- filling --------------------------------------------------------------------
    def band_view(self, cells: np.ndarray) -> np.ndarray:
        """This ensemble's rows of a full (H, W) raster, as a flat contiguous array."""
        a = cells.reshape(self.height, self.width)[self.row0:self.row0 + self.rows]
        return np.ascontiguousarray(a).reshape(-1)

    def stream(self, rasters, *, first: int = 0, variant: str = "2b-final",
               with_kernel: bool = False, reset_counts: bool = True, slot_wrap: int = 0,
               ids=None, already_banded: bool = False) -> StreamStats:
        """Upload rasters (uint8 arrays of this ensemble's band) through the variant's
        pipeline; slot of item i = first + (i % slot_wrap or i)."""
        arrays = []
        for r in rasters:
            a = getattr(r, "cells", r)
            if not already_banded and (self.row0 != 0 or self.rows != self.height):
                a = self.band_view(a)
            a = a.reshape(-1)
            if a.dtype != np.uint8 or a.size != self.pixels:
                raise ValueError(f"raster must be uint8 with {self.pixels} pixels")
            if not a.flags["C_CONTIGUOUS"]:
                a = np.ascontiguousarray(a)
            arrays.append(a)
        k = len(arrays)
        items = (N.StreamItem * max(k, 1))()
        rep = N.StreamReport(0.0, k, items)
        code = N.VARIANT_CODES[variant]
        N.call("fs_ensemble_stream", self._h, first, slot_wrap, N.ptr_array(arrays), k, code,
               int(with_kernel), int(reset_counts), C.byref(rep))
        span = min(slot_wrap, k) if slot_wrap else k
        for i in range(span):
            self.ids[first + i] = (ids[i] if ids is not None else
                                   getattr(rasters[i], "id", f"slot{first + i}"))
        return StreamStats(
            variant=variant, n=k, total_us=rep.total_us,
            host_us=[items[i].host_us for i in range(k)],
            copy_us=[items[i].copy_us for i in range(k)],
            xform_us=[items[i].xform_us for i in range(k)],
            kernel_us=[items[i].kernel_us for i in range(k)],
        )

    def upload(self, surfaces, *, first: int = 0, variant: str | None = None) -> StreamStats:
        """Upload surfaces into slots first.. (2b-final when the sources are pinned,
        2b-initial — pinned staging with a parallel host copy — when pageable)."""
        if variant is None:
            pinned = all(N.is_pinned(getattr(s, "cells", s)) for s in surfaces)
            variant = "2b-final" if pinned else "2b-initial"
        return self.stream(surfaces, first=first, variant=variant)

    def synth(self, first: int, k: int, *, seed: int, members: int, eps: float,
              mask_index0: int | None = None) -> None:
        """Generate flood-like synthetic masks (fs_synth_host's bytes) straight into
        slots first..first+k-1, for this ensemble's band."""
        mi = first if mask_index0 is None else mask_index0
        N.call("fs_ensemble_synth", self._h, first, k, seed, self.width, self.height, self.row0,
               members, float(eps), mi)
        for i in range(k):
            self.ids[first + i] = f"s{mi + i:04d}"

    # -- recompute ------------------------------------------------------------------
    def overlap(self, slots=None, *, cycles: int = 1, remainder: int = 0, counts: bool = True,
                bins: bool = True, rgba: bool = True, out_counts=None, out_rgba=None,
                out_bins=None, device_outputs: bool = False):
        """Fused counts / histogram / composite over ``slots`` (cycled to
        n = cycles*k + remainder).  Returns (counts[H_band, W], bins, rgba[H_band, W, 4])
        as numpy arrays (or the device pointers passed in when device_outputs)."""
        sl = self._slots(slots)
        k = int(sl.size)
        n_inputs = cycles * k + remainder
        if device_outputs:
            cp = int(out_counts) if (counts and out_counts is not None) else None
            rp = int(out_rgba) if (rgba and out_rgba is not None) else None
            bp = int(out_bins) if (bins and out_bins is not None) else None
            N.call("fs_ensemble_overlap", self._h, sl.ctypes.data_as(N._u32p), k, cycles,
                   remainder, cp, bp, rp, 1)
            return out_counts, out_bins, out_rgba
        c = (out_counts if out_counts is not None else
             np.empty((self.rows, self.width), dtype=np.uint32)) if counts else None
        r = (out_rgba if out_rgba is not None else
             np.empty((self.rows, self.width, 4), dtype=np.uint8)) if rgba else None
        b = (out_bins if out_bins is not None else
             np.empty(n_inputs + 1, dtype=np.int64)) if bins else None
        N.call("fs_ensemble_overlap", self._h, sl.ctypes.data_as(N._u32p), k, cycles, remainder,
               None if c is None else N.ptr(c), None if b is None else N.ptr(b),
               None if r is None else N.ptr(r), 0)
        return c, b, r

    def running_counts(self, n_inputs: int, *, bins: bool = True, rgba: bool = True):
        c = np.empty((self.rows, self.width), dtype=np.uint32)
        b = np.empty(n_inputs + 1, dtype=np.int64) if bins else None
        r = np.empty((self.rows, self.width, 4), dtype=np.uint8) if rgba else None
        N.call("fs_ensemble_running_counts", self._h, N.ptr(c), None if b is None else N.ptr(b),
               None if r is None else N.ptr(r), n_inputs, 0)
        return c, b, r

    def gram(self, slots=None, *, engine: str = "auto", out=None, device_outputs: bool = False):
        """int64 (k, k) intersection Gram of the slots' wet masks (this band's pixels)."""
        sl = self._slots(slots)
        k = int(sl.size)
        if device_outputs:
            N.call("fs_ensemble_gram", self._h, sl.ctypes.data_as(N._u32p), k,
                   _GRAM_ENGINES[engine], int(out), 1)
            return out
        g = out if out is not None else np.empty((k, k), dtype=np.int64)
        N.call("fs_ensemble_gram", self._h, sl.ctypes.data_as(N._u32p), k, _GRAM_ENGINES[engine],
               N.ptr(g), 0)
        return g

    def products(self, slots=None, *, engine: str = "auto", counts=True, bins=True, rgba=True,
                 gram=True, out_counts=None, out_bins=None, out_rgba=None, out_gram=None,
                 device_outputs: bool = False):
        """Counts, histogram, composite and Gram of ``slots`` in ONE call
        (fs_ensemble_recompute): with a tensor-core engine and k <= 256 the overlap
        products come out of the Gram kernel itself (one read of the packed masks).
        Returns (counts, bins, rgba, gram, fused)."""
        sl = self._slots(slots)
        k = int(sl.size)
        fused = C.c_int(0)
        if device_outputs:
            ptrs = [int(p) if (want and p is not None) else None
                    for want, p in ((counts, out_counts), (bins, out_bins), (rgba, out_rgba),
                                    (gram, out_gram))]
            N.call("fs_ensemble_recompute", self._h, sl.ctypes.data_as(N._u32p), k,
                   _GRAM_ENGINES[engine], *ptrs, 1, C.byref(fused))
            return out_counts, out_bins, out_rgba, out_gram, bool(fused.value)
        c = (out_counts if out_counts is not None else
             np.empty((self.rows, self.width), dtype=np.uint32)) if counts else None
        b = (out_bins if out_bins is not None else np.empty(k + 1, dtype=np.int64)) if bins else None
        r = (out_rgba if out_rgba is not None else
             np.empty((self.rows, self.width, 4), dtype=np.uint8)) if rgba else None
        g = (out_gram if out_gram is not None else np.empty((k, k), dtype=np.int64)) if gram else None
        N.call("fs_ensemble_recompute", self._h, sl.ctypes.data_as(N._u32p), k,
               _GRAM_ENGINES[engine], *[None if x is None else N.ptr(x) for x in (c, b, r, g)], 0,
               C.byref(fused))
        return c, b, r, g, bool(fused.value)

    def pipeline(self, slots=None, *, tau: float = 0.8, engine: str = "auto", depth: int = 3,
                 ids=None, comm=None) -> "NativePipeline":
        """Native frame loop over ``slots`` (fs_pipeline_*): recompute, device Jaccard /
        outliers, D2H and host linkage overlapped in C++.  ``comm`` (dist.NativeComm):
        this ensemble is one rank's row band and every frame sums the bands' partials."""
        return NativePipeline(self, self._slots(slots), tau=tau, engine=engine, depth=depth,
                              ids=ids, comm=comm)

    def recompute(self, slots=None, *, tau: float = 0.8, engine: str = "auto",
                  overlap: bool = True, pairwise: bool = True) -> Snapshot:
        """Full recompute of the working set: grid, histogram, composite, Gram,
        similarity, outlier scores and clusters."""
        sl = self._slots(slots)
        ids = [self.ids[i] if self.ids[i] is not None else f"slot{i}" for i in sl.tolist()]
        grid = hist = comp = gram = sim = outl = clus = None
        if overlap and pairwise:
            c, b, r, gram, _ = self.products(sl, engine=engine)
        elif overlap:
            c, b, r = self.overlap(sl)
        elif pairwise:
            gram = self.gram(sl, engine=engine)
        if overlap:
            grid = AccumulationGrid._from_device(self.width, self.rows, int(sl.size), c)
            hist = OverlapHistogram(bins=[int(x) for x in b])
            comp = CompositeImage(width=self.width, height=self.rows, pixels=r)
        if pairwise:
            sim = similarity_from_gram(gram)
            if len(ids) >= 2:
                outl = outliers_from_similarity(sim, ids)
            clus = cluster_from_similarity(sim, ids, tau)
        return Snapshot(grid, hist, comp, gram, sim, outl, clus)


class NativePipeline:
    """``depth`` frames in flight, C++ worker threads for the complete-linkage merge
    (include/floodstream.h, fs_pipeline_*).  ``run(n)`` returns the last frame's products."""

    def __init__(self, ens: DeviceEnsemble, slots: np.ndarray, *, tau: float, engine: str,
                 depth: int, ids=None, comm=None):
        self.ens = ens
        self.slots = np.ascontiguousarray(slots, dtype=np.uint32)
        self.k = int(self.slots.size)
        self.ids = list(ids) if ids is not None else [
            ens.ids[i] if ens.ids[i] is not None else f"slot{i}" for i in self.slots.tolist()]
        order = {s: r for r, s in enumerate(sorted(set(self.ids)))}
        self.rank = np.array([order[s] for s in self.ids], dtype=np.uint32)
        if not (0.0 < tau <= 1.0):
            raise ValueError("tau must be in (0, 1]")
        self.tau = float(tau)
        h = C.c_void_p()
        N.call("fs_pipeline_create", ens.handle, self.slots.ctypes.data_as(N._u32p), self.k,
               _GRAM_ENGINES[engine], self.tau, self.rank.ctypes.data_as(N._u32p), int(depth),
               C.byref(h))
        self._h = h
        self.comm = comm
        if comm is not None:
            N.call("fs_pipeline_set_comm", h, comm.handle)

    def run(self, n_frames: int) -> dict:
        k = self.k
        bins = np.empty(k + 1, np.int64)
        gram = np.empty((k, k), np.int64)
        sim = np.empty((k, k), np.float64)
        scores = np.empty(max(k, 1), np.float64)
        labels = np.empty(k, np.int32)
        ms = C.c_double()
        N.call("fs_pipeline_run", self._h, int(n_frames), N.ptr(bins), N.ptr(gram), N.ptr(sim),
               N.ptr(scores), N.ptr(labels), C.byref(ms))
        members: dict[int, list[str]] = {}
        for i, lab in enumerate(labels.tolist()):
            members.setdefault(lab, []).append(self.ids[i])
        clusters = sorted((sorted(m) for m in members.values()), key=lambda c: c[0])
        outliers = {sid: scores[i] for i, sid in enumerate(self.ids)} if k >= 2 else None
        return {"bins": bins, "gram": gram, "similarity": sim, "outliers": outliers,
                "clusters": clusters, "device_ms": ms.value, "frames": int(n_frames)}

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            N.load().fs_pipeline_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
