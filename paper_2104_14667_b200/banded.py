"""Spatial + iterative streaming for ensembles larger than the device budget.

The paper handles data that exceeds device memory by *spatial and iterative
subdivision* (PAPER.md:9); the reference implements only the iterative half (one
surface at a time, fs/analytics.py:119-120, cycled by fs/streaming.py:417-425) and
rejects rasters above 16384 px (fs/device.py:256-263).  ``BandedStream`` does both on
the B200: the raster is cut into spatial bands of ``band_rows`` rows; for each band
all k masks' rows are streamed from host memory through the dual-buffer upload
pipeline (H2D on the copy stream, binarize + bit-pack on the compute stream,
``fs_ensemble_stream``), then one fused recompute (``fs_ensemble_recompute``: counts,
histogram, composite and the Gram partial of that band) runs while the NEXT band
uploads into the other of two band ensembles.  The band's counts/RGBA go back to host
memory on a third stream (PCIe is full duplex), its int64 [histogram | Gram] partial
into a pinned slot; partials are summed exactly on the host at the end.  Device memory
is bounded by two bands, whatever the raster size.

Multi-GPU: each rank streams its own block of rows (``dist.band``) and the per-rank
[histogram | Gram] sums are combined by one all-reduce — the only exchange.  Results
are bit-identical to one device (integer sums), so Jaccard / outliers / clusters are
too (fs/analytics.py:165-240).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .analytics import cluster_from_similarity, outliers_from_similarity, similarity_from_gram
from .dist import band as row_band
from .dist import partial_layout


def default_band_rows(width: int, k: int, budget_bytes: int = 8 << 30) -> int:
    """Rows per band so two in-flight bands fit ``budget_bytes`` of device memory:
    per pixel and band, k/8 packed + 2 staging + 4 counts + 4 RGBA bytes."""
    per_px = 2 * (k / 8.0 + 2 + 8)
    return max(1, int(budget_bytes / per_px) // max(1, width))


def split_bands(rows: int, band_rows: int) -> list[tuple[int, int]]:
    """(offset, rows) of consecutive bands of ``band_rows`` rows covering ``rows``; the
    last band takes the remainder."""
    if band_rows < 1:
        raise ValueError("band_rows must be >= 1")
    return [(r, min(band_rows, rows - r)) for r in range(0, rows, band_rows)]


@dataclass
class BandStats:
    """Measured timings of one banded pass (device clock where noted)."""

    bands: int = 0
    rows_per_band: int = 0
    upload_us: list[float] = field(default_factory=list)  # per band: H2D + pack (events)
    wall_s: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


class BandedStream:
    """Rows [row0, row0 + rows) of a k-mask ensemble, processed band by band."""

    def __init__(self, width: int, height: int, k: int, *, row0: int = 0, rows: int | None = None,
                 band_rows: int | None = None, budget_bytes: int = 8 << 30,
                 device: int | None = None):
        import torch

        rows = height - row0 if rows is None else rows
        if width < 1 or height < 1 or k < 1 or rows < 0 or row0 < 0 or row0 + rows > height:
            raise ValueError("bad banded geometry")
        self.width, self.height, self.k = int(width), int(height), int(k)
        self.row0, self.rows = int(row0), int(rows)
        self.band_rows = int(band_rows) if band_rows else default_band_rows(width, k, budget_bytes)
        if self.band_rows < 1:
            raise ValueError("band_rows must be >= 1")
        dev = torch.cuda.current_device() if device is None else int(device)
        N.set_device(dev)
        self.device = torch.device("cuda", dev)
        self._ens: dict = {}
        self._streams = [torch.cuda.Stream(device=self.device) for _ in range(2)]
        self._d2h = torch.cuda.Stream(device=self.device)

    def bands(self) -> list[tuple[int, int]]:
        """(first row relative to row0, rows) of every band."""
        return split_bands(self.rows, self.band_rows)

    def close(self) -> None:
        for e in self._ens.values():
            e["ens"].close()
        self._ens.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- per-band device state: an ensemble of that band's size + its output buffers --
    def _slot(self, parity: int, nrows: int):
        import torch

        from .ensemble import DeviceEnsemble

        key = (parity, nrows)
        if key not in self._ens:
            px = nrows * self.width
            ens = DeviceEnsemble(self.width, nrows, self.k, device=self.device.index)
            ens.use_stream(self._streams[parity].cuda_stream)
            _, total = partial_layout(self.k)
            self._ens[key] = dict(
                ens=ens, stream=self._streams[parity],
                counts=torch.empty(px, dtype=torch.int32, device=self.device),
                rgba=torch.empty(px * 4, dtype=torch.uint8, device=self.device),
                part=torch.empty(total, dtype=torch.int64, device=self.device),
                drained=torch.cuda.Event())
            self._ens[key]["drained"].record(self._d2h)
        return self._ens[key]

    def run(self, source, *, engine: str = "auto", tau: float = 0.8, ids=None,
            counts_out=None, rgba_out=None, maps: bool = True, analytics: bool = True,
            group=None, variant: str | None = None) -> dict:
        """One pass over every band.

        ``source``: k host arrays holding this instance's rows (each (rows, width) or
        flat uint8; pinned memory uploads with the overlapped 2b-final DAG, pageable
        with 2b-initial), or a callable ``source(mask, r0, nrows) -> array`` returning
        rows [row0 + r0, row0 + r0 + nrows) of mask ``mask``.
        Returns counts (rows, width) uint32 / rgba (rows, width, 4) of these rows, the
        global int64 bins (k+1) and Gram (k, k) — summed over ranks of ``group`` when a
        process group is initialised — and the similarity / outliers / clusters.
        """
        import torch

        k, W = self.k, self.width
        nb, total = partial_layout(k)
        bands = self.bands()
        if maps:
            counts_out = _host_tensor(counts_out, (self.rows, W), torch.int32)
            rgba_out = _host_tensor(rgba_out, (self.rows, W, 4), torch.uint8)
        h_parts = torch.empty((max(1, len(bands)), total), dtype=torch.int64).pin_memory()
        h_parts.zero_()
        stats = BandStats(bands=len(bands), rows_per_band=self.band_rows)

        def rows_of(i, r0, n):
            if callable(source):
                a = source(i, r0, n)
            else:
                a = source[i]
                a = getattr(a, "cells", a)
                a = a.reshape(self.rows, W)[r0:r0 + n]
            a = np.asarray(a)
            if a.dtype != np.uint8 or a.size != n * W:
                raise ValueError(f"mask {i}: band rows must be uint8 with {n * W} pixels")
            return a.reshape(-1) if a.flags["C_CONTIGUOUS"] else np.ascontiguousarray(a).reshape(-1)

        slots = list(range(k))
        t0 = time.perf_counter()
        for b, (r0, n) in enumerate(bands):
            st = self._slot(b & 1, n)
            ens = st["ens"]
            arrays = [rows_of(i, r0, n) for i in range(k)]
            v = variant or ("2b-final" if all(N.is_pinned(a) for a in arrays) else "2b-initial")
            # the packed slots of this ensemble are rewritten only after its previous
            # band's recompute (same compute stream); its output buffers only after the
            # previous band's D2H drained
            rep = ens.stream(arrays, variant=v, already_banded=True)
            stats.upload_us.append(rep.total_us)
            stats.h2d_bytes += k * n * W
            st["stream"].wait_event(st["drained"])
            ens.products(slots, engine=engine, out_counts=st["counts"].data_ptr(),
                         out_rgba=st["rgba"].data_ptr(), out_bins=st["part"].data_ptr(),
                         out_gram=st["part"].data_ptr() + nb * 8, device_outputs=True)
            ready = torch.cuda.Event()
            ready.record(st["stream"])
            self._d2h.wait_event(ready)
            with torch.cuda.stream(self._d2h):
                h_parts[b].copy_(st["part"], non_blocking=True)
                if maps:
                    counts_out[r0:r0 + n].view(-1).copy_(st["counts"], non_blocking=True)
                    rgba_out[r0:r0 + n].view(-1).copy_(st["rgba"], non_blocking=True)
                    stats.d2h_bytes += 8 * n * W
                st["drained"].record(self._d2h)
        self._d2h.synchronize()
        part = h_parts.sum(dim=0) if bands else torch.zeros(total, dtype=torch.int64)
        _allreduce_cpu_or_device(part, group, self.device)
        stats.wall_s = time.perf_counter() - t0
        bins = part[:nb].numpy().copy()
        gram = part[nb:].numpy().reshape(k, k).copy()
        out = {"bins": bins, "gram": gram, "stats": stats}
        if maps:
            out["counts"] = counts_out.numpy().view(np.uint32).reshape(self.rows, W)
            out["rgba"] = rgba_out.numpy().reshape(self.rows, W, 4)
        if analytics:
            ids = list(ids) if ids is not None else [f"s{i:04d}" for i in range(k)]
            sim = similarity_from_gram(gram)
            out["similarity"] = sim
            out["outliers"] = outliers_from_similarity(sim, ids) if k >= 2 else None
            out["clusters"] = cluster_from_similarity(sim, ids, tau)
        return out


def _host_tensor(arr, shape, dtype):
    """Output buffer as a host torch tensor: a new pinned one, or a zero-copy view of
    the caller's numpy array (uint32 counts are viewed as int32)."""
    import torch

    if arr is None:
        return torch.empty(shape, dtype=dtype).pin_memory()
    if isinstance(arr, np.ndarray):
        if arr.dtype == np.uint32:
            arr = arr.view(np.int32)
        if arr.size != int(np.prod(shape)) or not arr.flags["C_CONTIGUOUS"]:
            raise ValueError(f"output must be a contiguous array of {int(np.prod(shape))} items")
        return torch.from_numpy(arr).view(shape)
    return arr.view(shape)


def _allreduce_cpu_or_device(part, group, device) -> None:
    """Sum a host int64 tensor over the ranks of ``group`` (NCCL via a device copy,
    gloo in place); no-op without an initialised multi-rank group."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    if dist.get_backend(group) == "nccl":
        d = part.to(device)
        dist.all_reduce(d, op=dist.ReduceOp.SUM, group=group)
        part.copy_(d.cpu())
    else:
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)


def rank_rows(height: int, group=None) -> tuple[int, int]:
    """This rank's block of rows (row0, rows) for a banded pass over ``height`` rows."""
    import torch.distributed as dist

    if not dist.is_initialized():
        return 0, height
    return row_band(height, dist.get_rank(group), dist.get_world_size(group))
