"""Ingest: decode surface files straight into pinned staging and stream them in
(SURVEY §8f row 4).

The reference decodes every surface into a fresh numpy array (``decode_surface_bytes``,
fs/rasters.py:60-117; ``SurfaceStore.surface``, fs/store.py:156-170) and the upload
then copies it again.  Here a PGM body is read from the file directly into a
page-locked buffer (one read, no intermediate array), PNGs are decoded by Pillow into
the same buffers, and decoding runs on a thread pool one batch ahead of the upload:
batch b+1 decodes while batch b streams through the 2b-final DAG (H2D + bit-pack on
the device) — the paper's host[i] -> copy[i] -> transform[i] overlap, from files.
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

from . import _native as N
from .rasters import RasterError, _Incomplete, _scan_pgm_header, decode_surface_bytes, pgm_header

_HEAD = 512  # first read for a header; long comment blocks fetch more


def probe(source) -> tuple[int, int]:
    """(width, height) of a PGM/PNG file path or bytes without decoding the body."""
    data = _head_bytes(source, 24)
    if data[:2] == b"P5":
        w, h, _, _ = _pgm_head(source)
        return w, h
    if data[:8] == b"\x89PNG\r\n\x1a\n":
        return int.from_bytes(data[16:20], "big"), int.from_bytes(data[20:24], "big")
    raise RasterError("unrecognised surface format (expected PGM P5 or PNG)")


def _head_bytes(source, n: int) -> bytes:
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source[:n])
    with open(source, "rb") as f:
        return f.read(n)


def _pgm_head(source) -> tuple[int, int, int, int]:
    """(width, height, maxval, body offset) of a PGM path or bytes: parse the first
    _HEAD bytes, and read further (x64 each time, up to the whole file) while the header
    is longer than what was read (e.g. long comment blocks)."""
    if isinstance(source, (bytes, bytearray, memoryview)):
        return pgm_header(source)
    n = _HEAD
    size = os.path.getsize(source)
    while True:
        head = _head_bytes(source, n)
        try:
            _scan_pgm_header(head)
            return pgm_header(head)
        except _Incomplete:
            if n >= size:
                raise RasterError("not a binary PGM (P5) file") from None
            n *= 64


def decode_into(source, out: np.ndarray) -> tuple[int, int]:
    """Decode one surface (path or bytes) into ``out`` (uint8, exactly W*H bytes, e.g.
    a pinned buffer).  PGM files are read straight into ``out``."""
    if out.dtype != np.uint8 or not out.flags["C_CONTIGUOUS"]:
        raise ValueError("out must be a contiguous uint8 array")
    flat = out.reshape(-1)
    if _head_bytes(source, 2) == b"P5":
        w, h, _, off = _pgm_head(source)
        if w * h != flat.size:
            raise RasterError(f"PGM is {w}x{h}, buffer holds {flat.size} px")
        if isinstance(source, (bytes, bytearray, memoryview)):
            body = memoryview(source)[off:off + w * h]
            if len(body) < w * h:
                raise RasterError(f"PGM truncated: expected {w * h} pixel bytes, got {len(body)}")
            flat[:] = np.frombuffer(body, dtype=np.uint8)
        else:
            with open(source, "rb") as f:
                f.seek(off)
                got = f.readinto(memoryview(flat))
            if got != w * h:
                raise RasterError(f"PGM truncated: expected {w * h} pixel bytes, got {got}")
        return w, h
    data = bytes(source) if isinstance(source, (bytes, bytearray, memoryview)) else Path(source).read_bytes()
    w, h, cells = decode_surface_bytes(data)
    if w * h != flat.size:
        raise RasterError(f"surface is {w}x{h}, buffer holds {flat.size} px")
    flat[:] = cells.reshape(-1)
    return w, h


_pool_lock = threading.Lock()
_pool: dict = {}  # (pixels, batch) -> two halves of pinned buffers, reused across calls


def _staging(P: int, batch: int):
    """Two batches of pinned staging buffers (page-locking 2 x batch x P bytes costs
    far more than a read, so they are kept for the next call of the same shape)."""
    with _pool_lock:
        bufs = _pool.pop((P, batch), None)
    return bufs or [[N.PinnedBuffer((P,)) for _ in range(batch)] for _ in range(2)]


def _release(P: int, batch: int, bufs) -> None:
    """Keep ``bufs`` for the next call; free whatever the pool held before (at most one
    shape stays page-locked)."""
    with _pool_lock:
        stale = list(_pool.values())
        _pool.clear()
        _pool[(P, batch)] = bufs
    for halves in stale:
        for half in halves:
            for buf in half:
                buf.free()


def stream_files(ens, sources, *, first: int = 0, batch: int = 16, workers: int | None = None,
                 ids=None) -> dict:
    """Decode ``sources`` (paths or bytes) into two pinned batches of ``batch`` buffers
    and stream them into ensemble slots first.. (2b-final), decoding batch b+1 on a
    thread pool while batch b uploads.  Returns timings (s) and bytes moved."""
    import time

    n = len(sources)
    if first + n > ens.capacity:
        raise ValueError("sources exceed the ensemble's capacity")
    P = ens.pixels
    batch = max(1, min(batch, n))
    bufs = _staging(P, batch)
    workers = workers or min(16, (os.cpu_count() or 4))
    t0 = time.perf_counter()
    upload_us = 0.0
    try:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            def decode_batch(b, half):
                lo = b * batch
                return [pool.submit(decode_into, sources[lo + i], bufs[half][i].array)
                        for i in range(min(batch, n - lo))]

            nb = -(-n // batch)
            pending = decode_batch(0, 0) if n else []
            for b in range(nb):
                for f in pending:
                    f.result()  # raises decode errors
                cur = [bufs[b & 1][i].array for i in range(len(pending))]
                pending = decode_batch(b + 1, (b + 1) & 1) if b + 1 < nb else []
                lo = b * batch
                st = ens.stream(cur, first=first + lo, variant="2b-final", already_banded=True,
                                ids=None if ids is None else ids[lo:lo + len(cur)])
                upload_us += st.total_us
    finally:
        _release(P, batch, bufs)
    wall = time.perf_counter() - t0
    return {"files": n, "bytes": n * P, "wall_s": wall, "upload_s": upload_us / 1e6,
            "rate_gbs": n * P / wall / 1e9 if wall > 0 else None}
