#!/usr/bin/env python
"""Ingest: surface files -> resident bit-packed ensemble.

Writes N PGM files of W x H (synthetic flood-like masks) to a scratch directory, then
times (JSON on stdout):
* b200: ingest.stream_files — PGM bodies read straight into pinned staging on a thread
  pool, one batch ahead of the 2b-final upload (H2D + bit-pack on the device);
* reference-style: the reference's per-surface decode (rasters.load_surface ->
  decode_surface_bytes, fs/rasters.py:104-117) into fresh arrays, then the upload
  from pageable memory (2b-initial), as SurfaceStore.surface + run_stream would.
"""
from __future__ import annotations

import argparse
import json
import shutil
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=8192)
    ap.add_argument("--height", type=int, default=8192)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--dir", default=None)
    args = ap.parse_args()

    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.ensemble import DeviceEnsemble
    from paper_2104_14667_b200.ingest import stream_files
    from paper_2104_14667_b200.rasters import load_surface, write_pgm
    from paper_2104_14667_b200.synth import synth_cells_gpu

    N.set_device(0)
    w, h, n = args.width, args.height, args.n
    d = Path(args.dir or tempfile.mkdtemp(prefix="fs_ingest_"))
    d.mkdir(parents=True, exist_ok=True)
    paths = []
    for i in range(n):
        p = d / f"s{i:04d}.pgm"
        p.write_bytes(write_pgm(synth_cells_gpu(w, h, i, seed=2104, members=8, eps=0.02)))
        paths.append(str(p))
    out = {"workload": f"{n} PGM files {w}x{h}", "bytes": n * w * h}
    try:
        with DeviceEnsemble(w, h, n) as ens:
            stream_files(ens, paths[: min(4, n)], batch=4)  # warm-up
            rep = stream_files(ens, paths, batch=16)
            out["b200_wall_s"] = round(rep["wall_s"], 4)
            out["b200_rate_gbs"] = round(rep["rate_gbs"], 3)
            t0 = time.perf_counter()
            surfaces = [load_surface(p) for p in paths]
            t1 = time.perf_counter()
            ens.upload(surfaces)
            t2 = time.perf_counter()
            out["reference_style_decode_s"] = round(t1 - t0, 4)
            out["reference_style_total_s"] = round(t2 - t0, 4)
            out["reference_style_rate_gbs"] = round(n * w * h / (t2 - t0) / 1e9, 3)
    finally:
        if args.dir is None:
            shutil.rmtree(d, ignore_errors=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
