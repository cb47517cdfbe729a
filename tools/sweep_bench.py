#!/usr/bin/env python
"""Config 5 (BASELINE.json configs[4]): the raster-dimension sweep of the transform,
measured on the B200 — the paper's dimension study (§6) on the real kernel.

Writes one JSON document (stdout or --out) with:
* two RateMaps (fs/bench.py:55-126 schema): a non-square / non-pow2 grid
  SweepSpec(512, 500, 16012) and the pow2-aligned SweepSpec(512, 512, 16384),
  rate = w*h / t_us / 1000 GB/s of uint8 raster, t = mean of `reps` launches of the
  binarize + bit-pack kernel on a raster already in HBM (CUDA events);
* the HBM roofline of the transform: 1.125 B/px (P read + P/8 write) vs the measured
  copy bandwidth in MEASURED_PEAKS.json;
* the pinned / pageable H2D transfer ladder (fs/bench.py:193-228, measured);
* the CPU point beside it: the reference's own binarization RasterSurface.wet_mask()
  (`cells > 0`, fs/rasters.py:50-51) timed with numpy on the host at a few sizes.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true", help="8x8 grids (smoke)")
    ap.add_argument("--engine", type=int, default=-1,
                    help="transform kernel: -1 default (4), 0 TMA bulk, 1 direct, 2 vector, 3 pipelined, 4 flat")
    args = ap.parse_args()

    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.sweep import (SweepSpec, run_transfer_baseline,
                                             run_transform_sweep)

    assert N.device_count() > 0, "needs a CUDA device"
    peaks = {}
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        peaks = json.loads(p.read_text())
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    specs = {"nonpow2": SweepSpec(512, 500, 16012), "pow2": SweepSpec(512, 512, 16384)}
    if args.quick:
        specs = {"nonpow2": SweepSpec(512, 2000, 16012), "pow2": SweepSpec(512, 2048, 16384)}
    doc = {"config": "c5: raster dimension sweep 512-16384 (non-square, non-pow2), iid p=0.5",
           "kernel": {-1: "library default", 0: "k_pack_bulk (TMA bulk-staged)",
                      1: "k_pack_direct", 2: "k_pack_vec (8 x 16-B loads in flight)",
                      3: "k_pack_pipe (next block's loads in flight, in-kernel tail)",
                      4: "k_pack_flat (one 4 KB block per warp, raster-sized grid, in-kernel tail)"}[args.engine]
                     + " binarize + bit-pack",
           "rate_def": "w*h / t_us / 1000 GB/s of uint8 raster (fs/bench.py:337-338)",
           "roofline": {"bound": "hbm", "bytes_per_px": 1.125, "peak_gbs": hbm,
                        "raster_rate_ceiling_gbs": round(hbm / 1.125, 1)}}
    for name, spec in specs.items():
        t0 = time.perf_counter()
        rm = run_transform_sweep(spec, reps=args.reps, engine=args.engine)
        r = rm.rates
        big = r[len(spec.points) // 2:, len(spec.points) // 2:]
        doc[name] = {"ratemap": rm.to_json(), "seconds": round(time.perf_counter() - t0, 2),
                     "rate_min": float(r.min()), "rate_max": float(r.max()),
                     "rate_median": float(np.median(r)),
                     "rate_median_upper_quadrant": float(np.median(big)),
                     "hbm_frac_upper_quadrant": round(float(np.median(big)) * 1.125 / hbm, 4)}
    ladder = [1 << s for s in range(16, 31, 2)]
    doc["transfer_pinned"] = run_transfer_baseline(points=ladder, repeats=3).to_json()
    doc["transfer_pageable"] = run_transfer_baseline(points=ladder[:-1], repeats=3,
                                                     pinned=False).to_json()
    # CPU point: the reference's binarization (cells > 0) with numpy, one thread
    rng = np.random.default_rng(0)
    cpu = []
    for (w, h) in [(512, 512), (2048, 1500), (4096, 4096), (8192, 8000)]:
        cells = (rng.random((h, w)) < 0.5).astype(np.uint8) * 7
        best = float("inf")
        for _ in range(3):
            t0 = time.perf_counter()
            _ = cells > 0
            best = min(best, time.perf_counter() - t0)
        cpu.append({"width": w, "height": h, "rate_gbps": w * h / best / 1e9, "cores": 1,
                    "op": "RasterSurface.wet_mask(): cells > 0 (numpy)"})
    doc["cpu_wet_mask"] = cpu
    text = json.dumps(doc)
    if args.out:
        Path(args.out).write_text(text)
    print(json.dumps({k: (v if k not in ("nonpow2", "pow2") else
                          {kk: vv for kk, vv in v.items() if kk != "ratemap"})
                      for k, v in doc.items() if not k.startswith("transfer")}))


if __name__ == "__main__":
    main()
