#!/usr/bin/env python
"""Run the REFERENCE implementation itself (baseline/_ref, its own analytics with its
NumPy backend, on the host) and this package (B200) on the same flood-like ensemble and
compare every product bit for bit: grid digest, histogram, composite bytes, the
similarity matrix, outlier scores (float hex) and cluster lists.  JSON on stdout.

Sizes are chosen so the reference's O(n^2 P) pair loop finishes in seconds."""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
REF = REPO / "baseline" / "_ref"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--height", type=int, default=768)
    ap.add_argument("--k", type=int, default=48)
    ap.add_argument("--members", type=int, default=6)
    ap.add_argument("--tau", type=float, default=0.8)
    args = ap.parse_args()
    if not (REF / "floodstream").exists():
        print(json.dumps({"unavailable": "baseline/_ref missing"}))
        return
    sys.path.insert(0, str(REPO))
    os.environ.pop("FLOODSTREAM_BACKEND", None)  # ours binds its "cuda" backend at import
    import paper_2104_14667_b200 as ours
    from paper_2104_14667_b200.synth import synth_cells

    os.environ["FLOODSTREAM_BACKEND"] = "numpy"  # the reference binds numpy at import
    sys.path.insert(0, str(REF))
    import floodstream as ref  # the reference package, unmodified

    w, h, k = args.width, args.height, args.k
    cells = [synth_cells(w, h, i, members=args.members, eps=0.03) for i in range(k)]
    ids = [f"s{i:03d}" for i in range(k)]
    rs = [ref.RasterSurface(id=i, name=i, width=w, height=h, cells=c) for i, c in zip(ids, cells)]
    us = [ours.RasterSurface(id=i, name=i, width=w, height=h, cells=c) for i, c in zip(ids, cells)]

    def products(m, surfaces):
        t0 = time.perf_counter()
        g = m.accumulate(surfaces)
        hist = m.overlap_histogram(g).bins
        comp = m.composite_map(g).pixels
        sim = m.similarity_matrix(surfaces)
        outl = m.outlier_scores(surfaces)
        clus = m.cluster_surfaces(surfaces, args.tau)
        return {"seconds": time.perf_counter() - t0, "digest": g.digest(), "bins": hist,
                "composite_sha": hashlib.sha256(comp.tobytes()).hexdigest(),
                "sim_sha": hashlib.sha256(sim.tobytes()).hexdigest(),
                "outliers": {s: float(v).hex() for s, v in outl.items()}, "clusters": clus}

    r = products(ref, rs)
    # ours, cold (first call: CUDA context, module load, allocations) and warm: a
    # warm-up on a DIFFERENT ensemble first, so nothing of the compared stack is
    # resident — the timed call still uploads it (once: the batched calls share the
    # device stack cache) and recomputes every product
    warm = [ours.RasterSurface(id=i, name=i, width=w, height=h,
                               cells=synth_cells(w, h, 1000 + n, members=args.members, eps=0.03))
            for n, i in enumerate(ids)]
    cold = products(ours, warm)["seconds"]
    o = products(ours, us)
    same = {key: r[key] == o[key] for key in ("digest", "bins", "composite_sha", "sim_sha",
                                              "outliers", "clusters")}
    print(json.dumps({"workload": f"{k} masks {w}x{h}, tau {args.tau}",
                      "reference": f"baseline/_ref floodstream {ref.__version__} (numpy backend)",
                      "identical": same, "all_identical": all(same.values()),
                      "reference_s": round(r["seconds"], 3), "b200_s": round(o["seconds"], 3),
                      "b200_cold_s": round(cold, 3),
                      "speedup": round(r["seconds"] / o["seconds"], 1),
                      "clusters": len(o["clusters"]), "digest": o["digest"]}))


if __name__ == "__main__":
    main()
