"""Generate the golden fixtures by running the REFERENCE package itself.

Imports ``floodstream`` from /root/reference/pkg/src (read-only, numpy backend) and,
when built, the reference's Cython accelerator from oracle/_ref, runs the hot-path
functions on seeded inputs and writes their outputs to tests/golden/*.json.  The
inputs are regenerated in the tests from the recorded recipes (numpy default_rng), and
their sha256 is stored so a generator drift is detected rather than silently passing.

Run here (the container that has /root/reference):  python tests/golden/make_golden.py
The fixtures are committed; /root/reference is never read at test time.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent))

import floodstream  # noqa: E402  (the reference)
from floodstream import analytics as ref  # noqa: E402
from floodstream import streaming as ref_stream  # noqa: E402
from floodstream.device import synthetic_default_profile  # noqa: E402
from floodstream.rasters import RasterSurface  # noqa: E402

from golden_inputs import (  # noqa: E402
    c1_cells,
    edge_cases,
    random_case,
    sha,
    stream_case,
)

assert floodstream.backends.kernels.NAME == "numpy", floodstream.backends.kernels.NAME


def surfaces_of(cells_list, ids=None):
    out = []
    for i, c in enumerate(cells_list):
        sid = ids[i] if ids else f"s{i:02d}"
        h, w = c.shape
        out.append(RasterSurface(id=sid, name=sid, width=w, height=h, cells=c))
    return out


def full_record(cells_list, ids, tau_list):
    surfaces = surfaces_of(cells_list, ids)
    grid = ref.accumulate(surfaces)
    hist = ref.overlap_histogram(grid)
    comp = ref.composite_map(grid)
    sim = ref.similarity_matrix(surfaces)
    k = len(surfaces)
    gram = np.zeros((k, k), dtype=np.int64)
    for i in range(k):
        for j in range(i, k):
            inter, union = ref.kernels.pair_counts(surfaces[i].cells.reshape(-1),
                                                   surfaces[j].cells.reshape(-1))
            gram[i, j] = gram[j, i] = inter
    rec = {
        "ids": ids,
        "input_sha": [sha(c) for c in cells_list],
        "counts_sha": sha(grid.counts),
        "digest": grid.digest(),
        "bins": hist.bins,
        "composite_sha": sha(comp.pixels),
        "gram": gram.tolist() if k <= 64 else None,
        "gram_sha": sha(gram),
        "sim_sha": sha(sim),
        "clusters": {repr(t): ref.cluster_surfaces(surfaces, t) for t in tau_list},
    }
    if k >= 2:
        scores = ref.outlier_scores(surfaces)
        rec["outliers"] = {sid: float(v).hex() for sid, v in scores.items()}
    return rec


def main():
    out = {}
    # ---- C1: bench.py:472-475 inputs, 16 x 2^20, seed 0, p = 0.5 ------------------
    cells = c1_cells()
    ids = [f"s{i:02d}" for i in range(16)]
    rec = full_record(cells, ids, [0.8, 0.3])
    flat = [c.reshape(-1) for c in cells]
    rec["pair01"] = list(ref.kernels.pair_counts(flat[0], flat[1]))
    out["c1"] = rec
    # cross-check with the reference's own Cython accelerator when built
    ref_dir = REPO / "oracle" / "_ref"
    if any(ref_dir.glob("_accel*.so")):
        sys.path.insert(0, str(ref_dir))
        import _accel  # the reference's Cython module

        counts = np.zeros(1 << 20, dtype=np.uint32)
        for f in flat:
            _accel.accumulate_into(counts, f)
        assert sha(counts.reshape(1024, 1024)) == rec["counts_sha"]
        assert list(_accel.overlap_counts(counts, 16)) == rec["bins"]
        assert list(_accel.pair_counts(flat[0], flat[1])) == rec["pair01"]
        rgba = np.zeros((1 << 20, 4), dtype=np.uint8)
        _accel.composite_fill(counts, 16, rgba)
        assert sha(rgba.reshape(1024, 1024, 4)) == rec["composite_sha"]
        out["c1"]["cython_agrees"] = True
    # ---- random small cases (test_acceptance.py:241-308 style) ------------------
    cases = []
    for case in range(40):
        cells, ids, tau = random_case(case)
        cases.append({"case": case, "tau": tau, **full_record(cells, ids, [tau])})
    out["random"] = cases
    # ---- edge cases --------------------------------------------------------------
    out["edge"] = {}
    for name, (cells, ids, taus) in edge_cases().items():
        out["edge"][name] = full_record(cells, ids, taus)
    # ---- run_stream cycling (streaming.py:417-433) --------------------------------
    streams = []
    for case in range(6):
        cells, n = stream_case(case)
        h, w = cells[0].shape
        surfaces = surfaces_of(cells)
        grid, _ = ref_stream.run_stream(ref_stream.StreamJob(
            variant=ref_stream.Variant.TWO_BUFFER_FINAL, n=n, width=w, height=h,
            profile=synthetic_default_profile(), surfaces=surfaces))
        streams.append({"case": case, "n": n, "digest": grid.digest(),
                        "counts_sha": sha(grid.counts),
                        "bins": ref.overlap_histogram(grid).bins,
                        "composite_sha": sha(ref.composite_map(grid).pixels)})
    out["stream"] = streams
    # ---- schedule DAGs -----------------------------------------------------------
    sched = {}
    for v in ref_stream.Variant:
        job = ref_stream.StreamJob(variant=v, n=5, width=100, height=60,
                                   profile=synthetic_default_profile())
        g = ref_stream.build_schedule(job)
        sched[v.value] = {"pairs": g.pairs, "nodes": [[n.id, n.kind.value, list(n.deps)]
                                                      for n in g.nodes]}
    out["schedule"] = sched
    # ---- closed form -------------------------------------------------------------
    out["closed_form"] = [
        [c, m, p, list(ref_stream.closed_form_times(c, m, p))]
        for c, m, p in ([[3, 3, 3], [2, 2, 2], [1, 1, 1]], [[10], [1], [1]],
                        [[1, 2, 3, 4], [4, 3, 2, 1], [1, 1, 1, 1]])
    ]
    path = HERE / "golden.json"
    path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
