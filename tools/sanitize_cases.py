#!/usr/bin/env python
"""Small invocations of every device kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck): protocol primitives, transform, fused and unfused
overlap, both tensor-core Gram kernels (single CTA incl. the fused overlap pass, and
the CTA-pair off-diagonal kernel), the CUDA-core Gram, streaming with per-item
accumulate, device synth.  Each result is checked against the oracle so a sanitizer
run is also a parity run."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))


def main():
    from oracle import fs_oracle as O
    from paper_2104_14667_b200 import _kernels_cuda as K
    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.ensemble import DeviceEnsemble
    from paper_2104_14667_b200.synth import synth_cells, synth_cells_gpu

    N.set_device(0)
    rng = np.random.default_rng(5)
    n = 4099
    a = rng.integers(0, 3, n).astype(np.uint8)
    b = rng.integers(0, 3, n).astype(np.uint8)
    counts = np.zeros(n, np.uint32)
    K.accumulate_into(counts, a)
    K.accumulate_into(counts, b)
    assert np.array_equal(counts, (a > 0).astype(np.uint32) + (b > 0))
    assert np.array_equal(np.asarray(K.overlap_counts(counts, 2)), O.overlap_counts(counts, 2))
    assert K.pair_counts(a, b) == O.pair_counts(a, b)
    out = np.zeros((n, 4), np.uint8)
    K.composite_fill(counts, 2, out)
    want = np.zeros((n, 4), np.uint8)
    O.composite_fill(counts, 2, want)
    assert np.array_equal(out, want)
    print("primitives ok", flush=True)

    # (1024, 1024, 144): the fused k <= 256 recompute with ~7 units per CTA, so both
    # expander groups, the operand ring and the partial rings wrap several times
    for (w, h, k) in [(130, 33, 20), (96, 20, 256), (1024, 1024, 144), (64, 40, 300)]:
        cells = [synth_cells(w, h, i, members=5, eps=0.05) for i in range(k)]
        with DeviceEnsemble(w, h, k) as ens:
            ens.stream(cells, variant="2b-final", with_kernel=True)
            c, bins, r = ens.overlap()
            want = O.accumulate(cells, w, h)
            assert np.array_equal(c, want)
            for eng in ("tc-f4", "tc", "popc"):
                g = ens.gram(engine=eng)
                assert np.array_equal(g, O.gram(cells)), eng
            c2, b2, r2, g2, fused = ens.products(engine="tc-f4")
            assert np.array_equal(c2, want) and np.array_equal(g2, O.gram(cells))
            rc, _, _ = ens.running_counts(k)
            assert np.array_equal(rc, want)
        print(f"ensemble {w}x{h} k={k} ok (fused={fused})", flush=True)
    got = synth_cells_gpu(257, 31, 3, members=2, eps=0.1)
    assert np.array_equal(got, synth_cells(257, 31, 3, members=2, eps=0.1))
    print("synth ok", flush=True)


if __name__ == "__main__":
    main()
