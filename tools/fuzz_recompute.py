#!/usr/bin/env python
"""Randomised parity sweep of the fused recompute (counts, histogram, composite, Gram)
against the oracle: random ensemble sizes (1..600 masks, so single narrow / 128 / 256
panels and several 256-mask panels with CTA pairs), random raster shapes, random slot
offsets and permutations, random depth values.  Runs for --seconds on one GPU and prints
one JSON line (cases, failures).  Test infrastructure: the oracle is the checker.

Usage: python tools/fuzz_recompute.py [--seconds 300] [--seed 1]
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
sys.path.insert(0, str(REPO / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300.0)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    from oracle import fs_oracle as O
    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.ensemble import DeviceEnsemble

    N.set_device(0)
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + args.seconds
    cases, failures = 0, []
    while time.time() < t_end:
        k = int(rng.choice([rng.integers(1, 130), rng.integers(120, 300), rng.integers(250, 600)]))
        budget = 6_000_000 // max(k, 1)  # keep the oracle Gram cheap
        h = int(rng.integers(1, max(2, int(np.sqrt(budget)) + 1)))
        w = int(rng.integers(1, max(2, budget // max(h, 1) + 1)))
        first = int(rng.integers(0, 4))
        p = rng.uniform(0.02, 0.98)
        cells = [(rng.random((h, w)) < p).astype(np.uint8) *
                 rng.integers(1, 256, (h, w)).astype(np.uint8) for _ in range(k)]
        want = O.accumulate(cells, w, h)
        gw = O.gram(cells)
        with DeviceEnsemble(w, h, k + first + int(rng.integers(0, 3))) as ens:
            ens.upload(cells, first=first)
            perm = rng.permutation(k) if rng.random() < 0.5 else np.arange(k)
            slots = [first + int(x) for x in perm]
            c, b, r, g, fused = ens.products(slots, engine="tc-f4")
        ok = (np.array_equal(c, want)
              and b.tolist() == O.overlap_counts(want.reshape(-1), k).tolist()
              and np.array_equal(r, O.composite(want, k))
              and np.array_equal(g, gw[np.ix_(perm, perm)]))
        cases += 1
        if not ok:
            failures.append({"k": k, "w": w, "h": h, "first": first, "fused": bool(fused)})
    print(json.dumps({"cases": cases, "failures": failures, "seed": args.seed,
                      "seconds": args.seconds}))
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
