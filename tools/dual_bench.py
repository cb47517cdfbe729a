#!/usr/bin/env python
"""The paper's dual-buffer study (Figs. 5-8) measured on the B200:
sweep.run_dual_buffer_suite over 2k / 4k / 8k images, the four strategies and
N in {10, 100, 1000}; JSON (BenchReport schema, suite "dual") on stdout."""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", nargs="*", default=["2k", "4k", "8k"])
    ap.add_argument("--n", nargs="*", type=int, default=[10, 100, 1000])
    ap.add_argument("--repeats", type=int, default=3)
    args = ap.parse_args()
    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.sweep import run_dual_buffer_suite

    N.set_device(0)
    rep = run_dual_buffer_suite(args.dims, args.n, repeats=args.repeats)
    doc = rep.to_json()
    doc["summary"] = {f"{r['dims']}/{r['variant']}/{r['n']}": round(r["efficiency"], 4)
                      for r in rep.rows}
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
