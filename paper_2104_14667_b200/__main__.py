"""``python -m paper_2104_14667_b200 bench <suite>`` — the reference's measurement suites
for this path (fs/cli.py:72-150 ``bench backends | dual | transfer | sweep``), run on the
device instead of the reference's cost model.  Reports use the reference's BenchReport /
RateMap schemas and the same ``--out file.{json,csv}`` convention; errors exit 2.
"""

from __future__ import annotations

import argparse
import json
import sys


def _write(report, out: str | None) -> None:
    if not out:
        return
    with open(out, "w") as f:
        if out.endswith(".csv"):
            f.write(report.to_csv())
        else:
            json.dump(report.to_json(), f, indent=1)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2104_14667_b200")
    top = ap.add_subparsers(dest="cmd", required=True)
    bench = top.add_parser("bench", help="measured benchmark suites (B200)")
    subs = bench.add_subparsers(dest="suite", required=True)
    b = subs.add_parser("backends", help="protocol vs batched backend (fs/cli.py:121-126)")
    b.add_argument("--pixels", type=int, default=1 << 20)
    b.add_argument("--surfaces", type=int, default=16)
    b.add_argument("--repeats", type=int, default=3)
    b.add_argument("--seed", type=int, default=0)
    d = subs.add_parser("dual", help="the four upload strategies, measured")
    d.add_argument("--dims", nargs="*", default=["2k", "4k", "8k"])
    d.add_argument("--n", nargs="*", type=int, default=[10, 100, 1000])
    d.add_argument("--repeats", type=int, default=3)
    t = subs.add_parser("transfer", help="pinned / pageable host->device ladder")
    t.add_argument("--min-bytes", type=int, default=64 << 10)
    t.add_argument("--max-bytes", type=int, default=64 << 20)
    t.add_argument("--step-bytes", type=int, default=4 << 20)
    t.add_argument("--repeats", type=int, default=5)
    t.add_argument("--pageable", action="store_true")
    s = subs.add_parser("sweep", help="transform rate over raster dimensions")
    s.add_argument("--start", type=int, default=512)
    s.add_argument("--step", type=int, default=500)
    s.add_argument("--stop", type=int, default=16012)
    s.add_argument("--reps", type=int, default=5)
    for p in (b, d, t, s):
        p.add_argument("--out", help="write the report to a .csv or .json file")
    args = ap.parse_args(argv)

    from . import sweep as S

    try:
        if args.suite == "backends":
            rep = S.run_backend_comparison(pixels=args.pixels, n_surfaces=args.surfaces,
                                           repeats=args.repeats, seed=args.seed)
            for row in rep.rows:
                print(f"{row['backend']:>13}: {row['mpix_per_s']:.1f} Mpx/s "
                      f"({row['best_s'] * 1e3:.2f} ms best of {args.repeats})")
        elif args.suite == "dual":
            rep = S.run_dual_buffer_suite(args.dims, args.n, repeats=args.repeats)
            for row in rep.rows:
                print(f"{row['dims']:>4} {row['variant']:>10} N={row['n']:<6} "
                      f"{row['total_us'] / 1e3:10.2f} ms  {row['rate_gbps']:6.2f} GB/s  "
                      f"eff {100 * row['efficiency']:5.1f}%")
        elif args.suite == "transfer":
            rep = S.run_transfer_baseline(args.min_bytes, args.max_bytes, args.step_bytes,
                                          args.repeats, pinned=not args.pageable)
            for row in rep.rows:
                print(f"{row['bytes']:>12} B  {row['rate_gbps']:6.2f} GB/s")
        else:
            rep = S.run_transform_sweep(S.SweepSpec(args.start, args.step, args.stop),
                                        reps=args.reps)
            r = rep.rates
            print(f"{r.shape[0]}x{r.shape[1]} cells, {r.min():.1f}..{r.max():.1f} GB/s")
        _write(rep, args.out)
        return 0
    except (ValueError, RuntimeError, MemoryError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
