#!/usr/bin/env python
"""Recompute cost across ensemble sizes on one B200: for k masks of P pixels (fixed
k * P = 2^34 mask-pixels, i.e. the C2 volume, plus C1-sized small cases) time one full
recompute — counts + histogram + composite + exact Gram (fs_ensemble_recompute, device
outputs, CUDA events on the ensemble stream) — and report mask-pixels/s, the Gram's
useful tensor ops k(k+1)P against 9 PFLOP/s FP4, and the overlap bytes against the
measured HBM bandwidth.  JSON lines on stdout."""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    import argparse

    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="", help="k:w:h,... (default: the built-in list)")
    ap.add_argument("--fused-only", action="store_true", help="skip the separate-pass timings")
    args = ap.parse_args()

    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.ensemble import DeviceEnsemble

    N.set_device(0)
    peaks = {}
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        peaks = json.loads(p.read_text())
    hbm = float(peaks.get("hbm_gbs", 6550.0))
    cases = [(16, 1024, 1024), (64, 4096, 4096), (128, 8192, 8192), (256, 8192, 8192),
             (384, 8192, 5461), (512, 8192, 4096), (1024, 4096, 4096), (2048, 4096, 2048),
             (4096, 4096, 1024)]
    if args.cases:
        cases = [tuple(int(x) for x in c.split(":")) for c in args.cases.split(",")]
    for k, w, h in cases:
        P = w * h
        with DeviceEnsemble(w, h, k) as ens:
            ens.synth(0, k, seed=2104, members=16, eps=0.02)
            d_c = torch.empty(P, dtype=torch.int32, device="cuda")
            d_r = torch.empty(P * 4, dtype=torch.uint8, device="cuda")
            d_b = torch.empty(k + 1, dtype=torch.int64, device="cuda")
            d_g = torch.empty(k * k, dtype=torch.int64, device="cuda")
            ms = []
            for it in range(8):
                fused = ens.products(list(range(k)), engine="tc-f4", out_counts=d_c.data_ptr(),
                                     out_rgba=d_r.data_ptr(), out_bins=d_b.data_ptr(),
                                     out_gram=d_g.data_ptr(), device_outputs=True)[4]
                if it >= 2:
                    ms.append(ens.kernel_ms("recompute"))
            t = statistics.median(ms)
            # the same products as separate passes: overlap kernel + Gram (tc-f4 / popc)
            alt = {}
            for eng in () if args.fused_only else ("tc-f4", "popc"):
                ov, gr = [], []
                for it in range(5):
                    ens.overlap(list(range(k)), out_counts=d_c.data_ptr(), out_rgba=d_r.data_ptr(),
                                out_bins=d_b.data_ptr(), device_outputs=True)
                    if it >= 1:
                        ov.append(ens.kernel_ms("overlap"))
                    if eng == "popc" and k > 512:
                        continue
                    ens.gram(list(range(k)), engine=eng, out=d_g.data_ptr(), device_outputs=True)
                    if it >= 1:
                        gr.append(ens.kernel_ms("gram"))
                alt["overlap_ms"] = round(statistics.median(ov), 4)
                if gr:
                    alt[f"gram_{eng}_ms"] = round(statistics.median(gr), 4)
            ops = float(k) * (k + 1) * P
            ov_bytes = k * P / 8 + 8 * P + 8 * (k + 1)
            print(json.dumps({"k": k, "width": w, "height": h, "mask_px": k * P,
                              "recompute_ms": round(t, 4), "fused": fused,
                              "tpx_per_s": round(k * P / t / 1e9, 3),
                              "gram_tflops": round(ops / t / 1e9, 1),
                              "fp4_frac": round(ops / t / 1e9 / 9000.0, 4),
                              "overlap_gbs": round(ov_bytes / t / 1e6, 1),
                              "hbm_frac": round(ov_bytes / t / 1e6 / hbm, 4), **alt}), flush=True)
            del d_c, d_r, d_b, d_g


if __name__ == "__main__":
    main()
