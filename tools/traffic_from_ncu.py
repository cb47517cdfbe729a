#!/usr/bin/env python
"""Per-launch DRAM traffic and pipe utilisation of a kernel, from one `ncu --set full`
capture, into profiles/traffic.json (bench.py's roofline "traffic" / "ncu" fields).

Usage: python tools/traffic_from_ncu.py <capture.ncu-rep> <key> [--ncu-key KEY]
  <key>       entry for dram__bytes_read.sum + dram__bytes_write.sum (bytes per launch)
  --ncu-key   entry for the utilisation summary (tensor pipe, FP4 issue, SMEM/L1TEX, DRAM)
Runs `ncu -i <capture> --page raw --csv` (the ncu CLI reads captures without a GPU).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import shutil
import subprocess
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
NCU = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"

_UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6}


def raw_metrics(rep: str) -> dict:
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def value(m: dict, name: str) -> float | None:
    if name not in m:
        return None
    v, u = m[name]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * _UNIT.get(u, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("capture")
    ap.add_argument("key")
    ap.add_argument("--ncu-key", default=None)
    args = ap.parse_args()
    m = raw_metrics(args.capture)
    rd, wr = value(m, "dram__bytes_read.sum"), value(m, "dram__bytes_write.sum")
    p = REPO / "profiles" / "traffic.json"
    doc = json.loads(p.read_text()) if p.exists() else {}
    doc[args.key] = int(rd + wr)
    rel = Path(args.capture).resolve()
    try:
        rel = rel.relative_to(REPO)
    except ValueError:
        pass
    if args.ncu_key:
        pick = {
            "tc_pipe_active_pct": "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
            "fp4_mma_ops_pct_of_peak_elapsed":
                "sm__ops_path_tensor_op_utcomma_src_fp4_dst_fp32_sparsity_off.avg."
                "pct_of_peak_sustained_elapsed",
            "l1tex_tensor_smem_wavefronts_pct":
                "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "duration_us": "gpu__time_duration.sum",
            "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
        }
        summ = {}
        for k, name in pick.items():
            x = value(m, name)
            if x is not None:
                summ[k] = round(x, 2 if k != "duration_us" else 1)
        summ["dram_read_bytes"] = int(rd)
        summ["dram_write_bytes"] = int(wr)
        summ["source"] = f"{rel} (ncu --set full, one launch)"
        doc[args.ncu_key] = summ
    doc["_source"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from ncu --set full "
                      "captures (tools/traffic_from_ncu.py); see each *_ncu entry's source")
    p.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps({args.key: doc[args.key], **({args.ncu_key: doc[args.ncu_key]}
                                                  if args.ncu_key else {})}))


if __name__ == "__main__":
    main()
