#!/usr/bin/env python
"""SM clock, power and throttle reasons while the C2 fused recompute runs back to back
(k_recompute_f4, 256 x 8192^2, device outputs) for a few seconds — the clock the tensor
roofline is met at.  NVML is sampled every 2 ms on a side thread; the kernel time comes
from CUDA events.  JSON on stdout.

Usage: python tools/clock_under_load.py [--seconds 4] [--k 256] [--size 8192]"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    import pynvml
    import torch

    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.ensemble import DeviceEnsemble

    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--k", type=int, default=256)
    ap.add_argument("--size", type=int, default=8192)
    args = ap.parse_args()
    N.set_device(0)
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    sm_max = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            try:
                samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
            except pynvml.NVMLError:
                pass
            time.sleep(0.002)

    k, w = args.k, args.size
    P = w * w
    with DeviceEnsemble(w, w, k) as ens:
        ens.synth(0, k, seed=2104, members=16, eps=0.02)
        d_c = torch.empty(P, dtype=torch.int32, device="cuda")
        d_r = torch.empty(P * 4, dtype=torch.uint8, device="cuda")
        d_b = torch.empty(k + 1, dtype=torch.int64, device="cuda")
        d_g = torch.empty(k * k, dtype=torch.int64, device="cuda")

        def one():
            ens.products(list(range(k)), engine="tc-f4", out_counts=d_c.data_ptr(),
                         out_rgba=d_r.data_ptr(), out_bins=d_b.data_ptr(),
                         out_gram=d_g.data_ptr(), device_outputs=True)

        for _ in range(5):
            one()
        torch.cuda.synchronize()
        th = threading.Thread(target=sampler, daemon=True)
        th.start()
        ms, n, t_end = [], 0, time.time() + args.seconds
        while time.time() < t_end:
            one()
            n += 1
            if n % 16 == 0:
                ms.append(ens.kernel_ms("recompute"))
        torch.cuda.synchronize()
        stop.set()
        th.join()
    clocks = [s[0] for s in samples]
    power = [s[1] for s in samples]
    reasons = 0
    for s in samples:
        reasons |= s[2]
    names = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake"}
    doc = {"workload": f"k_recompute_f4 back to back, {k} x {w}^2, device outputs",
           "launches": n, "seconds": args.seconds,
           "recompute_ms_median": round(statistics.median(ms), 4) if ms else None,
           "sm_mhz_median": statistics.median(clocks) if clocks else None,
           "sm_mhz_min": min(clocks) if clocks else None, "sm_max_mhz": sm_max,
           "power_w_median": round(statistics.median(power), 1) if power else None,
           "power_w_max": round(max(power), 1) if power else None,
           "throttle_reasons": [v for b, v in names.items() if reasons & b],
           "nvml_samples": len(samples)}
    if doc["sm_mhz_median"] and doc["recompute_ms_median"]:
        # the MMA stream of one launch at this clock: each of the 148 CTAs issues 4 stages
        # of 768 cycles (k <= 256 panel) per 1024-px unit it owns
        units_per_cta = -(-(P // 1024) // 148)
        doc["mma_floor_ms_at_this_clock"] = round(4 * units_per_cta * 768 /
                                                  (doc["sm_mhz_median"] * 1e3), 4)
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
