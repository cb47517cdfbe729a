#!/usr/bin/env python
"""Pinned host -> device bandwidth (SURVEY §8(d) BW_pcie, the reference's transfer ladder
fs/bench.py:193-228 measured): per visible GPU alone, then every visible GPU copying at
the same time (one host thread per GPU, each with its own pinned buffer; on an 8-GPU box
this shows whether the host's PCIe root complexes sustain all links at once), plus 1 / 2 /
4 concurrent copy streams on GPU 0 (is one DMA stream the PCIe limit?).  JSON on stdout.

Usage: python tools/h2d_probe.py [--gib 1] [--reps 3]"""
from __future__ import annotations

import argparse
import json
import threading
import time

import torch


def _one_gpu(dev: int, nbytes: int, reps: int, start=None) -> float:
    """best GB/s of `reps` pinned H2D copies of nbytes on device `dev`"""
    torch.cuda.set_device(dev)
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dev}")
    s = torch.cuda.Stream(device=dev)
    d.copy_(h)  # warm-up
    torch.cuda.synchronize(dev)
    if start is not None:
        start.wait()
    best = 0.0
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            d.copy_(h, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def streams(nstreams: int, total: int, reps: int) -> float:
    chunk = total // nstreams
    h = [torch.empty(chunk, dtype=torch.uint8).pin_memory() for _ in range(nstreams)]
    d = [torch.empty(chunk, dtype=torch.uint8, device="cuda:0") for _ in range(nstreams)]
    ss = [torch.cuda.Stream(device=0) for _ in range(nstreams)]
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize(0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in ss:
            s.wait_stream(torch.cuda.current_stream())
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i].copy_(h[i], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        best = max(best, chunk * nstreams / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    nbytes = int(args.gib * (1 << 30))
    ngpu = torch.cuda.device_count()
    doc = {"probe": "pinned H2D GB/s, best of reps, CUDA events per device",
           "bytes": nbytes, "gpus": ngpu,
           "per_gpu_alone": {str(g): round(_one_gpu(g, nbytes, args.reps), 2) for g in range(ngpu)}}
    # all GPUs at once: threads released together, each timing its own device's copies
    res = [0.0] * ngpu
    start = threading.Event()

    def worker(g):
        res[g] = _one_gpu(g, nbytes, args.reps, start)

    th = [threading.Thread(target=worker, args=(g,)) for g in range(ngpu)]
    for t in th:
        t.start()
    time.sleep(0.5)
    t0 = time.perf_counter()
    start.set()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    doc["all_gpus_concurrent"] = {"per_gpu": {str(g): round(res[g], 2) for g in range(ngpu)},
                                  "sum_gbs": round(sum(res), 2),
                                  "aggregate_wall_gbs": round(ngpu * nbytes * args.reps / wall / 1e9, 2)}
    doc["gpu0_copy_streams"] = {f"streams_{n}": round(streams(n, 4 << 30, args.reps), 2)
                                for n in (1, 2, 4)}
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
