#!/usr/bin/env python
"""Pinned H2D bandwidth with 1, 2 and 4 concurrent copy streams (is one DMA stream the
PCIe limit?).  JSON on stdout."""
import json
import sys

import torch


def run(nstreams, total=4 << 30, reps=3):
    chunk = total // nstreams
    h = [torch.empty(chunk, dtype=torch.uint8).pin_memory() for _ in range(nstreams)]
    d = [torch.empty(chunk, dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
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


print(json.dumps({f"streams_{n}": round(run(n), 2) for n in (1, 2, 4)}))
