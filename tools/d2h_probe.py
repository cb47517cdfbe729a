#!/usr/bin/env python
"""Device -> host copy rate on one B200 (the maps' read-back: counts + RGBA = 8 B/px), next
to host -> device, for pinned destinations: one cudaMemcpyAsync of N bytes, several
chunks on one stream, and chunks split over two streams.  CUDA events, best of 5.
JSON on stdout."""
from __future__ import annotations

import json


def main():
    import torch

    dev = torch.device("cuda", 0)
    out = {"probe": "pinned D2H / H2D copy rate (GB/s), CUDA events, best of 5", "rows": []}
    for mib in (64, 256, 512):
        n = mib << 20
        d = torch.empty(n, dtype=torch.uint8, device=dev)
        h = torch.empty(n, dtype=torch.uint8).pin_memory()
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def timed(fn):
            best = 1e30
            for _ in range(6):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                best = min(best, a.elapsed_time(b))
            return n / (best * 1e-3) / 1e9

        def d2h_one():
            h.copy_(d, non_blocking=True)

        def h2d_one():
            d.copy_(h, non_blocking=True)

        def d2h_two_streams():
            ev = torch.cuda.Event()
            ev.record()
            half = n // 2
            for st, sl in ((s1, slice(0, half)), (s2, slice(half, n))):
                st.wait_event(ev)
                with torch.cuda.stream(st):
                    h[sl].copy_(d[sl], non_blocking=True)
            for st in (s1, s2):
                torch.cuda.current_stream().wait_stream(st)

        out["rows"].append({"mib": mib, "d2h_gbs": round(timed(d2h_one), 2),
                            "h2d_gbs": round(timed(h2d_one), 2),
                            "d2h_two_streams_gbs": round(timed(d2h_two_streams), 2)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
