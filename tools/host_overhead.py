#!/usr/bin/env python
"""Host-side cost per recompute call at config 1 (16 x 1024^2): the C ABI call alone
(device outputs, no sync), and the full pipelined frame of ShardedEnsemble.run_frames.
JSON on stdout."""
import json
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    import torch

    from paper_2104_14667_b200 import _native as N
    from paper_2104_14667_b200.dist import ShardedEnsemble

    N.set_device(0)
    w = h = 1024
    k = 16
    sh = ShardedEnsemble(w, h, k)
    sh.ens.synth(0, k, seed=2104, members=1, eps=0.5)
    dev = torch.device("cuda", 0)
    d_c = torch.empty(w * h, dtype=torch.int32, device=dev)
    d_r = torch.empty(w * h * 4, dtype=torch.uint8, device=dev)
    d_p = torch.empty(k + 1 + k * k, dtype=torch.int64, device=dev)
    import numpy as np

    sl = np.arange(k, dtype=np.uint32)
    for _ in range(20):
        sh.ens.products(sl, out_counts=d_c.data_ptr(), out_rgba=d_r.data_ptr(),
                        out_bins=d_p.data_ptr(), out_gram=d_p.data_ptr() + (k + 1) * 8,
                        device_outputs=True)
    torch.cuda.synchronize()
    n = 500
    t0 = time.perf_counter()
    for _ in range(n):
        sh.ens.products(sl, out_counts=d_c.data_ptr(), out_rgba=d_r.data_ptr(),
                        out_bins=d_p.data_ptr(), out_gram=d_p.data_ptr() + (k + 1) * 8,
                        device_outputs=True)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out = {"abi_call_us": round((t1 - t0) / n * 1e6, 2),
           "device_us_per_recompute": round((t2 - t0) / n * 1e6, 2)}
    sh.run_frames(sl, 20, keep=False)
    t0 = time.perf_counter()
    sh.run_frames(sl, n, keep=False)
    out["run_frames_us_per_frame"] = round((time.perf_counter() - t0) / n * 1e6, 2)
    with sh.ens.pipeline(sl, depth=3) as pipe:
        pipe.run(20)
        t0 = time.perf_counter()
        r = pipe.run(n)
        out["native_pipeline_us_per_frame"] = round((time.perf_counter() - t0) / n * 1e6, 2)
        out["native_pipeline_device_us_per_frame"] = round(r["device_ms"] * 1e3 / n, 2)
    sh.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
