#!/usr/bin/env python
"""Probe: cost of cudaHostRegister/Unregister on pageable numpy arrays (the price of
zero-copy protocol calls).  JSON on stdout."""
import ctypes
import json
import time

import numpy as np

rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
rt.cudaHostUnregister.argtypes = [ctypes.c_void_p]
rt.cudaFree(None)
out = {}
for mb in (1, 4, 16, 64):
    a = np.ones(mb << 20, np.uint8)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        rc = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        t1 = time.perf_counter()
        rc2 = rt.cudaHostUnregister(a.ctypes.data)
        t2 = time.perf_counter()
        ts.append(((t1 - t0) * 1e6, (t2 - t1) * 1e6, rc, rc2))
    out[f"{mb}MB"] = {"register_us": round(min(t[0] for t in ts), 1),
                      "unregister_us": round(min(t[1] for t in ts), 1), "rc": ts[-1][2:]}
print(json.dumps(out))
