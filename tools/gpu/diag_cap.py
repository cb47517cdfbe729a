import sys, json
sys.path.insert(0, '.')
from paper_2104_14667_b200 import _native as N
from paper_2104_14667_b200.ensemble import DeviceEnsemble
import torch
N.set_device(0)
w = h = 8192
out = {}
for cap in (256, 264):
    with DeviceEnsemble(w, h, cap) as ens:
        ens.synth(0, 256, seed=2104, members=16, eps=0.02)
        d_c = torch.empty(w * h, dtype=torch.int32, device="cuda")
        d_r = torch.empty(w * h * 4, dtype=torch.uint8, device="cuda")
        d_p = torch.empty(257 + 256 * 256, dtype=torch.int64, device="cuda")
        ms = []
        for first in (0, 1, 0, 1, 0, 1):
            sl = list(range(first, first + 256)) if first + 256 <= cap else list(range(256))
            ens.products(sl, engine="tc-f4", out_counts=d_c.data_ptr(), out_rgba=d_r.data_ptr(),
                         out_bins=d_p.data_ptr(), out_gram=d_p.data_ptr() + 257 * 8, device_outputs=True)
            ms.append(round(ens.kernel_ms("recompute"), 4))
        out[cap] = ms
print(json.dumps(out))
