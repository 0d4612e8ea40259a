"""Per-phase cycle breakdown of the cluster panel kernel."""
import sys, ctypes
sys.path.insert(0, ".")
import torch
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import device as dv, _capi
from paper_2411_09859_b200.inputs import skew_lower
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
xd = dv.to_device_colmajor(skew_lower(n, 0))
import os
lib = _capi.load()
pk.ltlt_blk_piv_device(xd, b, "var1"); torch.cuda.synchronize()
buf = torch.zeros(160 * 16, dtype=torch.int64, device="cuda")
lib.skl_debug_set_panel_profile.argtypes = [ctypes.c_void_p]
lib.skl_debug_set_panel_profile(buf.data_ptr())
pk.ltlt_blk_piv_device(xd, b, "var1"); torch.cuda.synchronize()
lib.skl_debug_set_panel_profile(None)
p = buf.view(160, 16).cpu().numpy()
names = ["v+warp_argmax", "cta_cand+publish", "cluster_barrier", "winner+gather+rowread", "gemv(az)", "swap/scale/z"]
for c in ([0, 7, 15] if n <= 8192 else [0, 8, 63, 127]):
    steps = max(p[c, 6], 1)
    tot = p[c, :6].sum()
    print(f"cta {c}: {tot/steps:.0f} cyc/step over {steps} steps: " + ", ".join(f"{names[i]}={p[c,i]/steps:.0f}" for i in range(6))
          + (f"; kernel total {p[c,7]/1e6:.2f} Mcyc, outside the step loop {(p[c,7]-tot)/1e6:.2f} Mcyc"
             f" (prologue {p[c,8]/1e6:.2f}, loop-end..prof {p[c,9]/1e6:.2f}, start..gperm {p[c,10]/1e6:.2f}, pbuf {p[c,11]/1e6:.2f})" if p[c, 7] else "")
          + f"; phase 3 cumulative: winner {p[c,12]/steps:.0f}, gathers issued {p[c,13]/steps:.0f}, row poll {p[c,14]/steps:.0f}")
