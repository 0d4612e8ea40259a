"""Per-phase cycle breakdown of the panel kernel (profiling build)."""
import os, sys, ctypes
os.environ["SKEWLTL_B200_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_2411_09859_b200", "_lib", "libskewltl_b200_prof.so")
sys.path.insert(0, ".")
import torch
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import device as dv, _capi
from paper_2411_09859_b200.inputs import skew_lower
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
xd = dv.to_device_colmajor(skew_lower(n, 0))
pk.ltlt_blk_piv_device(xd, b, "var1"); torch.cuda.synchronize()
lib = _capi.load()
buf = (ctypes.c_ulonglong * 32)()
lib.skl_debug_panel_profile(buf)
base = list(buf)
pk.ltlt_blk_piv_device(xd, b, "var1"); torch.cuda.synchronize()
lib.skl_debug_panel_profile(buf)
names = ["gemv", "cta_argmax", "publish", "poll", "win_reduce", "fetch_row", "swap", "scale+gather"]
steps = n - 1
for c in range(2):
    tot = sum(buf[c*16+i] - base[c*16+i] for i in range(8))
    print(f"cta{'0' if c == 0 else 'last'}: total {tot/steps:.0f} cyc/step")
    for i, nm in enumerate(names):
        d = buf[c*16+i] - base[c*16+i]
        print(f"   {nm:14s} {d/steps:8.0f} cyc/step  {100*d/max(tot,1):5.1f}%")
ts = (ctypes.c_ulonglong * (8 * 160 * 4))()
lib.skl_debug_panel_ts(ts)
import numpy as np
a = np.array(list(ts), dtype=np.int64).reshape(8, 160, 4)[:, :148, :]
for s in range(8):
    start, pub, seen = a[s, :, 0], a[s, :, 1], a[s, :, 2]
    t0 = start.min()
    print(f"step {100+s}: start spread {start.max()-start.min()} ns, pub {pub.min()-t0}..{pub.max()-t0} (argmax cta {pub.argmax()}), seen {seen.min()-t0}..{seen.max()-t0} ns")
