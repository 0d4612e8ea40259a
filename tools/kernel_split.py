"""Per-kernel-class device time of one factorization (skl_timing hooks)."""
import sys, ctypes
sys.path.insert(0, ".")
import torch
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import device as dv, _capi
from paper_2411_09859_b200.inputs import skew_lower
n = int(sys.argv[1]); b = int(sys.argv[2]); fused = sys.argv[3] if len(sys.argv) > 3 else "var1"
dist = "uniform" if n == 16384 else "normal"
xd = dv.to_device_colmajor(skew_lower(n, 0, dist))
lib = _capi.load()
pk.ltlt_blk_piv_device(xd, b, fused); torch.cuda.synchronize()
lib.skl_timing_enable(1)
pk.ltlt_blk_piv_device(xd, b, fused); torch.cuda.synchronize()
ms = (ctypes.c_double * 4)(); cnt = (ctypes.c_int * 4)()
lib.skl_timing_read(ms, cnt); lib.skl_timing_enable(0)
names = ["panel", "pack", "gemm", "finalize"]
print(f"n={n} b={b} {fused}: " + ", ".join(f"{names[i]}={ms[i]:.2f}ms/{cnt[i]}" for i in range(4)), f"total={sum(ms):.2f}ms")
