"""Phase cycles of the batched kernel, CTA 0 (build: make variant V=bprof VFLAGS=-DSKL_BATCHED_PROF,
run with SKEWLTL_B200_LIB=paper_2411_09859_b200/_lib/libskewltl_b200_vbprof.so)."""
import sys, ctypes, numpy as np, torch
sys.path.insert(0, ".")
from paper_2411_09859_b200 import apps, _capi
from paper_2411_09859_b200.inputs import skew_lower
dt = np.float64 if (len(sys.argv) < 2 or sys.argv[1] == "f64") else np.float32
B = int(sys.argv[2]) if len(sys.argv) > 2 else 148
nm = int(sys.argv[3]) if len(sys.argv) > 3 else 1   # matrices CTA 0 factors in the call
xs = np.stack([skew_lower(256, i) for i in range(B)]).astype(dt)
xd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(xs, 1, 2))).cuda()
apps.ltlt_batched_piv_device(xd); torch.cuda.synchronize()
lib = _capi.load()
out = (ctypes.c_ulonglong * 8)()
lib.skl_debug_read_bprof(out)
names = ["load", "elim0", "gather1", "elim1", "fold", "pass", "fixup"]
tot = sum(out[:7])
print(dt.__name__, f"B={B}: {tot / nm:.0f} cyc/matrix (CTA 0):",
      ", ".join(f"{names[i]}={out[i] / nm:.0f}" for i in range(7)))
