"""Scratch GPU check of the unblocked two-step kernel vs the oracle."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle, torch
from paper_2411_09859_b200.unblocked import ltlt_unb_twostep, ltlt_unb_twostep_device
from paper_2411_09859_b200 import device as dv
from paper_2411_09859_b200.inputs import skew_lower
for n in (2, 3, 4, 5, 17, 64, 129, 512, 700, 1000):
    x = skew_lower(n, n)
    o = oracle.ltlt_unb_twostep(x, pivot=True)
    r = ltlt_unb_twostep(x, pivot=True)
    pe = np.array_equal(r.p.pivots, o.pivots)
    dt = np.max(np.abs(r.t.tau - o.tau)) / max(np.max(np.abs(o.tau)), 1e-300) if n > 1 else 0
    dl = np.max(np.abs(np.tril(r.l.data, -1) - np.tril(o.work, -1)))
    up = np.array_equal(np.triu(r.l.data), np.triu(x))
    fl = (r.flops.level2, r.flops.level3, r.flops.panel, r.flops.pivot) == tuple(o.flops[k] for k in ("level2","level3","panel","pivot"))
    print(f"twostep n={n}: piv_eq={pe} dtau={dt:.2e} dL={dl:.2e} upper_ok={up} flops_ok={fl}", flush=True)
# unpivoted on a matrix that needs no pivoting (diagonally... use worked example)
x = np.zeros((4, 4), order="F"); x[1,0],x[2,0],x[3,0],x[2,1],x[3,1],x[3,2] = 2,1,3,4,1,5
r = ltlt_unb_twostep(x); print("worked tau", r.t.tau)
x = np.zeros((3,3), order="F"); x[2,0] = 1.0
try:
    ltlt_unb_twostep(x); print("no ZeroPivot!")
except Exception as e: print("ZeroPivot ok:", type(e).__name__, getattr(e, "column", None))
xd = dv.to_device_colmajor(skew_lower(512, 0))
for _ in range(3): ltlt_unb_twostep_device(xd, True)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ltlt_unb_twostep_device(xd, True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"TIME twostep n=512: {ms:.3f} ms  {512**3/3/ms/1e6:.2f} GFLOP/s")
