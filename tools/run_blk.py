"""Run ltlt_blk_piv_device a few times (for ncu launch lists / profiles)."""
import sys, argparse
sys.path.insert(0, ".")
import torch
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import device as dv
from paper_2411_09859_b200.inputs import skew_lower
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096); ap.add_argument("--b", type=int, default=128)
ap.add_argument("--fused", default="var1"); ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
xd = dv.to_device_colmajor(skew_lower(a.n, 0))
for _ in range(a.reps):
    pk.ltlt_blk_piv_device(xd, a.b, a.fused)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); pk.ltlt_blk_piv_device(xd, a.b, a.fused); e1.record(); torch.cuda.synchronize()
print(f"n={a.n} b={a.b} {a.fused}: {e0.elapsed_time(e1):.3f} ms")
