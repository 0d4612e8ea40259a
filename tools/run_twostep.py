import sys, torch
sys.path.insert(0, ".")
from paper_2411_09859_b200.unblocked import ltlt_unb_twostep_device
from paper_2411_09859_b200 import device as dv
from paper_2411_09859_b200.inputs import skew_lower
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
xd = dv.to_device_colmajor(skew_lower(n, 0))
for _ in range(3): ltlt_unb_twostep_device(xd, True)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): ltlt_unb_twostep_device(xd, True)
e1.record(); torch.cuda.synchronize()
print(f"twostep n={n}: {e0.elapsed_time(e1)/5:.3f} ms")
