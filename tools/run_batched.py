import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2411_09859_b200 import apps
from paper_2411_09859_b200.inputs import skew_lower
dt = np.float64 if (len(sys.argv) < 2 or sys.argv[1] == "f64") else np.float32
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
xs = np.stack([skew_lower(256, i) for i in range(B)]).astype(dt)
xd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(xs, 1, 2))).cuda()
for _ in range(2): apps.ltlt_batched_piv_device(xd)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); apps.ltlt_batched_piv_device(xd); e1.record(); torch.cuda.synchronize()
print(f"{dt.__name__} batched {B}x256: {e0.elapsed_time(e1):.2f} ms")
