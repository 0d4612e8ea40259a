import sys, statistics, numpy as np, torch
sys.path.insert(0, ".")
from paper_2411_09859_b200 import apps
from paper_2411_09859_b200.inputs import skew_lower
xs = np.stack([skew_lower(256, i) for i in range(8192)])
for dt in (np.float64, np.float32):
    xd = torch.from_numpy(np.ascontiguousarray(np.swapaxes(xs.astype(dt), 1, 2))).cuda()
    for _ in range(2): apps.ltlt_batched_piv_device(xd)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    t = []
    for _ in range(5):
        e0.record(); apps.ltlt_batched_piv_device(xd); e1.record(); torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    ms = statistics.median(t)
    print(dt.__name__, f"batched 8192x256: {ms:.2f} ms (min {min(t):.2f} max {max(t):.2f}), {8192*256**3/3/ms/1e9:.2f} TFLOP/s", flush=True)
