"""Config-2b skr2k microbench driver (for ncu captures and A/B timing; L2 flushed like bench.py)."""
import sys, statistics
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2411_09859_b200 import _capi, kernels3, device as dv
N = 4096
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
lib = _capi.load()
rng = np.random.default_rng(0)
Bd = dv.to_device_colmajor(rng.standard_normal((N, 128)))
Wd = kernels3.form_w_device(Bd, torch.as_tensor(rng.standard_normal(127), device="cuda"))
Cd = dv.to_device_colmajor(rng.standard_normal((N, N)))
nb = lib.skl_skr2k_workspace_size(N, 128); ws = dv.workspace(nb)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for it in range(reps):
    flush.zero_(); torch.cuda.synchronize()
    e0.record()
    st = lib.skl_skr2k_lower(N, 128, 1.0, Bd.data_ptr(), N, Wd.data_ptr(), N, 1.0, Cd.data_ptr(), N, 1, ws.data_ptr(), nb, None, dv.stream_ptr())
    e1.record(); torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
    if reps <= 8:
        print(f"skr2k call {it}: {ms[-1]:.4f} ms -> {2146959360/ms[-1]/1e9:.2f} TFLOP/s")
m = statistics.median(ms[2:] if reps > 4 else ms)
print(f"skr2k median {m*1e3:.1f} us -> {2146959360/m/1e9:.2f} TFLOP/s ({100*2146959360/m/1e9/35.44:.1f} % of 35.44)")
