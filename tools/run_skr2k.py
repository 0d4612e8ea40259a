"""Config-2b skr2k microbench driver (for ncu captures)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2411_09859_b200 import _capi, kernels3, device as dv
N = 4096
lib = _capi.load()
rng = np.random.default_rng(0)
Bd = dv.to_device_colmajor(rng.standard_normal((N, 128)))
Wd = kernels3.form_w_device(Bd, torch.as_tensor(rng.standard_normal(127), device="cuda"))
Cd = dv.to_device_colmajor(rng.standard_normal((N, N)))
nb = lib.skl_skr2k_workspace_size(N, 128); ws = dv.workspace(nb)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(4):
    e0.record()
    st = lib.skl_skr2k_lower(N, 128, 1.0, Bd.data_ptr(), N, Wd.data_ptr(), N, 1.0, Cd.data_ptr(), N, 1, ws.data_ptr(), nb, None, dv.stream_ptr())
    e1.record(); torch.cuda.synchronize()
    print(f"skr2k call {it}: {e0.elapsed_time(e1):.4f} ms -> {2146959360/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s")
