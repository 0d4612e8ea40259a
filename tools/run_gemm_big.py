"""One large trailing update C(n lower) += -A T A^T (k columns) via the C ABI (ncu target)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2411_09859_b200 import _capi, device as dv
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 140
lib = _capi.load()
rng = np.random.default_rng(0)
A = dv.to_device_colmajor(rng.standard_normal((n, k)))
tau = torch.as_tensor(rng.standard_normal(k - 1), device="cuda")
C = dv.empty_colmajor(n, n, torch.float64); C.normal_()
nb = lib.skl_sktri_rankk_workspace_size(n, k); ws = dv.workspace(nb)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(3):
    e0.record()
    st = lib.skl_sktri_rankk_lower(n, k, -1.0, A.data_ptr(), n, tau.data_ptr(), 1.0, C.data_ptr(), n, ws.data_ptr(), nb, dv.stream_ptr())
    e1.record(); torch.cuda.synchronize(); assert st == 0
    ms = e0.elapsed_time(e1)
    print(f"rankk n={n} k={k}: {ms:.3f} ms -> {2*k*n*(n-1)/2/ms/1e9:.2f} TFLOP/s")
