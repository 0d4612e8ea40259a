"""Run skl_ltlt_unb_panel(n, width) a few times (ncu target for one panel launch)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2411_09859_b200 import _capi, device as dv
from paper_2411_09859_b200.inputs import skew_lower
n, w, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 3
lib = _capi.load()
x = dv.to_device_colmajor(skew_lower(n, 0))
L = dv.empty_colmajor(n, n, torch.float64)
tau = torch.zeros(n - 1, dtype=torch.float64, device="cuda")
piv = torch.zeros(n, dtype=torch.int64, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
nb = lib.skl_ltlt_unb_panel_workspace_size(n, w)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
for _ in range(reps):
    _capi.check(lib.skl_ltlt_unb_panel(n, w, 1, x.data_ptr(), n, L.data_ptr(), n, tau.data_ptr(), piv.data_ptr(),
                                       info.data_ptr(), ws.data_ptr(), nb, dv.stream_ptr()), "panel")
torch.cuda.synchronize()
print("ok", n, w)
