"""Time apps.solve's device part (skl_ltlt_solve) after one factorization."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import _capi, device as dv
from paper_2411_09859_b200.inputs import skew_lower
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
xd = dv.to_device_colmajor(skew_lower(n, 0))
L, tau, piv = pk.ltlt_blk_piv_device(xd, 128, "var1")
lib = _capi.load()
for nrhs in (1, 16, 128):
    B = dv.to_device_colmajor(np.random.default_rng(0).standard_normal((n, nrhs)))
    nb = lib.skl_ltlt_solve_workspace_size(n, nrhs); ws = dv.workspace(nb)
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(3):
        e0.record()
        lib.skl_ltlt_solve(n, nrhs, L.data_ptr(), n, tau.data_ptr(), piv.data_ptr(), B.data_ptr(), n, 10.0,
                           info.data_ptr(), ws.data_ptr(), nb, dv.stream_ptr())
        e1.record(); torch.cuda.synchronize()
    print(f"solve n={n} nrhs={nrhs}: {e0.elapsed_time(e1):.3f} ms (info {int(info.item())})")
