"""Phase clocks of panel_push_kernel (profiling build: make prof), one panel launch.
    SKEWLTL_B200_LIB=paper_2411_09859_b200/_lib/libskewltl_b200_prof.so python tools/push_phases.py 512:96 4096:96"""
import ctypes, json, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2411_09859_b200 import _capi, device as dv
from paper_2411_09859_b200.inputs import skew_lower
import os
NAMES = ["v+warp_argmax", "sync1", "cta_cand+push_issue", "cand_wait", "winner+gather+scale", "row_wait",
         "z+sync2", "gemv"]
if os.environ.get("MULTI_NAMES"):
    NAMES = ["v+argmax+sync", "cand_send", "cluster_wait", "publish", "record_poll+sync", "swap+gather+scale",
             "row_poll+z+sync", "gemv"]
lib = _capi.load()
for case in sys.argv[1:]:
    n, w = (int(v) for v in case.split(":"))
    x = dv.to_device_colmajor(skew_lower(n, 0))
    L = dv.empty_colmajor(n, n, torch.float64)
    tau = torch.zeros(n - 1, dtype=torch.float64, device="cuda")
    piv = torch.zeros(n, dtype=torch.int64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    nb = lib.skl_ltlt_unb_panel_workspace_size(n, w)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    def once():
        _capi.check(lib.skl_ltlt_unb_panel(n, w, 1, x.data_ptr(), n, L.data_ptr(), n, tau.data_ptr(), piv.data_ptr(),
                                           info.data_ptr(), ws.data_ptr(), nb, dv.stream_ptr()), "panel")
    once(); torch.cuda.synchronize()
    buf = torch.zeros(160 * 16, dtype=torch.int64, device="cuda")
    lib.skl_debug_set_panel_profile.argtypes = [ctypes.c_void_p]
    lib.skl_debug_set_panel_profile(buf.data_ptr()); once(); torch.cuda.synchronize()
    lib.skl_debug_set_panel_profile(None)
    p = buf.view(160, 16).cpu().numpy().astype(float)
    for c in ((0, 7, 15) if not os.environ.get("MULTI_NAMES") else (0, 50, 100)):
        st = max(p[c, 8], 1)
        print(json.dumps({"n": n, "w": w, "cta": c, "steps": int(st), "sum": round(p[c, :8].sum() / st),
                          **{NAMES[i]: round(p[c, i] / st) for i in range(8)},
                          "gemv_sub(zk,cached,uncached)": [round(p[c, 9 + i] / st) for i in range(3)],
                          "p1_sub(armed,v_done)": [round(p[c, 12 + i] / st) for i in range(2)]}))
    if not os.environ.get("MULTI_NAMES"):
        for c in (0, 7, 15):
            st = max(p[c, 8], 1)
            print(f"  n={n} cta {c} per warp [winner..scale, row_wait, z, sync2_wait]: " +
                  " ".join("w%d:%s" % (w, [round(p[32 + c * 8 + w, i] / st) for i in range(4)]) for w in range(8)))
