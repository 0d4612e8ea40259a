"""Per-step phase clocks of ONE pivoted panel launch (profiling build only).

    SKEWLTL_B200_LIB=paper_2411_09859_b200/_lib/libskewltl_b200_prof.so \
        python tools/panel_phases.py 4096:96 16384:128 [--json out.json]

Each n:width runs skl_ltlt_unb_panel (the first `width` columns of X, the same
panel plan the blocked driver uses for its first panel at that n) twice; the
second run's per-CTA clock64 phase counters are reported as cycles per
elimination step.  Phase boundaries are the CMARK points in panel_cluster.cu.
"""
import argparse
import ctypes
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2411_09859_b200 import _capi
from paper_2411_09859_b200 import device as dv
from paper_2411_09859_b200.inputs import skew_lower

NAMES = ["v+warp_argmax", "cta_cand+publish", "exchange_wait", "winner+gather+row", "gemv_az", "swap_scale_z"]


def run(n, width, lib):
    x = dv.to_device_colmajor(skew_lower(n, 0))
    L = dv.empty_colmajor(n, n, torch.float64)
    tau = torch.zeros(n - 1, dtype=torch.float64, device="cuda")
    piv = torch.zeros(n, dtype=torch.int64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    nbytes = lib.skl_ltlt_unb_panel_workspace_size(n, width)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

    def once():
        st = lib.skl_ltlt_unb_panel(n, width, 1, x.data_ptr(), n, L.data_ptr(), n, tau.data_ptr(), piv.data_ptr(),
                                    info.data_ptr(), ws.data_ptr(), nbytes, dv.stream_ptr())
        _capi.check(st, "panel")

    once()
    torch.cuda.synchronize()
    buf = torch.zeros(160 * 16, dtype=torch.int64, device="cuda")
    lib.skl_debug_set_panel_profile.argtypes = [ctypes.c_void_p]
    lib.skl_debug_set_panel_profile(buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    once()
    e1.record()
    torch.cuda.synchronize()
    lib.skl_debug_set_panel_profile(None)
    ms = e0.elapsed_time(e1)
    p = buf.view(160, 16).cpu().numpy().astype(np.float64)
    ctas = int(np.count_nonzero(p[:, 6]))
    out = {"n": n, "width": width, "ctas": ctas, "ms": ms, "steps": int(p[0, 6]),
           "us_per_step": 1e3 * ms / max(p[0, 6], 1), "cta": {}}
    for c in sorted({0, ctas // 2, ctas - 1}):
        steps = max(p[c, 6], 1)
        row = {NAMES[i]: round(p[c, i] / steps, 1) for i in range(6)}
        row["sum"] = round(p[c, :6].sum() / steps, 1)
        row["phase3_split"] = {"winner": round(p[c, 12] / steps, 1), "gathers_issued": round(p[c, 13] / steps, 1),
                               "row_ready": round(p[c, 14] / steps, 1)}
        row["outside_loop_Mcyc"] = round((p[c, 7] - p[c, :6].sum()) / 1e6, 3)
        out["cta"][c] = row
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="+")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    lib = _capi.load()
    res = []
    for c in args.cases:
        n, w = (int(v) for v in c.split(":"))
        r = run(n, w, lib)
        res.append(r)
        print(json.dumps(r), flush=True)
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
