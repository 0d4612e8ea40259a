"""Per-step cost of ONE pivoted panel launch as a function of rows and width.

    python tools/panel_sweep.py [--ns 256,512,1024,2048,4096] [--widths 16,32,64,96]

Each (n, width) runs skl_ltlt_unb_panel (first `width` columns) with the driver's
per-class CUDA-event timers on; the panel class (panel kernel + its two finish
kernels) divided by the steps is the per-elimination cost.  The finish kernels'
fixed cost is estimated from the smallest width and reported separately.
"""
import argparse
import ctypes
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2411_09859_b200 import _capi
from paper_2411_09859_b200 import device as dv
from paper_2411_09859_b200.inputs import skew_lower


def panel_ms(lib, n, width, reps=5):
    x = dv.to_device_colmajor(skew_lower(n, 0))
    L = dv.empty_colmajor(n, n, torch.float64)
    tau = torch.zeros(n - 1, dtype=torch.float64, device="cuda")
    piv = torch.zeros(n, dtype=torch.int64, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    nbytes = lib.skl_ltlt_unb_panel_workspace_size(n, width)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

    def once():
        _capi.check(lib.skl_ltlt_unb_panel(n, width, 1, x.data_ptr(), n, L.data_ptr(), n, tau.data_ptr(),
                                           piv.data_ptr(), info.data_ptr(), ws.data_ptr(), nbytes,
                                           dv.stream_ptr()), "panel")
    once()
    torch.cuda.synchronize()
    lib.skl_timing_enable(1)
    for _ in range(reps):
        once()
    torch.cuda.synchronize()
    ms = (ctypes.c_double * 4)()
    cnt = (ctypes.c_int * 4)()
    lib.skl_timing_read(ms, cnt)
    lib.skl_timing_enable(0)
    return ms[0] / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="256,512,1024,2048,4096")
    ap.add_argument("--widths", default="8,16,32,64,96")
    args = ap.parse_args()
    lib = _capi.load()
    out = []
    for n in (int(v) for v in args.ns.split(",")):
        row = {"n": n}
        for w in (int(v) for v in args.widths.split(",")):
            if w >= n:
                continue
            row[w] = round(panel_ms(lib, n, w) * 1e3, 2)   # microseconds per panel launch
        ws = sorted(k for k in row if k != "n")
        if len(ws) >= 2:
            a, b = ws[-2], ws[-1]
            row["us_per_step_marginal"] = round((row[b] - row[a]) / (b - a), 3)
        out.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
