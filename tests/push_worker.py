"""Subprocess body of test_gpu_push.py: factor a few matrices with the panel mode the
environment selects (SKL_PANEL_PUSH) and save L / tau / pivots to the given .npz."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2411_09859_b200 as pk  # noqa: E402
from paper_2411_09859_b200.inputs import skew_lower  # noqa: E402

out = {}
for n, b, fused in ((300, 64, "var1"), (1000, 128, "var2a"), (2049, 96, "var2b"), (512, 512, "var1")):
    r = pk.ltlt_blk_piv(pk.SkewMatrixLower(skew_lower(n, 11 * n)), b=b, fused=fused)
    out[f"L{n}"], out[f"t{n}"], out[f"p{n}"] = np.asarray(r.l.data), np.asarray(r.t.tau), np.asarray(r.p.pivots)
import os  # noqa: E402
if os.environ.get("SKL_TEST_BIG"):
    # crosses the 8192-trailing-row limit of the fused epilogue and the multi- / single-cluster
    # boundary inside one factorization
    n = 8600
    r = pk.ltlt_blk_piv(pk.SkewMatrixLower(skew_lower(n, 5)), b=256, fused="var1")
    out[f"L{n}"], out[f"t{n}"], out[f"p{n}"] = np.asarray(r.l.data), np.asarray(r.t.tau), np.asarray(r.p.pivots)
r = pk.ltlt_unb_twostep(pk.SkewMatrixLower(skew_lower(512, 0)), pivot=True)
out["Ltw"], out["ttw"], out["ptw"] = np.asarray(r.l.data), np.asarray(r.t.tau), np.asarray(r.p.pivots)
np.savez(sys.argv[1], **out)
print("PUSH_OK")
