"""Per-kernel-class device time of one config-5 factorization (n=49152, nb=512) on one GPU,
plus the panel plan (single- vs multi-cluster steps): the inputs of the multi-GPU timeline
model in DESIGN.md §7.  Uses the BASELINE matrix (host Philox rows, bit-identical to the golden)."""
import ctypes, json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import _capi
from paper_2411_09859_b200.blocked import gpu_panel_plan
from paper_2411_09859_b200.inputs import normal_scaled_rows, skew_device_from_rows
n, nb = 49152, 512
lib = _capi.load()
X = skew_device_from_rows(normal_scaled_rows(n, 0), torch)
pk.ltlt_blk_piv_device(X, nb, "var1")
torch.cuda.synchronize()
lib.skl_timing_enable(1)
pk.ltlt_blk_piv_device(X, nb, "var1")
torch.cuda.synchronize()
ms = (ctypes.c_double * 4)(); cnt = (ctypes.c_int * 4)()
lib.skl_timing_read(ms, cnt); lib.skl_timing_enable(0)
plan = gpu_panel_plan(n, nb, "var1")
multi = [p for p in plan if p["ctas"] > p["cluster_size"]]
out = {"panel_ms": ms[0], "pack_ms": ms[1], "gemm_ms": ms[2], "finalize_ms": ms[3], "launches": list(cnt),
       "panels": len(plan), "multi_cluster_panels": len(multi),
       "multi_cluster_steps": sum(p["nelim"] for p in multi), "steps": sum(p["nelim"] for p in plan),
       "first_panel": plan[0], "last_multi": multi[-1] if multi else None}
print(json.dumps(out))
