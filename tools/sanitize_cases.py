"""Small-n workload for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family of the library once, checked against the oracle so a sanitizer run also
shows the results stay correct.  The panel variant is chosen by the environment
(SKL_PANEL_V2=0: panel_cluster_kernel; SKL_FORCE_MULTI=1: multi-cluster exchange)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import oracle
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import apps, kernels3
from paper_2411_09859_b200.inputs import skew_lower
from paper_2411_09859_b200.unblocked import ltlt_unb_twostep

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
x = skew_lower(n, 5)
for fused in ("var1", "var2a"):
    r = pk.ltlt_blk_piv(pk.SkewMatrixLower(x), b=64, fused=fused)
    assert np.array_equal(r.p.pivots, oracle.ltlt_blk_piv(x, b=64, fused=fused).pivots), fused
xs = skew_lower(96, 6)
assert np.array_equal(ltlt_unb_twostep(xs, pivot=True).p.pivots, oracle.ltlt_unb_twostep(xs, pivot=True).pivots)
batch = np.stack([skew_lower(64, i) for i in range(4)])
for dt in (np.float64, np.float32):
    apps.pfaffian_batched(batch.astype(dt))
y = pk.solve(pk.SkewMatrixLower(x), np.linspace(-1, 1, n))
assert np.allclose(y, oracle.solve(x, np.linspace(-1, 1, n)), rtol=1e-8, atol=1e-10)
a = np.asfortranarray(np.random.default_rng(0).standard_normal((n, 16)))
c = np.asfortranarray(np.random.default_rng(1).standard_normal((n, n)))
kernels3.skew_rank2k(c, 1.0, a, np.asfortranarray(a[:, ::-1]), 1.0)
print("SANITIZE_CASES_OK", n)
