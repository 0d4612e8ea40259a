"""Subprocess body of test_gpu_multi.py: the driver's panel plan is read from the
environment once per process (SKL_FORCE_MULTI / SKL_MULTI_Q),
so every exchange variant runs in its own interpreter."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402  (checker only)
import paper_2411_09859_b200 as pk  # noqa: E402
from paper_2411_09859_b200.inputs import skew_lower  # noqa: E402


def check(r, o, n, pivoted):
    lg, lo = np.tril(np.asarray(r.l.data), -1), np.tril(o.work, -1)
    scale = max(1.0, float(np.max(np.abs(lo), initial=0.0)))
    growth = 1.0 if pivoted else scale
    assert np.array_equal(np.asarray(r.p.pivots), o.pivots), "pivots"
    assert np.max(np.abs(lg - lo), initial=0.0) <= 1e-10 * n * growth * scale, "L"
    tscale = max(1.0, float(np.max(np.abs(o.tau), initial=0.0)))
    assert np.max(np.abs(np.asarray(r.t.tau) - o.tau), initial=0.0) <= 1e-10 * n * growth * tscale, "tau"


def main():
    for n, b in [(300, 64), (1000, 128), (1537, 96)]:
        x = skew_lower(n, n + 7)
        for fused in ("var1", "var2a", "var2b"):
            r = pk.ltlt_blk_piv(pk.SkewMatrixLower(x), b=b, fused=fused)
            check(r, oracle.ltlt_blk_piv(x, b=b, fused=fused), n, True)
    x = skew_lower(301, 11)
    for driver in ("var1", "var2a", "twostep"):
        r = getattr(pk, f"ltlt_blk_{driver}")(pk.SkewMatrixLower(x), b=64)
        check(r, oracle.ltlt_blk(x, 64, driver, "ll"), 301, False)
    print("MULTI_OK")


if __name__ == "__main__":
    main()
