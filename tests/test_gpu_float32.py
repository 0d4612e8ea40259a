"""float32 input to the single-matrix drivers (SURVEY 8b "Dtypes": the reference
runs float32 end to end and L / tau keep the input dtype).  The GPU factors
float32 input in float64 and rounds L and tau back to float32, so the checker
is the oracle's own float32 run (the reference's arithmetic): identical pivots
on these inputs (a flip could only come from a float32-rounding near-tie) and
L / tau within the BASELINE float32 tolerance, 1e-3 relative."""
import math

import numpy as np
import pytest

import oracle
from paper_2411_09859_b200.inputs import skew_lower

pytestmark = pytest.mark.gpu


def pk():
    import paper_2411_09859_b200 as m
    return m


def close32(r, o):
    assert r.l.data.dtype == np.float32 and np.asarray(r.t.tau).dtype == np.float32
    assert np.array_equal(np.asarray(r.p.pivots), o.pivots)
    lo = np.tril(o.work, -1)
    assert np.max(np.abs(np.tril(np.asarray(r.l.data), -1) - lo)) <= 1e-3 * max(1.0, np.max(np.abs(lo)))
    assert np.max(np.abs(np.asarray(r.t.tau) - o.tau)) <= 1e-3 * max(1.0, np.max(np.abs(o.tau)))


@pytest.mark.parametrize("n,b,fused", [(64, 16, "var1"), (300, 64, "var2a"), (1000, 128, "var1")])
def test_blk_piv_float32(n, b, fused):
    x = skew_lower(n, n).astype(np.float32)
    close32(pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=b, fused=fused), oracle.ltlt_blk_piv(x, b=b, fused=fused))


def test_unb_twostep_and_ll_float32():
    x = skew_lower(200, 5).astype(np.float32)
    close32(pk().ltlt_unb_twostep(pk().SkewMatrixLower(x), pivot=True), oracle.ltlt_unb_twostep(x, pivot=True))
    close32(pk().ltlt_unb_ll(pk().SkewMatrixLower(x), pivot=True), oracle.ltlt_unb_ll(x, pivot=True))


def test_device_float32_input_stays_float32():
    import torch
    from paper_2411_09859_b200 import device as dv
    x = skew_lower(150, 9).astype(np.float32)
    xd = dv.to_device_colmajor(x)
    assert xd.dtype == torch.float32
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower(xd), b=32)
    assert r.l.data.dtype == torch.float32 and r.t.tau.dtype == torch.float32 and r.l.data.is_cuda
    o = oracle.ltlt_blk_piv(x, b=32)
    assert np.array_equal(np.asarray(r.p.pivots), o.pivots)
    assert np.max(np.abs(r.t.tau.cpu().numpy() - o.tau)) <= 1e-3 * max(1.0, np.max(np.abs(o.tau)))


def test_pfaffian_float32_overflows_like_the_reference():
    # n = 256 N(0,1): |Pf| ~ e^{400} overflows float32 (and the reference's product) but not slog
    x = skew_lower(256, 0).astype(np.float32)
    with np.errstate(over="ignore"):
        pf = pk().pfaffian(pk().SkewMatrixLower(x))
    o = oracle.ltlt_blk_piv(x, b=256)
    s, lg = oracle.pfaffian_slog(o.tau, o.pivots, 256)
    ref = np.float32(1.0) * (-1 if np.count_nonzero(o.pivots) % 2 else 1)
    with np.errstate(over="ignore"):
        for i in range(0, 255, 2):
            ref = ref * (-o.tau[i])
    assert math.isinf(float(pf)) and math.isinf(float(ref)) and np.sign(pf) == np.sign(ref) == s
    from paper_2411_09859_b200.apps import pfaffian_slog
    s2, lg2 = pfaffian_slog(pk().SkewMatrixLower(x))
    assert s2 == s and abs(lg2 - lg) <= 1e-3 * abs(lg)


def test_solve_float32_input():
    x = skew_lower(120, 3).astype(np.float32)
    rhs = np.arange(120, dtype=np.float64)
    y = pk().solve(pk().SkewMatrixLower(x), rhs)
    dense = oracle.skew_dense(x.astype(np.float64))
    assert np.linalg.norm(dense @ y - rhs) <= 1e-8 * np.linalg.norm(rhs) * np.linalg.cond(dense)
