"""GPU parity of the fused Wimmer two-step kernel (config 1) and the Pfaffian."""

import numpy as np
import pytest

import oracle
from conftest import EPS, worked_example
from paper_2411_09859_b200.inputs import skew_lower

pytestmark = pytest.mark.gpu


def unb():
    from paper_2411_09859_b200 import unblocked
    return unblocked


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 17, 64, 129, 300, 700])
@pytest.mark.parametrize("pivot", [True, False])
def test_twostep_vs_oracle(n, pivot):
    x = skew_lower(n, n)
    o = oracle.ltlt_unb_twostep(x, pivot=pivot)
    r = unb().ltlt_unb_twostep(x, pivot=pivot)
    if pivot:
        assert np.array_equal(r.p.pivots, o.pivots)
    else:
        assert len(r.p.pivots) == 0
    scale = max(np.max(np.abs(o.tau)), 1.0) if n > 1 else 1.0
    tol = 1e-10 * n if pivot else 1e-6  # unpivoted growth is unbounded; compare loosely
    assert np.max(np.abs(r.t.tau - o.tau), initial=0.0) <= tol * scale
    assert np.array_equal(np.triu(r.l.data), np.triu(x))
    from paper_2411_09859_b200 import FlopCounter
    assert r.flops == FlopCounter(**o.flops)


def test_config1_golden(golden):
    g = golden("cfg1_n512.npz")
    x = skew_lower(512, 0)
    r = unb().ltlt_unb_twostep(x, pivot=True)
    assert np.array_equal(r.p.pivots, g["piv"])
    assert np.allclose(r.t.tau, g["tau"], rtol=1e-10 * 512, atol=1e-10 * 512)
    il = np.tril_indices(512, -1)
    assert np.max(np.abs(r.l.data[il] - g["l_lower"])) <= 1e-10 * 512
    assert oracle.residual(x, r.l.data, r.t.tau, r.p.pivots) <= 10 * EPS * 512
    assert r.flops.level2 == int(g["flops"][0]) and r.flops.pivot == int(g["flops"][3])


def test_worked_example_and_zero_pivot():
    from paper_2411_09859_b200 import ZeroPivot
    r = unb().ltlt_unb_twostep(worked_example())
    assert r.t.tau.tolist() == [2.0, 4.0, 10.5]
    ld = r.l.dense()
    assert [ld[2, 1], ld[3, 1], ld[3, 2]] == [0.5, 1.5, 0.25]
    x = np.zeros((3, 3), order="F")
    x[2, 0] = 1.0
    with pytest.raises(ZeroPivot) as e:
        unb().ltlt_unb_twostep(x)
    assert e.value.column == 0
    z = np.zeros((3, 3), order="F")
    z[2, 1] = 4.0
    assert unb().ltlt_unb_twostep(z).t.tau.tolist() == [0.0, 4.0]


def test_pfaffian_api():
    from paper_2411_09859_b200 import apps
    assert np.isclose(apps.pfaffian(worked_example()), 21.0)
    x = np.zeros((2, 2), order="F")
    x[1, 0] = 3.0
    assert apps.pfaffian(x) == -3.0
    assert apps.pfaffian(skew_lower(5, 1)) == 0.0
    assert apps.pfaffian(np.zeros((0, 0))) == 1.0
    rng = np.random.default_rng(4)
    for m in (4, 6, 8):
        ints = rng.integers(-5, 6, size=(m, m)).astype(float)
        xm = np.asfortranarray(np.tril(ints - ints.T, -1))
        assert np.isclose(apps.pfaffian(xm), float(oracle.pfaffian_bruteforce(xm)), rtol=1e-9, atol=1e-9)
    s, lg = apps.pfaffian_slog(skew_lower(512, 0))  # reference pfaffian() overflows here
    o = oracle.ltlt_blk_piv(skew_lower(512, 0), b=256)
    so, lo = oracle.pfaffian_slog(o.tau, o.pivots, 512)
    assert s == so and abs(lg - lo) <= 1e-10 * abs(lo)
