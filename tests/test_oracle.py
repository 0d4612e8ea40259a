"""CPU: the oracle restatement pinned to the reference's golden vectors and
known-answer tests.  (The oracle is test infrastructure only.)"""

from fractions import Fraction

import numpy as np
import pytest

import oracle
from conftest import EPS, GOLDEN, lower, worked_example
from paper_2411_09859_b200.inputs import skew_lower


# ---- known answers from the reference's own tests --------------------------

def test_worked_example_unpivoted():
    # test_unblocked.py:22-34: tau = (2, 4, 10.5); L[2,1]=.5, L[3,1]=1.5, L[3,2]=.25
    r = oracle.ltlt_unb_twostep(worked_example())
    assert r.tau.tolist() == [2.0, 4.0, 10.5]
    ld = oracle.l_dense(r.work)
    assert [ld[2, 1], ld[3, 1], ld[3, 2]] == [0.5, 1.5, 0.25]


def test_worked_example_pivoted_first_pivot():
    # test_blocked.py:122-125: pi_1 = 2 (|3| is the largest of (2, 1, 3))
    r = oracle.ltlt_blk_piv(worked_example(), b=2)
    assert r.pivots[0] == 0 and r.pivots[1] == 2


def test_pfaffian_conventions():
    # test_apps.py:17-28: Pf([[0,-3],[3,0]]) = -3 with x10 = 3; worked example 21
    x = np.zeros((2, 2), order="F")
    x[1, 0] = 3.0
    assert oracle.pfaffian(x) == -3.0
    assert np.isclose(oracle.pfaffian(worked_example()), 21.0)
    assert oracle.pfaffian(skew_lower(3, 1)) == 0.0


def test_m2_and_zero_column():
    # test_unblocked.py:43-48 and 116-122
    x = np.zeros((2, 2), order="F")
    x[1, 0] = -3.5
    assert oracle.ltlt_blk_piv(x, b=1).tau.tolist() == [-3.5]
    z = np.zeros((3, 3), order="F")
    z[2, 1] = 4.0
    assert oracle.ltlt_unb_twostep(z).tau.tolist() == [0.0, 4.0]


def test_zero_pivot_unpivoted():
    # test_unblocked.py:108-114
    x = np.zeros((3, 3), order="F")
    x[2, 0] = 1.0
    with pytest.raises(ZeroDivisionError):
        oracle.ltlt_unb_twostep(x)


def test_s_splitting_and_w_pattern():
    # test_core.py:70-75 and test_kernels3.py:195-200
    assert set(oracle.form_s_entries(np.array([2.0, 3.0, 7.0]))) == {(0, 1, -2.0), (2, 1, 3.0), (2, 3, -7.0)}
    a = np.random.default_rng(0).standard_normal((5, 2))
    w = oracle.form_w(a, np.array([2.5]))
    assert not w[:, 0].any() and np.allclose(w[:, 1], -2.5 * a[:, 0])


def test_level2_kats():
    # test_kernels2.py:58-61 and 137-141
    a = np.zeros((2, 2), order="F")
    oracle.skew_rank2(a, 1.0, np.array([1.0, 0.0]), np.array([0.0, 1.0]))
    assert a[1, 0] == -1.0
    y = np.zeros(3)
    oracle.skew_tridiag_gemv(y, 1.0, np.eye(3), np.array([2.0, 3.0]), np.ones(3))
    assert y.tolist() == [-2.0, -1.0, 3.0]


# ---- exact rational cross-checks ------------------------------------------

@pytest.mark.parametrize("seed", range(6))
def test_float_oracle_matches_exact_elimination(seed):
    rng = np.random.default_rng(seed)
    m = 7
    ints = rng.integers(-9, 10, size=(m, m)).astype(float)
    x = np.tril(ints - ints.T, -1)
    lm, tau, piv = oracle.gauss_elim_exact(x, pivot=True)
    r = oracle.ltlt_unb_ll(np.asfortranarray(x), pivot=True)
    assert np.array_equal(r.pivots, piv)
    assert np.allclose(r.tau, np.array([float(t) for t in tau]), rtol=1e-12, atol=1e-12)
    ld = oracle.l_dense(r.work)
    assert np.allclose(ld, np.array([[float(v) for v in row] for row in lm]), atol=1e-12)


def test_pfaffian_bruteforce():
    x = worked_example()
    assert oracle.pfaffian_bruteforce(x) == Fraction(21)
    rng = np.random.default_rng(3)
    for m in (2, 4, 6, 8):
        ints = rng.integers(-5, 6, size=(m, m)).astype(float)
        xm = np.asfortranarray(np.tril(ints - ints.T, -1))
        assert np.isclose(oracle.pfaffian(xm), float(oracle.pfaffian_bruteforce(xm)), rtol=1e-9, atol=1e-9)


# ---- golden vectors produced by the unmodified reference ---------------------

def test_kat_fixture(golden):
    g = golden("kat.npz")
    r = oracle.ltlt_unb_twostep(g["worked_x"])
    assert np.array_equal(r.tau, g["worked_tau"])
    rp = oracle.ltlt_blk_piv(g["worked_x"], b=2)
    assert np.array_equal(rp.pivots, g["worked_piv_piv"])
    assert np.array_equal(rp.tau, g["worked_piv_tau"])
    assert np.array_equal(rp.work, g["worked_piv_L"])


def test_cfg1_fixture(golden):
    g = golden("cfg1_n512.npz")
    r = oracle.ltlt_unb_twostep(skew_lower(512, 0), pivot=True)
    assert np.array_equal(r.pivots, g["piv"])
    assert np.array_equal(r.tau, g["tau"])
    il = np.tril_indices(512, -1)
    assert np.array_equal(r.work[il], g["l_lower"])
    assert [r.flops[k] for k in ("level2", "level3", "panel", "pivot")] == g["flops"].tolist()


@pytest.mark.parametrize("n,b", [(64, 16), (300, 32), (513, 64), (1000, 128)])
@pytest.mark.parametrize("fused", ["var1", "var2a", "var2b"])
def test_blk_small_fixture(golden, n, b, fused):
    g = golden("blk_small.npz")
    key = f"n{n}_b{b}_{fused}_"
    r = oracle.ltlt_blk_piv(skew_lower(n, n), b=b, fused=fused)
    assert np.array_equal(r.pivots, g[key + "piv"])
    assert np.array_equal(r.tau, g[key + "tau"])
    rng_r = np.random.Generator(np.random.Philox(12345)).standard_normal(n)
    S = np.tril(r.work[:, :n - 1], -2)
    lr = rng_r + S @ rng_r[1:]
    assert np.allclose(lr, g[key + "lr"], rtol=1e-13, atol=1e-13)
    assert [r.flops[k] for k in ("level2", "level3", "panel", "pivot")] == g[key + "flops"].tolist()


def test_cfg2_fixture(golden):
    g = golden("cfg2_n4096_b128.npz")
    r = oracle.ltlt_blk_piv(skew_lower(4096, 0), b=128)
    assert np.array_equal(r.pivots, g["piv"])
    assert np.array_equal(g["piv"], g["piv_var2a"]) and np.array_equal(g["piv"], g["piv_var2b"])
    assert np.allclose(r.tau, g["tau"], rtol=1e-12, atol=1e-12)
    sign, lg = oracle.pfaffian_slog(r.tau, r.pivots, 4096)
    assert sign == g["sign"] and abs(lg - g["logpf"]) < 1e-9


@pytest.mark.parametrize("tag,dtype", [("f64", np.float64), ("f32", np.float32)])
def test_cfg4_fixture_prefix(golden, tag, dtype):
    g = golden(f"cfg4_batch_{tag}.npz")
    for i in range(6):
        x = skew_lower(256, i).astype(dtype)
        r = oracle.ltlt_blk_piv(x, b=256)
        assert np.array_equal(r.pivots, g["piv"][i])
        s, lg = oracle.pfaffian_slog(r.tau, r.pivots, 256)
        assert s == g["sign"][i] and abs(lg - g["logpf"][i]) < (1e-9 if tag == "f64" else 1e-3)


def test_residual_bound_small():
    for n in (10, 100, 300):
        x = skew_lower(n, 7)
        r = oracle.ltlt_blk_piv(x, b=32)
        assert oracle.residual(x, r.work, r.tau, r.pivots) <= 10 * EPS * n


# ---- unpivoted drivers pinned to the reference ----------

UNPIV_N = [(64, 16), (150, 32), (301, 64)]


def unpiv_cases():
    """(key suffix, oracle call) for every driver the unpiv fixture holds."""
    out = []
    for drv in ("var1", "var2a", "var2b", "twostep", "left"):
        for pv in ("ll", "rl", "twostep"):
            out.append((f"{drv}_{pv}", lambda x, b, fc, drv=drv, pv=pv: oracle.ltlt_blk(x, b, drv, pv)))
    out += [
        ("unb_rl", lambda x, b, fc: oracle.ltlt_unb_rl(x)),
        ("unb_rl_piv", lambda x, b, fc: oracle.ltlt_unb_rl(x, True)),
        ("unb_ll", lambda x, b, fc: oracle.ltlt_unb_ll(x)),
        ("unb_ll_first", lambda x, b, fc: oracle.ltlt_unb_ll(x, first_column=fc)),
        ("panel40_ll", lambda x, b, fc: oracle.ltlt_unb_panel(x, 40, "ll")),
        ("panel40_rl", lambda x, b, fc: oracle.ltlt_unb_panel(x, 40, "rl")),
        ("panel40_twostep", lambda x, b, fc: oracle.ltlt_unb_panel(x, 40, "twostep")),
        ("panel40_piv", lambda x, b, fc: oracle.ltlt_unb_panel(x, 40, "ll", True)),
        ("panel40_first", lambda x, b, fc: oracle.ltlt_unb_panel(x, 40, "ll", False, fc)),
    ]
    return out


def l_checksum(work, n, seed=12345):
    r = np.random.Generator(np.random.Philox(seed)).standard_normal(n)
    S = np.tril(work[:, :n - 1], -2)
    return r + S @ r[1:]


@pytest.mark.parametrize("n,b", UNPIV_N)
@pytest.mark.parametrize("case", unpiv_cases(), ids=lambda c: c[0])
def test_unpivoted_drivers_fixture(golden, n, b, case):
    """The oracle's unpivoted blocked / unblocked / panel drivers reproduce the
    unmodified reference bit for bit (tau, pivots, flop tallies, L)."""
    g = golden("unpiv_small.npz")
    name, call = case
    key = f"n{n}_{name}_"
    r = call(skew_lower(n, n), b, g[f"n{n}_first_column"])
    assert np.array_equal(r.tau, g[key + "tau"])
    assert np.array_equal(r.pivots, g[key + "piv"])
    assert [r.flops[k] for k in ("level2", "level3", "panel", "pivot")] == g[key + "flops"].tolist()
    assert np.array_equal(l_checksum(r.work, n), g[key + "lr"])
    if key + "first" in g:
        assert np.array_equal(r.first_column, g[key + "first"])
    if key + "l" in g:
        assert np.array_equal(r.work[np.tril_indices(n, -1)], g[key + "l"])


def test_unpivoted_zero_pivot_oracle():
    """Unpivoted breakdown: exact zero pivot with a nonzero tail (unblocked.py:83-85)."""
    x = np.zeros((4, 4), order="F")
    x[2, 0], x[3, 1] = 1.0, 2.0          # X[1, 0] == 0, X[2, 0] != 0
    with pytest.raises(ZeroDivisionError):
        oracle.ltlt_blk(x, 2, "var2a")
    z = np.zeros((3, 3), order="F")
    z[2, 1] = 4.0                        # all-zero first column: tau 0, continue
    r = oracle.ltlt_blk(z, 2, "var1")
    assert r.tau.tolist() == [0.0, 4.0]


# ---- solve pinned to the reference ------------------------

@pytest.mark.parametrize("n", [2, 8, 64, 300])
def test_solve_fixture(golden, n):
    g = golden("solve_small.npz")
    x = skew_lower(n, n)
    assert np.array_equal(oracle.solve(x, g[f"n{n}_b1"]), g[f"n{n}_y1"])
    assert np.array_equal(oracle.solve(x, g[f"n{n}_b3"]), g[f"n{n}_y3"])


@pytest.mark.parametrize("n", [3, 7])
def test_solve_singular_fixture(golden, n):
    g = golden("solve_small.npz")
    with pytest.raises(ZeroDivisionError, match=f"row {int(g[f'odd{n}_row'])}$"):
        oracle.solve(skew_lower(n, n), np.ones(n))


@pytest.mark.parametrize("i", range(9))
def test_skew_tridiag_gemm_fixture(golden, i):
    """oracle.skew_tridiag_gemm (beta = 1 restatement) vs the reference's
    kernels3.skew_tridiag_gemm outputs (l3_small.npz)."""
    import sys
    sys.path.insert(0, str(GOLDEN))
    from l3_cases import L3_CASES, l3_inputs
    g = golden("l3_small.npz")
    p, q, k, tril, alpha, beta = L3_CASES[i]
    a, b, tau, c = l3_inputs(i, p, q, k)
    assert np.array_equal(g[f"c{i}_meta"][:3], [p, q, k])
    want = g[f"c{i}_out"]
    got = c.copy(order="F")
    if beta != 1.0:   # the restatement has beta = 1; apply beta on the written part first
        mask = np.tril(np.ones((p, q), bool), -1) if tril else np.ones((p, q), bool)
        got[mask] *= beta
    oracle.skew_tridiag_gemm(got, alpha, a, tau, b, tril=tril)
    assert np.allclose(got, want, rtol=1e-13, atol=1e-13 * max(k, 1))
    if tril:   # nothing on or above the diagonal moves
        up = ~np.tril(np.ones((p, q), bool), -1)
        assert np.array_equal(want[up], c[up])
