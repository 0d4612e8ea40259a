"""GPU parity of the stand-alone kernels (kernels2/kernels3/core API) vs the oracle."""

import numpy as np
import pytest

import oracle
from conftest import lower

pytestmark = pytest.mark.gpu
RNG = np.random.default_rng(2024)


def k3():
    from paper_2411_09859_b200 import kernels3
    return kernels3


def k2():
    from paper_2411_09859_b200 import kernels2
    return kernels2


@pytest.mark.parametrize("n,k", [(1, 3), (2, 2), (37, 5), (300, 10), (513, 129), (1000, 64)])
@pytest.mark.parametrize("alpha,beta", [(1.0, 1.0), (-0.5, 2.0), (1.0, 0.0)])
def test_skew_rank2k(n, k, alpha, beta):
    a = RNG.standard_normal((n, k))
    w = oracle.form_w(a, RNG.standard_normal(max(k - 1, 0)))
    c = np.asfortranarray(RNG.standard_normal((n, n)))
    want = c.copy()
    keff = oracle.skew_rank2k(want, alpha, a, w) if beta == 1.0 else None
    if beta != 1.0:
        want = beta * c
        keff = oracle.skew_rank2k(want, alpha, a, w)
        want = np.where(np.tril(np.ones((n, n), bool), -1), want, c)
    got = c.copy()
    k3().skew_rank2k(got, alpha, a, w, beta)
    low = np.tril(np.ones((n, n), bool), -1)
    assert np.allclose(got[low], want[low], rtol=1e-12, atol=1e-12 * max(k, 1))
    assert np.array_equal(got[~low], c[~low])
    assert k3().last_keff == keff


def test_skew_rank2k_config2_microbench_shape():
    n, k = 4096, 128
    a = RNG.standard_normal((n, k))
    w = oracle.form_w(a, RNG.standard_normal(k - 1))
    c = np.asfortranarray(RNG.standard_normal((n, n)))
    want = c.copy()
    oracle.skew_rank2k(want, 1.0, a, w)
    got = c.copy()
    k3().skew_rank2k(got, 1.0, a, w, 1.0)
    assert k3().last_keff == 64
    low = np.tril(np.ones((n, n), bool), -1)
    assert np.max(np.abs(got[low] - want[low])) <= 1e-13 * k * np.max(np.abs(want[low]))


@pytest.mark.parametrize("n,k", [(5, 3), (33, 17), (1200, 40), (600, 600)])
def test_skew_rank2k_keep_list_edge_cases(n, k):
    """The one-launch prologue (flag bits per row block, grid barrier, ordered keep list) against
    kernels3.py:318-321: a column is kept only if it is nonzero in BOTH factors, wherever the
    nonzero sits (first row, last row, a row block of its own), with or without the skipping."""
    a = RNG.standard_normal((n, k))
    b = RNG.standard_normal((n, k))
    a[:, 0] = 0.0                      # zero in A only
    b[:, k - 1] = 0.0                  # zero in B only
    if k > 4:
        a[:, 2] = 0.0
        a[n - 1, 2] = 3.0              # a single nonzero, in the last row
        b[:, 3] = 0.0
        b[0, 3] = -2.0                 # a single nonzero, in the first row
        a[:, 4] = 0.0
        b[:, 4] = 0.0                  # zero in both
    for skip in (True, False):
        c = np.asfortranarray(RNG.standard_normal((n, n)))
        want = c.copy()
        keff = oracle.skew_rank2k(want, 0.75, a, b, skip_zero_columns=skip)
        got = c.copy()
        k3().skew_rank2k(got, 0.75, a, b, 1.0, skip_zero_columns=skip)
        low = np.tril(np.ones((n, n), bool), -1)
        assert k3().last_keff == keff
        assert np.allclose(got[low], want[low], rtol=1e-12, atol=1e-12 * k)
        assert np.array_equal(got[~low], c[~low])
    # nothing survives: C is only scaled
    z = np.zeros((n, k))
    c = np.asfortranarray(RNG.standard_normal((n, n)))
    got = c.copy()
    k3().skew_rank2k(got, 1.0, z, b, 2.0)
    assert k3().last_keff == 0
    low = np.tril(np.ones((n, n), bool), -1)
    assert np.array_equal(got[low], 2.0 * c[low]) and np.array_equal(got[~low], c[~low])


def test_skew_rank2k_alias_and_shape_errors():
    a = RNG.standard_normal((6, 6))
    with pytest.raises(ValueError):
        k3().skew_rank2k(a, 1.0, a, a.copy())
    with pytest.raises(ValueError):
        k3().skew_rank2k(np.zeros((5, 5)), 1.0, np.zeros((5, 2)), np.zeros((5, 3)))


@pytest.mark.parametrize("n,k", [(2, 1), (50, 4), (400, 129), (777, 256)])
def test_skew_tridiag_rankk(n, k):
    from paper_2411_09859_b200.core import SkewTridiagonal
    a = RNG.standard_normal((n, k))
    tau = RNG.standard_normal(k - 1)
    c = np.asfortranarray(RNG.standard_normal((n, n)))
    want = c.copy()
    oracle.skew_tridiag_rankk(want, -1.0, a, tau)
    got = c.copy()
    k3().skew_tridiag_rankk(got, -1.0, a, SkewTridiagonal(tau))
    low = np.tril(np.ones((n, n), bool), -1)
    assert np.allclose(got[low], want[low], rtol=1e-12, atol=1e-12 * k)
    assert np.array_equal(got[~low], c[~low])


@pytest.mark.parametrize("n,k", [(5, 2), (9, 7), (300, 128)])
def test_form_w_bit_exact(n, k):
    from paper_2411_09859_b200.core import SkewTridiagonal, form_s_splitting
    a = RNG.standard_normal((n, k))
    tau = RNG.standard_normal(k - 1)
    w = k3().form_w(a, form_s_splitting(SkewTridiagonal(tau)))
    assert np.array_equal(w, oracle.form_w(a, tau))


@pytest.mark.parametrize("n", [2, 3, 16, 64, 300])
def test_skew_rank2(n):
    a = np.asfortranarray(RNG.standard_normal((n, n)))
    x, y = RNG.standard_normal(n), RNG.standard_normal(n)
    want = 0.5 * lower(a) + 1.25 * lower(np.outer(x, y) - np.outer(y, x))
    got = a.copy()
    k2().skew_rank2(got, 1.25, x, y, 0.5)
    assert np.allclose(lower(got), want, rtol=1e-14, atol=1e-14)
    assert np.array_equal(np.triu(got), np.triu(a))
    two = np.zeros((2, 2), order="F")
    k2().skew_rank2(two, 1.0, np.array([1.0, 0.0]), np.array([0.0, 1.0]), 1.0)
    assert two[1, 0] == -1.0


def test_skew_tridiag_gemv():
    from paper_2411_09859_b200.core import SkewTridiagonal
    y = np.zeros(3)
    k2().skew_tridiag_gemv(y, 1.0, np.eye(3), SkewTridiagonal(np.array([2.0, 3.0])), np.ones(3), 0.0)
    assert y.tolist() == [-2.0, -1.0, 3.0]
    p, k = 40, 9
    a = RNG.standard_normal((p, k))
    tau, x = RNG.standard_normal(k - 1), RNG.standard_normal(k)
    y0 = RNG.standard_normal(p - 5)
    want = y0.copy()
    oracle.skew_tridiag_gemv(want, -1.0, a, tau, x, tail_from=5)
    got = y0.copy()
    k2().skew_tridiag_gemv(got, -1.0, a, SkewTridiagonal(tau), x, tail_from=5)
    assert np.allclose(got, want, rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("forward", [True, False])
def test_apply_row_pivots_bit_exact(forward):
    n, q = 60, 17
    piv = np.zeros(n, dtype=np.int64)
    for k in range(n):
        piv[k] = RNG.integers(0, n - k)
    block = np.asfortranarray(RNG.standard_normal((n, q)))
    want = block.copy()
    oracle.apply_row_pivots(want, piv, forward)
    got = block.copy()
    k2().apply_row_pivots(got, piv, forward)
    assert np.array_equal(got, want)


def test_apply_symmetric_pivot_bit_exact():
    from paper_2411_09859_b200.core import SkewMatrixLower, apply_symmetric_pivot
    n = 40
    x = np.asfortranarray(np.tril(RNG.standard_normal((n, n)), -1))
    for k, pi in [(0, 5), (3, 30), (10, 1), (38, 1), (7, 0)]:
        want = x.copy()
        oracle.sym_swap_lower(want, k, k + pi)
        sx = SkewMatrixLower(x.copy(order="F"))
        apply_symmetric_pivot(sx, k, pi)
        assert np.array_equal(sx.data, want)
    with pytest.raises(IndexError):
        apply_symmetric_pivot(SkewMatrixLower(x), 35, 10)


@pytest.mark.parametrize("i", range(9))
def test_skew_tridiag_gemm_vs_reference_fixture(golden, i):
    """skl_skew_tridiag_gemm (DMMA kernel, tile-table mode) vs the reference's
    kernels3.skew_tridiag_gemm on general and tril blocks (p < q, beta in
    {0, 2, -1}, alpha = 0, k up to 150); untouched entries bit-identical."""
    import sys
    from conftest import GOLDEN
    from paper_2411_09859_b200.core import SkewTridiagonal
    sys.path.insert(0, str(GOLDEN))
    from l3_cases import L3_CASES, l3_inputs
    g = golden("l3_small.npz")
    p, q, k, tril, alpha, beta = L3_CASES[i]
    a, b, tau, c = l3_inputs(i, p, q, k)
    want = g[f"c{i}_out"]
    got = c.copy(order="F")
    k3().skew_tridiag_gemm(got, alpha, a, SkewTridiagonal(tau), b, beta, tril=tril)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12 * max(k, 1))
    if tril:
        up = ~np.tril(np.ones((p, q), bool), -1)
        assert np.array_equal(got[up], c[up])


def test_skew_tridiag_gemm_device_tensors_and_alias():
    import torch
    from paper_2411_09859_b200 import device as dv
    from paper_2411_09859_b200.core import SkewTridiagonal
    p, q, k = 700, 300, 96
    a = RNG.standard_normal((p, k))
    b = RNG.standard_normal((k, q))
    tau = RNG.standard_normal(k - 1)
    c = np.asfortranarray(RNG.standard_normal((p, q)))
    want = c.copy()
    oracle.skew_tridiag_gemm(want, -1.0, a, tau, b, tril=True)
    cd = dv.to_device_colmajor(c)
    k3().skew_tridiag_gemm(cd, -1.0, dv.to_device_colmajor(a), SkewTridiagonal(torch.as_tensor(tau, device="cuda")),
                           dv.to_device_colmajor(b), 1.0, tril=True)
    assert np.allclose(dv.to_host_colmajor(cd), want, rtol=1e-12, atol=1e-12 * k)
    x = np.asfortranarray(RNG.standard_normal((8, 8)))
    with pytest.raises(ValueError):
        k3().skew_tridiag_gemm(x, 1.0, x, SkewTridiagonal(np.ones(7)), np.ones((8, 8)))
    with pytest.raises(ValueError):
        k3().skew_tridiag_gemm(np.zeros((5, 4)), 1.0, np.zeros((5, 3)), SkewTridiagonal(np.ones(2)),
                               np.zeros((3, 5)))


# ---- gen_rank2 / trapezoid_rank2 (kernels2.py:134-163, 274-312) -----------------

def test_gen_rank2_scalar_and_dense():
    from paper_2411_09859_b200 import instrument as ins
    from paper_2411_09859_b200.kernels2 import gen_rank2
    a = np.array([[2.0]])
    gen_rank2(a, 0.5, np.array([3.0]), np.array([4.0]), np.array([5.0]), np.array([6.0]), 1.0)
    assert a[0, 0] == 2.0 + 0.5 * (12.0 + 30.0)
    rng = np.random.default_rng(3)
    for p, q, beta in ((8, 4, 0.25), (1000, 37, 1.0), (3, 1, -1.0)):
        a = np.asfortranarray(rng.standard_normal((p, q)))
        x, y, u, v = rng.standard_normal(p), rng.standard_normal(p), rng.standard_normal(q), rng.standard_normal(q)
        want = beta * a + 2.0 * (np.outer(x, u) + np.outer(y, v))
        tr, fc = ins.CallTrace(), ins.FlopCounter()
        with ins.tracing(tr), ins.counting(fc):
            gen_rank2(a, 2.0, x, u, y, v, beta)
        assert np.allclose(a, want, rtol=1e-14, atol=1e-14)
        assert tr.calls == [("gen_rank2", "trailing")] and fc.level2 == 4 * p * q
    a = rng.standard_normal((4, 3))
    before = a.copy()
    gen_rank2(a, 0.0, np.ones(4), np.ones(3), np.ones(4), np.ones(3), 1.0)
    assert np.array_equal(a, before)
    with pytest.raises(ValueError):
        gen_rank2(a, 1.0, np.ones(3), np.ones(3), np.ones(4), np.ones(3), 1.0)


def test_trapezoid_rank2_matches_dense():
    from paper_2411_09859_b200.kernels2 import trapezoid_rank2
    rng = np.random.default_rng(4)
    for n, start, climit in ((10, 3, 7), (300, 20, 140), (50, 5, 50)):
        buf = np.asfortranarray(rng.standard_normal((n, n)))
        x, y = rng.standard_normal(n - start), rng.standard_normal(n - start)
        want = buf.copy()
        full = np.zeros((n, n))
        full[start:, start:] = np.outer(x, y) - np.outer(y, x)
        il, jl = np.tril_indices(n, -1)
        keep = (jl >= start) & (jl < climit)
        want[il[keep], jl[keep]] += full[il[keep], jl[keep]]
        trapezoid_rank2(buf, start, climit, 1.0, x, y)
        assert np.allclose(np.tril(buf, -1), np.tril(want, -1), rtol=1e-13, atol=1e-13)
        assert np.array_equal(np.triu(buf), np.triu(want))
    buf = np.asfortranarray(rng.standard_normal((4, 4)))
    before = buf.copy()
    trapezoid_rank2(buf, 3, 3, 1.0, np.ones(1), np.ones(1))
    assert np.array_equal(buf, before)


def test_kernel_wrappers_record_reference_calls():
    from paper_2411_09859_b200 import instrument as ins
    from paper_2411_09859_b200.core import SkewTridiagonal
    from paper_2411_09859_b200.kernels2 import skew_rank2, skew_tridiag_gemv
    from paper_2411_09859_b200.kernels3 import skew_tridiag_rankk
    rng = np.random.default_rng(5)
    n, k = 40, 6
    c = np.asfortranarray(rng.standard_normal((n, n)))
    a = np.asfortranarray(rng.standard_normal((n, k)))
    t = SkewTridiagonal(rng.standard_normal(k - 1))
    tr, fc = ins.CallTrace(), ins.FlopCounter()
    with ins.tracing(tr), ins.counting(fc), ins.scope("panel"):
        skew_rank2(c, 1.0, rng.standard_normal(n), rng.standard_normal(n))
        skew_tridiag_gemv(np.zeros(n - 5), -1.0, a, t, rng.standard_normal(k), 1.0, tail_from=5)
        skew_tridiag_rankk(c, -1.0, a, t, 1.0)
    assert tr.calls == [("skew_rank2", "panel"), ("skew_tridiag_gemv", "panel"), ("skew_tridiag_rankk", "panel")]
    assert fc.level2 == 2 * n * (n - 1) + 2 * (n - 5) * k + 4 * k
    assert fc.level3 == 2 * k * (n * (n - 1) // 2) + 4 * k * n
