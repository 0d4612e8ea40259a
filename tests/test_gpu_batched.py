"""GPU parity of the batched factorization + Pfaffian (config 4)."""

import numpy as np
import pytest

import oracle
from paper_2411_09859_b200.inputs import skew_lower

pytestmark = pytest.mark.gpu


def apps():
    from paper_2411_09859_b200 import apps as a
    return a


@pytest.mark.parametrize("n", [2, 3, 4, 7, 16, 33, 100, 256])
def test_batched_f64_vs_oracle(n):
    xs = np.stack([skew_lower(n, 100 + i) for i in range(6)])
    L, tau, piv, sign, logabs = apps().ltlt_batched_piv(xs)
    for i in range(6):
        o = oracle.ltlt_blk_piv(xs[i], b=max(n, 1))
        assert np.array_equal(piv[i], o.pivots)
        assert np.allclose(tau[i], o.tau, rtol=1e-10 * n, atol=1e-10 * n)
        assert np.max(np.abs(np.tril(L[i], -1) - np.tril(o.work, -1))) <= 1e-10 * n
        assert np.array_equal(np.triu(L[i]), np.triu(xs[i]))
        s, lg = oracle.pfaffian_slog(o.tau, o.pivots, n)
        assert sign[i] == s
        if n % 2 == 0:
            assert abs(logabs[i] - lg) <= 1e-10 * max(abs(lg), 1.0)


def test_batched_known_answers():
    x = np.zeros((4, 4))
    x[1, 0], x[2, 0], x[3, 0], x[2, 1], x[3, 1], x[3, 2] = 2, 1, 3, 4, 1, 5
    y = np.zeros((4, 4))
    y[1, 0] = 3.0  # singular 4x4: Pf = 0
    sign, logabs = apps().pfaffian_batched(np.stack([x, y]))
    assert sign[0] * np.exp(logabs[0]) == pytest.approx(21.0)
    assert sign[1] == 0.0
    z = np.zeros((1, 2, 2))
    z[0, 1, 0] = 3.0  # test_apps.py:17-20: Pf = -3
    s2, l2 = apps().pfaffian_batched(z)
    assert s2[0] * np.exp(l2[0]) == pytest.approx(-3.0)


def test_config4_f64_golden(golden):
    g = golden("cfg4_batch_f64.npz")
    xs = np.stack([skew_lower(256, i) for i in range(8192)])
    L, tau, piv, sign, logabs = apps().ltlt_batched_piv(xs)
    assert np.array_equal(piv[:128], g["piv"])
    assert np.allclose(tau[:128], g["tau"], rtol=1e-10 * 256, atol=1e-10 * 256)
    assert np.array_equal(sign, g["sign"])
    assert np.max(np.abs(logabs - g["logpf"]) / np.abs(g["logpf"])) <= 1e-10


def test_config4_f32_golden(golden):
    """fp32 (config 4) against the reference's own fp32 run (the pfaffian path,
    apps.py:12-30 -> ltlt_blk_piv(b=256) in float32): bit-exact pivot sequences
    for all 128 fixture matrices, identical Pfaffian signs for all 8192, and
    log|Pf| within the north star's fp32 tolerance (1e-3 relative).  On a pivot
    flip the message names the matrix, the step and the top-2 margin of that
    step (measured in fp64 on the same fp32 matrix) so the flip can be judged."""
    g = golden("cfg4_batch_f32.npz")
    xs = np.stack([skew_lower(256, i).astype(np.float32) for i in range(8192)])
    L, tau, piv, sign, logabs = apps().ltlt_batched_piv(xs)
    flips = [i for i in range(128) if not np.array_equal(piv[i], g["piv"][i])]
    if flips:
        i = flips[0]
        k = int(np.flatnonzero(piv[i] != g["piv"][i])[0])
        marg = oracle.pivot_margins(xs[i].astype(np.float64), b=256)
        pytest.fail(f"fp32 pivots differ in {len(flips)}/128 matrices; first: matrix {i} step {k} "
                    f"(gpu {piv[i][k]} vs reference {g['piv'][i][k]}), fp64 top-2 margin at step {k - 1}: "
                    f"{marg[k - 1]:.3e}")
    assert np.array_equal(sign, g["sign"])
    rel = np.abs(logabs - g["logpf"]) / np.abs(g["logpf"])
    assert np.median(rel) <= 1e-5 and np.max(rel) <= 1e-3
    assert np.allclose(tau[:128], g["tau"], rtol=1e-3, atol=1e-3 * np.abs(g["tau"]).max())


@pytest.mark.parametrize("n", [257, 300, 512])
def test_batched_two_rows_per_thread(n):
    """n > 256: every thread owns two physical rows (RPT = 2 instantiation)."""
    xs = np.stack([skew_lower(n, 300 + i) for i in range(3)])
    L, tau, piv, sign, logabs = apps().ltlt_batched_piv(xs)
    for i in range(3):
        o = oracle.ltlt_blk_piv(xs[i], b=n)
        assert np.array_equal(piv[i], o.pivots)
        assert np.allclose(tau[i], o.tau, rtol=1e-10 * n, atol=1e-10 * n)
        assert np.max(np.abs(np.tril(L[i], -1) - np.tril(o.work, -1))) <= 1e-10 * n
        assert np.array_equal(np.triu(L[i]), np.triu(xs[i]))
        s, lg = oracle.pfaffian_slog(o.tau, o.pivots, n)
        assert sign[i] == s
        if n % 2 == 0:
            assert abs(logabs[i] - lg) <= 1e-10 * max(abs(lg), 1.0)


def test_batched_zero_columns_and_rank_deficient():
    """All-zero subcolumns (tau = 0, elimination continues) and a rank-deficient
    matrix (Pf = 0) inside one batch, against the oracle."""
    n = 40
    a = skew_lower(n, 7)
    a[:, 5] = 0.0
    a[5, :] = 0.0          # row/column 5 zero: singular, a zero tau appears
    b = np.zeros((n, n))   # everything zero
    c = skew_lower(n, 8)
    xs = np.stack([a, b, c])
    L, tau, piv, sign, logabs = apps().ltlt_batched_piv(xs)
    for i in range(3):
        o = oracle.ltlt_blk_piv(xs[i], b=n)
        assert np.array_equal(piv[i], o.pivots)
        assert np.allclose(tau[i], o.tau, rtol=1e-10 * n, atol=1e-10 * n)
        assert np.max(np.abs(np.tril(L[i], -1) - np.tril(o.work, -1))) <= 1e-10 * n
    assert sign[0] == 0.0 and sign[1] == 0.0 and sign[2] != 0.0


def test_batched_rejects_aliasing_and_large_n():
    import torch
    from paper_2411_09859_b200 import _capi
    lib = _capi.load()
    xd = torch.zeros((2, 8, 8), dtype=torch.float64, device="cuda")
    tau = torch.empty((2, 8), dtype=torch.float64, device="cuda")
    piv = torch.empty((2, 8), dtype=torch.int64, device="cuda")
    st = lib.skl_ltlt_batched_piv(2, 8, _capi.SKL_F64, xd.data_ptr(), 8, 64, xd.data_ptr(), 8, 64, tau.data_ptr(),
                                  piv.data_ptr(), None, None, None)
    assert st == 3  # SKL_ALIAS
    big = torch.zeros((1, 513, 513), dtype=torch.float64, device="cuda")
    with pytest.raises(Exception):
        apps().ltlt_batched_piv_device(big)
        torch.cuda.synchronize()
