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
    """fp32: pivots/log|Pf| vs the reference's own fp32 run.  Rounding-level
    near-ties can flip an fp32 pivot in any implementation, so a small number
    of matrices may take a different (equally valid) pivot path; the Pfaffian
    magnitude must still agree to fp32 accuracy for all of them."""
    g = golden("cfg4_batch_f32.npz")
    xs = np.stack([skew_lower(256, i).astype(np.float32) for i in range(8192)])
    L, tau, piv, sign, logabs = apps().ltlt_batched_piv(xs)
    same = np.array([np.array_equal(piv[i], g["piv"][i]) for i in range(128)])
    assert same.mean() >= 0.95
    assert np.mean(sign == g["sign"]) >= 0.99
    rel = np.abs(logabs - g["logpf"]) / np.abs(g["logpf"])
    assert np.median(rel) <= 1e-5 and np.max(rel) <= 1e-3
