"""GPU parity of apps.solve (apps.py:33-100) against the
oracle (pinned to the reference in test_oracle.py): permuted unit-lower solve,
pivoted skew-tridiagonal solve, transposed solve, all on the device.

Tolerance: the solution is compared relative to its largest entry with
1e-10 * n * kappa_est, kappa_est = max|y| / max|b| (>= 1), and the residual
||X y - b|| / (||X|| ||y||) must stay <= 10 eps n."""

import numpy as np
import pytest

import oracle
from paper_2411_09859_b200.inputs import skew_lower

pytestmark = pytest.mark.gpu


def pk():
    import paper_2411_09859_b200 as m
    return m


@pytest.mark.parametrize("n", [2, 8, 64, 300, 1000])
@pytest.mark.parametrize("nrhs", [None, 1, 3, 17])
def test_solve_vs_oracle(n, nrhs):
    x = skew_lower(n, n + 11)
    rng = np.random.Generator(np.random.Philox(n))
    b = rng.standard_normal(n) if nrhs is None else rng.standard_normal((n, nrhs))
    y = pk().solve(pk().SkewMatrixLower(x), b)
    yo = oracle.solve(x, b)
    assert y.shape == yo.shape
    kappa = max(1.0, float(np.max(np.abs(yo))) / max(float(np.max(np.abs(b))), 1e-300))
    assert np.max(np.abs(y - yo)) <= 1e-10 * n * kappa * max(1.0, float(np.max(np.abs(yo))))
    X = oracle.skew_dense(x)
    r = X @ y.reshape(n, -1) - b.reshape(n, -1)
    eps = np.finfo(float).eps
    assert np.linalg.norm(r) <= 10 * eps * n * np.linalg.norm(X) * np.linalg.norm(y)


def test_solve_block_argument_and_device_rhs():
    import torch
    n = 200
    x = skew_lower(n, 3)
    b = np.random.Generator(np.random.Philox(1)).standard_normal((n, 2))
    y1 = pk().solve(pk().SkewMatrixLower(x), b, block=32)
    bd = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    y2 = pk().solve(pk().SkewMatrixLower(x), bd)
    assert y2.is_cuda and y2.shape == (n, 2)
    assert np.allclose(y1, y2.cpu().numpy(), rtol=1e-9, atol=1e-12)
    assert np.allclose(y1, oracle.solve(x, b, block=32), rtol=1e-8, atol=1e-10)


@pytest.mark.parametrize("n", [1, 3, 7, 65])
def test_solve_singular_odd(n):
    """Every odd m is singular: SingularT (apps.py:80-82)."""
    with pytest.raises(pk().SingularT):
        pk().solve(pk().SkewMatrixLower(skew_lower(n, n)), np.ones(n))


def test_solve_dimension_mismatch():
    with pytest.raises(ValueError):
        pk().solve(pk().SkewMatrixLower(skew_lower(8, 0)), np.ones(7))


@pytest.mark.parametrize("n,nrhs", [(8192, 1), (8192, 6), (16384, 2)])
def test_solve_large_n_residual(n, nrhs):
    """Sizes past the 48 KB default shared-memory window of the permutation
    composition (n > 6144): device-resident X and b, residual on the device."""
    import torch
    from paper_2411_09859_b200 import device as dv
    x = skew_lower(n, 3)
    xd = dv.to_device_colmajor(x)
    b = torch.randn(n, nrhs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(n))
    y = pk().solve(pk().SkewMatrixLower(xd), b)
    Xd = torch.tril(xd, -1)
    Xd = Xd - Xd.T
    r = Xd @ y - b
    eps = np.finfo(float).eps
    assert float(torch.linalg.norm(r)) <= 10 * eps * n * float(torch.linalg.norm(Xd)) * float(torch.linalg.norm(y))
