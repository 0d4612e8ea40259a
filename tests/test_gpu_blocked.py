"""GPU parity of the pivoted blocked driver (through the C ABI) against the
oracle and the reference's golden vectors."""

import numpy as np
import pytest

import oracle
from conftest import EPS, worked_example
from paper_2411_09859_b200.inputs import skew_lower

pytestmark = pytest.mark.gpu


def pk():
    import paper_2411_09859_b200 as m
    return m


def l_checksums(work, n, seed=12345):
    r = np.random.Generator(np.random.Philox(seed)).standard_normal(n)
    S = np.tril(work[:, :n - 1], -2)
    lr = r + S @ r[1:]
    return lr


def assert_matches_oracle(x, b, fused, rtol=1e-10):
    n = x.shape[0]
    o = oracle.ltlt_blk_piv(x, b=b, fused=fused)
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=b, fused=fused)
    assert np.array_equal(r.p.pivots, o.pivots), "pivot sequence must be bit-exact"
    scale = max(np.max(np.abs(o.tau)), 1.0) if n > 1 else 1.0
    # BASELINE tolerance: L and T elementwise within 1e-10 * n relative
    assert np.max(np.abs(r.t.tau - o.tau), initial=0.0) <= rtol * n * scale
    assert np.max(np.abs(np.tril(r.l.data, -1) - np.tril(o.work, -1)), initial=0.0) <= rtol * n
    assert np.array_equal(np.triu(r.l.data), np.triu(x))  # upper/diag untouched
    assert r.flops == pk().FlopCounter(**o.flops)
    return r, o


@pytest.mark.parametrize("n,b", [(1, 4), (2, 1), (2, 4), (3, 2), (5, 1), (10, 3), (17, 16), (64, 16),
                                 (100, 7), (300, 32), (513, 64), (1000, 128), (1100, 256)])
@pytest.mark.parametrize("fused", ["var1", "var2a", "var2b"])
def test_blocked_vs_oracle(n, b, fused):
    assert_matches_oracle(skew_lower(n, n + b), b, fused)


def test_worked_example():
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower(worked_example()), b=2)
    assert r.p.pivots.tolist()[:2] == [0, 2]
    o = oracle.ltlt_blk_piv(worked_example(), b=2)
    assert np.allclose(r.t.tau, o.tau, rtol=1e-15)


def test_zero_matrix_and_zero_column():
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower.zeros(5), b=2)
    assert not r.t.tau.any() and not r.p.pivots.any()
    assert np.array_equal(r.l.dense(), np.eye(5))
    z = np.zeros((3, 3), order="F")
    z[2, 1] = 4.0
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower(z), b=2)
    o = oracle.ltlt_blk_piv(z, b=2)
    assert np.array_equal(r.p.pivots, o.pivots) and np.array_equal(r.t.tau, o.tau)


def test_nan_poisoned_upper_triangle_never_read():
    # test_core.py:39-58: entries on/above the diagonal are never read
    n = 300
    x = skew_lower(n, 5)
    xp = x.copy(order="F")
    xp[np.triu_indices(n)] = np.nan
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower(xp), b=32)
    o = oracle.ltlt_blk_piv(x, b=32)
    assert np.array_equal(r.p.pivots, o.pivots)
    assert np.isfinite(np.tril(r.l.data, -1)).all() and np.isfinite(r.t.tau).all()
    assert np.isnan(r.l.data[np.triu_indices(n)]).all()


def test_input_not_mutated_and_deterministic():
    x = skew_lower(700, 9)
    keep = x.copy()
    r1 = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=64)
    r2 = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=64)
    assert np.array_equal(x, keep)
    assert np.array_equal(r1.l.data, r2.l.data) and np.array_equal(r1.t.tau, r2.t.tau)


def test_pivot_stability_and_residual():
    n = 800
    x = skew_lower(n, 11)
    x[2:, 0] *= 1e3  # engineered near-breakdown (test_unblocked.py:93-104)
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=64)
    assert r.l.max_abs() <= 1.0 + 1e-15
    assert oracle.residual(x, r.l.data, r.t.tau, r.p.pivots) <= 10 * EPS * n


def test_device_resident_entry():
    import torch
    from paper_2411_09859_b200 import device as dv
    n = 512
    x = skew_lower(n, 3)
    xd = dv.to_device_colmajor(x)
    L, tau, piv = pk().ltlt_blk_piv_device(xd, 64, "var2a")
    o = oracle.ltlt_blk_piv(x, b=64, fused="var2a")
    assert np.array_equal(piv.cpu().numpy(), o.pivots)
    assert torch.equal(xd, dv.to_device_colmajor(x))  # input untouched


@pytest.mark.parametrize("fused", ["var1", "var2a", "var2b"])
def test_golden_small(golden, fused):
    g = golden("blk_small.npz")
    for n, b in [(64, 16), (300, 32), (513, 64), (1000, 128)]:
        key = f"n{n}_b{b}_{fused}_"
        r = pk().ltlt_blk_piv(pk().SkewMatrixLower(skew_lower(n, n)), b=b, fused=fused)
        assert np.array_equal(r.p.pivots, g[key + "piv"])
        assert np.allclose(r.t.tau, g[key + "tau"], rtol=1e-10 * n, atol=1e-10 * n)
        assert np.allclose(l_checksums(r.l.data, n), g[key + "lr"], rtol=1e-10 * n, atol=1e-10 * n)


@pytest.mark.parametrize("fused", ["var1", "var2a", "var2b"])
def test_config2_golden(golden, fused):
    """Config 2 (n=4096, nb=128) at full size: bit-exact pivots vs the reference,
    tau, L checksums, Pfaffian (sign, log|Pf|) and the backward error."""
    g = golden("cfg2_n4096_b128.npz")
    n = 4096
    x = skew_lower(n, 0)
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=128, fused=fused)
    assert np.array_equal(r.p.pivots, g["piv"])
    assert np.allclose(r.t.tau, g["tau"], rtol=1e-10 * n, atol=1e-10 * n)
    assert np.allclose(l_checksums(r.l.data, n), g["lr"], rtol=1e-10 * n, atol=1e-10 * n)
    sign, lg = oracle.pfaffian_slog(r.t.tau, r.p.pivots, n)
    assert sign == g["sign"] and abs(lg - g["logpf"]) <= 1e-10 * abs(g["logpf"])
    if fused == "var1":
        assert r.flops.level3 == int(g["flops"][1])
        res = residual_gpu(x, r)
        assert res <= 10 * EPS * n


def residual_gpu(x, r):
    """||P X P^T - L T L^T||_F / ||X||_F on the GPU (library GEMMs)."""
    import torch
    from paper_2411_09859_b200.core import compose_permutation
    n = x.shape[0]
    dev = "cuda"
    X = torch.as_tensor(np.tril(x, -1), device=dev)
    X = X - X.T
    perm = torch.as_tensor(compose_permutation(r.p), device=dev)
    PX = X[perm][:, perm]
    L = torch.as_tensor(r.l.dense(), device=dev)
    T = torch.as_tensor(r.t.dense(), device=dev)
    R = PX - L @ T @ L.T
    return float(torch.linalg.norm(R) / torch.linalg.norm(X))


def test_config3_golden(golden):
    """Config 3 (n=16384, nb=256, U(-1,1)): pivots, tau and log|Pf| vs the reference run."""
    g = golden("cfg3_n16384_b256.npz")
    import torch
    from paper_2411_09859_b200 import device as dv
    n = 16384
    x = skew_lower(n, 0, "uniform")
    L, tau, piv = pk().ltlt_blk_piv_device(dv.to_device_colmajor(x), 256, "var1")
    piv = piv.cpu().numpy()
    tau = tau.cpu().numpy()
    assert np.array_equal(piv, g["piv"])
    assert np.allclose(tau, g["tau"], rtol=1e-10 * n, atol=1e-10 * n)
    sign, lg = oracle.pfaffian_slog(tau, piv, n)
    assert sign == g["sign"] and abs(lg - g["logpf"]) <= 1e-10 * abs(g["logpf"])
    # L checksum on the device
    rr = torch.as_tensor(np.random.Generator(np.random.Philox(12345)).standard_normal(n), device="cuda")
    S = torch.tril(L[:, : n - 1], -2)
    lr = rr + S @ rr[1:]
    assert np.allclose(lr.cpu().numpy(), g["lr"], rtol=1e-10 * n, atol=1e-10 * n)


@pytest.mark.parametrize("n,b,fused", [(1, 4, "var1"), (2, 1, "var1"), (300, 32, "var2a"), (640, 64, "var1"),
                                       (1000, 128, "var2b")])
def test_host_buffer_entry(n, b, fused):
    """skl_ltlt_blk_piv_host (pinned host in/out, lower-triangle copies) returns the
    device path's factors bit for bit, and in place reproduces the full buffer."""
    import torch
    x = skew_lower(n, 7 * n + b)
    x = np.asfortranarray(x)
    x[np.triu_indices(n)] = np.nan        # upper triangle + diagonal never read
    dev = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=b, fused=fused)
    xp = torch.empty((n, n), dtype=torch.float64).pin_memory().numpy().T
    xp[...] = x
    L, tau, piv = pk().ltlt_blk_piv_host(xp, b, fused)
    assert np.array_equal(np.tril(L, -1), np.tril(dev.l.data, -1))
    assert np.array_equal(tau, dev.t.tau) and np.array_equal(piv, dev.p.pivots)
    # L's upper triangle: X's values inside the 128x128 diagonal blocks, untouched (0) elsewhere
    for j in range(n):
        blk0 = (j // 128) * 128
        assert np.all(np.isnan(L[blk0:j + 1, j])) and not L[:blk0, j].any()
    # in place: the whole buffer equals the reference's work buffer
    L2, tau2, piv2 = pk().ltlt_blk_piv_host(xp, b, fused, out=(xp, np.empty(max(n - 1, 0)), np.empty(n, np.int64)))
    assert L2 is xp and np.array_equal(np.tril(xp, -1), np.tril(dev.l.data, -1))
    assert np.array_equal(np.isnan(np.triu(xp)), np.isnan(np.triu(x))) and np.array_equal(tau2, tau)
