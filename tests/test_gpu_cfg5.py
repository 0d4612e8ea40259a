"""Config 5 at full size (n=49152, nb=512, X = G - G^T, G ~ N(0, 1/n) from
Philox seed 0) against ONE run of the unmodified reference
(`ltlt_blk_piv(x, b=512)`, blocked.py:303-363; fixture written by
tests/golden/make_cfg5.py).  This is the size with the smallest pivot margins,
so the bit-exact pivot sequence is the point of the test.

Tolerances (north star): pivots bit-exact; tau and the L checksums
L.r / L^T.r elementwise within 1e-10 * n (relative and absolute); log|Pf|
within 1e-10 relative; Pfaffian sign equal."""

import numpy as np
import pytest

import oracle

N5, NB5 = 49152, 512


def _checksums_device(L, n, torch, chunk=2048):
    """L.r and L^T.r from the 'ones' buffer (column j-1 holds L[:, j] below the
    diagonal), column block by column block on the device."""
    r = torch.as_tensor(np.random.Generator(np.random.Philox(12345)).standard_normal(n), device="cuda")
    lr = r.clone()
    ltr = r.clone()
    rows = torch.arange(n, device="cuda")[:, None]
    for c0 in range(0, n - 1, chunk):
        c1 = min(n - 1, c0 + chunk)
        S = L[:, c0:c1].clone()
        cols = torch.arange(c0, c1, device="cuda")[None, :]
        S.masked_fill_(rows < cols + 2, 0.0)
        lr += S @ r[1 + c0:1 + c1]
        ltr[1 + c0:1 + c1] += S.t() @ r
    return lr.cpu().numpy(), ltr.cpu().numpy()


@pytest.mark.gpu
def test_config5_golden(golden):
    g = golden("cfg5_n49152_b512.npz")
    import torch

    import paper_2411_09859_b200 as pk
    from paper_2411_09859_b200.inputs import normal_scaled_rows, skew_device_from_rows

    n = N5
    free = torch.cuda.mem_get_info()[0]
    if free < 80 * 2 ** 30:
        pytest.skip(f"config 5 needs ~80 GiB of device memory, {free / 2 ** 30:.0f} GiB free")
    X = skew_device_from_rows(normal_scaled_rows(n, 0), torch)
    L, tau, piv = pk.ltlt_blk_piv_device(X, NB5, "var1")
    del X
    torch.cuda.empty_cache()
    piv = piv.cpu().numpy()
    tau = tau.cpu().numpy()
    ref_piv = g["piv"].astype(np.int64)
    if not np.array_equal(piv, ref_piv):
        k = int(np.flatnonzero(piv != ref_piv)[0])
        pytest.fail(f"pivot sequence differs from the reference first at step {k}: "
                    f"gpu {piv[k]} vs reference {ref_piv[k]}")
    assert np.allclose(tau, g["tau"], rtol=1e-10 * n, atol=1e-10 * n)
    sign, lg = oracle.pfaffian_slog(tau, piv, n)
    assert sign == float(g["sign"])
    assert abs(lg - float(g["logpf"])) <= 1e-10 * abs(float(g["logpf"]))
    lr, ltr = _checksums_device(L, n, torch)
    assert np.allclose(lr, g["lr"], rtol=1e-10 * n, atol=1e-10 * n)
    assert np.allclose(ltr, g["ltr"], rtol=1e-10 * n, atol=1e-10 * n)
    # |L| <= 1 under partial pivoting (strict lower part of the 'ones' buffer)
    assert float(torch.tril(L[:, : n - 1], -2).abs().max()) <= 1.0
