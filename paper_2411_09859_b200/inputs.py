"""Seeded synthetic inputs for the BASELINE.json configs.

The reference's own tests and CLI use seeded Philox matrices
(``core.py:87-97``, ``cli.py:110,137``); the configs use X = G - G^T with G
drawn from ``np.random.Generator(np.random.Philox(seed))``.  Inputs are
generated on the host so the oracle and the GPU see identical bits.
"""

from __future__ import annotations

import numpy as np

#: BASELINE.json configs as (name, n, nb, distribution, dtype)
CONFIGS = {
    1: dict(name="unb_twostep_n512", n=512, nb=None, dist="normal"),
    2: dict(name="blk_piv_n4096_nb128", n=4096, nb=128, dist="normal"),
    3: dict(name="blk_piv_n16384_nb256", n=16384, nb=256, dist="uniform"),
    4: dict(name="batched_8192x256", n=256, nb=256, dist="normal", batch=8192),
    5: dict(name="blk_piv_n49152_nb512", n=49152, nb=512, dist="normal_scaled"),
}


def skew_lower(n, seed=0, dist="normal", dtype=np.float64):
    """Strictly-lower column-major buffer of X = G - G^T (upper/diag zero)."""
    rng = np.random.Generator(np.random.Philox(seed))
    if dist == "normal":
        g = rng.standard_normal((n, n))
    elif dist == "uniform":
        g = rng.uniform(-1.0, 1.0, (n, n))
    elif dist == "normal_scaled":
        g = rng.standard_normal((n, n)) / np.sqrt(n)
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    x = g - g.T
    out = np.zeros((n, n), dtype=dtype, order="F")
    il, jl = np.tril_indices(n, -1)
    out[il, jl] = x[il, jl].astype(dtype)
    return out


def config_input(cfg, seed=0, dtype=np.float64):
    c = CONFIGS[cfg]
    return skew_lower(c["n"], seed, c["dist"], dtype)


def batched_inputs(batch, n=256, seed0=0, dtype=np.float64):
    """Config 4: matrix i uses seed seed0 + i; fp32 is the fp64 X cast."""
    out = np.zeros((batch, n, n), dtype=dtype)
    for i in range(batch):
        out[i] = skew_lower(n, seed0 + i, "normal", np.float64).astype(dtype).T
    # stored so that out[i].T is column-major: out[i][j, r] = X[r, j]
    return out


def normal_scaled_rows(n, seed=0, out=None, chunk=1024):
    """Config 5's G = Philox(seed).standard_normal((n, n)) / sqrt(n), row-major,
    drawn in row chunks (a chunked Philox draw equals one full draw)
    so no second n x n temporary is needed.  Bit-identical to skew_lower's G."""
    rng = np.random.Generator(np.random.Philox(seed))
    g = np.empty((n, n), dtype=np.float64) if out is None else out
    s = np.sqrt(n)
    for i0 in range(0, n, chunk):
        i1 = min(n, i0 + chunk)
        g[i0:i1] = rng.standard_normal((i1 - i0, n)) / s
    return g


def skew_device_from_rows(g, torch, chunk=2048):
    """Column-major CUDA tensor X = G - G^T from a row-major host G (the full skew
    matrix; only its strict lower triangle is read).  fp64 subtraction is
    correctly rounded on both sides, so X equals skew_lower's bit for bit."""
    n = g.shape[0]
    gd = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for i0 in range(0, n, chunk):
        gd[i0:i0 + chunk].copy_(torch.from_numpy(g[i0:i0 + chunk]))
    x = torch.empty((n, n), dtype=torch.float64, device="cuda").t()   # column-major
    for j0 in range(0, n, chunk):
        x[:, j0:j0 + chunk] = gd[:, j0:j0 + chunk] - gd[j0:j0 + chunk, :].t()
    del gd
    torch.cuda.empty_cache()
    return x
