"""Config-5 golden: ONE run of the UNMODIFIED reference at n=49152, nb=512.

    OPENBLAS_NUM_THREADS=8 python tests/golden/make_cfg5.py [--n 49152] [--b 512] [--tmp /tmp/cfg5]

Input: the BASELINE config-5 matrix, X = G - G^T with G = Philox(0).standard_normal((n, n)) / sqrt(n)
(SURVEY §8d).  G is drawn in row chunks (a chunked Philox draw equals one full draw) and
accumulated straight into a column-major memmap D: row chunk [i0, i1) adds G[i0:i1, :] to
D[i0:i1, :] and subtracts its transpose from D[:, i0:i1].  Each entry receives exactly one
addition of +G[i, j] and one of -G[j, i] onto 0, so D[i, j] == G[i, j] - G[j, i] bit for bit
whatever the order.  The upper triangle and diagonal are then zeroed (SkewMatrixLower.from_dense,
reference core.py:62-68).  D lives on disk so the reference's own work copy (unblocked.py:43-48)
is the only 18 GiB resident array.

Output `cfg5_n49152_b512.npz`: pivots, tau, sign, log|Pf| (from tau and the pivot
parity), the L checksums L.r and L^T.r for a fixed Philox vector (computed column-block-wise from
the 'ones' buffer, same definition as make_golden.checksums), the reference's flop tallies and the
wall time.  The GPU box never reads the reference; `tests/test_gpu_cfg5.py` reads this file.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)


def build_input(n, path, seed=0, chunk=1024):
    rng = np.random.Generator(np.random.Philox(seed))
    D = np.lib.format.open_memmap(path, mode="w+", dtype=np.float64, shape=(n, n), fortran_order=True)
    s = np.sqrt(n)
    for i0 in range(0, n, chunk):
        i1 = min(n, i0 + chunk)
        g = rng.standard_normal((i1 - i0, n)) / s
        D[i0:i1, :] += g
        D[:, i0:i1] -= g.T
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        for j in range(j0, j1):
            D[: j + 1, j] = 0.0
    D.flush()
    return D


def checksums_blockwise(work, n, seed=12345, chunk=1024):
    """L.r and L^T.r with L read from the 'ones' buffer: S = tril(work[:, :n-1], -2)."""
    r = np.random.Generator(np.random.Philox(seed)).standard_normal(n)
    lr = r.copy()
    ltr = r.copy()
    for c0 in range(0, n - 1, chunk):
        c1 = min(n - 1, c0 + chunk)
        S = np.array(work[:, c0:c1])
        rows = np.arange(n)[:, None]
        cols = np.arange(c0, c1)[None, :]
        S[rows < cols + 2] = 0.0
        lr += S @ r[1 + c0:1 + c1]
        ltr[1 + c0:1 + c1] += S.T @ r
    return lr, ltr


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=49152)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--tmp", default="/tmp/cfg5")
    ap.add_argument("--out", default=str(HERE / "cfg5_n49152_b512.npz"))
    args = ap.parse_args()
    import skewltl as sk
    sk.kernels2.set_workers(1)
    n = args.n
    os.makedirs(args.tmp, exist_ok=True)
    t0 = time.time()
    D = build_input(n, os.path.join(args.tmp, f"x{n}.npy"))
    print(f"input built in {time.time() - t0:.1f} s", flush=True)
    t0 = time.time()
    r = sk.ltlt_blk_piv(sk.SkewMatrixLower(D), b=args.b)
    dt = time.time() - t0
    print(f"reference ltlt_blk_piv(n={n}, b={args.b}) took {dt:.1f} s", flush=True)
    del D
    piv, tau = r.p.pivots, r.t.tau
    even = tau[0:n - 1:2]
    sign = (-1.0 if np.count_nonzero(piv) % 2 else 1.0) * float(np.prod(np.sign(-even)))
    logpf = float(np.sum(np.log(np.abs(even)))) if n % 2 == 0 else -np.inf
    lr, ltr = checksums_blockwise(r.l.data, n)
    fc = r.flops
    np.savez_compressed(args.out, piv=piv.astype(np.int32), tau=tau, lr=lr, ltr=ltr, sign=np.array(sign),
                        logpf=np.array(logpf),
                        flops=np.array([fc.level2, fc.level3, fc.panel, fc.pivot], dtype=np.int64),
                        seconds=np.array(dt), n=np.array(n), b=np.array(args.b))
    print("cfg5 golden written:", args.out, "sign", sign, "logpf", logpf, flush=True)


if __name__ == "__main__":
    main()
