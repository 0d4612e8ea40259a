"""Generate golden fixtures by running the UNMODIFIED reference `skewltl`.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py [--big]
The GPU box never imports the reference; tests read only the .npz files
written here.  Inputs come from paper_2411_09859_b200.inputs (the BASELINE
seeded generators), so the GPU path sees the identical bits.

Fixtures
  kat.npz              worked 4x4 / m=2 / zero-column known answers (pivoted and not)
  cfg1_n512.npz        ltlt_unb_twostep(pivot=True): pivots, tau, full strictly-lower L, flops
  blk_small.npz        ltlt_blk_piv at n in {64, 300, 513, 1000} x var1/2a/2b: pivots, tau, L checksums
  cfg2_n4096_b128.npz  ltlt_blk_piv(b=128) var1 (+ var2a/var2b pivots): pivots, tau, L.r / L^T.r, sign, log|Pf|
  cfg3_n16384_b256.npz (--big) same for config 3 (about 6 minutes of reference time)
  cfg4_batch.npz       (--big) pfaffian path per matrix (fp64 and fp32): sign, log|Pf| for all 8192,
                       pivots and tau for the first 128
  solve_small.npz      apps.solve: n in {2, 8, 64, 300}, 1 and 3 right-hand sides;
                       SingularT row for odd n
  mm_small.mtx         mmio.mm_write of a 9x9 skew matrix (the Matrix Market format)
  l3_small.npz         kernels3.skew_tridiag_gemm: general and tril blocks, several
                       (p, q, k, alpha, beta) incl. p < q, k = 0 and beta = 0: inputs and outputs
  unpiv_small.npz      unpivoted drivers: ltlt_blk_var1/2a/2b/twostep/left x panel
                       variants ll/rl/twostep, ltlt_unb_rl (+pivoted), ltlt_unb_ll (+first_column),
                       ltlt_unb_panel (ll/rl/twostep, pivoted, first_column) at n in {64, 150, 301}:
                       tau, pivots, flops, L checksums (full strictly-lower L at n=64)
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.path.insert(0, str(HERE.parent.parent))

from paper_2411_09859_b200.inputs import skew_lower  # noqa: E402

sys.path.insert(0, str(HERE))
from l3_cases import L3_CASES, l3_inputs  # noqa: E402


def ref():
    import skewltl
    return skewltl


def checksums(work, n, seed=12345):
    """L.r and L^T.r for a fixed Philox vector, from the 'ones' buffer."""
    r = np.random.Generator(np.random.Philox(seed)).standard_normal(n)
    S = np.tril(work[:, :n - 1], -2)  # S[i, j-1] = L[i, j] for i > j >= 1
    lr = r.copy()
    lr += S @ r[1:]
    ltr = r.copy()
    ltr[1:] += S.T @ r
    return lr, ltr


def slog(tau, piv, n):
    if n % 2:
        return 0.0, -np.inf
    even = np.asarray(tau[0:n - 1:2], dtype=np.float64)
    sign = (-1.0 if np.count_nonzero(piv) % 2 else 1.0) * float(np.prod(np.sign(-even)))
    return sign, float(np.sum(np.log(np.abs(even))))


def flops_tuple(fc):
    return np.array([fc.level2, fc.level3, fc.panel, fc.pivot], dtype=np.int64)


def make_kat(sk):
    out = {}
    x = sk.SkewMatrixLower.zeros(4)
    x.data[1, 0], x.data[2, 0], x.data[3, 0] = 2.0, 1.0, 3.0
    x.data[2, 1], x.data[3, 1] = 4.0, 1.0
    x.data[3, 2] = 5.0
    out["worked_x"] = x.data.copy()
    r = sk.ltlt_unb_twostep(x)
    out["worked_tau"] = r.t.tau
    out["worked_L"] = r.l.dense()
    rp = sk.ltlt_blk_piv(x, b=2)
    out["worked_piv_tau"] = rp.t.tau
    out["worked_piv_piv"] = rp.p.pivots
    out["worked_piv_L"] = rp.l.data
    out["worked_pf"] = np.array(sk.pfaffian(x))
    x2 = sk.SkewMatrixLower.zeros(2)
    x2.data[1, 0] = -3.5
    out["m2_x"] = x2.data.copy()
    out["m2_tau"] = sk.ltlt_blk_piv(x2, b=1).t.tau
    x3 = sk.SkewMatrixLower.zeros(2)
    x3.data[1, 0] = 3.0
    out["pf2_val"] = np.array(sk.pfaffian(x3))
    z = sk.SkewMatrixLower.zeros(3)
    z.data[2, 1] = 4.0
    out["zerocol_x"] = z.data.copy()
    out["zerocol_tau"] = sk.ltlt_blk_piv(z, b=2).t.tau
    return out


def make_blk(sk, n, b, fused, seed=0, store_l=False):
    x = skew_lower(n, seed)
    t0 = time.time()
    r = sk.ltlt_blk_piv(sk.SkewMatrixLower(x), b=b, fused=fused)
    dt = time.time() - t0
    lr, ltr = checksums(r.l.data, n)
    sign, lg = slog(r.t.tau, r.p.pivots, n)
    d = dict(piv=r.p.pivots.astype(np.int32), tau=r.t.tau, lr=lr, ltr=ltr, sign=np.array(sign),
             logpf=np.array(lg), flops=flops_tuple(r.flops), seconds=np.array(dt))
    if store_l:
        il = np.tril_indices(n, -1)
        d["l_lower"] = r.l.data[il]
    return d


def _batch_one(args):
    i, dtype = args
    sys.path.insert(0, REF)
    import skewltl as sk
    x = skew_lower(256, i).astype(dtype)
    r = sk.ltlt_blk_piv(sk.SkewMatrixLower(x), b=256)
    sign, lg = slog(r.t.tau, r.p.pivots, 256)
    return i, r.p.pivots.astype(np.int16), r.t.tau.astype(np.float64), sign, lg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    sk = ref()
    sk.kernels2.set_workers(1)
    only = set(args.only.split(",")) if args.only else None

    def want(name):
        return only is None or name in only

    if want("kat"):
        np.savez_compressed(HERE / "kat.npz", **make_kat(sk))
        print("kat ok", flush=True)
    if want("cfg1"):
        x = skew_lower(512, 0)
        t0 = time.time()
        r = sk.ltlt_unb_twostep(sk.SkewMatrixLower(x), pivot=True)
        il = np.tril_indices(512, -1)
        np.savez_compressed(HERE / "cfg1_n512.npz", piv=r.p.pivots.astype(np.int32), tau=r.t.tau,
                            l_lower=r.l.data[il], flops=flops_tuple(r.flops), seconds=np.array(time.time() - t0))
        print("cfg1 ok", flush=True)
    if want("small"):
        d = {}
        for n, b in [(64, 16), (300, 32), (513, 64), (1000, 128)]:
            for fused in ("var1", "var2a", "var2b"):
                g = make_blk(sk, n, b, fused, seed=n)
                for k, v in g.items():
                    d[f"n{n}_b{b}_{fused}_{k}"] = v
        np.savez_compressed(HERE / "blk_small.npz", **d)
        print("small ok", flush=True)
    if want("unpiv"):
        d = {}

        def put(key, r, n):
            lr, ltr = checksums(r.l.data, n)
            d[f"{key}_tau"] = r.t.tau
            d[f"{key}_piv"] = r.p.pivots.astype(np.int32)
            d[f"{key}_flops"] = flops_tuple(r.flops)
            d[f"{key}_lr"], d[f"{key}_ltr"] = lr, ltr
            if r.l.first_column is not None:
                d[f"{key}_first"] = r.l.first_column
            if n <= 64:
                d[f"{key}_l"] = r.l.data[np.tril_indices(n, -1)]

        for n, b in [(64, 16), (150, 32), (301, 64)]:
            X = sk.SkewMatrixLower(skew_lower(n, n))
            fcv = np.random.Generator(np.random.Philox(n)).standard_normal(n - 1) * 0.5
            d[f"n{n}_first_column"] = fcv
            for drv in ("var1", "var2a", "var2b", "twostep", "left"):
                fn = getattr(sk, f"ltlt_blk_{drv}")
                for pv in ("ll", "rl", "twostep"):
                    put(f"n{n}_{drv}_{pv}", fn(X, b=b, panel_variant=pv), n)
            put(f"n{n}_unb_rl", sk.ltlt_unb_rl(X), n)
            put(f"n{n}_unb_rl_piv", sk.ltlt_unb_rl(X, pivot=True), n)
            put(f"n{n}_unb_ll", sk.ltlt_unb_ll(X), n)
            put(f"n{n}_unb_ll_first", sk.ltlt_unb_ll(X, first_column=fcv), n)
            for pv in ("ll", "rl", "twostep"):
                put(f"n{n}_panel40_{pv}", sk.ltlt_unb_panel(X, 40, variant=pv), n)
            put(f"n{n}_panel40_piv", sk.ltlt_unb_panel(X, 40, pivot=True), n)
            put(f"n{n}_panel40_first", sk.ltlt_unb_panel(X, 40, first_column=fcv), n)
        np.savez_compressed(HERE / "unpiv_small.npz", **d)
        print("unpiv ok", flush=True)
    if want("l3"):
        d = {}
        # inputs are regenerated by the tests from Philox(1000 + i) in the order a, b, tau, c
        for i, (p_, q_, k_, tril, alpha, beta) in enumerate(L3_CASES):
            a, b, tau, c = l3_inputs(i, p_, q_, k_)
            out = c.copy(order="F")
            sk.kernels3.skew_tridiag_gemm(out, alpha, a, sk.SkewTridiagonal(tau), b, beta, tril=tril)
            d[f"c{i}_meta"] = np.array([p_, q_, k_, int(tril), alpha, beta])
            d[f"c{i}_out"] = out
        cases = L3_CASES
        d["ncases"] = np.array(len(cases))
        np.savez_compressed(HERE / "l3_small.npz", **d)
        print("l3 ok", flush=True)
    if want("solve"):
        d = {}
        for n in (2, 8, 64, 300):
            X = sk.SkewMatrixLower(skew_lower(n, n))
            b1 = np.random.Generator(np.random.Philox(n)).standard_normal(n)
            b3 = np.random.Generator(np.random.Philox(n + 1)).standard_normal((n, 3))
            d[f"n{n}_b1"], d[f"n{n}_b3"] = b1, b3
            d[f"n{n}_y1"], d[f"n{n}_y3"] = sk.solve(X, b1), sk.solve(X, b3)
        for n in (3, 7):
            try:
                sk.solve(sk.SkewMatrixLower(skew_lower(n, n)), np.ones(n))
                d[f"odd{n}_row"] = np.array(-1)
            except sk.SingularT as e:
                d[f"odd{n}_row"] = np.array(int(str(e).rsplit(" ", 1)[-1]))
        np.savez_compressed(HERE / "solve_small.npz", **d)
        print("solve ok", flush=True)
    if want("mmio"):
        x = sk.SkewMatrixLower(skew_lower(9, 4))
        x.data[5, 2] = 0.0                           # a structural zero is skipped
        sk.mm_write(HERE / "mm_small.mtx", x)
        print("mmio ok", flush=True)
    if want("cfg2"):
        g = make_blk(sk, 4096, 128, "var1")
        for fused in ("var2a", "var2b"):
            g2 = make_blk(sk, 4096, 128, fused)
            g[f"piv_{fused}"] = g2["piv"]
            g[f"tau_{fused}"] = g2["tau"]
        np.savez_compressed(HERE / "cfg2_n4096_b128.npz", **g)
        print("cfg2 ok", g["seconds"], flush=True)
    if args.big and want("cfg4"):
        for dtype, tag in ((np.float64, "f64"), (np.float32, "f32")):
            with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
                res = list(ex.map(_batch_one, [(i, dtype) for i in range(8192)], chunksize=64))
            res.sort(key=lambda t: t[0])
            np.savez_compressed(HERE / f"cfg4_batch_{tag}.npz",
                                sign=np.array([t[3] for t in res]), logpf=np.array([t[4] for t in res]),
                                piv=np.stack([t[1] for t in res[:128]]), tau=np.stack([t[2] for t in res[:128]]))
            print("cfg4", tag, "ok", flush=True)
    if args.big and want("cfg3"):
        x = skew_lower(16384, 0, "uniform")
        t0 = time.time()
        r = sk.ltlt_blk_piv(sk.SkewMatrixLower(x), b=256)
        dt = time.time() - t0
        lr, ltr = checksums(r.l.data, 16384)
        sign, lg = slog(r.t.tau, r.p.pivots, 16384)
        np.savez_compressed(HERE / "cfg3_n16384_b256.npz", piv=r.p.pivots.astype(np.int32), tau=r.t.tau, lr=lr,
                            ltr=ltr, sign=np.array(sign), logpf=np.array(lg), flops=flops_tuple(r.flops),
                            seconds=np.array(dt))
        print("cfg3 ok", dt, flush=True)


if __name__ == "__main__":
    main()
