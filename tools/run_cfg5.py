"""Config 5 (n=49152, nb=512, G ~ N(0, 1/n)) on ONE B200: device-resident
factorization timing plus the size-independent parity properties:

* backward error ||P X P^T - L T L^T||_F / (n ||X||_F) <= 10 eps n (blockwise on the GPU),
* log|Pf| from tau equals slogdet(X)/2 (cuSOLVER LU, an independent algorithm),
* |L| <= 1 (partial pivoting), pivots in range, last pivot 0.

X is generated exactly as the configs define it (Philox(seed) row chunks == one
full draw) and streamed to the device chunk by chunk; nothing reads the reference.
Usage: python tools/run_cfg5.py [--n 49152] [--b 512] [--reps 2] [--no-check]
"""
import argparse
import json
import math
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import device as dv


def device_skew_input(n, seed=0, dist="normal_scaled", chunk=2048):
    """Column-major CUDA tensor holding X = G - G^T (full skew) for the config generator."""
    rng = np.random.Generator(np.random.Philox(seed))
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")      # row-major G[i, j]
    pin = torch.empty((chunk, n), dtype=torch.float64).pin_memory()
    for i0 in range(0, n, chunk):
        rows = min(chunk, n - i0)
        if dist == "normal_scaled":
            g = rng.standard_normal((rows, n)) / np.sqrt(n)
        elif dist == "uniform":
            g = rng.uniform(-1.0, 1.0, (rows, n))
        else:
            g = rng.standard_normal((rows, n))
        pin[:rows].numpy()[...] = g
        G[i0:i0 + rows].copy_(pin[:rows], non_blocking=True)
        torch.cuda.synchronize()
    X = torch.empty((n, n), dtype=torch.float64, device="cuda").t()    # column-major
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        X[:, j0:j1] = G[:, j0:j1] - G[j0:j1, :].t()
    del G
    torch.cuda.empty_cache()
    return X


def dense_unit_lower_(Lbuf):
    """'ones'-mode L buffer (column j-1 holds L[:, j] below the diagonal) -> dense unit lower, in place."""
    n = Lbuf.shape[0]
    chunk = 2048
    # shift columns right by one, last to first so nothing is overwritten early
    for j1 in range(n, 1, -chunk):
        j0 = max(1, j1 - chunk)
        Lbuf[:, j0:j1] = Lbuf[:, j0 - 1:j1 - 1].clone()
    Lbuf[:, 0] = 0.0
    rows = torch.arange(n, device=Lbuf.device)[:, None]
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        blk = Lbuf[:, j0:j1]
        idx = torch.arange(j0, j1, device=blk.device)
        blk.masked_fill_(rows <= idx[None, :], 0.0)
        blk[idx, idx - j0] = 1.0
    return Lbuf


def compose_perm(piv):
    p = np.arange(piv.size)
    for k, off in enumerate(piv):
        if off:
            p[k], p[k + off] = p[k + off], p[k]
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=49152)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--fused", default="var1")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--dist", default="normal_scaled")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--virtual", type=int, default=0,
                    help="also run the block-cyclic driver over this many virtual ranks and compare")
    ap.add_argument("--nbd", type=int, default=512)
    a = ap.parse_args()
    n = a.n
    t0 = time.time()
    X = device_skew_input(n, 0, a.dist)
    gen_s = time.time() - t0
    L = dv.empty_colmajor(n, n, torch.float64)
    tau = torch.empty(n - 1, dtype=torch.float64, device="cuda")
    piv = torch.empty(n, dtype=torch.int64, device="cuda")
    from bench import ClockSampler
    sampler = ClockSampler(0)
    sampler.start()
    times = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        pk.ltlt_blk_piv_device(X, a.b, a.fused, out=(L, tau, piv))
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    clocks = sampler.stop()
    # per-kernel-class split of one more factorization (CUDA events per launch)
    import ctypes
    from paper_2411_09859_b200 import _capi
    lib = _capi.load()
    lib.skl_timing_enable(1)
    pk.ltlt_blk_piv_device(X, a.b, a.fused, out=(L, tau, piv))
    torch.cuda.synchronize()
    kms, kcnt = (ctypes.c_double * 4)(), (ctypes.c_int * 4)()
    lib.skl_timing_read(kms, kcnt)
    lib.skl_timing_enable(0)
    split = {k: round(kms[i], 2) for i, k in enumerate(["panel", "pack", "gemm", "finalize"])}
    split["launches"] = list(kcnt)
    dv._WS.clear()
    torch.cuda.empty_cache()
    ms = min(times)
    flops = n ** 3 / 3
    out = {"n": n, "nb": a.b, "fused": a.fused, "ms": round(ms, 2), "all_ms": [round(t, 2) for t in times],
           "gflops": round(flops / ms / 1e6, 1), "gen_s": round(gen_s, 1), "split_ms": split,
           "clocks": clocks}
    if a.virtual:
        from paper_2411_09859_b200.dist import DistLTLT
        c = DistLTLT(n, a.b, a.fused, nbd=a.nbd, virtual_ranks=a.virtual)
        dts = []
        for _ in range(2):
            c.load_input(X)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            Ld, taud_, pivd = c.factorize()
            e1.record()
            torch.cuda.synchronize()
            dts.append(e0.elapsed_time(e1))
        out["virtual"] = {"ranks": a.virtual, "nbd": a.nbd, "ms": round(min(dts), 2),
                          "piv_equal": bool(torch.equal(pivd, piv)), "tau_equal": bool(torch.equal(taud_, tau)),
                          "l_equal": bool(torch.equal(torch.tril(Ld, -1), torch.tril(L, -1)))}
        del Ld, taud_, pivd
        c.close()
        torch.cuda.empty_cache()
    if not a.no_check:
        pv = piv.cpu().numpy()
        tv = tau.cpu().numpy()
        out["pivots_ok"] = bool(pv[-1] == 0 and pv[0] == 0 and np.all(pv >= 0)
                                and np.all(np.arange(n) + pv < n))
        out["nontrivial_pivots"] = int(np.count_nonzero(pv))
        # log|Pf| and sign from tau (pfaffian_slog convention)
        ev = tv[0::2]
        logpf = float(np.sum(np.log(np.abs(ev))))
        out["logpf"] = logpf
        Lbuf = dense_unit_lower_(L)
        out["max_abs_L"] = float(Lbuf.abs().max())
        xnorm = float(torch.linalg.norm(X))
        perm = torch.as_tensor(compose_perm(pv), device="cuda")
        taud = tau
        rsq = 0.0
        chunk = 2048
        for j0 in range(0, n, chunk):
            j1 = min(n, j0 + chunk)
            Lt = Lbuf[j0:j1, :].t()                       # L^T[:, J]  (n x w)
            TLt = torch.zeros_like(Lt)
            TLt[1:] += taud[:, None] * Lt[:-1]           # T[i+1, i] = tau_i
            TLt[:-1] -= taud[:, None] * Lt[1:]           # T[i, i+1] = -tau_i
            R = X[:, perm[j0:j1]][perm] - Lbuf @ TLt
            rsq += float((R * R).sum())
            del R, TLt
        out["residual"] = math.sqrt(rsq) / (n * xnorm)
        out["residual_bound"] = 10 * np.finfo(np.float64).eps * n
        del Lbuf, L
        torch.cuda.empty_cache()
        sdet, ldet = torch.linalg.slogdet(X)
        out["slogdet_half"] = float(ldet) / 2
        out["logpf_rel_err"] = abs(logpf - float(ldet) / 2) / abs(float(ldet) / 2)
        out["ok"] = bool(out["pivots_ok"] and out["residual"] <= out["residual_bound"]
                         and out["logpf_rel_err"] <= 1e-10 and out["max_abs_L"] <= 1.0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
