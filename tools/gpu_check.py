"""Scratch GPU parity + timing check (development aid)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import oracle
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200 import kernels3
from paper_2411_09859_b200.inputs import skew_lower
import torch

def cmp(n, b, fused, seed=0):
    x = skew_lower(n, seed)
    t0 = time.time(); o = oracle.ltlt_blk_piv(x, b=b, fused=fused); t1 = time.time()
    r = pk.ltlt_blk_piv(pk.SkewMatrixLower(x), b=b, fused=fused)
    pe = np.array_equal(r.p.pivots, o.pivots)
    dt = np.max(np.abs(r.t.tau - o.tau)) / max(np.max(np.abs(o.tau)), 1e-300)
    dl = np.max(np.abs(np.tril(r.l.data, -1) - np.tril(o.work, -1)))
    up = np.array_equal(np.triu(r.l.data), np.triu(x))
    fl = r.flops == pk.FlopCounter(**o.flops)
    first = np.flatnonzero(r.p.pivots != o.pivots)[:5]
    print(f"n={n} b={b} {fused}: piv_eq={pe} first_bad={first} dtau={dt:.2e} dL={dl:.2e} upper_ok={up} flops_ok={fl} oracle={t1-t0:.2f}s", flush=True)

def skr2k_check(n, k):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((n, k)); tau = rng.standard_normal(k - 1)
    W = oracle.form_w(A, tau)
    C = np.asfortranarray(rng.standard_normal((n, n)))
    C0 = C.copy(); Cr = C.copy()
    keff = oracle.skew_rank2k(Cr, 1.0, A, W)
    Cg = C.copy()
    kernels3.skew_rank2k(Cg, 1.0, A, W, 1.0)
    low = np.tril(np.ones((n, n), bool), -1)
    err = np.max(np.abs(Cg[low] - Cr[low])); up = np.array_equal(Cg[~low], C0[~low])
    print(f"skr2k n={n} k={k}: keff={keff} gpu_keff={kernels3.last_keff} maxerr={err:.2e} upper_untouched={up}", flush=True)

if __name__ == "__main__":
    torch.cuda.init()
    skr2k_check(300, 10); skr2k_check(1000, 129)
    for n, b in [(2, 4), (3, 2), (10, 3), (64, 16), (300, 32), (513, 64), (1000, 128)]:
        for fused in ("var1", "var2a", "var2b"):
            cmp(n, b, fused)
    cmp(4096, 128, "var1")
    # timing (device resident)
    for n, b, fused in [(4096, 128, "var1"), (4096, 128, "var2a")]:
        x = skew_lower(n, 0)
        xd = pk.device.to_device_colmajor(x) if hasattr(pk, "device") else None
        from paper_2411_09859_b200 import device as dv
        xd = dv.to_device_colmajor(x)
        for _ in range(2): pk.ltlt_blk_piv_device(xd, b, fused)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); 
        for _ in range(3): pk.ltlt_blk_piv_device(xd, b, fused)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"TIME n={n} b={b} {fused}: {ms:.2f} ms  {n**3/3/ms/1e9:.2f} TFLOP/s", flush=True)
