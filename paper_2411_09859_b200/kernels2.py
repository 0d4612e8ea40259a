"""Level-2 kernels (drop-in for reference ``kernels2.py``).

``skew_rank2`` (kernels2.py:93-131), ``gen_rank2`` (kernels2.py:134-163),
``skew_tridiag_gemv`` (kernels2.py:178-229), ``apply_row_pivots``
(kernels2.py:232-271) and ``trapezoid_rank2`` / ``PanelView``
(kernels2.py:274-312) with the reference's signatures and in-place
semantics; the arithmetic runs in the CUDA library.  NumPy operands are
staged to the GPU and the output view written back; column-major torch CUDA
tensors are updated in place.  Every call is recorded in the active
``instrument`` trace / counter with the reference's flop rule.
"""

from __future__ import annotations

import numpy as np

from dataclasses import dataclass

from . import _capi
from . import device as dv
from . import instrument
from .core import SkewTridiagonal, _is_torch

JAM = 64                 # kernels2.py:24 (CPU column jamming; informational)
PIVOT_ROW_BLOCK = 512    # kernels2.py:27 (informational)


def set_workers(n):
    """Accepted for compatibility (kernels2.py:29-41); GPU parallelism is internal."""
    return None


def get_workers():
    return 1


def _vec(v):
    t = dv.torch()
    if _is_torch(v) and v.is_cuda:
        return v.to(t.float64).contiguous()
    return dv.vec_to_device(np.asarray(v, dtype=np.float64), t.float64)


def _mat(x):
    return x if dv.is_colmajor_cuda(x) else dv.to_device_colmajor(np.asarray(x, dtype=np.float64))


def skew_rank2(a, alpha, x, y, beta=1, workers=None):
    """A := beta A + alpha (x y^T - y x^T), strictly-lower triangle only."""
    n = a.shape[0]
    if a.shape[1] != n or len(x) != n or len(y) != n:
        raise ValueError("dimension mismatch")
    instrument.record_call("skew_rank2")
    instrument.add_flops("level2", 2 * n * max(n - 1, 0))
    if n <= 1 or (alpha == 0 and beta == 1):
        return
    dv.require_cuda()
    ad, xd, yd = _mat(a), _vec(x), _vec(y)
    st = _capi.load().skl_skew_rank2_lower(n, float(alpha), xd.data_ptr(), yd.data_ptr(), float(beta),
                                           ad.data_ptr(), dv.ld_of(ad), dv.stream_ptr())
    _capi.check(st, "skew_rank2")
    if not _is_torch(a):
        a[...] = dv.to_host_colmajor(ad)


def gen_rank2(a, alpha, x, u, y, v, beta=1, workers=None, fused=True):
    """A := beta A + alpha (x u^T + y v^T) on a p x q rectangle (kernels2.py:134-163).
    ``fused`` / ``workers`` are accepted for compatibility: one pass on the GPU."""
    p, q = a.shape
    if len(x) != p or len(y) != p or len(u) != q or len(v) != q:
        raise ValueError("dimension mismatch")
    instrument.record_call("gen_rank2")
    instrument.add_flops("level2", 4 * p * q)
    if p == 0 or q == 0 or (alpha == 0 and beta == 1):
        return
    dv.require_cuda()
    ad = _mat(a)
    xd, ud, yd, vd = _vec(x), _vec(u), _vec(y), _vec(v)
    st = _capi.load().skl_gen_rank2(p, q, float(alpha), xd.data_ptr(), ud.data_ptr(), yd.data_ptr(), vd.data_ptr(),
                                    float(beta), ad.data_ptr(), dv.ld_of(ad), dv.stream_ptr())
    _capi.check(st, "gen_rank2")
    if not _is_torch(a):
        a[...] = dv.to_host_colmajor(ad)


@dataclass
class PanelView:
    """Trapezoidal update region [start, n) x [start, climit) of a lower-stored
    skew matrix (kernels2.py:274-293): a square skew part plus the rectangle below."""

    buf: object
    start: int
    climit: int

    @property
    def square(self):
        return self.buf[self.start:self.climit, self.start:self.climit]

    @property
    def rect(self):
        return self.buf[self.climit:, self.start:self.climit]


def trapezoid_rank2(buf, start, climit, alpha, x, y, workers=None, fused=True):
    """alpha (x y^T - y x^T) on rows/cols [start, n) of ``buf``, columns < climit
    (kernels2.py:296-312): skew_rank2 on the square + gen_rank2 on the rectangle."""
    n = buf.shape[0]
    climit = min(climit, n)
    nsq = climit - start
    if nsq <= 0:
        return
    view = PanelView(buf, start, climit)
    skew_rank2(view.square, alpha, x[:nsq], y[:nsq], 1, workers=workers)
    if climit < n:
        gen_rank2(view.rect, alpha, x[nsq:], y[:nsq], -y[nsq:], x[:nsq], 1, workers=workers, fused=fused)


def tridiag_matvec(tau, x):
    """z = T x (kernels2.py:166-175); tiny O(k) host helper used for checks."""
    tau = np.asarray(tau)
    x = np.asarray(x)
    k = len(x)
    if len(tau) != max(k - 1, 0):
        raise ValueError("dimension mismatch")
    z = np.zeros(k, dtype=np.result_type(tau.dtype, x.dtype) if k else x.dtype)
    if k > 1:
        z[1:] = tau * x[:-1]
        z[:-1] -= tau * x[1:]
    return z


def skew_tridiag_gemv(y, alpha, a, t: SkewTridiagonal, x, beta=1, workers=None, fused=True, tail_from=0):
    """y := beta y + alpha (A (T x))[tail_from:]."""
    p, k = a.shape
    rows = p - tail_from
    if t.m != k or len(x) != k or len(y) != rows or rows < 0:
        raise ValueError("dimension mismatch")
    instrument.record_call("skew_tridiag_gemv")
    instrument.add_flops("level2", 2 * rows * k + 4 * k)
    if rows == 0:
        return
    dv.require_cuda()
    ad, xd = _mat(a), _vec(x)
    yd = _vec(y)
    taud = _vec(t.tau)
    st = _capi.load().skl_skew_tridiag_gemv(p, k, float(alpha), ad.data_ptr(), dv.ld_of(ad),
                                            taud.data_ptr() if taud.numel() else None, xd.data_ptr(),
                                            float(beta), yd.data_ptr(), int(tail_from), dv.stream_ptr())
    _capi.check(st, "skew_tridiag_gemv")
    if _is_torch(y):
        y.copy_(yd)
    else:
        y[...] = yd.cpu().numpy()


def apply_row_pivots(block, p, forward=True, workers=None):
    """Permute the rows of ``block`` by P(p) (or its inverse) as one gather."""
    n = block.shape[0]
    q = block.shape[1] if block.ndim == 2 else 1
    pivots = p.pivots if hasattr(p, "pivots") else np.asarray(p)
    idx = np.arange(n)
    for k, off in enumerate(pivots):
        if off:
            j = k + int(off)
            if j >= n or off < 0:
                raise IndexError("pivot out of range")
            idx[k], idx[j] = idx[j], idx[k]
    if not forward:
        inv = np.empty_like(idx)
        inv[idx] = np.arange(n)
        idx = inv
    moved = idx != np.arange(n)
    instrument.record_call("apply_row_pivots")
    instrument.add_flops("pivot", int(np.count_nonzero(moved)) * q)
    if not moved.any() or q == 0:
        return
    touched = np.flatnonzero(moved)
    lo, hi = int(touched[0]), int(touched[-1]) + 1
    t = dv.require_cuda()
    host = block if block.ndim == 2 else np.asarray(block).reshape(n, 1)
    bd = _mat(host) if not _is_torch(block) else (block if block.dim() == 2 else block.view(n, 1))
    idxd = t.as_tensor(idx.astype(np.int64), device="cuda")
    lib = _capi.load()
    nbytes = lib.skl_apply_row_pivots_workspace_size(q, lo, hi)
    ws = dv.workspace(nbytes)
    st = lib.skl_apply_row_pivots(n, q, bd.data_ptr(), dv.ld_of(bd), idxd.data_ptr(), lo, hi, ws.data_ptr(),
                                  nbytes, dv.stream_ptr())
    _capi.check(st, "apply_row_pivots")
    if not _is_torch(block):
        out = dv.to_host_colmajor(bd)
        if block.ndim == 2:
            block[...] = out
        else:
            block[...] = out[:, 0]
