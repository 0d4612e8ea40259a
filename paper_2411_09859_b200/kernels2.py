"""Level-2 kernels (drop-in for reference ``kernels2.py``).

``skew_rank2`` (kernels2.py:93-131), ``skew_tridiag_gemv`` (kernels2.py:178-229)
and ``apply_row_pivots`` (kernels2.py:232-271) with the reference's
signatures and in-place semantics; the arithmetic runs in the CUDA library.
NumPy operands are staged to the GPU and the output view written back;
column-major torch CUDA tensors are updated in place.
"""

from __future__ import annotations

import numpy as np

from . import _capi
from . import device as dv
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
    if n <= 1 or (alpha == 0 and beta == 1):
        return
    dv.require_cuda()
    ad, xd, yd = _mat(a), _vec(x), _vec(y)
    st = _capi.load().skl_skew_rank2_lower(n, float(alpha), xd.data_ptr(), yd.data_ptr(), float(beta),
                                           ad.data_ptr(), dv.ld_of(ad), dv.stream_ptr())
    _capi.check(st, "skew_rank2")
    if not _is_torch(a):
        a[...] = dv.to_host_colmajor(ad)


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
