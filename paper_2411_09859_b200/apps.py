"""Pfaffian on top of the pivoted factorization (drop-in for reference ``apps.py``).

``pfaffian(x, b=None)`` keeps the reference convention (apps.py:12-30):
Pf = sign(P) prod_{i even} (-tau_i), Pf([[0, a], [-a, 0]]) = a, odd m -> 0,
m == 0 -> 1.  Like the reference it can overflow to inf for large m, so
``pfaffian_slog`` returns the overflow-free (sign, log|Pf|).
``pfaffian_batched`` is the batched B200 path (config 4): many independent
matrices in one launch, (sign, log|Pf|) per matrix.  ``solve`` (apps.py:76-100)
runs the permuted triangular / tridiagonal solves on the device.
"""

from __future__ import annotations

import math

import numpy as np

from .blocked import DEFAULT_BLOCK, ltlt_blk_piv
from .core import SkewMatrixLower


def slog_from_factors(tau, pivots, m):
    """(sign, log|Pf|) from tau and the pivot parity."""
    if m == 0:
        return 1.0, 0.0
    if m % 2:
        return 0.0, -math.inf
    even = np.asarray(tau[0:m - 1:2], dtype=np.float64)
    if np.any(even == 0):
        return 0.0, -math.inf
    sign = (-1.0 if np.count_nonzero(pivots) % 2 else 1.0) * float(np.prod(np.sign(-even)))
    return sign, float(np.sum(np.log(np.abs(even))))


def pfaffian(x: SkewMatrixLower, b=None):
    """Pfaffian via the pivoted factorization (apps.py:12-30)."""
    if not isinstance(x, SkewMatrixLower):
        x = SkewMatrixLower(x)
    m = x.m
    if m == 0:
        return 1.0
    if m % 2:
        return 0.0
    res = ltlt_blk_piv(x, b=b or min(DEFAULT_BLOCK, m))
    tau = res.t.tau.detach().cpu().numpy() if hasattr(res.t.tau, "detach") else np.asarray(res.t.tau)
    # the product runs in tau's dtype, like the reference's numpy scalars: a float32
    # input overflows to inf exactly where the reference's does (pfaffian_slog does not)
    val = res.p.sign()
    for i in range(0, m - 1, 2):
        val = val * (-tau[i])
    return val


def solve(x: SkewMatrixLower, b, block=None, tol_scale=10.0):
    """Solve X y = b through the pivoted factorization (apps.py:76-100):
    permute, unit-lower solve, pivoted skew-tridiagonal solve, transposed
    unit-lower solve, permute back -- all on the device (``skl_ltlt_solve``
    after ``skl_ltlt_blk_piv``).  ``b`` may hold several right-hand sides as
    columns.  Raises SingularT for a numerically singular X (every odd m)."""
    from . import _capi
    from . import device as dv
    from .blocked import _device_input, ltlt_blk_piv_device
    from .core import SingularT

    if not isinstance(x, SkewMatrixLower):
        x = SkewMatrixLower(x)
    m = x.m
    t = dv.require_cuda()
    if not dv.is_colmajor_cuda(x.data) and np.asarray(x.data).dtype not in (np.float64, np.float32):
        x = SkewMatrixLower(np.asarray(x.data, dtype=np.float64))
    bd_in = b if dv._is_cuda_tensor(b) else None
    bh = None if bd_in is not None else np.asarray(b, dtype=float)
    one_d = (bd_in.dim() if bd_in is not None else bh.ndim) == 1
    if bd_in is not None:
        rhs = bd_in.reshape(m, -1) if one_d else bd_in
        if rhs.shape[0] != m:
            raise ValueError("dimension mismatch")
        bdev = dv.empty_colmajor(m, rhs.shape[1], t.float64)
        bdev.copy_(rhs)
    else:
        rhs = bh.reshape(m, -1) if one_d else bh
        if rhs.shape[0] != m:
            raise ValueError("dimension mismatch")
        bdev = dv.to_device_colmajor(rhs)
    nrhs = int(bdev.shape[1])
    xd, _, _ = _device_input(x, "solve")
    L, tau, piv = ltlt_blk_piv_device(xd, b=block or min(DEFAULT_BLOCK, m), fused="var1")
    if nrhs == 0:
        out = bdev
    else:
        lib = _capi.load()
        nbytes = lib.skl_ltlt_solve_workspace_size(m, nrhs)
        ws = dv.workspace(nbytes)
        info = t.zeros(1, dtype=t.int32, device="cuda")
        st = lib.skl_ltlt_solve(m, nrhs, L.data_ptr(), dv.ld_of(L), tau.data_ptr() if m > 1 else None,
                                piv.data_ptr(), bdev.data_ptr(), dv.ld_of(bdev), float(tol_scale), info.data_ptr(),
                                ws.data_ptr(), nbytes, dv.stream_ptr())
        _capi.check(st, "solve")
        code = int(info.item())
        if code:
            raise SingularT(f"tridiagonal pivot at row {code - 1}")
        out = bdev
    if bd_in is not None:
        return out.reshape(-1) if one_d else out
    res = dv.to_host_colmajor(out)
    return res.ravel() if one_d else res


def pfaffian_slog(x: SkewMatrixLower, b=None):
    """Overflow-free Pfaffian: (sign, log|Pf|)."""
    if not isinstance(x, SkewMatrixLower):
        x = SkewMatrixLower(x)
    m = x.m
    if m == 0 or m % 2:
        return slog_from_factors(np.zeros(0), np.zeros(0), m)
    res = ltlt_blk_piv(x, b=b or min(DEFAULT_BLOCK, m))
    tau = res.t.tau.detach().cpu().numpy() if hasattr(res.t.tau, "detach") else res.t.tau
    return slog_from_factors(tau, res.p.pivots, m)


def _batched_device(xd, dtype_code, stream=None):
    from . import _capi
    from . import device as dv
    t = dv.require_cuda()
    batch, n, _ = xd.shape
    L = t.empty_like(xd)
    tau = t.empty((batch, max(n - 1, 1)), dtype=xd.dtype, device=xd.device)
    piv = t.empty((batch, n), dtype=t.int64, device=xd.device)
    sign = t.empty(batch, dtype=t.float64, device=xd.device)
    logabs = t.empty(batch, dtype=t.float64, device=xd.device)
    st = _capi.load().skl_ltlt_batched_piv(batch, n, dtype_code, xd.data_ptr(), n, n * n, L.data_ptr(), n, n * n,
                                          tau.data_ptr(), piv.data_ptr(), sign.data_ptr(), logabs.data_ptr(),
                                          dv.stream_ptr(stream))
    _capi.check(st, "ltlt_batched_piv")
    return L, tau[:, : n - 1], piv, sign, logabs


def ltlt_batched_piv_device(xd, stream=None):
    """Device entry for many independent matrices.

    ``xd``: CUDA tensor (batch, n, n), float64 or float32, with xd[b, j, i] =
    X_b[i, j] (each matrix column-major, ld = n).  Returns device tensors
    (L, tau, piv, sign, logabs) without synchronising; L has the layout of xd.
    """
    from . import _capi
    from . import device as dv
    t = dv.require_cuda()
    if xd.dim() != 3 or xd.shape[1] != xd.shape[2] or not xd.is_contiguous():
        raise ValueError("xd must be a contiguous (batch, n, n) CUDA tensor")
    if xd.dtype == t.float64:
        code = _capi.SKL_F64
    elif xd.dtype == t.float32:
        code = _capi.SKL_F32
    else:
        raise TypeError("batched factorization supports float64 and float32")
    return _batched_device(xd, code, stream)


def pfaffian_batched(xs):
    """(sign, log|Pf|) of every matrix in ``xs`` ((batch, m, m) NumPy array of
    lower-stored skew matrices, xs[b] indexed [row, col]); one launch.  The
    per-matrix factorization is that of ``pfaffian`` (apps.py:12-30)."""
    from . import device as dv
    t = dv.require_cuda()
    xs = np.asarray(xs)
    if xs.ndim != 3 or xs.shape[1] != xs.shape[2]:
        raise ValueError("xs must be (batch, m, m)")
    if xs.dtype not in (np.float64, np.float32):
        raise TypeError("float64 or float32 required")
    m = xs.shape[1]
    if m == 0:
        return np.ones(xs.shape[0]), np.zeros(xs.shape[0])
    xd = t.from_numpy(np.ascontiguousarray(np.swapaxes(xs, 1, 2))).to("cuda")
    _L, _tau, _piv, sign, logabs = ltlt_batched_piv_device(xd)
    return sign.cpu().numpy(), logabs.cpu().numpy()


def ltlt_batched_piv(xs):
    """Batched drop-in: per-matrix (L buffer, tau, pivots) as NumPy arrays plus
    (sign, log|Pf|); each matrix's factors are those of ltlt_blk_piv(x_b, b=m)."""
    from . import device as dv
    t = dv.require_cuda()
    xs = np.asarray(xs)
    xd = t.from_numpy(np.ascontiguousarray(np.swapaxes(xs, 1, 2))).to("cuda")
    L, tau, piv, sign, logabs = ltlt_batched_piv_device(xd)
    Lh = np.swapaxes(L.cpu().numpy(), 1, 2)
    return Lh, tau.cpu().numpy(), piv.cpu().numpy(), sign.cpu().numpy(), logabs.cpu().numpy()
