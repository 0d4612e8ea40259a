"""Level-3 sandwiched kernels (drop-in for reference ``kernels3.py``).

Same signatures and in-place semantics as the reference:
``skew_rank2k`` (kernels3.py:305-351), ``skew_tridiag_rankk``
(kernels3.py:151-209), ``skew_tridiag_gemm`` (kernels3.py:239-302),
``form_w`` (kernels3.py:354-364).  Operands may be
NumPy arrays (copied to the GPU and the output view written back) or
column-major torch CUDA tensors (updated in place on the device).  Every
call is recorded in the active ``instrument`` trace / counter with the
reference's flop rule.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _capi
from . import device as dv
from . import instrument
from .core import SkewTridiagonal, SSplitting, _is_torch


@dataclass(frozen=True)
class BlockConfig:
    """CPU cache-blocking constants (kernels3.py:28-41), kept for compatibility:
    the GPU tiles are fixed by the kernels (128x128 DMMA tiles), so these only
    round-trip through set_block_config / get_block_config."""

    m_c: int = 128
    k_c: int = 256
    n_c: int = 256
    m_r: int = 8
    n_r: int = 4


_config = BlockConfig()


def set_block_config(**kw):
    global _config
    _config = replace(_config, **kw)
    return _config


def get_block_config() -> BlockConfig:
    return _config


last_keff = 0


def _check_alias(c, a, name):
    if a is None:
        return
    if _is_torch(c) or _is_torch(a):
        return  # checked by the C ABI (SKL_ALIAS)
    if np.shares_memory(c, a):
        raise ValueError(f"output aliases operand {name}")


def _dev(x):
    return x if dv.is_colmajor_cuda(x) else dv.to_device_colmajor(np.asarray(x, dtype=np.float64))


def _writeback(c, cd):
    if not _is_torch(c):
        c[...] = dv.to_host_colmajor(cd)


def skew_rank2k(c, alpha, a, b, beta=1, *, workers=None, skip_zero_columns=True):
    """C_lower := beta C + alpha (A B^T - B A^T), zero columns skipped."""
    global last_keff
    n, k = a.shape
    if tuple(b.shape) != (n, k) or c.shape[0] != n or c.shape[1] != n:
        raise ValueError("dimension mismatch")
    _check_alias(c, a, "a")
    _check_alias(c, b, "b")
    instrument.record_call("skew_rank2k")
    t = dv.require_cuda()
    cd, ad, bd = _dev(c), _dev(a), _dev(b)
    lib = _capi.load()
    nbytes = lib.skl_skr2k_workspace_size(n, k)
    ws = dv.workspace(nbytes)
    keff = t.zeros(1, dtype=t.int32, device="cuda")
    st = lib.skl_skr2k_lower(n, k, float(alpha), ad.data_ptr(), dv.ld_of(ad), bd.data_ptr(), dv.ld_of(bd),
                             float(beta), cd.data_ptr(), dv.ld_of(cd), 1 if skip_zero_columns else 0,
                             ws.data_ptr(), nbytes, keff.data_ptr(), dv.stream_ptr())
    _capi.check(st, "skew_rank2k")
    _writeback(c, cd)
    last_keff = int(keff.item())
    instrument.add_flops("level3", 4 * last_keff * (n * (n - 1) // 2))
    return None


def skew_tridiag_rankk(c, alpha, a, t: SkewTridiagonal, beta=1, *, fused=True, workers=None):
    """C_lower := beta C + alpha A T A^T (T skew tridiagonal)."""
    n, k = a.shape
    if c.shape[0] != n or c.shape[1] != n or t.m != k:
        raise ValueError("dimension mismatch")
    _check_alias(c, a, "a")
    instrument.record_call("skew_tridiag_rankk")
    instrument.add_flops("level3", 2 * k * (n * (n - 1) // 2) + 4 * k * n)
    tt = dv.require_cuda()
    cd, ad = _dev(c), _dev(a)
    tau = t.tau if _is_torch(t.tau) else dv.vec_to_device(np.asarray(t.tau, dtype=np.float64), tt.float64)
    lib = _capi.load()
    nbytes = lib.skl_sktri_rankk_workspace_size(n, k)
    ws = dv.workspace(nbytes)
    st = lib.skl_sktri_rankk_lower(n, k, float(alpha), ad.data_ptr(), dv.ld_of(ad),
                                   tau.data_ptr() if tau.numel() else None, float(beta), cd.data_ptr(),
                                   dv.ld_of(cd), ws.data_ptr(), nbytes, dv.stream_ptr())
    _capi.check(st, "skew_tridiag_rankk")
    _writeback(c, cd)
    return None


def skew_tridiag_gemm(c, alpha, a, t: SkewTridiagonal, b, beta=1, *, tril=False, fused=True, workers=None):
    """C := beta*C + alpha * A (T B) on a general p x q block (kernels3.py:239-302);
    ``tril=True`` writes only the entries with row > col.  ``fused`` and
    ``workers`` are accepted for signature compatibility: T B is always formed
    inside the operand pack (the fused form) and the CUDA grid replaces the pool."""
    p, k = a.shape
    kb, q = b.shape
    if kb != k or tuple(c.shape) != (p, q) or t.m != k:
        raise ValueError("dimension mismatch")
    _check_alias(c, a, "a")
    _check_alias(c, b, "b")
    instrument.record_call("skew_tridiag_gemm")
    written = (min(p, q) * (min(p, q) - 1) // 2 + max(p - q, 0) * q) if tril else p * q
    instrument.add_flops("level3", 2 * k * written + 4 * k * q)
    tt = dv.require_cuda()
    cd, ad, bd = _dev(c), _dev(a), _dev(b)
    tau = t.tau if _is_torch(t.tau) else dv.vec_to_device(np.asarray(t.tau, dtype=np.float64), tt.float64)
    lib = _capi.load()
    nbytes = lib.skl_skew_tridiag_gemm_workspace_size(p, q, k)
    ws = dv.workspace(nbytes)
    st = lib.skl_skew_tridiag_gemm(p, q, k, float(alpha), ad.data_ptr() if ad.numel() else None, dv.ld_of(ad),
                                   tau.data_ptr() if tau.numel() else None, bd.data_ptr() if bd.numel() else None,
                                   dv.ld_of(bd), float(beta), cd.data_ptr(), dv.ld_of(cd), 1 if tril else 0,
                                   ws.data_ptr(), nbytes, dv.stream_ptr())
    _capi.check(st, "skew_tridiag_gemm")
    _writeback(c, cd)
    return None


def form_w(a, s):
    """W = A S (every other column zero, starting with the first)."""
    n, kdim = a.shape
    if s.m != kdim:
        raise ValueError("dimension mismatch")
    instrument.record_call("form_w")
    instrument.add_flops("level3", 2 * n * len(s.entries))
    tt = dv.require_cuda()
    # recover tau from the splitting (core.py:153-169 pattern)
    tau = np.zeros(max(kdim - 1, 0), dtype=np.float64)
    for i, j, v in s.entries:
        if j == i - 1:
            tau[i - 1] = v
        elif j == i + 1:
            tau[i] = -v
    ad = _dev(a)
    taud = dv.vec_to_device(tau, tt.float64)
    wd = dv.empty_colmajor(n, kdim, tt.float64)
    st = _capi.load().skl_form_w(n, kdim, ad.data_ptr(), dv.ld_of(ad), taud.data_ptr() if tau.size else None,
                                 wd.data_ptr(), max(n, 1), dv.stream_ptr())
    _capi.check(st, "form_w")
    return wd if _is_torch(a) else dv.to_host_colmajor(wd)


def form_w_device(a, tau):
    """Device form of W = A S straight from tau (no SSplitting object)."""
    tt = dv.require_cuda()
    n, kdim = a.shape
    wd = dv.empty_colmajor(n, kdim, tt.float64)
    st = _capi.load().skl_form_w(n, kdim, a.data_ptr(), dv.ld_of(a), tau.data_ptr() if tau.numel() else None,
                                 wd.data_ptr(), max(n, 1), dv.stream_ptr())
    _capi.check(st, "form_w")
    return wd


__all__ = ["skew_rank2k", "skew_tridiag_rankk", "skew_tridiag_gemm", "form_w", "form_w_device", "SSplitting"]
