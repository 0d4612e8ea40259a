"""Unblocked drivers (drop-in for reference ``unblocked.py``).

* ``ltlt_unb_twostep(x, pivot)`` (unblocked.py:229-240): the Wimmer two-step
  driver, run by the fused single-cluster CUDA kernel ``skl_ltlt_unb_twostep``
  (eliminations, symmetric interchanges, fold and skew rank-2 updates of
  each pair in one launch).
* ``ltlt_unb_ll(x, pivot)`` (unblocked.py:205-226): left-looking; with
  pivoting it is the pivoted blocked driver with one panel spanning the
  whole matrix (blocked.py:341-362 with b >= m - 1 is exactly _panel_ll over
  all columns), served by the same panel kernel.
"""

from __future__ import annotations

import numpy as np

from . import _capi
from . import device as dv
from .blocked import FactorizationResult, ltlt_blk_piv_device
from .core import (PermutationVector, SkewMatrixLower, SkewTridiagonal, UnitLowerFactor, ZeroPivot,
                   _is_torch)
from .instrument import FlopCounter, flops_unb_twostep


def _prep(x):
    if not isinstance(x, SkewMatrixLower):
        x = SkewMatrixLower(x)
    if x.m < 1:
        raise ValueError("m >= 1 required")
    if dv.is_colmajor_cuda(x.data):
        if x.data.dtype != dv.torch().float64:
            raise TypeError("the GPU path computes in float64")
        return x, x.data, True
    host = np.asarray(x.data)
    if host.dtype == object:
        raise TypeError("exact (object) dtypes are served by the reference, not the GPU path")
    if host.dtype != np.float64:
        raise TypeError("the GPU path computes in float64")
    return x, dv.to_device_colmajor(host), False


def ltlt_unb_twostep_device(xd, pivot=False, out=None, stream=None):
    """Device entry: returns (L, tau, piv, info) CUDA tensors without syncing."""
    t = dv.require_cuda()
    m = xd.shape[0]
    if out is None:
        L = dv.empty_colmajor(m, m, t.float64)
        tau = t.empty(max(m - 1, 0), dtype=t.float64, device="cuda")
        piv = t.zeros(m, dtype=t.int64, device="cuda")
    else:
        L, tau, piv = out
    info = t.zeros(1, dtype=t.int32, device="cuda")
    lib = _capi.load()
    nbytes = lib.skl_ltlt_unb_twostep_workspace_size(m)
    ws = dv.workspace(nbytes)
    st = lib.skl_ltlt_unb_twostep(m, 1 if pivot else 0, xd.data_ptr(), dv.ld_of(xd), L.data_ptr(), dv.ld_of(L),
                                  tau.data_ptr() if m > 1 else None, piv.data_ptr(), info.data_ptr(),
                                  ws.data_ptr(), nbytes, dv.stream_ptr(stream))
    _capi.check(st, "ltlt_unb_twostep")
    return L, tau, piv, info


def ltlt_unb_twostep(x: SkewMatrixLower, pivot=False) -> FactorizationResult:
    """Two-step right-looking factorization (unblocked.py:229-240)."""
    x, xd, on_device = _prep(x)
    m = x.m
    L, tau, piv, info = ltlt_unb_twostep_device(xd, pivot)
    code = int(info.item())
    if code:
        raise ZeroPivot(code - 1)
    tau_h = tau.cpu().numpy()
    piv_h = piv.cpu().numpy() if pivot else np.zeros(0, dtype=np.int64)
    flops = flops_unb_twostep(m, piv.cpu().numpy(), tau_h, pivot=pivot)
    l_out = L if on_device else dv.to_host_colmajor(L)
    t_out = tau if on_device else tau_h
    return FactorizationResult(UnitLowerFactor(l_out, "ones"), SkewTridiagonal(t_out), PermutationVector(piv_h, m),
                               flops)


def ltlt_unb_ll(x: SkewMatrixLower, pivot=False, first_column=None) -> FactorizationResult:
    """Left-looking (modified Aasen) factorization (unblocked.py:205-226).

    The pivoted form runs the panel kernel over all columns at once.  The
    unpivoted form is outside the GPU hot path and raises.
    """
    if pivot and first_column is not None:
        raise ValueError("first_column is only supported without pivoting")
    if not pivot or first_column is not None:
        raise NotImplementedError("unpivoted left-looking driver is not on the B200 hot path")
    x, xd, on_device = _prep(x)
    m = x.m
    L, tau, piv = ltlt_blk_piv_device(xd, b=max(m, 1), fused="var1")
    tau_h = tau.cpu().numpy()
    piv_h = piv.cpu().numpy()
    fc = FlopCounter()
    # unblocked accounting (no panel scope): eliminations + gemvs + swaps
    for g in range(m - 1):
        if g >= 2:
            fc.level2 += 2 * (m - g - 1) * g + 4 * g
        off = int(piv_h[g + 1])
        if off:
            a = g + 1
            b = a + off
            fc.pivot += 2 * (a + (m - b - 1) + (b - a - 1)) + 1
        if tau_h[g] != 0:
            fc.level2 += max(m - g - 2, 0)
    l_out = L if on_device else dv.to_host_colmajor(L)
    t_out = tau if on_device else tau_h
    return FactorizationResult(UnitLowerFactor(l_out, "ones"), SkewTridiagonal(t_out), PermutationVector(piv_h, m), fc)


__all__ = ["ltlt_unb_twostep", "ltlt_unb_twostep_device", "ltlt_unb_ll", "_is_torch"]
