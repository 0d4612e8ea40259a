"""Unblocked drivers (drop-in for reference ``unblocked.py``).

* ``ltlt_unb_twostep(x, pivot)`` (unblocked.py:229-240): the Wimmer two-step
  driver, entered through ``skl_ltlt_unb_twostep``.  From n = 128 up it runs
  the blocked GPU driver (lean cluster panel ``panel_push_kernel`` + DMMA
  trailing update), which computes the same L, T and pivots and is faster
  (config 1, n=512: 0.83 ms vs 2.9 ms for the fused right-looking kernel);
  below n = 128 the fused single-cluster two-step kernel (``twostep.cu``:
  eliminations, interchanges, fold and skew rank-2 of each pair in one
  launch) serves it.  DESIGN.md §1 records the decision.
* ``ltlt_unb_ll(x, pivot, first_column)`` (unblocked.py:205-226): one
  left-looking panel over the whole matrix = the blocked driver with
  b >= m - 1 (blocked.py:341-362), served by the same panel kernel, pivoted
  or not; ``first_column`` is applied up front on the device.
* ``ltlt_unb_rl(x, pivot)`` (unblocked.py:192-202): same factors through the
  same GPU driver, right-looking flop tally.
* ``ltlt_unb_panel(x, width, variant, pivot, first_column)``
  (unblocked.py:243-275): ``skl_ltlt_unb_panel`` (first ``width`` columns).
"""

from __future__ import annotations

import numpy as np

from . import _capi
from . import device as dv
from .blocked import (PANEL_VARIANTS, FactorizationResult, _device_input, _narrow, ltlt_blk_device,
                      ltlt_blk_piv_device)
from .core import (InvalidVariant, PermutationVector, SkewMatrixLower, SkewTridiagonal, UnitLowerFactor,
                   ZeroPivot, _is_torch)
from .instrument import flops_unb_ll, flops_unb_panel, flops_unb_rl, flops_unb_twostep


def _prep(x):
    """-> (x, float64 column-major CUDA input, on_device, dt); float32 input is
    factored in float64 and rounded back (blocked._device_input / _narrow)."""
    if not isinstance(x, SkewMatrixLower):
        x = SkewMatrixLower(x)
    if x.m < 1:
        raise ValueError("m >= 1 required")
    xd, on_device, dt = _device_input(x)
    return x, xd, on_device, dt


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
        from .blocked import _check_out_device
        _check_out_device(xd, m, L, tau, piv)
    info = t.zeros(1, dtype=t.int32, device="cuda")
    lib = _capi.load()
    nbytes = lib.skl_ltlt_unb_twostep_workspace_size(m)
    ws = dv.workspace(nbytes, stream=stream)
    st = lib.skl_ltlt_unb_twostep(m, 1 if pivot else 0, xd.data_ptr(), dv.ld_of(xd), L.data_ptr(), dv.ld_of(L),
                                  tau.data_ptr() if m > 1 else None, piv.data_ptr(), info.data_ptr(),
                                  ws.data_ptr(), nbytes, dv.stream_ptr(stream))
    _capi.check(st, "ltlt_unb_twostep")
    return L, tau, piv, info


def ltlt_unb_twostep(x: SkewMatrixLower, pivot=False) -> FactorizationResult:
    """Two-step right-looking factorization (unblocked.py:229-240)."""
    x, xd, on_device, dt = _prep(x)
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
    return _narrow(FactorizationResult(UnitLowerFactor(l_out, "ones"), SkewTridiagonal(t_out),
                                       PermutationVector(piv_h, m), flops), dt)


def _apply_first_column_device(xd, first_column):
    """Non-default first L column (unblocked.py:182-189) on a device copy of X:
    X[1:, 1:] += f x0^T - x0 f^T with x0 = X[1:, 0], through skl_skew_rank2_lower."""
    t = dv.require_cuda()
    m = xd.shape[0]
    fcvec = np.asarray(first_column)
    if fcvec.shape != (m - 1,):
        raise ValueError("first_column must have length m - 1")
    fcvec = fcvec.astype(np.float64, copy=True)
    work = dv.empty_colmajor(m, m, t.float64)
    work.copy_(xd)
    if m > 2:
        fd = t.as_tensor(fcvec, device="cuda")
        x0 = work[1:, 0].clone()
        sub = work[1:, 1:]
        st = _capi.load().skl_skew_rank2_lower(m - 1, 1.0, fd.data_ptr(), x0.data_ptr(), 1.0, sub.data_ptr(),
                                               dv.ld_of(sub), dv.stream_ptr())
        _capi.check(st, "first_column")
    return work, fcvec


def _unpivoted_full(xd, m):
    """Unpivoted factorization of all columns: one reference panel spanning the
    matrix (unblocked.py:205-226 / 192-202), run by skl_ltlt_blk (pivot = 0)."""
    L, tau, _piv, info = ltlt_blk_device(xd, b=max(m, 1), fused="var2a", pivot=False)
    code = int(info.item())
    if code:
        raise ZeroPivot(code - 1)
    return L, tau


def _result(L, tau_h, tau, piv_h, m, fc, on_device, first_column=None, dt=None):
    l_out = L if on_device else dv.to_host_colmajor(L)
    t_out = tau if on_device else tau_h
    return _narrow(FactorizationResult(UnitLowerFactor(l_out, "ones", first_column), SkewTridiagonal(t_out),
                                       PermutationVector(piv_h, m), fc), dt)


def ltlt_unb_ll(x: SkewMatrixLower, pivot=False, first_column=None) -> FactorizationResult:
    """Left-looking (modified Aasen) factorization (unblocked.py:205-226).

    One left-looking panel spanning the matrix is exactly the blocked driver
    with b >= m - 1, so the GPU runs skl_ltlt_blk (pivoted or not; the GPU
    splits the panel to fit the cluster).  ``first_column`` (unpivoted only)
    applies its transform up front on the device (skl_skew_rank2_lower).
    """
    if pivot and first_column is not None:
        raise ValueError("first_column is only supported without pivoting")
    x, xd, on_device, dt = _prep(x)
    m = x.m
    fcvec = None
    if pivot:
        L, tau, piv = ltlt_blk_piv_device(xd, b=max(m, 1), fused="var1")
        piv_h = piv.cpu().numpy()
    else:
        if first_column is not None:
            xd, fcvec = _apply_first_column_device(xd, first_column)
        L, tau = _unpivoted_full(xd, m)
        piv_h = np.zeros(0, dtype=np.int64)
    tau_h = tau.cpu().numpy()
    fc = flops_unb_ll(m, tau_h, piv_h if pivot else None, first_column=fcvec is not None)
    return _result(L, tau_h, tau, piv_h, m, fc, on_device, fcvec, dt)


def ltlt_unb_rl(x: SkewMatrixLower, pivot=False) -> FactorizationResult:
    """Right-looking (modified Parlett-Reid) factorization (unblocked.py:192-202).

    Same factors and pivots as the left-looking order in exact arithmetic; the
    GPU computes them with the blocked left-looking-panel driver and reports
    the right-looking tally (instrument.flops_unb_rl).
    """
    x, xd, on_device, dt = _prep(x)
    m = x.m
    if pivot:
        L, tau, piv = ltlt_blk_piv_device(xd, b=max(m, 1), fused="var1")
        piv_h = piv.cpu().numpy()
    else:
        L, tau = _unpivoted_full(xd, m)
        piv_h = np.zeros(0, dtype=np.int64)
    tau_h = tau.cpu().numpy()
    fc = flops_unb_rl(m, tau_h, piv_h if pivot else None)
    return _result(L, tau_h, tau, piv_h, m, fc, on_device, dt=dt)


def ltlt_unb_panel(x: SkewMatrixLower, panel_width, variant="ll", pivot=False,
                   first_column=None) -> FactorizationResult:
    """Factor only the first ``panel_width`` columns (unblocked.py:243-275):
    skl_ltlt_unb_panel.  Only L columns [0, width) are returned (zeros
    elsewhere, like the reference's lbuf), with tau and pivots[:width+1]."""
    if variant not in PANEL_VARIANTS:
        raise InvalidVariant(f"unknown panel variant {variant!r}")
    if pivot and variant != "ll":
        raise InvalidVariant("a pivoted panel factorization must be left-looking")
    if pivot and first_column is not None:
        raise ValueError("first_column is only supported without pivoting")
    x, xd, on_device, dt = _prep(x)
    m = x.m
    t = dv.require_cuda()
    fcvec = None
    if first_column is not None:
        xd, fcvec = _apply_first_column_device(xd, first_column)
    nelim = min(int(panel_width), m - 1)
    L = dv.empty_colmajor(m, m, t.float64)
    tau = t.zeros(max(m - 1, 0), dtype=t.float64, device="cuda")
    piv = t.zeros(m, dtype=t.int64, device="cuda")
    info = t.zeros(1, dtype=t.int32, device="cuda")
    if nelim >= 1:
        lib = _capi.load()
        nbytes = lib.skl_ltlt_unb_panel_workspace_size(m, nelim)
        if nbytes == 0:
            raise InvalidVariant("configuration not supported by the GPU panel kernel")
        ws = dv.workspace(nbytes)
        st = lib.skl_ltlt_unb_panel(m, nelim, 1 if pivot else 0, xd.data_ptr(), dv.ld_of(xd), L.data_ptr(),
                                    dv.ld_of(L), tau.data_ptr(), piv.data_ptr() if pivot else None,
                                    info.data_ptr(), ws.data_ptr(), nbytes, dv.stream_ptr())
        _capi.check(st, "ltlt_unb_panel")
        code = int(info.item())
        if code:
            raise ZeroPivot(code - 1)
    L[:, max(nelim, 0):] = 0.0
    tau_h = tau.cpu().numpy()
    piv_h = piv.cpu().numpy()[:nelim + 1] if pivot else np.zeros(0, dtype=np.int64)
    pfull = piv.cpu().numpy() if pivot else None
    fc = flops_unb_panel(m, int(panel_width), variant, tau_h, pfull, first_column=fcvec is not None)
    return _result(L, tau_h, tau, piv_h, m, fc, on_device, fcvec, dt)


__all__ = ["ltlt_unb_twostep", "ltlt_unb_twostep_device", "ltlt_unb_ll", "ltlt_unb_rl", "ltlt_unb_panel", "_is_torch"]
