"""Pivoted blocked LTL^T on the B200 (drop-in for reference ``blocked.py``).

``ltlt_blk_piv`` keeps the reference signature (blocked.py:303-363) and
returns the same ``FactorizationResult`` (L in the "ones" working layout,
tau, relative pivot offsets, flop tally).  The computation is entirely the
CUDA library's ``skl_ltlt_blk_piv``: pivoted left-looking panel kernel,
packed operand formation and the lower-triangular DMMA trailing GEMM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _capi
from . import device as dv
from .core import (InvalidVariant, PermutationVector, PivotUnsupported, SkewMatrixLower, SkewTridiagonal,
                   UnitLowerFactor, ZeroPivot, _is_torch)
from .instrument import FlopCounter, flops_blk_piv, flops_blk_unpivoted

DEFAULT_BLOCK = 256                               # blocked.py:34
PIVOTED_FUSED = ("var1", "var2a", "var2b")       # blocked.py:35
PANEL_VARIANTS = ("ll", "rl", "twostep")         # unblocked.py VARIANTS


@dataclass
class Features:
    """Accepted for signature compatibility (blocked.py:38-62); GPU tiling is
    internal, so the CPU optimisation-ladder toggles have no effect."""

    fused_l2: bool = True
    parallel_l2: bool = False
    external_t: bool = True
    fused_l3: bool = True

    @property
    def l2_workers(self):
        return None if self.parallel_l2 else 1


#: optimisation ladder (blocked.py:67-75): cumulative CPU feature steps, accepted
#: by every driver; the GPU kernels are the same at every step
LADDER = {
    "step0": Features(fused_l2=False, parallel_l2=False, external_t=False, fused_l3=False),
    "step1": Features(fused_l2=True, parallel_l2=False, external_t=False, fused_l3=False),
    "step2": Features(fused_l2=True, parallel_l2=True, external_t=False, fused_l3=False),
    "step3": Features(fused_l2=True, parallel_l2=True, external_t=True, fused_l3=False),
    "step4": Features(fused_l2=True, parallel_l2=True, external_t=True, fused_l3=True),
    "step5": Features(fused_l2=True, parallel_l2=True, external_t=True, fused_l3=True),
}
LADDER_VARIANT = {name: ("blk-var2b" if name == "step5" else "blk-var1") for name in LADDER}


@dataclass
class FactorizationResult:
    """L, T, pivots and the flop tally of one factorization (unblocked.py:30-40)."""

    l: UnitLowerFactor
    t: SkewTridiagonal
    p: PermutationVector
    flops: FlopCounter


def _device_input(x, who="the GPU path"):
    """SkewMatrixLower data -> (column-major float64 CUDA tensor, on_device, dt).

    float32 input (the reference runs it end to end, SURVEY 8b "Dtypes") is
    factored in float64 on the device and the factors are rounded back to float32
    (``dt``; None for float64) by ``_narrow``: L and tau keep the input dtype like
    the reference's, computed with fp64 arithmetic.  Pivots can then differ from
    the reference's float32 run only at float32-rounding near-ties."""
    if dv.is_colmajor_cuda(x.data):
        t = dv.torch()
        if x.data.dtype == t.float64:
            return x.data, True, None
        if x.data.dtype == t.float32:
            xd = dv.empty_colmajor(x.m, x.m, t.float64)
            xd.copy_(x.data)
            return xd, True, t.float32
        raise TypeError(f"{who} serves float64 and float32")
    host = np.asarray(x.data)
    if host.dtype == object:
        raise TypeError("exact (object) dtypes are served by the reference, not the GPU path")
    if host.dtype == np.float64:
        return dv.to_device_colmajor(host), False, None
    if host.dtype == np.float32:
        return dv.to_device_colmajor(host.astype(np.float64)), False, np.float32
    raise TypeError(f"{who} serves float64 and float32")


def _narrow(res, dt):
    """Round a FactorizationResult's L and tau to the input dtype (float32 input)."""
    if dt is None:
        return res
    L, tau = res.l.data, res.t.tau
    if _is_torch(L):
        L, tau = L.to(dt), tau.to(dt)
    else:
        L, tau = np.asarray(L, dtype=dt, order="F"), np.asarray(tau, dtype=dt)
    return FactorizationResult(UnitLowerFactor(L, res.l.mode, res.l.first_column), SkewTridiagonal(tau), res.p,
                               res.flops)


def _check_block(b):
    if b < 1:
        raise ValueError("block size must be >= 1")


def gpu_panel_plan(m, b=DEFAULT_BLOCK, fused="var1"):
    """The GPU panel schedule of ltlt_blk_piv for (m, b, fused): one dict per panel
    (first column r, columns eliminated, kind "cluster"/"grid", CTAs, cluster size).
    The GPU panel width can be narrower than b when the panel block would not fit
    on-chip; pivots, L and T are invariant to it."""
    import ctypes as C
    if fused not in PIVOTED_FUSED:
        raise InvalidVariant(f"fused must be one of {PIVOTED_FUSED}, got {fused!r}")
    dv.require_cuda()
    lib = _capi.load()
    cap = max(int(m), 1)
    bufs = [(C.c_int * cap)() for _ in range(5)]
    cnt = lib.skl_ltlt_blk_piv_plan(int(m), int(b), _capi.VARIANT_CODES[fused], *bufs, cap)
    if cnt < 0:
        raise InvalidVariant("configuration not supported by the GPU panel kernel")
    r, ne, kind, ctas, cs = (list(v)[:cnt] for v in bufs)
    return [{"r": r[i], "nelim": ne[i], "kind": "cluster" if kind[i] else "grid", "ctas": ctas[i],
             "cluster_size": cs[i]} for i in range(cnt)]


def _check_out_device(x, m, L, tau, piv):
    """out=(L, tau, piv) buffers cross the C ABI as raw pointers: check them here."""
    t = dv.torch()
    if not (dv.is_colmajor_cuda(L) and L.dtype == t.float64 and tuple(L.shape) == (m, m) and L.device == x.device):
        raise ValueError("out L must be a column-major float64 (m, m) CUDA tensor on x's device")
    for name, v, dt, size in (("tau", tau, t.float64, m - 1), ("piv", piv, t.int64, m)):
        if v is None and name == "piv":
            continue
        if not (dv._is_cuda_tensor(v) and v.dtype == dt and v.dim() == 1 and v.numel() >= size
                and v.is_contiguous() and v.device == x.device):
            raise ValueError(f"out {name} must be a contiguous {dt} CUDA tensor of length {size} on x's device")


def ltlt_blk_piv_device(x, b=DEFAULT_BLOCK, fused="var1", out=None, stream=None):
    """Device-resident entry: ``x`` is a column-major float64 CUDA tensor.

    Returns ``(L, tau, piv)`` CUDA tensors without synchronising.  ``out``
    may supply preallocated ``(L, tau, piv)`` (L may be ``x`` itself for an
    in-place factorization).
    """
    if fused not in PIVOTED_FUSED:
        raise InvalidVariant(f"fused must be one of {PIVOTED_FUSED}, got {fused!r}")
    _check_block(b)
    t = dv.require_cuda()
    if not dv.is_colmajor_cuda(x) or x.dtype != t.float64:
        raise ValueError("x must be a column-major float64 CUDA tensor")
    m = x.shape[0]
    if m < 1:
        raise ValueError("m >= 1 required")
    if out is None:
        L = dv.empty_colmajor(m, m, t.float64)
        tau = t.empty(max(m - 1, 0), dtype=t.float64, device=x.device)
        piv = t.empty(m, dtype=t.int64, device=x.device)
    else:
        L, tau, piv = out
        _check_out_device(x, m, L, tau, piv)
    lib = _capi.load()
    code = _capi.VARIANT_CODES[fused]
    nbytes = lib.skl_ltlt_blk_piv_workspace_size(m, int(b), code)
    if nbytes == 0:
        raise InvalidVariant("configuration not supported by the GPU panel kernel")
    ws = dv.workspace(nbytes, stream=stream)
    st = lib.skl_ltlt_blk_piv(m, int(b), code, x.data_ptr(), dv.ld_of(x), L.data_ptr(), dv.ld_of(L),
                              tau.data_ptr() if m > 1 else None, piv.data_ptr(), ws.data_ptr(), nbytes,
                              dv.stream_ptr(stream))
    _capi.check(st, "ltlt_blk_piv")
    return L, tau, piv


def ltlt_blk_piv_host(x, b=DEFAULT_BLOCK, fused="var1", out=None, stream=None, sync=True):
    """Host-buffer entry (``skl_ltlt_blk_piv_host``): H2D of X's lower part,
    factorization, D2H of L's lower part, tau and piv in one stream-ordered call.

    ``x`` is an F-ordered float64 numpy array (a view of pinned memory for
    asynchronous copies).  ``out = (L, tau, piv)`` numpy arrays (L F-ordered,
    may be ``x`` for an in-place factorization) are written: L's strict lower
    triangle and its 128x128 diagonal blocks (see the header); the rest of
    L's upper triangle is left untouched.  Returns ``(L, tau, piv)``.
    """
    if fused not in PIVOTED_FUSED:
        raise InvalidVariant(f"fused must be one of {PIVOTED_FUSED}, got {fused!r}")
    _check_block(b)
    x = np.asarray(x)
    if x.dtype != np.float64 or x.ndim != 2 or x.shape[0] != x.shape[1] or not x.flags.f_contiguous:
        raise ValueError("x must be a square F-ordered float64 array")
    m = x.shape[0]
    if m < 1:
        raise ValueError("m >= 1 required")
    if out is None:
        L = np.zeros((m, m), dtype=np.float64, order="F")
        tau = np.empty(max(m - 1, 0), dtype=np.float64)
        piv = np.empty(m, dtype=np.int64)
    else:
        L, tau, piv = out
        if not (isinstance(L, np.ndarray) and L.flags.f_contiguous and L.dtype == np.float64 and L.shape == (m, m)):
            raise ValueError("out L must be an F-ordered float64 (m, m) array")
        if not (isinstance(tau, np.ndarray) and tau.dtype == np.float64 and tau.ndim == 1
                and tau.size >= m - 1 and tau.flags.c_contiguous):
            raise ValueError("out tau must be a contiguous float64 array of length m - 1")
        if not (isinstance(piv, np.ndarray) and piv.dtype == np.int64 and piv.ndim == 1
                and piv.size >= m and piv.flags.c_contiguous):
            raise ValueError("out piv must be a contiguous int64 array of length m")
    lib = _capi.load()
    code = _capi.VARIANT_CODES[fused]
    nbytes = lib.skl_ltlt_blk_piv_host_workspace_size(m, int(b), code)
    if nbytes == 0:
        raise InvalidVariant("configuration not supported by the GPU panel kernel")
    ws = dv.workspace(nbytes, stream=stream)
    st = lib.skl_ltlt_blk_piv_host(m, int(b), code, x.ctypes.data, m, L.ctypes.data, m,
                                   tau.ctypes.data if m > 1 else None, piv.ctypes.data, ws.data_ptr(), nbytes,
                                   dv.stream_ptr(stream))
    _capi.check(st, "ltlt_blk_piv_host")
    if sync:
        (stream if stream is not None else dv.require_cuda().cuda.current_stream()).synchronize()
    return L, tau, piv


def ltlt_blk_piv(x: SkewMatrixLower, b=DEFAULT_BLOCK, fused="var1", features=None) -> FactorizationResult:
    """Pivoted blocked right-looking factorization (blocked.py:303-363).

    The input is never mutated.  NumPy input returns NumPy factors (drop-in);
    a torch CUDA ``data`` buffer returns device-resident L and tau.
    """
    if fused not in PIVOTED_FUSED:
        raise InvalidVariant(f"fused must be one of {PIVOTED_FUSED}, got {fused!r}")
    _check_block(b)
    if fused != "var1" and features is not None and not features.external_t:
        # blocked.py:326-327: the fused pivoted schedules need tau in an external vector
        raise InvalidVariant(f"pivoted blk-{fused} needs tau in an external vector (external_t)")
    if not isinstance(x, SkewMatrixLower):
        x = SkewMatrixLower(x)
    m = x.m
    if m < 1:
        raise ValueError("m >= 1 required")
    xd, on_device, dt = _device_input(x, "the blocked GPU path")
    L, tau, piv = ltlt_blk_piv_device(xd, b, fused)
    piv_h = piv.cpu().numpy()
    tau_h = tau.cpu().numpy()
    flops = flops_blk_piv(m, b, fused, piv_h, tau_h)
    if on_device:
        return _narrow(FactorizationResult(UnitLowerFactor(L, "ones"), SkewTridiagonal(tau),
                                           PermutationVector(piv_h, m), flops), dt)
    return _narrow(FactorizationResult(UnitLowerFactor(dv.to_host_colmajor(L), "ones"), SkewTridiagonal(tau_h),
                                       PermutationVector(piv_h, m), flops), dt)


# ---------------------------------------------------------------------------
# Unpivoted blocked drivers: blocked.py:162-290.  They run
# the same GPU driver as ltlt_blk_piv with the pivot row fixed (skl_ltlt_blk,
# pivot = 0); the panel is always the left-looking cluster kernel and the
# trailing update the DMMA GEMM, which compute the same factorization as the
# reference's rl / twostep panels and rank-2k couplings (equal in exact
# arithmetic; the flop tally returned is the reference's for the requested
# driver and panel variant, replayed by instrument.flops_blk_unpivoted).
# ---------------------------------------------------------------------------

_GPU_SCHEDULE = {"var1": "var1", "var2a": "var2a", "var2b": "var2b", "twostep": "var2a", "left": "left"}


def _prep_input(x):
    if not isinstance(x, SkewMatrixLower):
        x = SkewMatrixLower(x)
    m = x.m
    if m < 1:
        raise ValueError("m >= 1 required")
    xd, on_device, dt = _device_input(x, "the blocked GPU path")
    return x, xd, on_device, dt


def ltlt_blk_device(x, b=DEFAULT_BLOCK, fused="var1", pivot=False, out=None, stream=None):
    """Device entry of skl_ltlt_blk: returns ``(L, tau, piv, info)`` CUDA tensors
    without synchronising (``piv`` is None when unpivoted; ``info`` int32[1]:
    first zero-pivot column + 1, 0 = success).  ``fused="left"`` (unpivoted only)
    runs the blocked left-looking driver: skew_tridiag_gemm(tril) into each
    panel, no trailing update (blocked.py:236-265)."""
    if fused not in PIVOTED_FUSED and not (fused == "left" and not pivot):
        raise InvalidVariant(f"fused must be one of {PIVOTED_FUSED}, got {fused!r}")
    _check_block(b)
    t = dv.require_cuda()
    m = x.shape[0]
    if out is None:
        L = dv.empty_colmajor(m, m, t.float64)
        tau = t.empty(max(m - 1, 0), dtype=t.float64, device=x.device)
    else:
        L, tau = out
        _check_out_device(x, m, L, tau, None)
    piv = t.empty(m, dtype=t.int64, device=x.device) if pivot else None
    info = t.zeros(1, dtype=t.int32, device=x.device)
    lib = _capi.load()
    code = _capi.SKL_LEFT if fused == "left" else _capi.VARIANT_CODES[fused]
    nbytes = lib.skl_ltlt_blk_piv_workspace_size(m, int(b), code)
    if nbytes == 0:
        raise InvalidVariant("configuration not supported by the GPU panel kernel")
    ws = dv.workspace(nbytes, stream=stream)
    st = lib.skl_ltlt_blk(m, int(b), code, 1 if pivot else 0, x.data_ptr(), dv.ld_of(x), L.data_ptr(), dv.ld_of(L),
                          tau.data_ptr() if m > 1 else None, piv.data_ptr() if pivot else None, info.data_ptr(),
                          ws.data_ptr(), nbytes, dv.stream_ptr(stream))
    _capi.check(st, "ltlt_blk")
    return L, tau, piv, info


def _blk_unpivoted(x, b, driver, panel_variant, features, who):
    _check_block(b)
    if panel_variant not in PANEL_VARIANTS:
        raise InvalidVariant(f"unknown panel variant {panel_variant!r}")
    f = features or Features()
    if driver != "var1" and not f.external_t:
        raise InvalidVariant(f"{who} needs tau in an external vector (external_t)")
    x, xd, on_device, dt = _prep_input(x)
    m = x.m
    L, tau, _piv, info = ltlt_blk_device(xd, b, _GPU_SCHEDULE[driver], pivot=False)
    code = int(info.item())
    if code:
        raise ZeroPivot(code - 1)
    tau_h = tau.cpu().numpy()
    l_host = None if on_device and driver != "twostep" else dv.to_host_colmajor(L)
    flops = flops_blk_unpivoted(m, b, driver, panel_variant, tau_h, l_host)
    l_out = L if on_device else l_host
    return _narrow(FactorizationResult(UnitLowerFactor(l_out, "ones"), SkewTridiagonal(tau if on_device else tau_h),
                                       PermutationVector(np.zeros(0, dtype=np.int64), m), flops), dt)


def ltlt_blk_var1(x: SkewMatrixLower, b=DEFAULT_BLOCK, panel_variant="ll", features=None) -> FactorizationResult:
    """Blocked right-looking Variant 1 without pivoting (blocked.py:162-184)."""
    return _blk_unpivoted(x, b, "var1", panel_variant, features, "blk-var1")


def ltlt_blk_var2a(x: SkewMatrixLower, b=DEFAULT_BLOCK, panel_variant="ll", features=None) -> FactorizationResult:
    """Fused Variant 2a without pivoting (blocked.py:187-208)."""
    return _blk_unpivoted(x, b, "var2a", panel_variant, features, "blk-var2a")


def ltlt_blk_var2b(x: SkewMatrixLower, b=DEFAULT_BLOCK, panel_variant="ll", features=None) -> FactorizationResult:
    """Fused Variant 2b without pivoting (blocked.py:211-233)."""
    return _blk_unpivoted(x, b, "var2b", panel_variant, features, "blk-var2b")


def ltlt_blk_twostep(x: SkewMatrixLower, b=DEFAULT_BLOCK, panel_variant="ll", features=None) -> FactorizationResult:
    """Blocked two-step path (blocked.py:268-290): Variant 2a's iteration whose
    sandwich the reference realises as W = A S + skew rank-2k; the GPU runs the
    same coupling through the one DMMA GEMM (Q = A T^T packed on the fly)."""
    return _blk_unpivoted(x, b, "twostep", panel_variant, features, "blk-2step")


def ltlt_blk_left(x: SkewMatrixLower, b=DEFAULT_BLOCK, pivot=False, panel_variant="ll",
                  features=None) -> FactorizationResult:
    """Blocked left-looking factorization (blocked.py:236-265): before each panel
    the GPU pulls every prior coupling into the panel's columns with the
    skew_tridiag_gemm(tril) kernel (kernels3.py:239-302) and never touches the
    trailing matrix.  Pivoting is impossible at the blocked level
    (PivotUnsupported, blocked.py:247-248)."""
    if pivot:
        raise PivotUnsupported("a blocked pivoted left-looking algorithm cannot exist")
    return _blk_unpivoted(x, b, "left", panel_variant, features, "blk-left")
