"""ctypes binding of libskewltl_b200.so (the C ABI in include/skewltl_b200.h).

This module is the only place the shared library is loaded.  There is no
fallback: if the library is missing or no CUDA device is present, every
compute entry point raises ``NativeUnavailable`` instead of silently running
something else.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_lib" / "libskewltl_b200.so"

SKL_OK, SKL_ZERO_PIVOT, SKL_BAD_ARGUMENT, SKL_ALIAS, SKL_CUDA_ERROR, SKL_UNSUPPORTED, SKL_BAD_PIVOT = range(7)
SKL_VAR1, SKL_VAR2A, SKL_VAR2B, SKL_LEFT = 0, 1, 2, 3
SKL_F64, SKL_F32 = 0, 1
VARIANT_CODES = {"var1": SKL_VAR1, "var2a": SKL_VAR2A, "var2b": SKL_VAR2B}

#: exported symbol -> (restype, argtypes); mirrors include/skewltl_b200.h
_i, _ll, _d, _sz, _p = C.c_int, C.c_longlong, C.c_double, C.c_size_t, C.c_void_p
SIGNATURES = {
    "skl_version": (C.c_char_p, []),
    "skl_last_error": (C.c_char_p, []),
    "skl_skr2k_workspace_size": (_sz, [_i, _i]),
    "skl_skr2k_lower": (_i, [_i, _i, _d, _p, _ll, _p, _ll, _d, _p, _ll, _i, _p, _sz, _p, _p]),
    "skl_sktri_rankk_workspace_size": (_sz, [_i, _i]),
    "skl_sktri_rankk_lower": (_i, [_i, _i, _d, _p, _ll, _p, _d, _p, _ll, _p, _sz, _p]),
    "skl_form_w": (_i, [_i, _i, _p, _ll, _p, _p, _ll, _p]),
    "skl_skew_tridiag_gemm_workspace_size": (_sz, [_i, _i, _i]),
    "skl_skew_tridiag_gemm": (_i, [_i, _i, _i, _d, _p, _ll, _p, _p, _ll, _d, _p, _ll, _i, _p, _sz, _p]),
    "skl_skew_rank2_lower": (_i, [_i, _d, _p, _p, _d, _p, _ll, _p]),
    "skl_gen_rank2": (_i, [_i, _i, _d, _p, _p, _p, _p, _d, _p, _ll, _p]),
    "skl_skew_tridiag_gemv": (_i, [_i, _i, _d, _p, _ll, _p, _p, _d, _p, _i, _p]),
    "skl_apply_row_pivots_workspace_size": (_sz, [_i, _i, _i]),
    "skl_apply_row_pivots": (_i, [_i, _i, _p, _ll, _p, _i, _i, _p, _sz, _p]),
    "skl_apply_symmetric_pivot": (_i, [_i, _p, _ll, _i, _ll, _p]),
    "skl_pack_factor": (_i, [_i, _p, _ll, _p, _p, _ll, _p]),
    "skl_unpack_factor": (_i, [_i, _p, _ll, _p, _ll, _p, _p]),
    "skl_ltlt_blk_piv_workspace_size": (_sz, [_i, _i, _i]),
    "skl_ltlt_blk_piv_plan": (_i, [_i, _i, _i, _p, _p, _p, _p, _p, _i]),
    "skl_ltlt_blk_piv": (_i, [_i, _i, _i, _p, _ll, _p, _ll, _p, _p, _p, _sz, _p]),
    "skl_ltlt_blk": (_i, [_i, _i, _i, _i, _p, _ll, _p, _ll, _p, _p, _p, _p, _sz, _p]),
    "skl_ltlt_unb_panel_workspace_size": (_sz, [_i, _i]),
    "skl_ltlt_unb_panel": (_i, [_i, _i, _i, _p, _ll, _p, _ll, _p, _p, _p, _p, _sz, _p]),
    "skl_ltlt_solve_workspace_size": (_sz, [_i, _i]),
    "skl_ltlt_solve": (_i, [_i, _i, _p, _ll, _p, _p, _p, _ll, _d, _p, _p, _sz, _p]),
    "skl_ltlt_blk_piv_host_workspace_size": (_sz, [_i, _i, _i]),
    "skl_ltlt_blk_piv_host": (_i, [_i, _i, _i, _p, _ll, _p, _ll, _p, _p, _p, _sz, _p]),
    "skl_ltlt_unb_twostep_workspace_size": (_sz, [_i]),
    "skl_ltlt_unb_twostep": (_i, [_i, _i, _p, _ll, _p, _ll, _p, _p, _p, _p, _sz, _p]),
    "skl_ltlt_batched_piv": (_i, [_i, _i, _i, _p, _ll, _ll, _p, _ll, _ll, _p, _p, _p, _p, _p]),
    "skl_ltlt_dist_shared_size": (_sz, [_i, _i, _i]),
    "skl_ltlt_dist_workspace_size": (_sz, [_i, _i, _i, _i]),
    "skl_ltlt_dist_offsets": (_i, [_i, _i, _i, _p, _p, _p, _p]),
    "skl_ltlt_blk_piv_dist": (_i, [_i, _i, _i, _i, _i, _i, _i, _p, _ll, _p, _ll, _p, _p, _sz, _p, _p, _p]),
    "skl_dist_owner_table": (_i, [_i, _ll, _i, _i, _i, _p, _sz]),
    "skl_vmm_available": (_i, []),
    "skl_vmm_last_result": (_i, []),
    "skl_vmm_granularity": (_i, [_i, _p]),
    "skl_vmm_create": (_i, [_sz, _i, _i, _p]),
    "skl_vmm_export_fd": (_i, [C.c_ulonglong, _p]),
    "skl_vmm_import_fd": (_i, [_i, _p]),
    "skl_vmm_release": (_i, [C.c_ulonglong]),
    "skl_vmm_reserve": (_i, [_sz, _sz, _p]),
    "skl_vmm_free_va": (_i, [C.c_ulonglong, _sz]),
    "skl_vmm_map": (_i, [C.c_ulonglong, _sz, C.c_ulonglong, _sz, _i]),
    "skl_vmm_unmap": (_i, [C.c_ulonglong, _sz]),
    "skl_nccl_available": (_i, []),
    "skl_nccl_unique_id": (_i, [_p, _sz]),
    "skl_nccl_barrier_create": (_i, [_i, _i, _p, _p]),
    "skl_nccl_barrier": (_i, [_p, _p]),
    "skl_nccl_barrier_destroy": (_i, [_p]),
    "skl_timing_enable": (_i, [_i]),
    "skl_timing_read": (_i, [_p, _p]),
    "skl_launch_count": (_ll, []),
    "skl_debug_set_panel_profile": (_i, [_p]),
}


#: C type of skl_barrier_fn (a host callback may implement the cross-rank barrier)
BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing (there is no CPU fallback)."""


class NativeError(RuntimeError):
    """A CUDA error reported through the C ABI."""


_lib = None


def load(path=None):
    """Load (once) and return the ctypes handle, with signatures applied."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("SKEWLTL_B200_LIB", LIB_PATH))
    if not p.exists():
        raise NativeUnavailable(f"{p} not built; run __graft_entry__.build()")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error():
    return load().skl_last_error().decode()


def check(status, what=""):
    """Map a C-ABI status to the reference's exception types."""
    if status == SKL_OK:
        return
    from .core import InvalidVariant  # local import: core does not need ctypes
    if status == SKL_BAD_ARGUMENT:
        raise ValueError(f"{what}: dimension mismatch or bad argument")
    if status == SKL_ALIAS:
        raise ValueError(f"{what}: output aliases operand")
    if status == SKL_UNSUPPORTED:
        raise InvalidVariant(f"{what}: unsupported variant/configuration ({last_error()})")
    if status == SKL_BAD_PIVOT:
        raise IndexError("pivot index out of range")
    if status == SKL_CUDA_ERROR:
        raise NativeError(f"{what}: {last_error()}")
    raise NativeError(f"{what}: status {status}")
