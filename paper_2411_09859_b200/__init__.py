"""paper_2411_09859_b200: B200-native pivoted LTL^T of skew-symmetric matrices.

Drop-in for the reference ``skewltl`` hot path (arXiv 2411.09859): the same
public names and result types, computed by hand-written sm_100a CUDA kernels
behind the C ABI in ``include/skewltl_b200.h``.  There is no CPU fallback.
"""

from .core import (InvalidVariant, PermutationVector, PivotUnsupported, SingularT,  # noqa: F401
                   SkewMatrixLower, SkewTridiagonal, SSplitting, UnitLowerFactor, ZeroPivot,
                   apply_symmetric_pivot, compose_permutation, form_s_splitting, invert_permutation,
                   pack_in_place, random_skew, reconstruct, unpack_in_place)
from .instrument import CallTrace, FlopCounter  # noqa: F401
from .blocked import (DEFAULT_BLOCK, LADDER, FactorizationResult, Features, ltlt_blk_device,  # noqa: F401
                      ltlt_blk_left, ltlt_blk_piv, ltlt_blk_piv_device, ltlt_blk_piv_host, ltlt_blk_twostep,
                      ltlt_blk_var1, ltlt_blk_var2a, ltlt_blk_var2b)
from .unblocked import ltlt_unb_ll, ltlt_unb_panel, ltlt_unb_rl, ltlt_unb_twostep  # noqa: F401
from .apps import pfaffian, solve  # noqa: F401
from .mmio import mm_read, mm_write  # noqa: F401

__version__ = "0.1.0"
