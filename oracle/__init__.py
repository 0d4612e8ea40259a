"""CPU oracle for the pivoted LTL^T hot path -- TEST INFRASTRUCTURE ONLY.

This package is a NumPy restatement of the reference `skewltl` algorithms
(arXiv 2411.09859 artefact, mounted read-only at /root/reference during
development).  Each function cites the reference file:line it follows.

It is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import it.  The GPU package
``paper_2411_09859_b200`` never imports, calls or falls back to anything here.

Parity pinning: the restatement is checked against golden vectors produced by
the unmodified reference (``tests/golden/make_golden.py``, run in the build
container where /root/reference exists) and against the reference's own
known-answer tests (worked 4x4 example, m=2, zero-column, S/W patterns,
Pfaffian conventions).  See tests/test_oracle.py.
"""

from .ltlt import (  # noqa: F401
    OracleResult,
    apply_row_pivots,
    compose_permutation,
    eliminate,
    form_s_entries,
    form_w,
    ltlt_blk,
    ltlt_blk_piv,
    ltlt_unb_ll,
    ltlt_unb_panel,
    ltlt_unb_rl,
    ltlt_unb_twostep,
    skew_tridiag_gemm,
    solve,
    tridiag_solve,
    l_dense,
    pfaffian,
    pfaffian_slog,
    pivot_margins,
    reconstruct_dense,
    residual,
    skew_dense,
    skew_rank2,
    skew_rank2k,
    skew_tridiag_gemv,
    skew_tridiag_rankk,
    sym_swap_lower,
    tridiag_matvec,
)
from .exact import gauss_elim_exact, pfaffian_bruteforce  # noqa: F401
