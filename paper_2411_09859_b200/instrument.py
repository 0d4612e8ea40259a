"""FlopCounter and the closed-form counts the GPU drivers report.

The reference tallies flops by having every kernel call ``add_flops`` on a
module-global counter (``instrument.py:14-40,101-113``).  The GPU path does
not call back into Python per kernel; instead the same tallies are computed
on the host from (m, b, variant) and the returned pivots/tau, replaying the
reference's accounting rules exactly:

* ``_eliminate``: level2 += rows below the pivot, only if tau != 0
  (unblocked.py:86-89); symmetric swap: pivot += 2(a + (n-b-1) + (b-a-1)) + 1
  in the swap view's coordinates (core.py:324);
* ``skew_tridiag_gemv``: 2 rows k + 4k (kernels2.py:559);
* ``apply_row_pivots``: pivot += moved rows x columns (kernels2.py:615-617);
* ``skew_tridiag_rankk``: level3 += 2k n(n-1)/2 + 4kn (kernels3.py:164);
* ``skew_rank2``: level2 += 2n(n-1) (kernels2.py:466);
* blocked panels accrue non-pivot work to ``panel`` (blocked.py:331,347).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class FlopCounter:
    """Per-class operation tallies (instrument.py:14-40)."""

    level2: int = 0
    level3: int = 0
    panel: int = 0
    pivot: int = 0

    @property
    def total(self) -> int:
        return self.level2 + self.level3 + self.panel + self.pivot

    def __add__(self, other: "FlopCounter") -> "FlopCounter":
        return FlopCounter(self.level2 + other.level2, self.level3 + other.level3,
                           self.panel + other.panel, self.pivot + other.pivot)


def _lower(n):
    return n * (n - 1) // 2


def _swap_moves(nview, a, b):
    return 2 * (a + (nview - b - 1) + (b - a - 1)) + 1


def _row_pivot_moves(rows, sub):
    idx = np.arange(rows)
    for k, off in enumerate(sub):
        if off:
            j = k + int(off)
            idx[k], idx[j] = idx[j], idx[k]
    return int(np.count_nonzero(idx != np.arange(rows)))


def reference_schedule(m, b, fused):
    """Panels (r, nelim, lo, c0) of ltlt_blk_piv (blocked.py:325-362);
    c0 is the first tau index of the trailing couplings."""
    out = []
    if fused == "var2b":
        done, first = 0, True
        while done < m - 1:
            nelim = min(b + (1 if first else 0), m - 1 - done)
            lo = 0 if first else done - 1
            out.append((done, nelim, lo, 1 if first else done))
            done += nelim
            first = False
    else:
        r, pending = 0, False
        while r < m - 1:
            be = min(b, m - 1 - r)
            lo = r - 1 if (fused == "var2a" and pending) else r
            c0 = r + 1 if (fused == "var1" or not pending) else r
            out.append((r, be, lo, c0))
            r += be
            pending = True
    return out


def flops_blk_piv(m, b, fused, pivots, tau):
    """FlopCounter of ltlt_blk_piv(x, b, fused) given its pivots and tau."""
    fc = FlopCounter()
    pivots = np.asarray(pivots)
    tau = np.asarray(tau)
    for r, nelim, lo, c0 in reference_schedule(m, b, fused):
        for g in range(r, r + nelim):
            k = g - lo
            if k >= 2:
                rows = m - g - 1
                fc.panel += 2 * rows * k + 4 * k
            off = int(pivots[g + 1])
            if off:
                a = g + 1 - lo
                fc.pivot += _swap_moves(m - lo, a, a + off)
            if tau[g] != 0:
                fc.panel += max(m - g - 2, 0)
        if lo > 0 and nelim > 0:
            sub = pivots[r + 1:r + nelim + 1]
            if np.any(sub):
                fc.pivot += _row_pivot_moves(m - r - 1, sub) * lo
        rt = r + nelim
        if m - rt >= 2 and rt - c0 >= 1:
            n = m - rt
            k = rt - c0 + 1
            fc.level3 += 2 * k * _lower(n) + 4 * k * n
        if fused == "var1" and m - rt >= 2:
            n = m - rt - 1
            fc.level2 += 2 * n * max(n - 1, 0)
    return fc


def flops_unb_twostep(m, pivots, tau, pivot=True):
    """FlopCounter of ltlt_unb_twostep (unblocked.py:136-171,229-240)."""
    fc = FlopCounter()
    pivots = np.asarray(pivots)
    tau = np.asarray(tau)

    def elim(g):
        if pivot:
            off = int(pivots[g + 1])
            if off:
                fc.pivot += _swap_moves(m, g + 1, g + 1 + off)
        if tau[g] != 0:
            fc.level2 += max(m - g - 2, 0)

    def skr2(start):
        nsq = m - start
        if nsq > 0:
            fc.level2 += 2 * nsq * max(nsq - 1, 0)

    end = m - 1
    g = 0
    while g < end:
        if g + 1 >= end:
            elim(g)
            skr2(g + 2)
            g += 1
            continue
        elim(g)
        elim(g + 1)
        s = g + 3
        if g + 2 < m:
            fc.level2 += 6 * max(m - s, 0)
            skr2(s)
        g += 2
    return fc


def flop_model(variant, m, b=None):
    """Leading-order flop model used for GFLOP/s (oracle.py:164-172, cli.py:146)."""
    if variant in ("unb-rl", "rl"):
        return 2 * m ** 3 / 3
    return m ** 3 / 3
