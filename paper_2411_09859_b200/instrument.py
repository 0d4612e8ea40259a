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

from contextlib import contextmanager
from dataclasses import dataclass, field

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


@dataclass
class CallTrace:
    """Chronological (kernel, scope) record of the reference's kernel calls
    (instrument.py:44-54).  The GPU drivers run fused kernels, so the trace a
    driver emits is the reference's call sequence replayed from the same
    schedule and the returned pivots / tau (like the flop tallies below)."""

    calls: list = field(default_factory=list)

    def count(self, kernel=None, scope=None):
        return sum(1 for k, s in self.calls if (kernel is None or k == kernel) and (scope is None or s == scope))


# module-global accounting state, caller-serialised like the reference's (instrument.py:57-59)
_counter = None
_trace = None
_scope = "trailing"


@contextmanager
def counting(counter):
    """Route the tallies of the drivers called inside into ``counter`` (instrument.py:62-71)."""
    global _counter
    saved, _counter = _counter, counter
    try:
        yield counter
    finally:
        _counter = saved


@contextmanager
def tracing(trace):
    """Record the (replayed) kernel calls of the drivers called inside (instrument.py:74-84)."""
    global _trace
    saved, _trace = _trace, trace
    try:
        yield trace
    finally:
        _trace = saved


@contextmanager
def scope(name):
    global _scope
    saved, _scope = _scope, name
    try:
        yield
    finally:
        _scope = saved


def current_scope():
    return _scope


def add_flops(kind, n):
    """instrument.py:101-113: adds to the active counter (if any)."""
    if _counter is not None:
        setattr(_counter, kind, getattr(_counter, kind) + int(n))


def record_call(kernel):
    if _trace is not None:
        _trace.calls.append((kernel, _scope))


def _emit(fc, calls):
    """Hand a replayed driver's tally and call sequence to the active counter / trace."""
    if _counter is not None:
        for kind in ("level2", "level3", "panel", "pivot"):
            add_flops(kind, getattr(fc, kind))
    if _trace is not None:
        _trace.calls.extend(calls)
    return fc


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
    calls = []
    outer = _scope
    pivots = np.asarray(pivots)
    tau = np.asarray(tau)
    for r, nelim, lo, c0 in reference_schedule(m, b, fused):
        for g in range(r, r + nelim):
            k = g - lo
            if k >= 2:
                rows = m - g - 1
                fc.panel += 2 * rows * k + 4 * k
                calls.append(("skew_tridiag_gemv", "panel"))
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
                calls.append(("apply_row_pivots", outer))
        rt = r + nelim
        if m - rt >= 2 and rt - c0 >= 1:
            n = m - rt
            k = rt - c0 + 1
            fc.level3 += 2 * k * _lower(n) + 4 * k * n
            calls.append(("skew_tridiag_rankk", outer))
        if fused == "var1" and m - rt >= 2:
            n = m - rt - 1
            fc.level2 += 2 * n * max(n - 1, 0)
            calls.append(("skew_rank2", outer))
    return _emit(fc, calls)


def flops_unb_twostep(m, pivots, tau, pivot=True):
    """FlopCounter of ltlt_unb_twostep (unblocked.py:136-171,229-240)."""
    fc = FlopCounter()
    calls = []
    outer = _scope
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
            calls.append(("skew_rank2", outer))

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
    return _emit(fc, calls)


def flop_model(variant, m, b=None):
    """Leading-order flop model used for GFLOP/s (oracle.py:164-172, cli.py:146)."""
    if variant in ("unb-rl", "rl"):
        return 2 * m ** 3 / 3
    return m ** 3 / 3


# ---------------------------------------------------------------------------
# Flop replay of the unpivoted / unblocked drivers.  The
# counts depend only on shapes, tau (eliminations skip the scaling when tau
# is 0), the pivots and -- for the rank-2k couplings -- which operand columns
# are nonzero; each helper cites the reference routine whose tally it replays.
# ---------------------------------------------------------------------------

class _Tally:
    def __init__(self):
        self.fc = FlopCounter()
        self.in_panel = False
        self.calls = []
        self.outer = _scope

    def call(self, kernel):
        self.calls.append((kernel, "panel" if self.in_panel else self.outer))

    def done(self):
        return _emit(self.fc, self.calls)

    def add(self, kind, n):
        n = int(n)
        if self.in_panel and kind != "pivot":
            self.fc.panel += n
        else:
            setattr(self.fc, kind, getattr(self.fc, kind) + n)


def _t_elim(t, m, g, tau, pivots=None, swap_from=0):
    """_eliminate (unblocked.py:63-91): swap moves + scaling of the tail."""
    if pivots is not None and len(pivots):
        off = int(pivots[g + 1])
        if off:
            a = g + 1 - swap_from
            t.add("pivot", _swap_moves(m - swap_from, a, a + off))
    if tau[g] != 0:
        t.add("level2", max(m - g - 2, 0))


def _t_skew_rank2(t, n):
    """skew_rank2 (kernels2.py:93-131)."""
    t.call("skew_rank2")
    t.add("level2", 2 * n * max(n - 1, 0))


def _t_trapezoid(t, m, start, climit):
    """trapezoid_rank2 (kernels2.py:296-312): square skew part + rectangle."""
    climit = min(climit, m)
    nsq = climit - start
    if nsq <= 0:
        return
    _t_skew_rank2(t, nsq)
    if climit < m:
        t.call("gen_rank2")
        t.add("level2", 4 * (m - climit) * nsq)


def _t_panel_ll(t, m, tau, base, nelim, lo, pivots=None, swap_from=None):
    """_panel_ll (unblocked.py:94-119)."""
    swap_from = lo if swap_from is None else swap_from
    for g in range(base, base + nelim):
        k = g - lo
        if k >= 2:
            t.call("skew_tridiag_gemv")
            t.add("level2", 2 * (m - g - 1) * k + 4 * k)
        _t_elim(t, m, g, tau, pivots, swap_from)


def _t_panel_rl(t, m, tau, base, nelim, climit, pivots=None, swap_from=None):
    """_panel_rl (unblocked.py:122-133)."""
    swap_from = base if swap_from is None else swap_from
    for g in range(base, base + nelim):
        _t_elim(t, m, g, tau, pivots, swap_from)
        _t_trapezoid(t, m, g + 2, climit)


def _t_panel_twostep(t, m, tau, base, nelim, climit):
    """_panel_twostep (unblocked.py:136-171), unpivoted."""
    end = base + nelim
    g = base
    while g < end:
        if g + 1 >= end:
            _t_elim(t, m, g, tau)
            _t_trapezoid(t, m, g + 2, climit)
            g += 1
            continue
        _t_elim(t, m, g, tau)
        _t_elim(t, m, g + 1, tau)
        s = g + 3
        if g + 2 < min(climit, m):
            t.add("level2", 6 * max(m - s, 0))
            _t_trapezoid(t, m, s, climit)
        g += 2


def _t_run_panel(t, m, tau, base, nelim, variant, carry):
    """_run_panel (blocked.py:88-105), unpivoted, inside the panel scope."""
    climit = base + nelim
    lo = base - 1 if carry else base
    t.in_panel = True
    if variant == "ll":
        _t_panel_ll(t, m, tau, base, nelim, lo)
    elif variant == "rl":
        if carry:
            _t_trapezoid(t, m, base + 1, climit)   # _apply_pending (unblocked.py:174-179)
        _t_panel_rl(t, m, tau, base, nelim, climit)
    else:
        if carry:
            _t_trapezoid(t, m, base + 1, climit)
        _t_panel_twostep(t, m, tau, base, nelim, climit)
    t.in_panel = False


def _t_rankk(t, n, k):
    """skew_tridiag_rankk (kernels3.py:164)."""
    t.call("skew_tridiag_rankk")
    t.add("level3", 2 * k * _lower(n) + 4 * k * n)


def _s_entries(k):
    """number of entries of S for T of order k (core.py:153-169)."""
    return sum((1 if row >= 2 else 0) + (1 if row + 1 < k else 0) for row in range(0, k, 2))


def rank2k_keff(a, tau):
    """keff of skew_rank2k(C, 1, A, W) with W = form_w(A, S(tau)) (kernels3.py:318-321):
    columns nonzero in both A and W, W formed exactly as form_w does."""
    a = np.asarray(a)
    n, k = a.shape
    w = np.zeros_like(a)
    for row in range(0, k, 2):                     # core.py:163-168 entries (row, col, v)
        if row >= 2:
            w[:, row - 1] += tau[row - 1] * a[:, row]
        if row + 1 < k:
            w[:, row + 1] += -tau[row] * a[:, row]
    return int(np.count_nonzero((a != 0).any(axis=0) & (w != 0).any(axis=0)))


def flops_blk_unpivoted(m, b, driver, panel_variant, tau, work=None):
    """FlopCounter of ltlt_blk_{var1,var2a,var2b,twostep,left} (blocked.py:162-290).

    ``work`` (the returned "ones" buffer, host) is needed by the twostep driver
    only: its rank-2k couplings skip zero columns (kernels3.py:318-321)."""
    t = _Tally()
    tau = np.asarray(tau)
    if driver == "var2b":
        done, first = 0, True
        while done < m - 1:
            nelim = min(b + (1 if first else 0), m - 1 - done)
            _t_run_panel(t, m, tau, done, nelim, panel_variant, not first)
            new = done + nelim
            c0 = 1 if first else done
            if m - new >= 2 and new - c0 >= 1:
                _t_rankk(t, m - new, new - c0 + 1)
            done, first = new, False
    elif driver == "left":
        r = 0
        while r < m - 1:
            be = min(b, m - 1 - r)
            if r >= 2:   # skew_tridiag_gemm(tril) (kernels3.py:239-259): p = m-r, q = be, k = r
                p, q, k = m - r, be, r
                written = _lower(min(p, q)) + max(p - q, 0) * q
                t.call("skew_tridiag_gemm")
                t.add("level3", 2 * k * written + 4 * k * q)
            _t_run_panel(t, m, tau, r, be, panel_variant, r > 0)
            r += be
    else:
        r, pending = 0, False
        while r < m - 1:
            be = min(b, m - 1 - r)
            carry = driver != "var1" and pending
            _t_run_panel(t, m, tau, r, be, panel_variant, carry)
            rt = r + be
            c0 = r + 1 if (driver == "var1" or not pending) else r
            if m - rt >= 2 and rt - c0 >= 1:
                n, k = m - rt, rt - c0 + 1
                if driver == "twostep":
                    a = np.asarray(work)[rt:, c0 - 1:rt]
                    t.call("form_w")
                    t.add("level3", 2 * n * _s_entries(k))              # form_w (kernels3.py:364)
                    t.call("skew_rank2k")
                    t.add("level3", 4 * rank2k_keff(a, tau[c0:rt]) * _lower(n))
                else:
                    _t_rankk(t, n, k)
            if driver == "var1" and m - rt >= 2:
                _t_skew_rank2(t, m - rt - 1)
            pending = True
            r = rt
    return t.done()


def flops_unb_rl(m, tau, pivots=None):
    """FlopCounter of ltlt_unb_rl (unblocked.py:192-202)."""
    t = _Tally()
    _t_panel_rl(t, m, np.asarray(tau), 0, m - 1, m, pivots, 0)
    return t.done()


def flops_unb_ll(m, tau, pivots=None, first_column=False):
    """FlopCounter of ltlt_unb_ll (unblocked.py:205-226)."""
    t = _Tally()
    if first_column:
        _t_skew_rank2(t, m - 1)
    _t_panel_ll(t, m, np.asarray(tau), 0, m - 1, 0, pivots, 0)
    return t.done()


def flops_unb_panel(m, width, variant, tau, pivots=None, first_column=False):
    """FlopCounter of ltlt_unb_panel (unblocked.py:243-275)."""
    t = _Tally()
    tau = np.asarray(tau)
    nelim = min(width, m - 1)
    climit = min(width, m)
    if first_column:
        _t_skew_rank2(t, m - 1)
    t.in_panel = True
    if variant == "ll":
        _t_panel_ll(t, m, tau, 0, nelim, 0, pivots, 0)
    elif variant == "rl":
        _t_panel_rl(t, m, tau, 0, nelim, climit)
    else:
        _t_panel_twostep(t, m, tau, 0, nelim, climit)
    t.in_panel = False
    return t.done()
