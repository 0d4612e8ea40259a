"""NumPy restatement of the reference pivoted LTL^T path (TEST ORACLE ONLY).

Follows the reference `skewltl` package (``/root/reference/pkg/src/skewltl``)
function by function; every routine names the file:line it restates.  The
loop structure, blocking constants and elementwise operation order are kept
so the oracle's rounding tracks the reference closely (pivots bit-exact,
factors to ~1e-13 relative).

Storage conventions (reference ``core.py:37-44``, ``unblocked.py:6-11``):
the skew matrix is held as the strictly-lower triangle of an m x m
column-major buffer; the factorization overwrites that buffer so that buffer
column g holds L column g+1 (rows g+2..) with an explicit 1.0 at [g+1, g];
tau (length m-1) is the subdiagonal of T; pivots[k] is the relative offset of
the transposition (k, k+pivots[k]), pivots[0] == 0.

Flop tallies mirror ``instrument.py:14-40,101-113``: a dict with keys
level2/level3/panel/pivot, where work done inside a blocked driver's panel
accrues to ``panel`` (``blocked.py:331,347``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# reference constants: kernels2.py:24 (JAM), kernels3.py:36-38 (BlockConfig)
JAM = 64
M_C, K_C, N_C = 128, 256, 256
DEFAULT_BLOCK = 256          # blocked.py:34
PIVOTED_FUSED = ("var1", "var2a", "var2b")   # blocked.py:35


class _Counter:
    """Flop/data-movement tally (instrument.py:14-40, 101-113)."""

    def __init__(self):
        self.level2 = 0
        self.level3 = 0
        self.panel = 0
        self.pivot = 0
        self.in_panel = False

    def add(self, kind, n):
        if self.in_panel and kind != "pivot":
            self.panel += int(n)
        else:
            setattr(self, kind, getattr(self, kind) + int(n))

    def as_dict(self):
        return {"level2": self.level2, "level3": self.level3,
                "panel": self.panel, "pivot": self.pivot}


_NULL = _Counter()


@dataclass
class OracleResult:
    """Work buffer holding L ("ones" layout), tau, pivots, flop tally."""

    work: np.ndarray
    tau: np.ndarray
    pivots: np.ndarray
    flops: dict = field(default_factory=dict)
    first_column: np.ndarray = None


# ----------------------------------------------------------------------------
# core.py restatements
# ----------------------------------------------------------------------------

def sym_swap_lower(buf, a, b, fc=_NULL):
    """X := P X P^T for the transposition (a, b), lower storage.

    Restates core.py:294-324 (row swap left of a, column swap below b, the
    crossing segment that changes sign, and the negated (b, a) entry).
    """
    if a == b:
        return
    if a > b:
        a, b = b, a
    n = buf.shape[0]
    if b >= n or a < 0:
        raise IndexError("pivot index out of range")
    if a > 0:
        row = buf[a, :a].copy()
        buf[a, :a] = buf[b, :a]
        buf[b, :a] = row
    if b + 1 < n:
        col = buf[b + 1:, a].copy()
        buf[b + 1:, a] = buf[b + 1:, b]
        buf[b + 1:, b] = col
    if b - a > 1:
        seg = buf[a + 1:b, a].copy()
        buf[a + 1:b, a] = -buf[b, a + 1:b]
        buf[b, a + 1:b] = -seg
    buf[b, a] = -buf[b, a]
    fc.add("pivot", 2 * (a + (n - b - 1) + (b - a - 1)) + 1)


def compose_permutation(pivots):
    """perm with (P x)[i] = x[perm[i]] (core.py:274-285)."""
    pivots = np.asarray(pivots, dtype=np.int64)
    idx = np.arange(len(pivots))
    for k, off in enumerate(pivots):
        if off:
            j = k + int(off)
            idx[k], idx[j] = idx[j], idx[k]
    return idx


def form_s_entries(tau):
    """Sparse S with T = S - S^T (core.py:153-169): list of (i, j, v)."""
    m = len(tau) + 1
    out = []
    for row in range(0, m, 2):
        if row >= 2:
            out.append((row, row - 1, tau[row - 1]))
        if row + 1 < m:
            out.append((row, row + 1, -tau[row]))
    return out


def skew_dense(lower):
    low = np.tril(np.asarray(lower), -1)
    return low - low.T


def l_dense(work):
    """Dense unit-lower L from the "ones" buffer (core.py:211-220)."""
    m = work.shape[0]
    out = np.eye(m, dtype=work.dtype)
    for j in range(1, m):
        out[j + 1:, j] = work[j + 1:, j - 1]
    return out


def tridiag_dense(tau):
    m = len(tau) + 1
    t = np.zeros((m, m), dtype=np.asarray(tau).dtype if len(tau) else np.float64)
    if m > 1:
        i = np.arange(m - 1)
        t[i + 1, i] = tau
        t[i, i + 1] = -np.asarray(tau)
    return t


def reconstruct_dense(work, tau, pivots=None):
    """P^T L T L^T P as a dense skew matrix (core.py:336-346)."""
    ld = l_dense(work).astype(np.float64)
    full = ld @ tridiag_dense(np.asarray(tau, dtype=np.float64)) @ ld.T
    if pivots is not None and len(pivots) and np.any(pivots):
        perm = compose_permutation(pivots)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm))
        full = full[np.ix_(inv, inv)]
    return full


def residual(x_lower, work, tau, pivots=None):
    """||P X P^T - L T L^T||_F / ||X||_F (tests/helpers.py:9-14 style)."""
    ref = skew_dense(np.asarray(x_lower, dtype=np.float64))
    rec = reconstruct_dense(work, tau, pivots)
    rec = skew_dense(rec)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(rec - ref) / (den if den else 1.0))


# ----------------------------------------------------------------------------
# kernels2.py restatements (level-2)
# ----------------------------------------------------------------------------

def skew_rank2(a, alpha, x, y, fc=_NULL):
    """A_lower += alpha (x y^T - y x^T) (kernels2.py:93-131, JAM blocking)."""
    n = a.shape[0]
    fc.add("level2", 2 * n * max(n - 1, 0))
    if n <= 1 or alpha == 0:
        return
    for j0 in range(0, n, JAM):
        j1 = min(j0 + JAM, n)
        for j in range(j0, j1):
            if j + 1 < j1:
                a[j + 1:j1, j] += alpha * (x[j + 1:j1] * y[j] - y[j + 1:j1] * x[j])
        if j1 < n:
            a[j1:, j0:j1] += alpha * (np.outer(x[j1:], y[j0:j1]) - np.outer(y[j1:], x[j0:j1]))


def gen_rank2(a, alpha, x, u, y, v, fc=_NULL):
    """A += alpha (x u^T + y v^T) on a rectangle (kernels2.py:134-163)."""
    p, q = a.shape
    fc.add("level2", 4 * p * q)
    if p == 0 or q == 0 or alpha == 0:
        return
    a += alpha * (np.outer(x, u) + np.outer(y, v))


def trapezoid_rank2(buf, start, climit, alpha, x, y, fc=_NULL):
    """Square skew rank-2 plus rectangular part (kernels2.py:296-312)."""
    n = buf.shape[0]
    climit = min(climit, n)
    nsq = climit - start
    if nsq <= 0:
        return
    skew_rank2(buf[start:climit, start:climit], alpha, x[:nsq], y[:nsq], fc)
    if climit < n:
        gen_rank2(buf[climit:, start:climit], alpha, x[nsq:], y[:nsq], -y[nsq:], x[:nsq], fc)


def tridiag_matvec(tau, x):
    """z = T x for the skew tridiagonal with subdiagonal tau (kernels2.py:166-175)."""
    k = len(x)
    z = np.zeros(k, dtype=np.result_type(np.asarray(tau).dtype, x.dtype) if k else x.dtype)
    if k > 1:
        z[1:] = tau * x[:-1]
        z[:-1] -= tau * x[1:]
    return z


def skew_tridiag_gemv(y, alpha, a, tau, x, tail_from=0, fc=_NULL):
    """y += alpha (A (T x))[tail_from:] (kernels2.py:178-229).

    Like the reference's fused fast path (kernels2.py:572-582) the product
    is formed at the full column height of A and the head rows dropped.
    """
    p, k = a.shape
    rows = p - tail_from
    fc.add("level2", 2 * rows * k + 4 * k)
    if alpha == 0 or rows == 0:
        return
    z = tridiag_matvec(tau, x)
    acc = a.dot(z)
    y += alpha * acc[tail_from:]


def apply_row_pivots(block, pivots, forward=True, fc=_NULL):
    """Permute rows of ``block`` by P(p) as one gather (kernels2.py:232-271)."""
    n = block.shape[0]
    q = block.shape[1] if block.ndim == 2 else 1
    idx = np.arange(n)
    for k, off in enumerate(np.asarray(pivots)):
        if off:
            j = k + int(off)
            if j >= n or off < 0:
                raise IndexError("pivot out of range")
            idx[k], idx[j] = idx[j], idx[k]
    if not forward:
        inv = np.empty_like(idx)
        inv[idx] = np.arange(n)
        idx = inv
    moved_mask = idx != np.arange(n)
    moved = int(np.count_nonzero(moved_mask))
    fc.add("pivot", moved * q)
    if moved == 0 or q == 0:
        return
    touched = np.flatnonzero(moved_mask)
    lo, hi = int(touched[0]), int(touched[-1]) + 1
    block[lo:hi] = block[idx[lo:hi]]


# ----------------------------------------------------------------------------
# kernels3.py restatements (level-3, sandwiched)
# ----------------------------------------------------------------------------

def _lower_entries(n):
    return n * (n - 1) // 2


def _k_panels(k, k_c=K_C):
    """k-panel boundaries with the 1.25 k_c tail merge (kernels3.py:69-80)."""
    out, pc = [], 0
    while pc < k:
        rem = k - pc
        step = rem if rem <= k_c + k_c // 4 else k_c
        out.append((pc, pc + step))
        pc += step
    return out


def _merge_tile(tile, contrib, alpha, row_off):
    """tile += alpha*contrib on strictly-lower entries (kernels3.py:101-118)."""
    mask = np.tril(np.ones(tile.shape, dtype=bool), k=row_off - 1)
    if alpha == 1:
        np.add(tile, contrib, out=tile, where=mask)
    elif alpha == -1:
        np.subtract(tile, contrib, out=tile, where=mask)
    else:
        np.add(tile, alpha * contrib, out=tile, where=mask)


def _accum_tile(tile, contrib, alpha):
    if alpha == 1:
        np.add(tile, contrib, out=tile)
    elif alpha == -1:
        np.subtract(tile, contrib, out=tile)
    else:
        tile += alpha * contrib


def _pack_bt(tau, a, jc, j1, pc, p1):
    """Rows [pc, p1) of B = T A^T for C-columns [jc, j1) (kernels3.py:134-148)."""
    k = a.shape[1]
    bp = np.zeros((p1 - pc, j1 - jc), dtype=a.dtype)
    lo1 = max(pc, 1)
    if lo1 < p1:
        bp[lo1 - pc:, :] = tau[lo1 - 1:p1 - 1, None] * a[jc:j1, lo1 - 1:p1 - 1].T
    hi2 = min(p1, k - 1)
    if hi2 > pc:
        bp[:hi2 - pc, :] -= tau[pc:hi2, None] * a[jc:j1, pc + 1:hi2 + 1].T
    return bp


def skew_tridiag_rankk(c, alpha, a, tau, fc=_NULL):
    """C_lower += alpha A T A^T (kernels3.py:151-209), beta = 1."""
    n, k = a.shape
    fc.add("level3", 2 * k * _lower_entries(n) + 4 * k * n)
    if n <= 1 or alpha == 0 or k == 0:
        return
    for jc in range(0, n, N_C):
        j1 = min(jc + N_C, n)
        for pc, p1 in _k_panels(k):
            bp = _pack_bt(tau, a, jc, j1, pc, p1)
            ak = a[:, pc:p1]
            for ic in range(jc, n, M_C):
                i1 = min(ic + M_C, n)
                contrib = ak[ic:i1].dot(bp)
                tile = c[ic:i1, jc:j1]
                if ic >= j1:
                    _accum_tile(tile, contrib, alpha)
                else:
                    _merge_tile(tile, contrib, alpha, ic - jc)


def skew_rank2k(c, alpha, a, b, skip_zero_columns=True, fc=_NULL):
    """C_lower += alpha (A B^T - B A^T), zero columns skipped (kernels3.py:305-351)."""
    n, k = a.shape
    if skip_zero_columns and k:
        keep = np.flatnonzero((a != 0).any(axis=0) & (b != 0).any(axis=0))
    else:
        keep = np.arange(k)
    keff = len(keep)
    fc.add("level3", 4 * keff * _lower_entries(n))
    if n <= 1 or alpha == 0 or keff == 0:
        return keff
    for jc in range(0, n, N_C):
        j1 = min(jc + N_C, n)
        for pc, p1 in _k_panels(keff):
            cols = keep[pc:p1]
            at_p = np.ascontiguousarray(a[jc:j1, cols].T)
            bt_p = np.ascontiguousarray(b[jc:j1, cols].T)
            for ic in range(jc, n, M_C):
                i1 = min(ic + M_C, n)
                contrib = a[ic:i1][:, cols].dot(bt_p) - b[ic:i1][:, cols].dot(at_p)
                tile = c[ic:i1, jc:j1]
                if ic >= j1:
                    _accum_tile(tile, contrib, alpha)
                else:
                    _merge_tile(tile, contrib, alpha, ic - jc)
    return keff


def form_w(a, tau, fc=_NULL):
    """W = A S with T = S - S^T (kernels3.py:354-364, core.py:153-169)."""
    n, kdim = a.shape
    ent = form_s_entries(tau)
    w = np.zeros((n, kdim), dtype=a.dtype, order="F")
    for i, j, v in ent:
        w[:, j] += v * a[:, i]
    fc.add("level3", 2 * n * len(ent))
    return w


def _pack_tb(tau, b, jc, j1, pc, p1):
    """Rows [pc, p1) of T B for B-columns [jc, j1) (kernels3.py:226-236)."""
    k = b.shape[0]
    bp = np.zeros((p1 - pc, j1 - jc), dtype=b.dtype)
    lo1 = max(pc, 1)
    if lo1 < p1:
        bp[lo1 - pc:, :] = tau[lo1 - 1:p1 - 1, None] * b[lo1 - 1:p1 - 1, jc:j1]
    hi2 = min(p1, k - 1)
    if hi2 > pc:
        bp[:hi2 - pc, :] -= tau[pc:hi2, None] * b[pc + 1:hi2 + 1, jc:j1]
    return bp


def skew_tridiag_gemm(c, alpha, a, tau, b, tril=False, fc=_NULL):
    """C += alpha A (T B) on a p x q block, beta = 1, fused packing
    (kernels3.py:239-302); tril writes only row > col entries."""
    p, k = a.shape
    q = b.shape[1]
    written = _lower_entries(min(p, q)) + max(p - q, 0) * q if tril else p * q
    fc.add("level3", 2 * k * written + 4 * k * q)
    if p == 0 or q == 0 or alpha == 0 or k == 0:
        return
    for jc in range(0, q, N_C):
        j1 = min(jc + N_C, q)
        row0 = jc if tril else 0
        tiles = [(ic, min(ic + M_C, p)) for ic in range(row0, p, M_C)]
        if not tiles:
            continue
        for pc, p1 in _k_panels(k):
            bp = _pack_tb(tau, b, jc, j1, pc, p1)
            ak = a[:, pc:p1]
            for ic, i1 in tiles:
                tile = c[ic:i1, jc:j1]
                contrib = ak[ic:i1].dot(bp)
                if not tril or ic >= j1:
                    _accum_tile(tile, contrib, alpha)
                else:
                    _merge_tile(tile, contrib, alpha, ic - jc)


# ----------------------------------------------------------------------------
# unblocked.py restatements
# ----------------------------------------------------------------------------

def _workbuf(x):
    x = np.asarray(x)
    if x.ndim != 2 or x.shape[0] != x.shape[1]:
        raise ValueError("square 2-D buffer required")
    if x.shape[0] < 1:
        raise ValueError("m >= 1 required")
    work = np.array(x, order="F")
    tau = np.zeros(max(x.shape[0] - 1, 0), dtype=work.dtype)
    return work, tau


def eliminate(work, tau, g, pivot=False, pivots=None, swap_from=0, fc=_NULL):
    """Column g -> L column g+1, tau[g] (unblocked.py:63-91).

    iamax with ties to the lowest index (np.argmax), symmetric swap over
    columns >= swap_from, explicit unit at [g+1, g].
    """
    if pivot:
        off = int(np.argmax(np.abs(work[g + 1:, g])))
        if pivots is not None:
            pivots[g + 1] = off
        if off:
            a = g + 1 - swap_from
            sym_swap_lower(work[swap_from:, swap_from:], a, a + off, fc)
    piv = work[g + 1, g]
    tau[g] = piv
    below = work[g + 2:, g]
    if piv == 0:
        if not pivot and below.size and np.any(below != 0):
            raise ZeroDivisionError(f"zero pivot while eliminating column {g}")
    else:
        below /= piv
        fc.add("level2", below.size)
    work[g + 1, g] = 1


def panel_ll(work, tau, base, nelim, lo, pivot=False, pivots=None, swap_from=None, fc=_NULL):
    """Left-looking eliminations of [base, base+nelim) (unblocked.py:94-119)."""
    if swap_from is None:
        swap_from = lo
    for g in range(base, base + nelim):
        if g - lo >= 2:
            skew_tridiag_gemv(work[g + 1:, g], -1, work[:, lo:g], tau[lo + 1:g],
                              work[g, lo:g], tail_from=g + 1, fc=fc)
        eliminate(work, tau, g, pivot, pivots, swap_from, fc)


def panel_twostep(work, tau, base, nelim, climit, pivot=False, pivots=None,
                  swap_from=None, fc=_NULL):
    """Wimmer two-step eliminations (unblocked.py:136-171)."""
    if swap_from is None:
        swap_from = base
    m = work.shape[0]
    end = base + nelim
    g = base
    while g < end:
        if g + 1 >= end:
            eliminate(work, tau, g, pivot, pivots, swap_from, fc)
            trapezoid_rank2(work, g + 2, climit, 1, work[g + 2:, g], work[g + 2:, g + 1], fc)
            g += 1
            continue
        eliminate(work, tau, g, pivot, pivots, swap_from, fc)
        eliminate(work, tau, g + 1, pivot, pivots, swap_from, fc)
        s = g + 3
        if g + 2 < min(climit, m):
            lcol1 = work[s:, g]
            lcol2 = work[s:, g + 1]
            work[s:, g + 2] -= tau[g + 1] * (work[g + 2, g] * lcol2 - lcol1)
            wv = work[s:, g + 2] - tau[g + 1] * lcol1
            fc.add("level2", 6 * max(m - s, 0))
            trapezoid_rank2(work, s, climit, -1, wv, lcol2, fc)
        g += 2


def panel_rl(work, tau, base, nelim, climit, pivot=False, pivots=None, swap_from=None, fc=_NULL):
    """Right-looking eliminations of [base, base+nelim), rank-2 updates
    restricted to columns < climit (unblocked.py:122-133)."""
    if swap_from is None:
        swap_from = base
    for g in range(base, base + nelim):
        eliminate(work, tau, g, pivot, pivots, swap_from, fc)
        s = g + 2
        trapezoid_rank2(work, s, climit, 1, work[s:, g], work[s:, g + 1], fc)


def apply_pending(work, base, climit, fc=_NULL):
    """Delayed coupling of the previous block (unblocked.py:174-179)."""
    s = base + 1
    trapezoid_rank2(work, s, climit, 1, work[s:, base - 1], work[s:, base], fc)


def apply_first_column(work, first_column, fc=_NULL):
    """Non-default first L column: its transform applied up front (unblocked.py:182-189)."""
    m = work.shape[0]
    fcvec = np.asarray(first_column)
    if fcvec.shape != (m - 1,):
        raise ValueError("first_column must have length m - 1")
    fcvec = fcvec.astype(work.dtype, copy=True)
    skew_rank2(work[1:, 1:], 1, fcvec, work[1:, 0], fc)
    return fcvec


def ltlt_unb_rl(x, pivot=False):
    """Unblocked right-looking (modified Parlett-Reid) driver (unblocked.py:192-202)."""
    work, tau = _workbuf(x)
    m = work.shape[0]
    pivots = np.zeros(m, dtype=np.int64) if pivot else np.zeros(0, dtype=np.int64)
    fc = _Counter()
    panel_rl(work, tau, 0, m - 1, m, pivot, pivots if pivot else None, 0, fc)
    return OracleResult(work, tau, pivots, fc.as_dict())


def ltlt_unb_panel(x, panel_width, variant="ll", pivot=False, first_column=None):
    """First ``panel_width`` columns only (unblocked.py:243-275)."""
    if variant not in ("ll", "rl", "twostep"):
        raise ValueError(f"unknown panel variant {variant!r}")
    if pivot and variant != "ll":
        raise ValueError("a pivoted panel factorization must be left-looking")
    if pivot and first_column is not None:
        raise ValueError("first_column is only supported without pivoting")
    work, tau = _workbuf(x)
    m = work.shape[0]
    nelim = min(panel_width, m - 1)
    climit = min(panel_width, m)
    pivots = np.zeros(m, dtype=np.int64) if pivot else None
    fc = _Counter()
    fcvec = apply_first_column(work, first_column, fc) if first_column is not None else None
    fc.in_panel = True
    if variant == "ll":
        panel_ll(work, tau, 0, nelim, 0, pivot, pivots, 0, fc)
    elif variant == "rl":
        panel_rl(work, tau, 0, nelim, climit, fc=fc)
    else:
        panel_twostep(work, tau, 0, nelim, climit, fc=fc)
    fc.in_panel = False
    lbuf = np.zeros_like(work)
    lbuf[:, :nelim] = work[:, :nelim]
    ptrim = pivots[:nelim + 1] if pivots is not None else np.zeros(0, dtype=np.int64)
    return OracleResult(lbuf, tau, ptrim, fc.as_dict(), fcvec)


def ltlt_unb_twostep(x, pivot=False):
    """Unblocked two-step driver (unblocked.py:229-240)."""
    work, tau = _workbuf(x)
    m = work.shape[0]
    pivots = np.zeros(m, dtype=np.int64) if pivot else np.zeros(0, dtype=np.int64)
    fc = _Counter()
    panel_twostep(work, tau, 0, m - 1, m, pivot, pivots if pivot else None, 0, fc)
    return OracleResult(work, tau, pivots, fc.as_dict())


def ltlt_unb_ll(x, pivot=False, first_column=None):
    """Unblocked left-looking (modified Aasen) driver (unblocked.py:205-226)."""
    if pivot and first_column is not None:
        raise ValueError("first_column is only supported without pivoting")
    work, tau = _workbuf(x)
    m = work.shape[0]
    pivots = np.zeros(m, dtype=np.int64) if pivot else np.zeros(0, dtype=np.int64)
    fc = _Counter()
    fcvec = apply_first_column(work, first_column, fc) if first_column is not None else None
    panel_ll(work, tau, 0, m - 1, 0, pivot, pivots if pivot else None, 0, fc)
    return OracleResult(work, tau, pivots, fc.as_dict(), fcvec)


# ----------------------------------------------------------------------------
# blocked.py restatements
# ----------------------------------------------------------------------------

def _apply_couplings(work, tau, c0, c1, region, fc):
    """C := C - A T~ A^T on [region:, region:) (blocked.py:108-125)."""
    m = work.shape[0]
    if m - region < 2 or c1 - c0 < 1:
        return
    a = work[region:, c0 - 1:c1]
    skew_tridiag_rankk(work[region:, region:], -1, a, tau[c0:c1], fc)


def _straggler(work, tau, rt, fc):
    """Var1 trailing rank-2 of the panel's last transform (blocked.py:128-134)."""
    m = work.shape[0]
    if m - rt < 2:
        return
    skew_rank2(work[rt + 1:, rt + 1:], 1, work[rt + 1:, rt - 1], work[rt + 1:, rt], fc)


def _block_pivots(work, pivots, base, nelim, lo, fc):
    """Row-swap older L columns by the panel's pivots (blocked.py:293-300)."""
    if lo <= 0 or nelim == 0:
        return
    sub = pivots[base + 1: base + nelim + 1]
    if np.any(sub):
        apply_row_pivots(work[base + 1:, :lo], sub, True, fc)


def _panel(work, tau, base, nelim, lo, pivots, fc):
    fc.in_panel = True
    try:
        panel_ll(work, tau, base, nelim, lo, True, pivots, lo, fc)
    finally:
        fc.in_panel = False


def ltlt_blk_piv(x, b=DEFAULT_BLOCK, fused="var1"):
    """Pivoted blocked right-looking driver (blocked.py:303-363)."""
    if fused not in PIVOTED_FUSED:
        raise ValueError(f"fused must be one of {PIVOTED_FUSED}, got {fused!r}")
    if b < 1:
        raise ValueError("block size must be >= 1")
    work, tau = _workbuf(x)
    m = work.shape[0]
    pivots = np.zeros(m, dtype=np.int64)
    fc = _Counter()
    if fused == "var2b":
        done, first = 0, True
        while done < m - 1:
            nelim = min(b + (1 if first else 0), m - 1 - done)
            lo = 0 if first else done - 1
            _panel(work, tau, done, nelim, lo, pivots, fc)
            _block_pivots(work, pivots, done, nelim, lo, fc)
            new = done + nelim
            _apply_couplings(work, tau, 1 if first else done, new, new, fc)
            done, first = new, False
    else:
        r, pending = 0, False
        while r < m - 1:
            be = min(b, m - 1 - r)
            carry = fused == "var2a" and pending
            lo = r - 1 if carry else r
            _panel(work, tau, r, be, lo, pivots, fc)
            _block_pivots(work, pivots, r, be, lo, fc)
            rt = r + be
            if fused == "var1":
                _apply_couplings(work, tau, r + 1, rt, rt, fc)
                _straggler(work, tau, rt, fc)
            else:
                _apply_couplings(work, tau, r if pending else r + 1, rt, rt, fc)
            pending = True
            r = rt
    return OracleResult(work, tau, pivots, fc.as_dict())


def _panel_variant(work, tau, base, nelim, variant, carry, fc):
    """_run_panel without pivoting (blocked.py:88-105)."""
    climit = base + nelim
    lo = base - 1 if carry else base
    fc.in_panel = True
    try:
        if variant == "ll":
            panel_ll(work, tau, base, nelim, lo, False, None, lo, fc)
        elif variant == "rl":
            if carry:
                apply_pending(work, base, climit, fc)
            panel_rl(work, tau, base, nelim, climit, fc=fc)
        elif variant == "twostep":
            if carry:
                apply_pending(work, base, climit, fc)
            panel_twostep(work, tau, base, nelim, climit, fc=fc)
        else:
            raise ValueError(f"unknown panel variant {variant!r}")
    finally:
        fc.in_panel = False


def _couplings_rank2k(work, tau, c0, c1, region, fc):
    """_apply_couplings(rank2k=True): W = A S then skew rank-2k (blocked.py:118-121)."""
    m = work.shape[0]
    if m - region < 2 or c1 - c0 < 1:
        return
    a = work[region:, c0 - 1:c1]
    w = form_w(a, tau[c0:c1], fc)
    skew_rank2k(work[region:, region:], 1, a, w, True, fc)


def ltlt_blk(x, b=DEFAULT_BLOCK, driver="var1", panel_variant="ll"):
    """Unpivoted blocked drivers (blocked.py:162-290): driver in var1, var2a,
    var2b (right-looking), twostep (2a with W = A S + skew rank-2k), left
    (left-looking: trapezoidal sandwiched gemm from the left, no trailing update)."""
    if b < 1:
        raise ValueError("block size must be >= 1")
    work, tau = _workbuf(x)
    m = work.shape[0]
    fc = _Counter()
    if driver == "var2b":
        done, first = 0, True
        while done < m - 1:
            nelim = min(b + (1 if first else 0), m - 1 - done)
            _panel_variant(work, tau, done, nelim, panel_variant, not first, fc)
            new = done + nelim
            _apply_couplings(work, tau, 1 if first else done, new, new, fc)
            done, first = new, False
    elif driver == "left":
        r = 0
        while r < m - 1:
            be = min(b, m - 1 - r)
            if r >= 2:
                skew_tridiag_gemm(work[r:, r:r + be], -1, work[r:, 0:r], tau[1:r],
                                  work[r:r + be, 0:r].T, True, fc)
            _panel_variant(work, tau, r, be, panel_variant, r > 0, fc)
            r += be
    elif driver in ("var1", "var2a", "twostep"):
        r, pending = 0, False
        while r < m - 1:
            be = min(b, m - 1 - r)
            carry = driver != "var1" and pending
            _panel_variant(work, tau, r, be, panel_variant, carry, fc)
            rt = r + be
            if driver == "var1":
                _apply_couplings(work, tau, r + 1, rt, rt, fc)
                _straggler(work, tau, rt, fc)
            elif driver == "var2a":
                _apply_couplings(work, tau, r if pending else r + 1, rt, rt, fc)
            else:
                _couplings_rank2k(work, tau, r if pending else r + 1, rt, rt, fc)
            pending = True
            r = rt
    else:
        raise ValueError(f"unknown driver {driver!r}")
    return OracleResult(work, tau, np.zeros(0, dtype=np.int64), fc.as_dict())


# ----------------------------------------------------------------------------
# apps.py restatement + Pfaffian in (sign, log|Pf|) form
# ----------------------------------------------------------------------------

def pfaffian(x, b=None):
    """Pf via the pivoted factorization (apps.py:12-30); may overflow to inf."""
    x = np.asarray(x)
    m = x.shape[0]
    if m == 0:
        return 1.0
    if m % 2:
        return 0.0
    res = ltlt_blk_piv(x, b=b or min(DEFAULT_BLOCK, m))
    val = -1 if np.count_nonzero(res.pivots) % 2 else 1
    for i in range(0, m - 1, 2):
        val = val * (-res.tau[i])
    return val


def tridiag_solve(tau, rhs, tol_scale=10.0):
    """T y = rhs by Gaussian elimination with partial pivoting, one extra
    superdiagonal of fill (apps.py:33-73).  Raises ZeroDivisionError where the
    reference raises SingularT (pivot at or below tol_scale eps max|tau|)."""
    m = len(tau) + 1
    x = np.array(rhs, dtype=float)
    if x.shape[0] != m:
        raise ValueError("dimension mismatch")
    d = np.zeros(m)
    e = np.zeros(m)
    f2 = np.zeros(m)
    sub = np.array(tau, dtype=float)
    if m > 1:
        e[:m - 1] = -sub
    big = float(np.max(np.abs(sub))) if m > 1 else 0.0
    thresh = tol_scale * np.finfo(float).eps * big
    for k in range(m - 1):
        if abs(sub[k]) > abs(d[k]):
            d[k], sub[k] = sub[k], d[k]
            e[k], d[k + 1] = d[k + 1], e[k]
            if k + 2 < m:
                f2[k], e[k + 1] = e[k + 1], f2[k]
            x[[k, k + 1]] = x[[k + 1, k]]
        if abs(d[k]) <= thresh:
            raise ZeroDivisionError(f"tridiagonal pivot at row {k}")
        mult = sub[k] / d[k]
        d[k + 1] -= mult * e[k]
        if k + 2 < m:
            e[k + 1] -= mult * f2[k]
        x[k + 1] -= mult * x[k]
    if abs(d[m - 1]) <= thresh:
        raise ZeroDivisionError(f"tridiagonal pivot at row {m - 1}")
    x[m - 1] /= d[m - 1]
    if m > 1:
        x[m - 2] = (x[m - 2] - e[m - 2] * x[m - 1]) / d[m - 2]
    for k in range(m - 3, -1, -1):
        x[k] = (x[k] - e[k] * x[k + 1] - f2[k] * x[k + 2]) / d[k]
    return x


def solve(x, b, block=None, tol_scale=10.0):
    """X y = b through the pivoted factorization (apps.py:76-100): permute,
    unit-lower solve, pivoted tridiagonal solve, transposed unit-lower solve,
    permute back.  Multiple right-hand sides as columns."""
    from scipy.linalg import solve_triangular
    x = np.asarray(x)
    m = x.shape[0]
    b = np.asarray(b, dtype=float)
    one_d = b.ndim == 1
    rhs = b.reshape(m, -1) if one_d else b
    if rhs.shape[0] != m:
        raise ValueError("dimension mismatch")
    res = ltlt_blk_piv(x, b=block or min(DEFAULT_BLOCK, m))
    perm = compose_permutation(res.pivots)
    z = rhs[perm]
    ld = l_dense(res.work)
    z = solve_triangular(ld, z, lower=True, unit_diagonal=True)
    z = tridiag_solve(res.tau, z, tol_scale=tol_scale)
    z = solve_triangular(ld, z, trans="T", lower=True, unit_diagonal=True)
    out = np.empty_like(z)
    out[perm] = z
    return out.ravel() if one_d else out


def pfaffian_slog(tau, pivots, m):
    """(sign, log|Pf|) from tau and the pivot parity; overflow-free form of
    apps.py:26-30.  Pf = sign(P) prod_{i even} (-tau_i)."""
    if m == 0:
        return 1.0, 0.0
    if m % 2:
        return 0.0, -math.inf
    sign = -1.0 if np.count_nonzero(pivots) % 2 else 1.0
    even = np.asarray(tau[0:m - 1:2], dtype=np.float64)
    if np.any(even == 0):
        return 0.0, -math.inf
    sign *= float(np.prod(np.sign(-even)))
    return sign, float(np.sum(np.log(np.abs(even))))


def pivot_margins(x, b=DEFAULT_BLOCK):
    """Top-2 relative margin of every argmax in a pivoted factorization
    (diagnostic for pivot parity; reruns the var1 driver with a hook)."""
    work, tau = _workbuf(np.asarray(x, dtype=np.float64))
    m = work.shape[0]
    pivots = np.zeros(m, dtype=np.int64)
    margins = np.full(m, np.inf)
    r = 0
    while r < m - 1:
        be = min(b, m - 1 - r)
        for g in range(r, r + be):
            if g - r >= 2:
                skew_tridiag_gemv(work[g + 1:, g], -1, work[:, r:g], tau[r + 1:g],
                                  work[g, r:g], tail_from=g + 1)
            col = np.abs(work[g + 1:, g])
            if col.size >= 2:
                top = np.partition(col, -2)[-2:]
                hi = max(top)
                margins[g] = (hi - min(top)) / hi if hi else np.inf
            eliminate(work, tau, g, True, pivots, r)
        _block_pivots(work, pivots, r, be, r, _NULL)
        rt = r + be
        _apply_couplings(work, tau, r + 1, rt, rt, _NULL)
        _straggler(work, tau, rt, _NULL)
        r = rt
    return margins
