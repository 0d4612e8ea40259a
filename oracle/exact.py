"""Exact-arithmetic references (TEST ORACLE ONLY; small sizes, pure Python).

Restates the reference's rational Gauss-transform elimination
(``oracle.py:79-134``) and brute-force Pfaffian (``oracle.py:137-161``).
They carry the full mirrored matrix and fractions.Fraction entries, so they
are independent of both BLAS and the lower-storage drivers.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

EXACT_SIZE_CAP = 16          # oracle.py:18
PFAFFIAN_BRUTE_CAP = 12      # oracle.py:19


def _full_exact(lower):
    m = lower.shape[0]
    full = [[Fraction(0)] * m for _ in range(m)]
    for j in range(m):
        for i in range(j + 1, m):
            v = lower[i, j]
            f = v if isinstance(v, Fraction) else Fraction(v.item() if hasattr(v, "item") else v)
            full[i][j] = f
            full[j][i] = -f
    return full


def gauss_elim_exact(lower, pivot=False):
    """L T L^T by explicit Gauss transforms in exact arithmetic.

    Returns (L as list-of-lists of Fraction, tau list, pivots int64 array).
    Ties in the pivot search resolve to the lowest index (strict '>'),
    as in oracle.py:103-108.
    """
    lower = np.asarray(lower, dtype=object)
    m = lower.shape[0]
    if m > EXACT_SIZE_CAP:
        raise ValueError(f"exact elimination capped at m={EXACT_SIZE_CAP}")
    x = _full_exact(lower)
    lmat = [[Fraction(int(i == j)) for j in range(m)] for i in range(m)]
    tau = [Fraction(0)] * max(m - 1, 0)
    pivots = np.zeros(m, dtype=np.int64)
    for k in range(m - 1):
        if pivot:
            off, best = 0, abs(x[k + 1][k])
            for i in range(1, m - k - 1):
                v = abs(x[k + 1 + i][k])
                if v > best:
                    best, off = v, i
            pivots[k + 1] = off
            if off:
                a, b = k + 1, k + 1 + off
                x[a], x[b] = x[b], x[a]
                for row in x:
                    row[a], row[b] = row[b], row[a]
                for c in range(k + 1):
                    lmat[a][c], lmat[b][c] = lmat[b][c], lmat[a][c]
        piv = x[k + 1][k]
        tau[k] = piv
        if piv == 0:
            if any(x[i][k] != 0 for i in range(k + 2, m)):
                raise ZeroDivisionError(f"zero pivot while eliminating column {k}")
            continue
        for i in range(k + 2, m):
            li = x[i][k] / piv
            if li == 0:
                continue
            lmat[i][k + 1] = li
            x[i] = [x[i][c] - li * x[k + 1][c] for c in range(m)]
            for r in range(m):
                x[r][i] = x[r][i] - li * x[r][k + 1]
    return lmat, tau, pivots


def pfaffian_bruteforce(lower):
    """Signed sum over perfect matchings by first-row expansion."""
    lower = np.asarray(lower, dtype=object)
    m = lower.shape[0]
    if m % 2:
        return 0
    if m > PFAFFIAN_BRUTE_CAP:
        raise ValueError(f"brute-force Pfaffian capped at m={PFAFFIAN_BRUTE_CAP}")
    full = _full_exact(lower)

    def pf(rows):
        if not rows:
            return Fraction(1)
        r0 = rows[0]
        acc = Fraction(0)
        for pos in range(1, len(rows)):
            sign = 1 if pos % 2 else -1
            rest = rows[1:pos] + rows[pos + 1:]
            acc += sign * full[r0][rows[pos]] * pf(rest)
        return acc

    return pf(list(range(m)))
