"""O2 -- exact mini-oracle: the paper's formulas written out literally in exact arithmetic.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Pure-Python loops; only for tiny images.
Independent of fic_oracle.c: it uses the literal definitions, not the integer-moment form.

  Eq. (1)  E(R,D) = sum_i (s d_i + o - r_i)^2                     (§2, line 30)
  Eq. (2)  s* = <R - Rbar, D - Dbar> / ||D - Dbar||^2              (line 34)
  Eq. (3)  o = Rbar - s Dbar                                       (line 36)
  Eq. (4)  p_i = q_i / (number of pixels)                          (§3, line 52)
  Eq. (5)  entropy = -sum p_i ln p_i                               (line 56)
  decimation: d = mean of each 2x2 cell, kept exact                (line 30; reading R1)
  isometries: numpy rot90 (clockwise) and fliplr (horizontal mirror) (line 28; reading R2)
"""
from __future__ import annotations

from fractions import Fraction

import mpmath
import numpy as np


def lut_entry(c: int) -> int:
    """round-half-even(c * log2(c) * 2^32) at 200-bit precision (closed form of the key LUT)."""
    if c < 2:
        return 0
    with mpmath.workprec(200):
        v = mpmath.mpf(c) * mpmath.log(c, 2) * mpmath.mpf(2) ** 32
        fl = mpmath.floor(v)
        frac = v - fl
        r = int(fl)
        half = mpmath.mpf(1) / 2
        if frac > half or (frac == half and (r % 2 == 1)):
            r += 1
        return r


def entropy(values) -> mpmath.mpf:
    """Eq. (4)-(5): -sum p ln p over the gray levels present (natural log), 100-bit."""
    vals, counts = np.unique(np.asarray(values).ravel(), return_counts=True)
    m = int(counts.sum())
    with mpmath.workprec(100):
        return -mpmath.fsum(mpmath.mpf(int(q)) / m * mpmath.log(mpmath.mpf(int(q)) / m)
                            for q in counts)


def isometry(X: np.ndarray, k: int) -> np.ndarray:
    """k = 0..3: clockwise rotation by 90k degrees; k = 4..7: the same, then a horizontal mirror."""
    Y = np.rot90(np.asarray(X), -(k % 4))
    if k >= 4:
        Y = np.fliplr(Y)
    return np.ascontiguousarray(Y)


def decimated(img: np.ndarray, x: int, y: int, B: int):
    """B x B list of Fractions: mean of each 2x2 cell of the 2B x 2B block at (x, y)."""
    blk = np.asarray(img[y:y + 2 * B, x:x + 2 * B], dtype=np.int64)
    return [[Fraction(int(blk[2 * i, 2 * j] + blk[2 * i, 2 * j + 1] + blk[2 * i + 1, 2 * j]
                          + blk[2 * i + 1, 2 * j + 1]), 4) for j in range(B)] for i in range(B)]


def eq1_error(R, D, s) -> Fraction:
    """Eq. (1) with o from Eq. (3); R, D are flat sequences of Fractions/ints, s a float."""
    s = Fraction(s)
    n = len(R)
    Rbar = Fraction(sum(R), n)
    Dbar = Fraction(sum(D), n)
    o = Rbar - s * Dbar
    return sum((s * d + o - r) ** 2 for d, r in zip(D, R))


def eq2_s(R, D):
    """Eq. (2), clamped to [0,1]; s* = 0 for a flat domain (reading R12)."""
    n = len(R)
    Rbar = Fraction(sum(R), n)
    Dbar = Fraction(sum(D), n)
    num = sum((r - Rbar) * (d - Dbar) for r, d in zip(R, D))
    den = sum((d - Dbar) ** 2 for d in D)
    if den == 0:
        return Fraction(0)
    return min(max(num / den, Fraction(0)), Fraction(1))


def eq1_error_exact_s(R, D, s: Fraction) -> Fraction:
    n = len(R)
    Rbar = Fraction(sum(R), n)
    Dbar = Fraction(sum(D), n)
    o = Rbar - s * Dbar
    return sum((s * d + o - r) ** 2 for d, r in zip(D, R))


def score_scale(R, D, s) -> Fraction:
    """Magnitude of the terms of the expanded Eq. (1) (bounds binary64 cancellation error)."""
    s = Fraction(s)
    n = len(R)
    Rbar = Fraction(sum(R), n)
    Dbar = Fraction(sum(D), n)
    srr = sum((r - Rbar) ** 2 for r in R)
    srd = abs(sum((r - Rbar) * (d - Dbar) for r, d in zip(R, D)))
    sdd = sum((d - Dbar) ** 2 for d in D)
    return srr + 2 * s * srd + s * s * sdd


def brute_force_range(img, rx, ry, B, L, kept, s_list):
    """All (c, k, j) of one range with their exact Eq. (1) error.

    Returns (Emin, winners, table) where table[(c,k,j)] = exact E and winners is the set of
    (c,k,j) with E == Emin.
    """
    N = img.shape[0]
    A = (N - 2 * B) // L + 1
    R = [int(v) for v in np.asarray(img[ry:ry + B, rx:rx + B]).ravel()]
    table = {}
    for c, cand in enumerate(kept):
        x, y = (int(cand) % A) * L, (int(cand) // A) * L
        Dm = np.array(decimated(img, x, y, B), dtype=object)
        for k in range(8):
            Dk = list(isometry(Dm, k).ravel())
            for j, s in enumerate(s_list):
                table[(c, k, j)] = eq1_error(R, Dk, s)
    Emin = min(table.values())
    winners = {key for key, v in table.items() if v == Emin}
    return Emin, winners, table
