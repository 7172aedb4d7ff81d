"""Pins of the 5-bit closed-form s mode (NEXT-2; Eq. 2; reading R28): the s set is the 32
levels j/31 and the oracle searches them exhaustively.  Because Eq. (1) is a parabola in s with
its vertex at Eq. (2)'s s*, the winner must be the level nearest to the clamped s* -- checked here
against Eq. (2) and Eq. (1) literally in exact rationals (oracle/exact.py), not against the grid
search itself."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import exact
from fic_inputs import CLOSED5_S, make_image


def nearest_level(s_star):
    """Index of the level j/31 nearest to s* in [0, 1] (exact); ties -> None (either is optimal)."""
    best = min(range(32), key=lambda j: abs(Fraction(CLOSED5_S[j]) - s_star))
    d0 = abs(Fraction(CLOSED5_S[best]) - s_star)
    for j in (best - 1, best + 1):
        if 0 <= j < 32 and abs(Fraction(CLOSED5_S[j]) - s_star) == d0:
            return None
    return best


@pytest.mark.parametrize("seed,B", [(0, 4), (1, 4), (2, 2), (3, 8)])
def test_closed5_winner_is_nearest_level_to_eq2(seed, B):
    N, L = 24 if B < 8 else 32, 2
    img = make_image(N, 300 + seed)
    A = oracle.axis_candidates(N, B, L)
    kept = np.arange(A * A, dtype=np.int32)
    rng = np.random.default_rng(seed)
    G = N // B
    picks = rng.choice(G * G, 4, replace=False)
    ranges = np.stack([(picks % G) * B, (picks // G) * B], 1).astype(np.int32)
    recs = oracle.encode_level(img, B, L, kept, ranges, CLOSED5_S, 8.0, False)
    for (rx, ry), rec in zip(ranges, recs):
        R = [int(v) for v in img[ry:ry + B, rx:rx + B].ravel()]
        best_e, table = None, {}
        for c in range(A * A):
            x, y = (c % A) * L, (c // A) * L
            D = np.array(exact.decimated(img, x, y, B), dtype=object)   # d = D'/4 (Fractions)
            for k in range(8):
                Dk = list(exact.isometry(D, k).ravel())
                s_star = exact.eq2_s(R, Dk)                     # Eq. (2), clamped to [0, 1]
                j = nearest_level(s_star)
                js = [j] if j is not None else [jj for jj in range(32)
                                                 if abs(Fraction(CLOSED5_S[jj]) - s_star) <= Fraction(1, 62)]
                e = min(exact.eq1_error_exact_s(R, Dk, Fraction(CLOSED5_S[jj])) for jj in js)
                table[(c, k)] = (e, j)
                best_e = e if best_e is None or e < best_e else best_e
        c0, k0, j0 = int(rec["dom"]), int(rec["iso"]), int(rec["s_idx"])
        e_rec, j_near = table[(c0, k0)]
        scale = max(1.0, float(best_e))
        assert abs(rec["err"] - float(best_e)) <= 1e-9 * scale     # err = Eq. (1) at the optimum
        assert abs(float(e_rec) - float(best_e)) <= 1e-9 * scale   # the choice attains the minimum
        if j_near is not None:
            assert j0 == j_near                                    # ... at the level nearest s*


def test_closed5_levels():
    assert len(CLOSED5_S) == 32 and CLOSED5_S[0] == 0.0 and CLOSED5_S[-1] == 1.0
    assert np.allclose(np.diff(CLOSED5_S), 1 / 31)
