"""The error the decoder sees: the collage error with the QUANTISED offset (reading R10).

The encoder (oracle and GPU alike) chooses and accepts a leaf by E = sum (s d + o - r)^2 with the
exact o = Rbar - s Dbar (§2 Eq. 1 and 3); the code stores o through the 8-bit
quantiser (R11) and the decoder uses its cell centre o_hat (R23).  Because o minimises E for the
leaf's s, sum (s d + o - r) = 0, so

    E_q = sum (s d + o_hat - r)^2 = E + n (o_hat - o)^2                                  (*)

and |o_hat - o| <= w / 2 (w = 510/256) whenever o lies inside the quantiser's range.  These tests
pin (*) by brute force on every accepted leaf of an oracle encode (recomputing each leaf's
domain block, isometry and sums from the image, independently of the oracle's moment form) and
report how often an accepted leaf's RMS exceeds the tolerance once o is quantised (SPEC's
quantised-error rule binds SPEC's CPU program, not this encoder: DESIGN.md R10).
"""
import numpy as np

import oracle
from fic_inputs import config, image_for

W = 510.0 / 256.0


def iso_np(X, k):
    """out(i, j) = X(f_k(i, j)), reading R2 (the oracle's isometry order)."""
    b = X.shape[0] - 1
    out = np.empty_like(X)
    for i in range(X.shape[0]):
        for j in range(X.shape[1]):
            si, sj = [(i, j), (b - j, i), (b - i, b - j), (j, b - i), (i, b - j), (j, i), (b - i, j), (b - j, b - i)][k]
            out[i, j] = X[si, sj]
    return out


def quantised_errors(cfg):
    img = image_for(cfg)
    rec = oracle.encode_cfg(cfg, img)
    levels = [cfg["B_max"] >> l for l in range(len(cfg["s"]))]
    rows = []
    for r in rec:
        B = int(r["B"])
        s = cfg["s"][levels.index(B)][int(r["s_idx"])]
        R = img[r["ry"]:r["ry"] + B, r["rx"]:r["rx"] + B].astype(np.float64)
        Dp = img[r["dy"]:r["dy"] + 2 * B, r["dx"]:r["dx"] + 2 * B].astype(np.float64)
        d = (Dp[0::2, 0::2] + Dp[0::2, 1::2] + Dp[1::2, 0::2] + Dp[1::2, 1::2]) / 4.0  # R1
        d = iso_np(d, int(r["iso"]))
        n = B * B
        o = R.mean() - s * d.mean()
        o_hat = oracle.o_value(int(r["o_code"]))
        E_direct = float(((s * d + o - R) ** 2).sum())
        Eq_direct = float(((s * d + o_hat - R) ** 2).sum())
        rows.append((B, n, s, o, o_hat, float(r["err"]), E_direct, Eq_direct, bool(r["accepted"])))
    return rows


def test_quantised_error_identity_c2():
    cfg = config("C2")
    rows = quantised_errors(cfg)
    assert len(rows) > 1000
    for B, n, s, o, o_hat, E, E_d, Eq_d in (r[:8] for r in rows):
        scale = max(1.0, E_d, Eq_d)
        assert abs(E - E_d) <= 1e-9 * scale                     # the record's err is the plain SSE
        assert abs(Eq_d - (E_d + n * (o_hat - o) ** 2)) <= 1e-9 * scale   # (*)
        if -255.0 <= o <= 255.0:
            assert abs(o_hat - o) <= W / 2 + 1e-12


def test_quantised_rms_excess_is_bounded_c2():
    # how often an accepted leaf exceeds the tolerance once o is quantised, and by how much:
    # RMS_q^2 = E / n + (o_hat - o)^2 <= t^2 + (w/2)^2 for in-range o
    t = 8.0
    cfg = config("C2", t=t)
    # leaves accepted by the tolerance test (the last level's leaves are accepted unconditionally, R15)
    rows = [r for r in quantised_errors(cfg) if r[8] and r[5] <= t * t * r[1]]
    over = [r for r in rows if r[7] > t * t * r[1] * (1 + 1e-12)]
    frac = len(over) / len(rows)
    worst = max(np.sqrt(r[7] / r[1]) for r in rows)
    print(f"C2 t={t}: {len(over)} of {len(rows)} accepted leaves ({100 * frac:.2f}%) exceed the RMS "
          f"tolerance with the quantised o; worst RMS {worst:.4f} (bound {np.sqrt(t * t + (W / 2) ** 2):.4f})")
    in_range = [r for r in rows if -255.0 <= r[3] <= 255.0]
    assert all(np.sqrt(r[7] / r[1]) <= np.sqrt(t * t + (W / 2) ** 2) + 1e-9 for r in in_range)
    assert frac < 0.5
