"""Pins of the oracle's PIFS decoder and PSNR (readings R23-R26).

The paper only encodes; decoding is the standard PIFS iteration implied by P:28-30 and PSNR is
the metric of P:136-175.  Each check compares the oracle with something other than itself:
the quantiser cell geometry, closed forms (s = 0 codes, the scalar recursion a uniform code
reduces to, PSNR at MSE = 1), numpy's rot90/fliplr/reshape re-derivation of one pass, and
composition / contraction invariants.
"""
import math

import numpy as np
import pytest

import oracle
from fic_inputs import config, image_for, make_image

W = 510.0 / 256.0


def rand_code(rng, N, sizes, s_sets, B_max):
    """A random quadtree-shaped code: top blocks of B_max, each either a leaf or split once."""
    recs = []
    for ty in range(0, N, B_max):
        for tx in range(0, N, B_max):
            split = len(sizes) > 1 and rng.random() < 0.5
            B = sizes[1] if split else sizes[0]
            for y in range(ty, ty + B_max, B):
                for x in range(tx, tx + B_max, B):
                    l = sizes.index(B)
                    recs.append((x, y, B, 0, int(rng.integers(0, N - 2 * B + 1)),
                                 int(rng.integers(0, N - 2 * B + 1)), int(rng.integers(0, 8)),
                                 int(rng.integers(0, len(s_sets[l]))), int(rng.integers(0, 256)), 1, 0.0))
    return np.array(recs, dtype=oracle.RECORD_DTYPE)


def iso_np(X, k):
    """T_k by numpy primitives (reading R2): rotations clockwise, k >= 4 mirrored after."""
    Y = np.rot90(X, -(k & 3))
    return np.fliplr(Y) if k >= 4 else Y


# ----------------------------------------------------------------------------- o dequantiser
def test_o_value_is_cell_centre():
    assert oracle.o_value(128) == 0.99609375          # o = 0 -> code 128 (R11)
    assert oracle.o_value(0) == -254.00390625         # o = -255 -> code 0
    assert oracle.o_value(255) == 254.00390625
    for c in range(256):
        assert oracle.o_code(oracle.o_value(c)) == c  # the centre lies in its own cell
    rng = np.random.default_rng(3)
    for o in rng.uniform(-255, 255, 2000):
        assert abs(oracle.o_value(oracle.o_code(o)) - o) <= W / 2


# ----------------------------------------------------------------------------- closed forms
def test_s_zero_code_is_constant_per_range():
    rng = np.random.default_rng(5)
    N, s_sets = 32, [(0.0,), (0.0,)]
    code = rand_code(rng, N, [8, 4], s_sets, 8)
    want = np.zeros((N, N), np.uint8)
    for r in code:
        want[r["ry"]:r["ry"] + r["B"], r["rx"]:r["rx"] + r["B"]] = min(255, max(0, round_half_even(
            (r["o_code"] - 127.5) * W)))
    for it in (1, 2, 5):
        for init in (None, make_image(N, 9)):
            assert np.array_equal(oracle.decode(code, N, s_sets, 8, it, init), want)


def round_half_even(x):
    f = math.floor(x)
    d = x - f
    if d > 0.5 or (d == 0.5 and f % 2 == 1):
        return f + 1
    return f


def test_uniform_code_follows_scalar_recursion():
    # every record has the same (s, o): a constant image stays constant and each pixel follows
    # x <- clamp(rint(s x + o^)) (reading R24) from x0 = 128, whatever the domains and isometries
    for s, c in [(0.9, 140), (0.5, 60), (0.3, 255), (0.8, 0)]:
        rng = np.random.default_rng(c)
        N = 32
        code = rand_code(rng, N, [8, 4], [(s,), (s,)], 8)
        code["o_code"] = c
        x = 128
        for it in range(16):
            got = oracle.decode(code, N, [(s,), (s,)], 8, it)
            assert np.all(got == x), (s, c, it, x)
            x = min(255, max(0, round_half_even(s * x + (c - 127.5) * W)))


# ----------------------------------------------------------------------------- one pass by numpy
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_one_pass_matches_numpy(seed):
    rng = np.random.default_rng(seed)
    N = 32
    s_sets = [(0.2, 0.4), (0.3, 0.8)]
    code = rand_code(rng, N, [8, 4], s_sets, 8)
    prev = make_image(N, 40 + seed)
    want = prev.copy()
    for r in code:
        B = int(r["B"])
        blk = prev[r["dy"]:r["dy"] + 2 * B, r["dx"]:r["dx"] + 2 * B].astype(np.int64)
        d = blk.reshape(B, 2, B, 2).sum(axis=(1, 3)) / 4.0
        s = s_sets[[8, 4].index(B)][r["s_idx"]]
        v = np.rint(s * iso_np(d, int(r["iso"])) + (int(r["o_code"]) - 127.5) * W)
        want[r["ry"]:r["ry"] + B, r["rx"]:r["rx"] + B] = np.clip(v, 0, 255).astype(np.uint8)
    assert np.array_equal(oracle.decode(code, N, s_sets, 8, 1, prev), want)


# ----------------------------------------------------------------------------- PSNR
def test_psnr_closed_forms():
    a = make_image(16, 1)
    assert oracle.psnr(a, a) == math.inf
    b = a.astype(np.int32)
    b = np.where(b < 255, b + 1, b - 1).astype(np.uint8)          # |diff| = 1 everywhere: MSE = 1
    assert oracle.psnr(a, b) == pytest.approx(10 * math.log10(255 ** 2), abs=1e-12)
    c = a.copy()
    c[3, 5] = (int(c[3, 5]) + 16) % 256 if c[3, 5] < 240 else int(c[3, 5]) - 16   # one pixel off by 16
    assert oracle.psnr(a, c) == pytest.approx(10 * math.log10(255 ** 2 / (256 / 256)), abs=1e-12)


# ----------------------------------------------------------------------------- encode -> decode
def test_encode_decode_sanity_c2():
    cfg = config("C2")
    img = image_for(cfg)
    code = oracle.encode_cfg(cfg, img)
    outs = [oracle.decode(code, cfg["N"], cfg["s"], cfg["B_max"], it) for it in range(1, 13)]
    # composition: one more pass from decode(n) equals decode(n + 1)
    assert np.array_equal(oracle.decode(code, cfg["N"], cfg["s"], cfg["B_max"], 1, outs[4]), outs[5])
    # contraction (empirical contract, all s <= 0.9): max change nonincreasing after pass 2
    deltas = [int(np.abs(outs[i + 1].astype(int) - outs[i].astype(int)).max()) for i in range(len(outs) - 1)]
    assert all(deltas[i + 1] <= deltas[i] for i in range(1, len(deltas) - 1)), deltas
    assert deltas[-1] <= 1
    # sanity (not a paper value: different images): a t = 8 code decodes to a usable image
    assert oracle.psnr(img, outs[-1]) > 24.0
