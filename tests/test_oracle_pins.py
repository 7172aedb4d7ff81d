"""Pins of the CPU oracle (oracle/) against what the paper and mathematics fix.

Every check here compares the oracle with something other than itself: closed forms, values the
paper prints (tests/golden/paper_constants.json), library routines (numpy rot90/fliplr, mpmath),
exact-rational literal Eq. (1)-(5) brute force (oracle/exact.py), and invariants.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import exact
from fic_inputs import PREDEFINED_S, GRID_S, random_image, ramp_image, constant_image, make_image

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))
TWO32 = 2 ** 32
W = Fraction(510, 256)


# ----------------------------------------------------------------------------- paper constants
def test_s_schedule_matches_paper():
    g = GOLD["s_schedule"]
    for B in (16, 8, 4, 2):
        assert tuple(g[str(B)]) == PREDEFINED_S[B]
    assert GRID_S[0] == 0.0 and GRID_S[-1] == 1.0 and len(GRID_S) == 16


@pytest.mark.parametrize("N,n", GOLD["counts"]["cases"])
def test_candidate_and_range_counts(N, n):
    # (N - 2n + 1)^2 domain blocks at step 1, (N/n)^2 range blocks
    assert oracle.axis_candidates(N, n, 1) ** 2 == (N - 2 * n + 1) ** 2
    for L in (2, 3, 4):
        A = oracle.axis_candidates(N, n, L)
        xs = [x for x in range(0, N) if x % L == 0 and x + 2 * n <= N]
        assert A == len(xs)


def test_c4_domain_count():
    assert oracle.axis_candidates(1024, 8, 1) ** 2 == 1009 ** 2 == 1018081


# ----------------------------------------------------------------------------- entropy
def test_lut_correctly_rounded_mpmath():
    lut = oracle.lut(4096)
    for c in list(range(0, 1100)) + list(range(1100, 4097, 97)) + [4095, 4096]:
        assert int(lut[c]) == exact.lut_entry(c), c


def _single_block_keys(block):
    # an image that is exactly one 2B x 2B candidate (N = 2B, step 1)
    side = block.shape[0]
    keys, keep, H = oracle.entropy_keys(block.astype(np.uint8), side // 2, 1, -1.0)
    assert keys.size == 1
    return int(keys[0]), float(H[0])


def test_entropy_closed_forms():
    # constant -> 0 ; two symbols 8/8 -> ln 2 ; 16 distinct -> ln 16 (Eq. 4-5)
    k, H = _single_block_keys(np.full((4, 4), 9))
    assert k == 0 and H == 0.0
    two = np.array([3] * 8 + [200] * 8).reshape(4, 4)
    k, H = _single_block_keys(two)
    assert k == 16 * TWO32 and abs(H - math.log(2)) < 1e-15
    k, H = _single_block_keys(np.arange(16).reshape(4, 4) * 7)
    assert k == 64 * TWO32 and abs(H - math.log(16)) < 1e-14
    # 256 distinct levels in a 16x16 block -> ln 256
    k, H = _single_block_keys(np.random.default_rng(0).permutation(256).reshape(16, 16))
    assert k == 256 * 8 * TWO32 and abs(H - math.log(256)) < 1e-13


@pytest.mark.parametrize("B", [2, 4, 8])
def test_entropy_keys_vs_exact(B):
    img = random_image(4 * B, seed=B, lo=0, hi=15 if B > 2 else 255)
    keys, keep, H = oracle.entropy_keys(img, B, B // 2 if B > 1 else 1, -1.0)
    A = oracle.axis_candidates(img.shape[0], B, B // 2)
    m = 4 * B * B
    for c in range(keys.size):
        x, y = (c % A) * (B // 2), (c // A) * (B // 2)
        Hx = exact.entropy(img[y:y + 2 * B, x:x + 2 * B])
        assert abs(float(Hx) - H[c]) < 1e-12
        assert abs(int(keys[c]) * math.log(2) / (m * TWO32) - float(Hx)) < 1e-9


def test_entropy_invariance_isometry_and_permutation():
    # P:96 "all permutations constructed by rearranging pixels of the block have the same entropy"
    rng = np.random.default_rng(5)
    blk = rng.integers(0, 40, size=(8, 8))
    k0, _ = _single_block_keys(blk)
    for k in range(8):
        assert _single_block_keys(exact.isometry(blk, k))[0] == k0
    for _ in range(5):
        assert _single_block_keys(rng.permutation(blk.ravel()).reshape(8, 8))[0] == k0


def test_keep_is_strict_threshold():
    img = make_image(64, 3)
    keys, _, H = oracle.entropy_keys(img, 4, 2, -1.0)
    for tau in (2.0, 3.0, 3.5, 3.9):
        _, keep, _ = oracle.entropy_keys(img, 4, 2, tau)
        for c in range(keys.size):
            Hx = int(keys[c]) * math.log(2) / (64 * TWO32)
            if abs(Hx - tau) > 1e-9:
                assert bool(keep[c]) == (Hx > tau)
    _, keep, _ = oracle.entropy_keys(img, 4, 2, -1.0)
    assert keep.all()
    # the two-symbol block sits exactly at ln 2: "greater than" drops it
    two = np.array([3] * 8 + [200] * 8).reshape(4, 4).astype(np.uint8)
    assert oracle.entropy_keys(two, 2, 1, 0.6931)[1][0] == 1
    assert oracle.entropy_keys(two, 2, 1, 0.6932)[1][0] == 0


def test_pool_monotone_in_tau():
    img = make_image(64, 4)
    k1 = set(oracle.kept_list(img, 4, 2, 3.0).tolist())
    k2 = set(oracle.kept_list(img, 4, 2, 3.6).tolist())
    assert k2 <= k1 and len(k2) < len(k1)


# ----------------------------------------------------------------------------- decimation, isometries
def test_decimate_examples():
    img = np.array([[0, 2], [4, 6]], np.uint8)
    pad = np.zeros((4, 4), np.uint8)
    pad[:2, :2] = img
    D = oracle.decimate(pad, 0, 0, 1)  # a single 2x2 cell
    assert D[0, 0] == 12  # sum; mean 3
    assert (oracle.decimate(np.full((8, 8), 7, np.uint8), 0, 0, 4) == 28).all()
    pad[:2, :2] = [[0, 0], [0, 1]]
    assert oracle.decimate(pad, 0, 0, 1)[0, 0] == 1  # mean 0.25


def test_decimate_isometry_equivariant():
    rng = np.random.default_rng(1)
    blk = rng.integers(0, 256, size=(16, 16)).astype(np.uint8)
    for k in range(8):
        lhs = oracle.decimate(np.ascontiguousarray(exact.isometry(blk, k)).astype(np.uint8), 0, 0, 8)
        rhs = oracle.isometry(oracle.decimate(blk, 0, 0, 8), k)
        assert (lhs == rhs).all()


def test_isometry_example_and_library():
    X = np.array([[1, 2], [3, 4]])
    assert (oracle.isometry(X, 1) == [[3, 1], [4, 2]]).all()  # clockwise 90
    rng = np.random.default_rng(2)
    for B in (2, 3, 4, 8, 16, 32):
        X = rng.integers(0, 1000, size=(B, B))
        for k in range(8):
            assert (oracle.isometry(X, k) == exact.isometry(X, k)).all(), (B, k)


def test_isometry_group_closure():
    X = np.arange(16).reshape(4, 4)
    imgs = [oracle.isometry(X, k) for k in range(8)]
    keys = [im.tobytes() for im in imgs]
    assert len(set(keys)) == 8  # 8 distinct maps (original + 7 new)
    for a in range(8):
        for b in range(8):
            assert oracle.isometry(imgs[a], b).tobytes() in keys
    Y = X
    for _ in range(4):
        Y = oracle.isometry(Y, 1)
    assert (Y == X).all()
    for k in range(4, 8):  # mirrors are involutions
        assert (oracle.isometry(oracle.isometry(X, k), k) == X).all()


# ----------------------------------------------------------------------------- quantiser
def _exact_code(o: Fraction) -> int:
    if o >= 0:
        mu = o / W
        j = 0 if mu == 0 else math.ceil(mu) - 1
        return 128 + min(j, 127)
    mu = -o / W
    return 127 - min(math.ceil(mu) - 1, 127)


def test_o_code_quantiser():
    rng = np.random.default_rng(3)
    vals = list(rng.uniform(-255, 255, 2000)) + [-255.0, -254.0, -1.9921875, -1.0, -1e-12, 0.0,
                                                1e-12, 1.9921875, 2.0, 255.0]
    vals += [k * 1.9921875 for k in range(-128, 129)]
    prev = None
    for o in sorted(vals):
        code = oracle.o_code(o)
        assert code == _exact_code(Fraction(o))
        assert 0 <= code <= 255
        ohat = (Fraction(code) - Fraction(255, 2)) * W
        assert abs(ohat - Fraction(o)) <= W / 2 + Fraction(1, 10 ** 9) or abs(o) > 254
        if prev is not None:
            assert code >= prev
        prev = code
    assert oracle.o_code(0.0) == 128 and oracle.o_code(-255.0) == 0 and oracle.o_code(255.0) == 255


# ----------------------------------------------------------------------------- Eq. (1)-(3) brute force
def _check_level_vs_bruteforce(img, B, L, s_list, tau=-1.0):
    N = img.shape[0]
    kept = oracle.kept_list(img, B, L, tau)
    ranges = np.array([(u * B, v * B) for v in range(N // B) for u in range(N // B)], np.int32)
    rec = oracle.encode_level(img, B, L, kept, ranges, s_list, 0.0, True)
    A = oracle.axis_candidates(N, B, L)
    for r, (rx, ry) in enumerate(ranges):
        Emin, winners, table = exact.brute_force_range(img, int(rx), int(ry), B, L, kept, s_list)
        c, k, j = int(rec["dom"][r]), int(rec["iso"][r]), int(rec["s_idx"][r])
        R = [int(v) for v in img[ry:ry + B, rx:rx + B].ravel()]
        cand = int(kept[c])
        D = np.array(exact.decimated(img, (cand % A) * L, (cand // A) * L, B), dtype=object)
        Dk = list(exact.isometry(D, k).ravel())
        scale = exact.score_scale(R, Dk, s_list[j])
        tol = float(scale) * 2.0 ** -48 + 1e-300
        Echoice = table[(c, k, j)]
        # the oracle's choice is an exact minimiser up to binary64 rounding of Eq. (1)
        assert float(Echoice - Emin) <= tol, (rx, ry)
        assert abs(float(rec["err"][r]) - float(Echoice)) <= tol
        # E >= 0 (Eq. 1 is a sum of squares), up to rounding
        assert rec["err"][r] >= -tol
        # dominance of the closed form (Eq. 2) over any s in [0, 1]
        sstar = exact.eq2_s(R, Dk)
        assert exact.eq1_error_exact_s(R, Dk, sstar) <= Echoice
        # uniqueness: when the exact minimiser is unique and well separated it must be chosen
        if len(winners) == 1:
            second = min(v for key, v in table.items() if key not in winners)
            if float(second - Emin) > 4 * tol:
                assert (c, k, j) in winners
        # dx, dy, o (Eq. 3), o-code
        assert rec["dx"][r] == (cand % A) * L and rec["dy"][r] == (cand // A) * L
        o = Fraction(sum(R), B * B) - Fraction(s_list[j]) * Fraction(sum(sum(x) for x in D.tolist()), B * B)
        assert rec["o_code"][r] == _exact_code(o)


def test_level_bruteforce_b2_predefined():
    img = make_image(16, 11)
    _check_level_vs_bruteforce(img, 2, 2, PREDEFINED_S[2])


def test_level_bruteforce_b2_grid_random():
    img = random_image(12, 12)
    _check_level_vs_bruteforce(img, 2, 2, GRID_S)


def test_level_bruteforce_b4_entropy_filtered():
    img = make_image(24, 13)
    _check_level_vs_bruteforce(img, 4, 4, PREDEFINED_S[4], tau=2.5)


def test_level_bruteforce_b8_odd_step():
    img = random_image(24, 14, 0, 60)
    _check_level_vs_bruteforce(img, 8, 3, PREDEFINED_S[8])


def test_ls_dominance_random_blocks():
    rng = np.random.default_rng(7)
    for _ in range(200):
        B = int(rng.choice([2, 4, 8]))
        R = [int(v) for v in rng.integers(0, 256, B * B)]
        D = [Fraction(int(v), 4) for v in rng.integers(0, 1021, B * B)]
        sstar = exact.eq2_s(R, D)
        Estar = exact.eq1_error_exact_s(R, D, sstar)
        assert Estar >= 0
        for s in list(PREDEFINED_S[B]) + list(GRID_S):
            assert exact.eq1_error(R, D, s) >= Estar


# ----------------------------------------------------------------------------- degenerate cases
def test_ramp_zero_error():
    img = ramp_image(64)
    N, B, L = 64, 2, 2
    kept = oracle.kept_list(img, B, L, -1.0)
    ranges = np.array([(u * B, v * B) for v in range(N // B) for u in range(N // B)], np.int32)
    rec = oracle.encode_level(img, B, L, kept, ranges, PREDEFINED_S[2], 0.0, True)
    assert (rec["err"] == 0.0).all()
    assert (rec["dom"] == 0).all() and (rec["iso"] == 0).all() and (rec["s_idx"] == 0).all()


def test_constant_image_no_split():
    img = constant_image(64, 77)
    rec = oracle.encode(img, 16, 2, 4, [-1.0] * 4, [PREDEFINED_S[b] for b in (16, 8, 4, 2)],
                        [0.0] * 4)
    assert len(rec) == 16 and (rec["B"] == 16).all() and (rec["err"] == 0.0).all()
    # constant range: e = s^2 C / 16 = 0 for every domain -> lowest (c, k, j) = (0, 0, 0)
    assert (rec["dom"] == 0).all() and (rec["iso"] == 0).all() and (rec["s_idx"] == 0).all()


def test_constant_range_grid_s0_wins():
    img = make_image(32, 21)
    img[0:4, 0:4] = 100
    kept = oracle.kept_list(img, 4, 2, -1.0)
    rec = oracle.encode_level(img, 4, 2, kept, np.array([[0, 0]], np.int32), GRID_S, 0.0, True)
    assert rec["err"][0] == 0.0 and rec["dom"][0] == 0 and rec["iso"][0] == 0 and rec["s_idx"][0] == 0
    # predefined s: e = s^2 C/16 -> the flattest domain (min C), lowest index, k = 0, j = 0
    rec = oracle.encode_level(img, 4, 2, kept, np.array([[0, 0]], np.int32), PREDEFINED_S[4], 0.0, True)
    A = oracle.axis_candidates(32, 4, 2)
    Cs = []
    for c in kept:
        D = oracle.decimate(img, (c % A) * 2, (c // A) * 2, 4).astype(np.int64)
        Cs.append(16 * int((D * D).sum()) - int(D.sum()) ** 2)
    assert rec["dom"][0] == int(np.argmin(Cs)) and rec["iso"][0] == 0 and rec["s_idx"][0] == 0


def _affine_copy_image(seed, N=32, B=2, L=2, s=0.5, n_copies=12):
    """Left half: pixel-doubled even values (each 2x2 cell constant, even) so d = D'/4 is an even
    integer; right half: ranges written as exact affine copies r = s * T_k(d) + o of left-half
    domains (reading of the north star's "exact affine copies of its own decimated domains")."""
    rng = np.random.default_rng(seed)
    img = rng.integers(0, 256, size=(N, N)).astype(np.int64)
    cells = rng.integers(0, 128, size=(N // 2, N // 4)) * 2
    img[:, : N // 2] = np.kron(cells, np.ones((2, 2), np.int64))
    targets = []
    A = (N - 2 * B) // L + 1
    right = [(u, v) for v in range(N // B) for u in range(N // B) if u * B >= N // 2]
    picks = rng.choice(len(right), size=n_copies, replace=False)
    for p in picks:
        u, v = right[p]
        while True:
            a, b = int(rng.integers(0, A)), int(rng.integers(0, A))
            if a * L + 2 * B <= N // 2:
                break
        k = int(rng.integers(0, 8))
        d = img[b * L:b * L + 2 * B:2, a * L:a * L + 2 * B:2]  # pixel-doubled: d equals a sample
        dk = exact.isometry(d, k)
        vals = (s * dk).astype(np.int64)
        o = int(rng.integers(0, 256 - int(vals.max())))
        img[v * B:(v + 1) * B, u * B:(u + 1) * B] = vals + o
        targets.append((u * B, v * B))
    return img.astype(np.uint8), targets


def test_exact_affine_copies_zero_error():
    img, targets = _affine_copy_image(31)
    B, L = 2, 2
    kept = oracle.kept_list(img, B, L, -1.0)
    ranges = np.array(targets, np.int32)
    rec = oracle.encode_level(img, B, L, kept, ranges, PREDEFINED_S[2], 0.0, True)
    for r, (rx, ry) in enumerate(targets):
        assert rec["err"][r] == 0.0
        Emin, winners, table = exact.brute_force_range(img, rx, ry, B, L, kept, PREDEFINED_S[2])
        assert Emin == 0
        zero = sorted(key for key, v in table.items() if v == 0)
        assert (int(rec["dom"][r]), int(rec["iso"][r]), int(rec["s_idx"][r])) == zero[0]


# ----------------------------------------------------------------------------- quadtree
FIELDS = ("rx", "ry", "B", "dom", "dx", "dy", "iso", "s_idx", "o_code", "accepted", "err")


def same_records(a, b):
    return len(a) == len(b) and all(np.array_equal(a[f], b[f]) for f in FIELDS)


def _paint(rec, N):
    cov = np.zeros((N, N), np.int32)
    for r in rec:
        cov[r["ry"]:r["ry"] + r["B"], r["rx"]:r["rx"] + r["B"]] += 1
    return cov


@pytest.mark.parametrize("t", [0.0, 4.0, 8.0, 1e9])
def test_quadtree_invariants(t):
    N = 64
    img = make_image(N, 9)
    s_sets = [PREDEFINED_S[b] for b in (16, 8, 4, 2)]
    rec = oracle.encode(img, 16, 2, 4, [-1.0] * 4, s_sets, [t] * 4)
    assert (_paint(rec, N) == 1).all()  # leaves tile the image
    n = rec["B"].astype(np.float64) ** 2
    above = rec["B"] > 2
    assert (rec["err"][above] <= t * t * n[above]).all()
    assert (rec["accepted"] == 1).all()
    order = list(zip(-rec["B"], rec["ry"], rec["rx"]))
    assert order == sorted(order)  # canonical output order
    if t == 1e9:
        assert (rec["B"] == 16).all()
    if t == 0.0:
        assert (rec["err"][above] == 0.0).all()


def test_quadtree_children_match_single_levels():
    """Level-by-level re-derivation: ranges at level B/2 are the children of rejected ranges."""
    N, t = 64, 6.0
    img = make_image(N, 10)
    s_sets = [PREDEFINED_S[b] for b in (16, 8, 4, 2)]
    full = oracle.encode(img, 16, 2, 4, [-1.0] * 4, s_sets, [t] * 4)
    ranges = [(u * 16, v * 16) for v in range(N // 16) for u in range(N // 16)]
    got = []
    for li, B in enumerate((16, 8, 4, 2)):
        kept = oracle.kept_list(img, B, 4, -1.0)
        rec = oracle.encode_level(img, B, 4, kept, np.array(ranges, np.int32), s_sets[li], t, B == 2)
        got += [r for r in rec if r["accepted"]]
        rej = [(int(r["rx"]), int(r["ry"])) for r in rec if not r["accepted"]]
        h = B // 2
        ranges = sorted([(x + dx, y + dy) for (x, y) in rej for dy in (0, h) for dx in (0, h)],
                        key=lambda p: (p[1], p[0]))
    got = np.array(got, dtype=oracle.RECORD_DTYPE)
    assert same_records(got, full)


def test_shards_union_is_whole():
    N = 64
    img = make_image(N, 12)
    s_sets = [PREDEFINED_S[b] for b in (16, 8, 4, 2)]
    full = oracle.encode(img, 16, 2, 4, [-1.0] * 4, s_sets, [8.0] * 4)
    parts = np.concatenate([oracle.encode(img, 16, 2, 4, [-1.0] * 4, s_sets, [8.0] * 4, sh, 3)
                            for sh in range(3)])
    order = np.lexsort((parts["rx"], parts["ry"], -parts["B"]))
    assert same_records(parts[order], full)


# ----------------------------------------------------------------------------- C7 bit pattern
C7 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c7_score_bits.json")))


def _c7_image():
    """8x8 image: range R at (0, 0) (B = 2), and at (4, 4) a raw 4x4 domain whose 2x2 sums are
    the worked example's D' (each cell four equal pixels D'/4)."""
    img = np.zeros((8, 8), np.uint8)
    img[0:2, 0:2] = np.array(C7["R"])
    D = np.array(C7["Dprime"])
    for i in range(2):
        for j in range(2):
            img[4 + 2 * i: 6 + 2 * i, 4 + 2 * j: 6 + 2 * j] = D[i, j] // 4
    return img


@pytest.mark.parametrize("s", sorted(C7["e_bits"]))
def test_c7_score_bits_golden(s):
    """The binary64 bits of the canonical score (reading C7) on the SURVEY §8(c) worked example:
    a reordering of the same real expression (e.g. (A + t2) - hs Bq) changes the err bits the
    GPU parity tests compare for equality, and fails here.  Single kept domain (candidate 3 at
    L = 4 = (4, 4)), single s: the record's err * n (exact, n = 4) is e."""
    img = _c7_image()
    assert np.array_equal(oracle.decimate(img, 4, 4, 2), np.array(C7["Dprime"]))
    rec = oracle.encode_level(img, 2, 4, np.array([3], np.int32), np.array([[0, 0]], np.int32),
                              (float(s),), 8.0, True)[0]
    assert (rec["dx"], rec["dy"], rec["dom"]) == (4, 4, 0)
    assert rec["iso"] == C7["winner_iso_predefined"]          # k = 3 and 7 tie on SRD: lowest k
    assert float(rec["err"]) * 4 == float(C7["e_bits"][s])    # exact scaling by n = 4
    assert repr(float(rec["err"]) * 4) == C7["e_bits"][s]


def test_c7_worked_example_pair_and_grid():
    img = _c7_image()
    kept = np.array([3], np.int32)
    r = np.array([[0, 0]], np.int32)
    rec = oracle.encode_level(img, 2, 4, kept, r, (0.5, 0.9), 8.0, True)[0]
    assert (rec["iso"], rec["s_idx"], rec["o_code"]) == (3, 0, C7["o_code"])
    assert float(rec["err"]) == 1125.0 / 4 == 281.25
    assert oracle.o_value(C7["o_code"]) == C7["o_hat"]
    g = oracle.encode_level(img, 2, 4, kept, r, GRID_S, 8.0, True)[0]
    assert g["s_idx"] == C7["grid_j15"]["j"] and repr(GRID_S[5]) == C7["grid_j15"]["s"]
    assert repr(float(g["err"]) * 4) == C7["grid_j15"]["e"]
    # the SRD_k list of the worked example, via the isometries of the oracle
    Rm = np.array(C7["R"])
    Dm = np.array(C7["Dprime"])
    assert [int((Rm * oracle.isometry(Dm, k)).sum()) for k in range(8)] == C7["SRD_k"]


# ----------------------------------------------------------------------------- tiny s
def test_tiny_s_first_minimiser_is_not_the_srd_argmax():
    """At s = 1e-16 the binary64 scores of distinct cross terms SRD_k round to the same value,
    so the first minimiser of (E; dom, k, j) (C8) is often a lower k than the isometry with the
    largest SRD, which wins at any licensed s (SURVEY §8(c) 'Licensed GPU shortcut' holds only for s above
    a floor; DESIGN.md §6 'Exactness').  This is the case the GPU's finalize re-derives; the
    GPU test test_tiny_s_parity compares it with this oracle."""
    img = make_image(32, 5)
    B, L = 4, 4
    kept = oracle.kept_list(img, B, L, -1.0)
    ranges = np.array([(u * B, v * B) for v in range(32 // B) for u in range(32 // B)], np.int32)
    tiny = oracle.encode_level(img, B, L, kept, ranges, (1e-16,), 8.0, True)
    differ = 0
    for r, (rx, ry) in zip(tiny, ranges):
        c = int(kept[r["dom"]])
        A = oracle.axis_candidates(32, B, L)
        D = oracle.decimate(img, (c % A) * L, (c // A) * L, B)
        R = img[ry:ry + B, rx:rx + B].astype(np.int64)
        srd = [int((R * oracle.isometry(D, k)).sum()) for k in range(8)]
        differ += int(np.argmax(srd)) != int(r["iso"])
        # the chosen isometry attains the domain's minimal score: re-scoring that domain alone
        # under the SRD-argmax isometry gives the same err
        one = oracle.encode_level(img, B, L, np.array([c], np.int32), np.array([[rx, ry]], np.int32),
                                  (1e-16,), 8.0, True)[0]
        assert one["err"] == r["err"]
    assert differ > 0
