"""Pins of the oracle's top-K pool selection (the paper's "pool size" axis, Tables 1-2 P:154-166,
Fig. 4; reading R27: K largest entropies, ties to the lower row-major index, kept list in
row-major order).  Checked against brute-force entropy ranking (Eq. 4-5 by numpy histograms),
the threshold selection it must agree with, and set invariants."""
import math

import numpy as np
import pytest

import oracle
from fic_inputs import config, image_for, make_image, constant_image


def entropies(img, B, L):
    """Eq. (4)-(5) per candidate, natural log, by numpy histograms (row-major candidates)."""
    N = img.shape[0]
    A = oracle.axis_candidates(N, B, L)
    H = np.zeros(A * A)
    for c in range(A * A):
        x, y = (c % A) * L, (c // A) * L
        blk = img[y:y + 2 * B, x:x + 2 * B]
        cnt = np.sort(np.bincount(blk.ravel(), minlength=256))  # canonical order: equal
        p = cnt[cnt > 0] / blk.size                              # histograms -> equal floats
        H[c] = -math.fsum(p * np.log(p))
    return H


def test_spec_example_two_of_four_tiles():
    img = make_image(64, 7)
    H = entropies(img, 16, 32)            # 64x64, domain 32, step 32: four tiles
    assert H.size == 4
    want = np.sort(np.argsort(-H, kind="stable")[:2])
    assert np.array_equal(oracle.kept_list_topk(img, 16, 32, 2), want)


@pytest.mark.parametrize("N,B,L,K", [(48, 4, 3, 17), (64, 2, 5, 40), (64, 8, 4, 9), (40, 4, 1, 100)])
def test_brute_force_ranking(N, B, L, K):
    img = make_image(N, N + B + L)
    H = entropies(img, B, L)
    # exact ranking: m H = m ln m - sum_v c_v ln c_v, so H descending <=> prod_v c_v^c_v ascending
    # (big integers: exact, ties such as {4,4,4,4} ~ {8,2,2,2,2} are genuine and go to the lower index)
    A = oracle.axis_candidates(N, B, L)
    prod = []
    for c in range(A * A):
        x, y = (c % A) * L, (c // A) * L
        cnt = np.bincount(img[y:y + 2 * B, x:x + 2 * B].ravel(), minlength=256)
        prod.append(math.prod(int(v) ** int(v) for v in cnt if v > 0))
    order = sorted(range(A * A), key=lambda c: (prod[c], c))
    assert np.allclose(np.sort(H)[::-1], H[order])  # same ranking as the float entropies
    assert np.array_equal(oracle.kept_list_topk(img, B, L, K), np.sort(order[:min(K, A * A)]))


def test_all_kept_and_prefix():
    img = image_for(config("C2"))
    n_c = oracle.axis_candidates(256, 8, 4) ** 2
    assert np.array_equal(oracle.kept_list_topk(img, 8, 4, n_c + 5), np.arange(n_c))
    prev = set()
    for K in (1, 5, 32, 64, 256, 1000):
        cur = set(oracle.kept_list_topk(img, 8, 4, K))
        assert len(cur) == K and prev <= cur
        prev = cur


def test_agrees_with_threshold_selection():
    img = image_for(config("C2"))
    for B, L in ((16, 4), (4, 4)):
        keys, _, H = oracle.entropy_keys(img, B, L)
        hs = np.unique(H)
        for q in (0.2, 0.5, 0.9):
            i = int(q * (hs.size - 1))
            tau = (hs[i] + hs[i + 1]) / 2  # strictly between two distinct entropies
            thr = oracle.kept_list(img, B, L, tau)
            assert np.array_equal(oracle.kept_list_topk(img, B, L, thr.size), thr)


def test_ties_take_lower_indices():
    img = constant_image(32, 77)          # every key is 0
    assert np.array_equal(oracle.kept_list_topk(img, 4, 2, 7), np.arange(7))


def test_encode_with_topk_equals_equivalent_thresholds():
    cfg = config("C2")
    img = image_for(cfg)
    Ks = [64, 256, 512, 1024]
    taus = []
    for l, B in enumerate((16, 8, 4, 2)):
        _, _, H = oracle.entropy_keys(img, B, cfg["L"])
        hs = np.sort(H)[::-1]
        while hs[Ks[l] - 1] - hs[Ks[l]] < 1e-9:  # move K to a strict entropy gap
            Ks[l] += 1
        taus.append((hs[Ks[l] - 1] + hs[Ks[l]]) / 2)
    a = oracle.encode(img, 16, 2, cfg["L"], cfg["tau"], cfg["s"], cfg["rms_tol"], topk=Ks)
    b = oracle.encode(img, 16, 2, cfg["L"], taus, cfg["s"], cfg["rms_tol"])
    assert len(a) == len(b)
    for f in a.dtype.names:  # field by field (struct padding bytes are not part of a record)
        assert np.array_equal(a[f], b[f]), f


def test_sampled10_set():
    # P:106 "a 10-member set of s, sampled from [0,1]" (the paper's baseline); SPEC's reading:
    # ten uniform mid-point samples {0.05, 0.15, ..., 0.95}
    from fic_inputs import SAMPLED10_S
    assert len(SAMPLED10_S) == 10 and SAMPLED10_S[0] == 0.05 and SAMPLED10_S[-1] == 0.95
    assert np.allclose(np.diff(SAMPLED10_S), 0.1) and all(0 < s < 1 for s in SAMPLED10_S)
