"""GPU parity of the B = 2 level's windowed searches against the CPU oracle, record by record.

b2wink_kernel (fic_b2.cu) serves uniform grids of 3..16 positive s (the 16-value grid, sampled10,
offset grids, with or without s = 0 listed); larger or non-uniform sets fall back to the two-pass
scan.  Every case compares all record fields (err included) with the oracle's exhaustive loop
(§2 Eq. 1-3, readings R17 / C7), on images chosen to stress the windows: textured
(narrow windows), pure noise (wide ones), a constant image (C = 0 for every domain, so the window
centres collapse onto the first sorted position), a ramp (exact affine copies, best = 0).
"""
import numpy as np
import pytest

import oracle
from fic_inputs import make_image, random_image, ramp_image, constant_image, GRID_S, SAMPLED10_S

pytestmark = pytest.mark.gpu

FIELDS = ("rx", "ry", "B", "dom", "dx", "dy", "iso", "s_idx", "o_code", "accepted", "err")


@pytest.fixture(scope="module")
def fic():
    import torch
    from paper_1501_04140_b200 import build as b
    b.build()
    import paper_1501_04140_b200 as p
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    ctx = p.Context(0, timing=True)
    yield p, ctx, torch
    ctx.close()


def run_level(fic, img, s, L=2, tau=-1.0, ranges=None):
    p, ctx, torch = fic
    N = img.shape[0]
    if ranges is None:
        ranges = np.array([(u * 2, v * 2) for v in range(N // 2) for u in range(N // 2)], np.int32)
    dimg = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    pool = ctx.build_domain_pool(dimg, 2, L, tau)
    out = ctx.encode_level(dimg, pool, torch.from_numpy(ranges.reshape(-1, 2)).cuda(), s, 8.0, False)
    got = p.records_to_numpy(out)
    ref = oracle.encode_level(img, 2, L, oracle.kept_list(img, 2, L, tau), ranges, s, 8.0, False)
    assert len(got) == len(ref)
    for f in FIELDS:
        if not np.array_equal(got[f], ref[f]):
            bad = np.nonzero(got[f] != ref[f])[0][:5]
            raise AssertionError(f"s={s}: field {f} differs at {bad}: gpu {got[bad[0]]} oracle {ref[bad[0]]}")
    return ctx.stats()


SETS = {
    "grid16": GRID_S,                                          # 15 positive + s = 0
    "sampled10": SAMPLED10_S,                                  # 10 positive, no zero
    "grid3": (1 / 3, 2 / 3, 1.0),                              # the smallest windowed set
    "offset8": tuple(0.2 + 0.1 * j for j in range(8)),         # a != h
    "zero+4": (0.0, 0.25, 0.5, 0.75, 1.0),
    "grid16pos": tuple(j / 16.0 for j in range(1, 17)),       # 16 positive: the largest windowed set
    "grid17": tuple(j / 17.0 for j in range(1, 18)),          # 17: falls back to the scan
    "nonuniform": (0.1, 0.3, 0.35, 0.8, 0.95),                 # not a grid: the scan
}


@pytest.mark.parametrize("name", list(SETS))
def test_b2_window_sets_textured(fic, name):
    run_level(fic, make_image(96, 41, texture=True), SETS[name])


@pytest.mark.parametrize("name", ["grid16", "sampled10", "offset8"])
@pytest.mark.parametrize("kind", ["noise", "constant", "ramp"])
def test_b2_window_sets_extreme_images(fic, name, kind):
    img = {"noise": random_image(64, 9), "constant": constant_image(48, 77), "ramp": ramp_image(64)}[kind]
    run_level(fic, img, SETS[name], L=1)


def test_b2_window_entropy_filtered_ragged(fic):
    # an entropy-filtered pool (n_k not a multiple of the tile size) and a ragged range subset
    img = make_image(120, 8, texture=True)
    rng = np.random.default_rng(3)
    allr = np.array([(u * 2, v * 2) for v in range(60) for u in range(60)], np.int32)
    ranges = allr[np.sort(rng.choice(len(allr), size=1999, replace=False))]
    for name in ("grid16", "sampled10"):
        run_level(fic, img, SETS[name], L=3, tau=2.4, ranges=ranges)


def test_b2_window_prunes(fic):
    # the windows skip pairs without scoring them (full encode of C2 in grid mode, whose small
    # pools -- ~4k domains at L = 4 -- leave little to prune: ~70% scanned; C3 scans ~18%)
    from fic_inputs import config, image_for
    p, ctx, torch = fic
    cfg = config("C2", s_mode="grid")
    rec = ctx.encode_cfg(cfg, torch.from_numpy(image_for(cfg)).cuda())
    got = p.records_to_numpy(rec)
    ref = oracle.encode_cfg(cfg)
    assert len(got) == len(ref) and all(np.array_equal(got[f], ref[f]) for f in FIELDS)
    lv = [x for x in ctx.stats() if x["B"] == 2][0]
    scanned = lv["pairs_scanned"] / max(1, lv["n_ranges"] * lv["n_kept"])
    assert scanned < 0.8, scanned
