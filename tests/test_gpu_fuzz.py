"""Randomized end-to-end parity (GPU vs oracle) over shapes the named configs do not reach:
image sizes that leave ragged domain tiles and few range groups, odd steps L, 1-4 levels, every
s mode, random entropy thresholds and tolerances, and small persistent grids (FIC_TC_CTAS) so
that the search plan splits groups across runs; B_max up to 32, occasionally an s below 2^-20.  Every record field must match bit for bit.
FIC_FUZZ_N=n widens the sweep (n cases, n // 3 top-K + shard cases; default 48)."""
import os

import numpy as np
import pytest

import oracle
from fic_inputs import make_image
from fic_inputs.configs import PREDEFINED_S, GRID_S, SAMPLED10_S, CLOSED5_S

pytestmark = pytest.mark.gpu

FIELDS = ("rx", "ry", "B", "dom", "dx", "dy", "iso", "s_idx", "o_code", "accepted", "err")


@pytest.fixture(scope="module")
def fic():
    import torch
    from paper_1501_04140_b200 import build as b
    b.build()
    import paper_1501_04140_b200 as p
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    ctx = p.Context(0)
    yield p, ctx, torch
    ctx.close()


def case(seed):
    rng = np.random.default_rng(1000 + seed)
    B_max = int(rng.choice([4, 8, 16, 32]))
    B_min = int(rng.choice([b for b in (2, 4, 8, 16, 32) if b <= B_max]))
    N = B_max * int(rng.integers(2, 6))
    L = int(rng.integers(1, 4))
    levels = []
    B = B_max
    while B >= B_min:
        levels.append(B)
        B //= 2
    mode = ["predefined", "grid", "sampled10", "closed5"][seed % 4]
    sets = {"grid": GRID_S, "sampled10": SAMPLED10_S, "closed5": CLOSED5_S}
    s_sets = [tuple(PREDEFINED_S.get(B, (0.1,))) if mode == "predefined" else sets[mode] for B in levels]
    if rng.random() < 0.15:  # s below the licensed floor (finalize re-derives (k, j))
        s_sets = [(1e-15,) + tuple(x) for x in s_sets] if mode == "predefined" else s_sets
    tau = [float(rng.choice([-1.0, 0.5, 1.5])) for _ in levels]
    tol = [float(rng.choice([2.0, 6.0, 12.0]))] * len(levels)
    img = make_image(N, 77 + seed, texture=bool(seed % 2))
    ctas = int(rng.choice([3, 7, 148]))
    return img, B_max, B_min, L, tau, s_sets, tol, mode, ctas


@pytest.mark.parametrize("seed", range(int(os.environ.get("FIC_FUZZ_N", "48"))))
def test_random_config_parity(fic, monkeypatch, seed):
    p, ctx, torch = fic
    img, B_max, B_min, L, tau, s_sets, tol, mode, ctas = case(seed)
    monkeypatch.setenv("FIC_TC_CTAS", str(ctas))
    try:
        ref = oracle.encode(img, B_max, B_min, L, tau, s_sets, tol)
    except Exception as e:  # e.g. an empty pool at a level with ranges: the GPU must refuse too
        with pytest.raises(p.FicError):
            ctx.encode(torch.from_numpy(img).cuda(), B_max, B_min, L, tau, s_sets, tol)
        return
    got = p.records_to_numpy(ctx.encode(torch.from_numpy(img).cuda(), B_max, B_min, L, tau, s_sets, tol))
    what = f"seed {seed}: N={img.shape[0]} B {B_max}->{B_min} L={L} {mode} tau={tau} tol={tol[0]} ctas={ctas}"
    assert len(got) == len(ref), what
    for f in FIELDS:
        assert np.array_equal(got[f], ref[f]), f"{what}: field {f}"


@pytest.mark.parametrize("seed", range(int(os.environ.get("FIC_FUZZ_N", "48")) // 3))
def test_random_topk_and_shards(fic, seed):
    """Random pool sizes (top-K, reading R27) and a random shard count: every shard's code and
    the merged code against the oracle's."""
    p, ctx, torch = fic
    img, B_max, B_min, L, tau, s_sets, tol, mode, _ = case(100 + seed)
    rng = np.random.default_rng(seed)
    K = [int(rng.integers(1, 300)) for _ in s_sets]
    W = int(rng.integers(1, 5))
    dimg = torch.from_numpy(img).cuda()
    parts = []
    for r in range(W):
        ref = oracle.encode(img, B_max, B_min, L, tau, s_sets, tol, shard=r, n_shards=W, topk=K)
        got = ctx.encode(dimg, B_max, B_min, L, tau, s_sets, tol, shard=r, n_shards=W, topk=K)
        g = p.records_to_numpy(got)
        assert len(g) == len(ref), (seed, r)
        for f in FIELDS:
            assert np.array_equal(g[f], ref[f]), (seed, r, f)
        parts.append(got.clone())
    counts = [x.shape[0] for x in parts]
    stride = max(max(counts), 1)
    buf = torch.zeros((W * stride, 40), dtype=torch.uint8, device="cuda")
    for r, x in enumerate(parts):
        buf[r * stride: r * stride + x.shape[0]] = x
    merged = p.records_to_numpy(ctx.merge_shards(buf, counts, stride))
    full = oracle.encode(img, B_max, B_min, L, tau, s_sets, tol, topk=K)
    assert len(merged) == len(full)
    for f in FIELDS:
        assert np.array_equal(merged[f], full[f]), (seed, "merged", f)
