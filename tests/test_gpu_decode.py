"""GPU parity of the PIFS decoder and PSNR (fic_decode / fic_psnr, readings R23-R26) against the
CPU oracle: decoded images byte-identical, PSNR identical (both from the exact integer SSE)."""
import numpy as np
import pytest

import oracle
from fic_inputs import config, image_for, make_image

pytestmark = pytest.mark.gpu


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


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rec_dev(torch, recs):
    return dev(torch, np.ascontiguousarray(recs).view(np.uint8).reshape(-1, 40))


def rand_code(rng, N, sizes, s_sets, B_max):
    recs = []
    for ty in range(0, N, B_max):
        for tx in range(0, N, B_max):
            B = sizes[1] if (len(sizes) > 1 and rng.random() < 0.5) else sizes[0]
            for y in range(ty, ty + B_max, B):
                for x in range(tx, tx + B_max, B):
                    l = sizes.index(B)
                    recs.append((x, y, B, 0, int(rng.integers(0, N - 2 * B + 1)),
                                 int(rng.integers(0, N - 2 * B + 1)), int(rng.integers(0, 8)),
                                 int(rng.integers(0, len(s_sets[l]))), int(rng.integers(0, 256)), 1, 0.0))
    return np.array(recs, dtype=oracle.RECORD_DTYPE)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
@pytest.mark.parametrize("iters", [0, 1, 2, 7])
def test_random_code_parity(fic, seed, iters):
    p, ctx, torch = fic
    rng = np.random.default_rng(seed)
    N = 64
    s_sets = [(0.1,), (0.2, 0.4), (0.3, 0.8), (0.5, 0.9)]
    code = rand_code(rng, N, [16, 8], s_sets, 16)
    init = make_image(N, 100 + seed)
    for ini in (None, init):
        got = ctx.decode(rec_dev(torch, code), N, 16, s_sets, iters,
                         None if ini is None else dev(torch, ini)).cpu().numpy()
        want = oracle.decode(code, N, s_sets, 16, iters, ini)
        assert np.array_equal(got, want), (seed, iters, ini is None)


@pytest.mark.parametrize("name,smode", [("C1", "predefined"), ("C1", "grid"), ("C2", "predefined"),
                                        ("C2", "grid"), ("C3", "predefined")])
def test_encode_decode_parity(fic, name, smode):
    p, ctx, torch = fic
    cfg = config(name, s_mode=smode)
    img = image_for(cfg)
    recs = ctx.encode_cfg(cfg, dev(torch, img))
    code = p.records_to_numpy(recs)
    got = ctx.decode(recs, cfg["N"], cfg["B_max"], cfg["s"], 12)
    want = oracle.decode(code, cfg["N"], cfg["s"], cfg["B_max"], 12)
    assert np.array_equal(got.cpu().numpy(), want)
    assert ctx.psnr(got, dev(torch, img)) == oracle.psnr(want, img)


def test_psnr_edge_cases(fic):
    p, ctx, torch = fic
    a = make_image(64, 3)
    assert ctx.psnr(dev(torch, a), dev(torch, a)) == float("inf")
    b = np.where(a < 255, a.astype(int) + 1, a.astype(int) - 1).astype(np.uint8)
    assert ctx.psnr(dev(torch, a), dev(torch, b)) == oracle.psnr(a, b)


def test_decode_errors(fic):
    p, ctx, torch = fic
    rng = np.random.default_rng(9)
    s_sets = [(0.5,), (0.5,)]
    code = rand_code(rng, 32, [8, 4], s_sets, 8)
    bad = code.copy()
    bad[3]["dx"] = 30  # 2B x 2B block past the edge
    with pytest.raises(p.FicError) as ei:
        ctx.decode(rec_dev(torch, bad), 32, 8, s_sets, 2)
    assert ei.value.status == 1
    bad = code.copy()
    bad[0]["s_idx"] = 3  # beyond the level's s list
    with pytest.raises(p.FicError):
        ctx.decode(rec_dev(torch, bad), 32, 8, s_sets, 2)
    # the context stays usable
    got = ctx.decode(rec_dev(torch, code), 32, 8, s_sets, 2).cpu().numpy()
    assert np.array_equal(got, oracle.decode(code, 32, s_sets, 8, 2))


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_decoder_convergence(fic, name):
    """SPEC acceptance 5 on the GPU decoder (readings R23-R25): from the constant 128 image the
    pass-to-pass change max |x_{i+1} - x_i| never grows after pass 2 and is at most one gray level
    by pass 16 (the passes round to 8 bits, so the real-valued "< 1" becomes "<= 1": a rounding
    limit cycle of one level can remain; the codes use s <= 0.9, a contraction up to rounding)."""
    p, ctx, torch = fic
    cfg = config(name)
    recs = ctx.encode_cfg(cfg, torch.from_numpy(image_for(cfg)).cuda())
    prev = ctx.decode(recs, cfg["N"], cfg["B_max"], cfg["s"], 0)
    deltas = []
    for it in range(1, 17):
        cur = ctx.decode(recs, cfg["N"], cfg["B_max"], cfg["s"], 1, init=prev)
        deltas.append(int((cur.int() - prev.int()).abs().max()))
        prev = cur
    assert deltas[-1] <= 1, deltas
    assert all(b <= a for a, b in zip(deltas[1:], deltas[2:])), deltas
