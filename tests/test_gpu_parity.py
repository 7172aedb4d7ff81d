"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (DESIGN.md §"Parity"): keep masks, entropy keys, kept lists, and every record field
(rx, ry, B, dom, dx, dy, iso, s_idx, o_code, accepted) bit-exact; err identical (both sides
evaluate the same binary64 expression; BASELINE.json allows 1e-12 relative, we require equality).
Full-size configs (C3, C4, C5) run the GPU in the launch configuration bench.py times and are
checked on seeded samples the oracle computes one by one, plus whole-output properties.
"""
import numpy as np
import pytest

import oracle
from fic_inputs import (config, image_for, make_image, random_image, ramp_image, constant_image,
                        sample_indices, PREDEFINED_S, GRID_S, SAMPLED10_S, CLOSED5_S)

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


def dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_same(gpu, orc, what=""):
    assert len(gpu) == len(orc), f"{what}: {len(gpu)} vs {len(orc)} records"
    for f in FIELDS:
        g, o = gpu[f], orc[f]
        if not np.array_equal(g, o):
            bad = np.nonzero(g != o)[0][:5]
            raise AssertionError(f"{what}: field {f} differs at {bad}: gpu {g[bad]} oracle {o[bad]}"
                                 f"\n gpu rec {gpu[bad[0]]}\n orc rec {orc[bad[0]]}")


# ------------------------------------------------------------------------------- pools
@pytest.mark.parametrize("N,B,L,tau", [
    (64, 4, 2, -1.0), (64, 2, 1, 2.0), (40, 8, 3, 3.0), (256, 16, 4, 5.10914), (256, 2, 4, 2.6),
    (96, 16, 1, 4.9), (512, 8, 2, 4.753761), (33, 4, 5, -1.0)])
def test_pool_parity(fic, N, B, L, tau):
    p, ctx, torch = fic
    img = make_image(N, N + B, texture=(N == 512))
    pool = ctx.build_domain_pool(dev(torch, img), B, L, tau)
    info = pool.info()
    keys, keep, _ = oracle.entropy_keys(img, B, L, tau)
    assert info["n_candidates"] == keys.size
    assert np.array_equal(info["keys"].cpu().numpy(), keys)
    assert np.array_equal(info["keep"].cpu().numpy(), keep)
    assert np.array_equal(info["kept"].cpu().numpy(), oracle.kept_list(img, B, L, tau))


def test_empty_pool_is_an_error(fic):
    p, ctx, torch = fic
    img = constant_image(32, 5)
    with pytest.raises(p.FicError) as ei:
        ctx.build_domain_pool(dev(torch, img), 4, 2, 0.5)
    assert ei.value.status == 3


# ------------------------------------------------------------------------------- one level
def level_case(fic, img, B, L, tau, s, tol=8.0, is_min=True, ranges=None):
    p, ctx, torch = fic
    N = img.shape[0]
    if ranges is None:
        ranges = np.array([(u * B, v * B) for v in range(N // B) for u in range(N // B)], np.int32)
    dimg = dev(torch, img)
    pool = ctx.build_domain_pool(dimg, B, L, tau)
    out = ctx.encode_level(dimg, pool, dev(torch, ranges.reshape(-1, 2)), s, tol, is_min)
    got = p.records_to_numpy(out)
    kept = oracle.kept_list(img, B, L, tau)
    ref = oracle.encode_level(img, B, L, kept, ranges, s, tol, is_min)
    assert_same(got, ref, f"B={B} L={L} tau={tau} s={s}")
    return got, ctx.stats()


@pytest.mark.parametrize("B", [2, 4, 8, 16])
@pytest.mark.parametrize("smode", ["predefined", "grid", "sampled10", "closed5"])
def test_level_parity_synthetic(fic, B, smode):
    img = make_image(96, 100 + B)
    s = {"predefined": PREDEFINED_S[B], "grid": GRID_S, "sampled10": SAMPLED10_S, "closed5": CLOSED5_S}[smode]
    level_case(fic, img, B, 2, -1.0, s, tol=6.0, is_min=False)


@pytest.mark.parametrize("B,N,L", [(2, 50, 3), (4, 72, 1), (8, 88, 5), (16, 80, 3)])
def test_level_parity_ragged_random(fic, B, N, L):
    # N not a multiple of the tile sizes, n_k not a multiple of 128, n_r not a multiple of 8
    img = random_image(N, 7 * B + N)
    n = (N // B) * B
    rng = np.random.default_rng(B)
    ranges = np.array([(u * B, v * B) for v in range(n // B) for u in range(n // B)], np.int32)
    keep = np.sort(rng.choice(len(ranges), size=len(ranges) * 2 // 3 + 1, replace=False))
    ranges = ranges[keep]
    level_case(fic, img, B, L, -1.0, PREDEFINED_S[B], ranges=ranges)


def test_level_parity_entropy_filtered(fic):
    img = make_image(128, 5, texture=True)
    for B, tau in ((16, 5.0), (8, 4.6), (4, 3.8), (2, 2.6)):
        level_case(fic, img, B, 2, tau, PREDEFINED_S[B])


def test_level_odd_s_lists(fic):
    img = make_image(64, 17)
    level_case(fic, img, 4, 2, -1.0, (0.0,))               # only s = 0
    level_case(fic, img, 4, 2, -1.0, (0.7, 0.0, 0.7, 1.0))  # duplicates, zero in the middle
    level_case(fic, img, 4, 2, -1.0, (1.0,))
    level_case(fic, img, 2, 2, -1.0, tuple(np.linspace(0, 1, 16)))


def test_level_zero_error_ramp(fic):
    got, _ = level_case(fic, ramp_image(64), 2, 2, -1.0, PREDEFINED_S[2])
    assert (got["err"] == 0.0).all() and (got["dom"] == 0).all() and (got["iso"] == 0).all()


def test_level_single_range_and_empty(fic):
    p, ctx, torch = fic
    img = make_image(64, 3)
    level_case(fic, img, 8, 2, -1.0, PREDEFINED_S[8], ranges=np.array([[24, 40]], np.int32))
    dimg = dev(torch, img)
    pool = ctx.build_domain_pool(dimg, 8, 2, -1.0)
    out = ctx.encode_level(dimg, pool, torch.zeros((0, 2), dtype=torch.int32, device="cuda"),
                           PREDEFINED_S[8], 8.0, True)
    assert out.shape[0] == 0


# ------------------------------------------------------------------------------- full encodes
def encode_both(fic, cfg, img=None):
    p, ctx, torch = fic
    if img is None:
        img = image_for(cfg)
    got = p.records_to_numpy(ctx.encode_cfg(cfg, dev(torch, img)))
    return img, got


@pytest.mark.parametrize("smode", ["predefined", "grid"])
def test_c1_full_parity(fic, smode):
    cfg = config("C1", s_mode=smode)
    img, got = encode_both(fic, cfg)
    assert_same(got, oracle.encode_cfg(cfg, img), f"C1 {smode}")


@pytest.mark.parametrize("seed", [0, 1])
def test_c2_full_parity(fic, seed):
    cfg = config("C2", seed=seed)
    img, got = encode_both(fic, cfg)
    assert_same(got, oracle.encode_cfg(cfg, img), f"C2 seed {seed}")


@pytest.mark.parametrize("t", [0.0, 4.0, 12.0, 1e9])
def test_quadtree_thresholds_parity(fic, t):
    cfg = config("C2", t=t)
    cfg["N"] = 128
    img = make_image(128, 77, texture=True)
    cfg["tau"] = [-1.0, 4.7, -1.0, 2.6]
    img, got = encode_both(fic, cfg, img)
    assert_same(got, oracle.encode_cfg(cfg, img), f"t={t}")


def test_constant_image(fic):
    cfg = config("C2")
    cfg["tau"] = [-1.0] * 4
    img = constant_image(256, 200)
    img, got = encode_both(fic, cfg, img)
    assert len(got) == 256 and (got["B"] == 16).all() and (got["err"] == 0.0).all()
    assert_same(got, oracle.encode_cfg(cfg, img), "constant")


def test_determinism_and_host_api(fic):
    p, ctx, torch = fic
    cfg = config("C2", seed=2)
    img = image_for(cfg)
    a = ctx.encode_cfg(cfg, dev(torch, img)).cpu().numpy().tobytes()
    b = ctx.encode_cfg(cfg, dev(torch, img)).cpu().numpy().tobytes()
    assert a == b
    h = ctx.encode_host(img, cfg["B_max"], cfg["B_min"], cfg["L"], cfg["tau"], cfg["s"], cfg["rms_tol"])
    assert h.tobytes() == a
    # a pinned output buffer: the kernels write the records into it directly (no final copy)
    cap = (cfg["N"] // cfg["B_min"]) ** 2
    pinned = torch.empty(cap * p.RECORD_BYTES, dtype=torch.uint8, pin_memory=True)
    hp = ctx.encode_host(img, cfg["B_max"], cfg["B_min"], cfg["L"], cfg["tau"], cfg["s"], cfg["rms_tol"],
                         out=pinned.numpy().view(p.RECORD_DTYPE))
    assert hp.tobytes() == a
    c3 = config("C3")  # a multi-level code: records from the side stream and the last finalize
    img3 = image_for(c3)
    ref = ctx.encode_cfg(c3, dev(torch, img3)).cpu().numpy().tobytes()
    cap3 = (c3["N"] // c3["B_min"]) ** 2
    pinned3 = torch.zeros(cap3 * p.RECORD_BYTES, dtype=torch.uint8, pin_memory=True)
    hp3 = ctx.encode_host(img3, c3["B_max"], c3["B_min"], c3["L"], c3["tau"], c3["s"], c3["rms_tol"],
                          out=pinned3.numpy().view(p.RECORD_DTYPE))
    assert hp3.tobytes() == ref


def test_shards_merge_equals_single(fic):
    p, ctx, torch = fic
    cfg = config("C2", seed=3)
    img = image_for(cfg)
    dimg = dev(torch, img)
    full = ctx.encode_cfg(cfg, dimg).cpu().numpy().tobytes()
    for W in (2, 3, 8):
        parts = [ctx.encode_cfg(cfg, dimg, shard=r, n_shards=W).clone() for r in range(W)]
        counts = [x.shape[0] for x in parts]
        stride = max(counts)
        buf = torch.zeros((W * stride, 40), dtype=torch.uint8, device="cuda")
        for r, x in enumerate(parts):
            buf[r * stride: r * stride + x.shape[0]] = x
        merged = ctx.merge_shards(buf, counts, stride).cpu().numpy().tobytes()
        assert merged == full, W


def test_errors(fic):
    p, ctx, torch = fic
    img = dev(torch, make_image(64, 1))
    with pytest.raises(p.FicError) as ei:  # N not a multiple of B_max
        ctx.encode(dev(torch, make_image(72, 1)), 16, 2, 2, [-1] * 4, [(0.5,)] * 4, [8.0] * 4)
    assert ei.value.status == 2
    with pytest.raises(p.FicError) as ei:  # s outside [0, 1]
        ctx.encode(img, 16, 2, 2, [-1] * 4, [(1.5,)] * 4, [8.0] * 4)
    assert ei.value.status == 1
    with pytest.raises(p.FicError) as ei:  # B_min not a power of two
        ctx.encode(img, 16, 3, 2, [-1] * 4, [(0.5,)] * 4, [8.0] * 4)
    assert ei.value.status == 1
    with pytest.raises(p.FicError) as ei:  # empty pool
        ctx.encode(dev(torch, constant_image(64, 3)), 16, 2, 2, [0.1] * 4, [(0.5,)] * 4, [8.0] * 4)
    assert ei.value.status == 3


# ------------------------------------------------------------------ full-size, sampled checks
def kept_for(img, cfg, li, B):
    if cfg.get("topk"):
        return oracle.kept_list_topk(img, B, cfg["L"], cfg["topk"][li])
    return oracle.kept_list(img, B, cfg["L"], cfg["tau"][li])


def sampled_level_check(fic, img, cfg, got, per_level=24, seed=0, parents=8):
    """Sampled records of a GPU encode re-derived one by one by the oracle at their level, plus
    sampled parents re-derived as rejected; leaves tile the image."""
    N = img.shape[0]
    cov = np.zeros((N, N), np.int32)
    for r in got:
        cov[r["ry"]:r["ry"] + r["B"], r["rx"]:r["rx"] + r["B"]] += 1
    assert (cov == 1).all()
    levels = [cfg["B_max"] >> i for i in range(len(cfg["s"]))]
    for li, B in enumerate(levels):
        sel = got[got["B"] == B]
        if len(sel) == 0:
            continue
        kept = kept_for(img, cfg, li, B)
        idx = sample_indices(len(sel), per_level, seed + li)
        ranges = np.stack([sel["rx"][idx], sel["ry"][idx]], 1).astype(np.int32)
        ref = oracle.encode_level(img, B, cfg["L"], kept, ranges, cfg["s"][li], cfg["rms_tol"][li],
                                  B == cfg["B_min"])
        assert_same(sel[idx], ref, f"sampled level B={B}")
        if li > 0 and parents:
            P = 2 * B
            pk = kept_for(img, cfg, li - 1, P)
            pi = sample_indices(len(sel), parents, seed + 100 + li)
            par = np.unique(np.stack([(sel["rx"][pi] // P) * P, (sel["ry"][pi] // P) * P], 1), axis=0)
            pref = oracle.encode_level(img, P, cfg["L"], pk, par.astype(np.int32), cfg["s"][li - 1],
                                       cfg["rms_tol"][li - 1], False)
            assert not pref["accepted"].any()


@pytest.mark.parametrize("smode,t", [("predefined", 4.0), ("predefined", 8.0), ("predefined", 12.0),
                                     ("grid", 8.0), ("closed5", 8.0)])
def test_c3_sampled(fic, smode, t):
    cfg = config("C3", s_mode=smode, t=t)
    img, got = encode_both(fic, cfg)
    # pools: full keep masks
    p, ctx, torch = fic
    for li, B in enumerate([16, 8, 4, 2]):
        pool = ctx.build_domain_pool(dev(torch, img), B, cfg["L"], cfg["tau"][li])
        _, keep, _ = oracle.entropy_keys(img, B, cfg["L"], cfg["tau"][li])
        assert np.array_equal(pool.info()["keep"].cpu().numpy(), keep)
    sampled_level_check(fic, img, cfg, got, per_level=16)


def test_c4_subset_1024(fic):
    """C4 (1024^2, exhaustive single level B = 8, L = 1: all 1009^2 domains x 8 isometries): the
    GPU encodes every range in the bench's launch configuration; the oracle re-derives the seeded
    subset of 1024 ranges BASELINE.json configs[3] names (8.3e9 pairs)."""
    p, ctx, torch = fic
    cfg = config("C4")
    img = image_for(cfg)
    B, L = 8, 1
    dimg = dev(torch, img)
    pool = ctx.build_domain_pool(dimg, B, L, -1.0)
    assert pool.info()["n_kept"] == 1009 ** 2
    ranges = np.array([(u * B, v * B) for v in range(128) for u in range(128)], np.int32)
    got = p.records_to_numpy(ctx.encode_level(dimg, pool, dev(torch, ranges), PREDEFINED_S[8], 8.0, True))
    idx = np.sort(sample_indices(len(ranges), 1024, 4))
    assert len(np.unique(idx)) == 1024
    kept = np.arange(1009 ** 2, dtype=np.int32)
    ref = oracle.encode_level(img, B, L, kept, ranges[idx], PREDEFINED_S[8], 8.0, True)
    assert_same(got[idx], ref, "C4 1024-range subset")


@pytest.mark.slow
def test_c5_sampled(fic):
    cfg = config("C5")
    img, got = encode_both(fic, cfg)
    sampled_level_check(fic, img, cfg, got, per_level=3, parents=2)


# ------------------------------------------------------------------ every search implementation
def test_b2_scan_parity(fic):
    """FIC_B2_WINDOW=0 runs the B = 2 two-pass scan (the path of the large s sets) for the
    predefined sets too instead of the Cauchy-Schwarz C windows: bit-exact as well."""
    import os
    p, _, torch = fic
    old = os.environ.get("FIC_B2_WINDOW")
    os.environ["FIC_B2_WINDOW"] = "0"
    try:
        ctx = p.Context(0)
        for smode in ("predefined", "grid"):
            cfg = config("C2", s_mode=smode, t=6.0)
            cfg["N"] = 128
            cfg["tau"] = [-1.0, 4.6, 3.6, 2.6]
            img = make_image(128, 91, texture=True)
            got = p.records_to_numpy(ctx.encode_cfg(cfg, dev(torch, img)))
            assert_same(got, oracle.encode_cfg(cfg, img), f"b2scan {smode}")
        ctx.close()
    finally:
        if old is None:
            os.environ.pop("FIC_B2_WINDOW", None)
        else:
            os.environ["FIC_B2_WINDOW"] = old


def test_capacity_error_reports_count(fic):
    p, ctx, torch = fic
    cfg = config("C2")
    img = image_for(cfg)
    full = ctx.encode_cfg(cfg, dev(torch, img))
    small = torch.empty((10, 40), dtype=torch.uint8, device="cuda")
    import ctypes as C
    n_out = C.c_int64()
    tau, n_s, s_flat, tol = ctx._cfg_arrays(cfg["tau"], cfg["s"], cfg["rms_tol"])
    from paper_1501_04140_b200.fic import _dptr, _ptr
    st = ctx.lib.fic_encode(ctx.handle, _dptr(dev(torch, img)), cfg["N"], cfg["B_max"], cfg["B_min"], cfg["L"],
                            _ptr(tau), _ptr(s_flat), _ptr(n_s), _ptr(tol), 0, 1, _dptr(small), 10,
                            C.byref(n_out))
    assert st == 4 and n_out.value == full.shape[0]
    # the first records written are the canonical first ones
    assert small.cpu().numpy().tobytes() == full[:10].cpu().numpy().tobytes()


def test_b64_and_bad_args(fic):
    p, ctx, torch = fic
    img = dev(torch, make_image(128, 2))
    with pytest.raises(p.FicError) as ei:  # B_max > 32
        ctx.encode(img, 64, 2, 2, [-1] * 6, [(0.5,)] * 6, [8.0] * 6)
    assert ei.value.status == 1
    with pytest.raises(p.FicError) as ei:  # more than 32 contrast values
        ctx.encode(img, 16, 2, 2, [-1] * 4, [tuple(np.linspace(0, 1, 33))] * 4, [8.0] * 4)
    assert ei.value.status == 1
    with pytest.raises(p.FicError):
        ctx.encode(img, 16, 2, 2, [-1] * 4, [(0.5,)] * 4, [8.0] * 4, shard=3, n_shards=2)


# ------------------------------------------------------------------ top-K pools (NEXT-1, R27)
@pytest.mark.parametrize("N,B,L,K", [(64, 4, 2, 100), (96, 8, 3, 37), (128, 2, 2, 1000), (64, 16, 4, 5),
                                     (80, 4, 1, 10 ** 6)])
def test_topk_pool_parity(fic, N, B, L, K):
    p, ctx, torch = fic
    img = make_image(N, N + K % 97)
    pool = ctx.build_domain_pool(dev(torch, img), B, L, topk=K)
    info = pool.info()
    want = oracle.kept_list_topk(img, B, L, K)
    assert np.array_equal(info["kept"].cpu().numpy(), want)
    keep = np.zeros(info["n_candidates"], np.uint8)
    keep[want] = 1
    assert np.array_equal(info["keep"].cpu().numpy(), keep)


def test_topk_ties_and_errors(fic):
    p, ctx, torch = fic
    img = constant_image(64, 77)  # every entropy key is 0: the K lowest indices
    pool = ctx.build_domain_pool(dev(torch, img), 4, 2, topk=9)
    assert np.array_equal(pool.info()["kept"].cpu().numpy(), np.arange(9))
    with pytest.raises(p.FicError) as ei:
        ctx.build_domain_pool(dev(torch, img), 4, 2, topk=0)
    assert ei.value.status == 1


@pytest.mark.parametrize("name,K,smode", [("C2", [256, 256, 256, 256], "predefined"),
                                          ("C2", [32, 64, 256, 512], "grid"),
                                          ("C2", [64, 64, 64, 64], "sampled10")])
def test_encode_topk_parity(fic, name, K, smode):
    p, ctx, torch = fic
    cfg = config(name, s_mode=smode, topk=K)
    img = image_for(cfg)
    got = p.records_to_numpy(ctx.encode_cfg(cfg, dev(torch, img)))
    assert_same(got, oracle.encode_cfg(cfg, img), f"{name} top-{K} {smode}")


def test_c3_topk_sampled(fic):
    p, ctx, torch = fic
    cfg = config("C3", topk=256)  # the paper's Table 1-2 pool size 256 at the paper's image size
    img, got = encode_both(fic, cfg)
    sampled_level_check(fic, img, cfg, got, per_level=40, parents=4)


@pytest.mark.parametrize("smode", ["closed5", "sampled10"])
def test_c2_full_parity_large_s_sets(fic, smode):
    cfg = config("C2", s_mode=smode)
    img, got = encode_both(fic, cfg)
    assert_same(got, oracle.encode_cfg(cfg, img), f"C2 {smode}")


def test_more_than_32_s_values_rejected(fic):
    p, ctx, torch = fic
    img = dev(torch, make_image(64, 5))
    with pytest.raises(p.FicError) as ei:
        ctx.encode(img, 16, 2, 2, [-1] * 4, [tuple(np.linspace(0, 1, 33))] * 4, [8.0] * 4)
    assert ei.value.status == 1


# ------------------------------------------------------------------ native NCCL path (8(e))
def test_native_nccl_single_rank(fic):
    """fic_ctx_create_nccl / fic_encode_nccl on a one-rank communicator (the box has one GPU):
    the shard / all-gather / merge path returns the one-GPU code byte for byte.  The multi-rank
    protocol (t % W shards, gather, canonical merge) is covered by the gloo tests and by
    test_shards_merge_equals_single."""
    p, ctx, torch = fic
    cfg = config("C2", seed=4)
    img = dev(torch, image_for(cfg))
    ref = ctx.encode_cfg(cfg, img)
    nctx = p.Context(0, nccl=(p.nccl_unique_id(), 1, 0))
    try:
        got = nctx.encode_nccl(img, cfg["B_max"], cfg["B_min"], cfg["L"], cfg["tau"], cfg["s"], cfg["rms_tol"])
        assert got.cpu().numpy().tobytes() == ref.cpu().numpy().tobytes()
        import ctypes as C
        from paper_1501_04140_b200.fic import _dptr, _ptr
        small = torch.empty((5, 40), dtype=torch.uint8, device="cuda")
        tau, n_s, s_flat, tol = nctx._cfg_arrays(cfg["tau"], cfg["s"], cfg["rms_tol"])
        n_out = C.c_int64()
        st = nctx.lib.fic_encode_nccl(nctx.handle, _dptr(img), cfg["N"], cfg["B_max"], cfg["B_min"], cfg["L"],
                                      _ptr(tau), _ptr(s_flat), _ptr(n_s), _ptr(tol), _dptr(small), 5,
                                      C.byref(n_out))
        assert st == 4 and n_out.value == ref.shape[0]  # capacity error reports the full count
    finally:
        nctx.close()
    with pytest.raises(p.FicError) as ei:  # no communicator on a plain context
        ctx.encode_nccl(img, cfg["B_max"], cfg["B_min"], cfg["L"], cfg["tau"], cfg["s"], cfg["rms_tol"])
    assert ei.value.status == 1


# ------------------------------------------------------------- persistent search plan (fic_tc.cu)
_C2_ORACLE = {}


@pytest.mark.parametrize("ctas,lockstep", [(16, 1), (7, 0), (3, 1), (148, 1)])
def test_persistent_plan_parity(fic, monkeypatch, ctas, lockstep):
    """The tcgen05 search runs as persistent CTAs whose work is full lockstep rounds of range
    groups plus a flattened (group, tile) tail cut into equal runs (partials per run, unused slots
    filled).  Small grids (FIC_TC_CTAS) and forced lockstep (FIC_TC_LOCKSTEP) put C2's levels
    through several full rounds, tails split across CTAs and groups split into many slots; the
    code must equal the oracle's bit for bit in every case."""
    monkeypatch.setenv("FIC_TC_CTAS", str(ctas))
    monkeypatch.setenv("FIC_TC_LOCKSTEP", str(lockstep))
    cfg = config("C2")
    img, got = encode_both(fic, cfg)
    if "C2" not in _C2_ORACLE:
        _C2_ORACLE["C2"] = oracle.encode_cfg(cfg, img)
    assert_same(got, _C2_ORACLE["C2"], f"C2 ctas={ctas} lockstep={lockstep}")


# ------------------------------------------------------------------ tiny s (below kSLicensed)
@pytest.mark.parametrize("B", [2, 4, 8, 16])
@pytest.mark.parametrize("s", [(1e-16,), (1e-18, 0.5), (0.0, 1e-14), (1e-15, 1e-16, 0.3)])
def test_tiny_s_parity(fic, B, s):
    """s below the licensed floor 2^-20 (DESIGN.md §6 'Exactness'): distinct SRD_k may give equal
    binary64 scores, so the winning isometry is no longer the SRD argmax; finalize re-derives
    (k, j) from the definition (C8).  Must equal the oracle bit for bit."""
    img = make_image(64, 40 + B)
    level_case(fic, img, B, 2, -1.0, s, is_min=True)


def test_tiny_s_full_encode(fic):
    cfg = config("C2", seed=1)
    cfg["s"] = [(1e-16,), (1e-17, 0.2), (0.3, 1e-15), (0.0, 1e-18)]
    img, got = encode_both(fic, cfg)
    assert_same(got, oracle.encode_cfg(cfg, img), "C2 tiny s")


# ------------------------------------------------------------------ full-output parity, timed configs
@pytest.mark.parametrize("smode", ["predefined", "grid"])
def test_c3_full_parity(fic, smode):
    """The whole C3 code (the configuration bench.py times: 512^2 + texture, 16->2, L = 2, entropy
    pools, t = 8), every record field, against the oracle's whole encode (§2 lines
    28-40; ~10-20 s of oracle time on the box's host cores)."""
    cfg = config("C3", s_mode=smode, t=8.0)
    img, got = encode_both(fic, cfg)
    assert_same(got, oracle.encode_cfg(cfg, img), f"C3 {smode} full")


def test_native_nccl_error_status_and_topk(fic):
    """fic_encode_nccl exchanges a failing shard's status through the count all-gather (every
    rank returns it instead of blocking in the record all-gather): on a one-rank communicator an
    empty pool comes back as FIC_ERR_EMPTY_POOL, and the context stays usable.  The top-K variant
    (fic_encode_nccl_topk) returns the one-GPU top-K code."""
    p, ctx, torch = fic
    nctx = p.Context(0, nccl=(p.nccl_unique_id(), 1, 0))
    try:
        bad = dev(torch, constant_image(64, 3))
        with pytest.raises(p.FicError) as ei:
            nctx.encode_nccl(bad, 16, 2, 2, [0.1] * 4, [(0.5,)] * 4, [8.0] * 4)
        assert ei.value.status == 3
        cfg = config("C2", topk=[64, 128, 256, 512])
        img = dev(torch, image_for(cfg))
        ref = ctx.encode_cfg(cfg, img)
        got = nctx.encode_nccl_cfg(cfg, img)
        assert got.cpu().numpy().tobytes() == ref.cpu().numpy().tobytes()
        with pytest.raises(p.FicError) as ei:
            nctx.encode_nccl(img, 16, 2, 4, [-1.0] * 4, cfg["s"], cfg["rms_tol"], topk=[64, 0, 1, 1])
        assert ei.value.status == 1
    finally:
        nctx.close()


# ------------------------------------------------------------------ B = 32 ranges ("B is a predefined parameter")
@pytest.mark.parametrize("smode", ["predefined", "grid", "closed5"])
@pytest.mark.parametrize("N,L,tau", [(96, 2, -1.0), (128, 3, 4.76), (80, 1, -1.0)])
def test_level_parity_b32(fic, smode, N, L, tau):
    img = make_image(N, 300 + N + L, texture=True)
    s = {"predefined": (0.1,), "grid": GRID_S, "closed5": CLOSED5_S}[smode]
    level_case(fic, img, 32, L, tau, s, tol=6.0, is_min=False)


@pytest.mark.parametrize("t", [4.0, 16.0])
def test_encode_b32_quadtree(fic, t):
    """Quadtree 32 -> 2 on the C2 image (every 32x32 range searched, then split) ..."""
    cfg = config("C2", t=t)
    cfg["B_max"] = 32
    cfg["tau"] = [5.2] + list(cfg["tau"])
    cfg["s"] = [(0.1,)] + list(cfg["s"])
    cfg["rms_tol"] = [t] * 5
    img, got = encode_both(fic, cfg)
    assert_same(got, oracle.encode_cfg(cfg, img), f"B_max=32 t={t}")


def test_encode_b32_accepts_on_ramp(fic):
    """... and on a ramp with noise-free affine copies, where 32x32 leaves are accepted."""
    cfg = config("C2", t=1.0)
    cfg["N"] = 128
    cfg["B_max"] = 32
    cfg["tau"] = [-1.0] * 5
    cfg["s"] = [(0.5, 0.9)] * 5
    cfg["rms_tol"] = [1.0] * 5
    img = ramp_image(128)
    img, got = encode_both(fic, cfg, img)
    assert (got["B"] == 32).all() and (got["err"] == 0.0).all()
    assert_same(got, oracle.encode_cfg(cfg, img), "B_max=32 ramp")


@pytest.mark.parametrize("B,N,L", [(16, 70, 3), (32, 66, 1), (16, 97, 2), (8, 75, 3), (4, 41, 1)])
def test_level_parity_unaligned_rows(fic, B, N, L):
    """Image widths that are not a multiple of 4 (rows not word-aligned): the pool kernels that
    read words fall back to bytes."""
    img = random_image(N, 11 * B + N)
    n = (N // B) * B
    ranges = np.array([(u * B, v * B) for v in range(n // B) for u in range(n // B)], np.int32)
    level_case(fic, img, B, L, -1.0, (0.1, 0.6) if B >= 16 else PREDEFINED_S[B], ranges=ranges)
