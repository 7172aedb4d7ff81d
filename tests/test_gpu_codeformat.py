"""FIC1 writer on the GPU (fic_serialize, NEXT-3) against the oracle's serializer
(oracle/codeformat.py, pinned in test_oracle_codeformat.py): the same bytes for the same code."""
import ctypes as C

import numpy as np
import pytest

import oracle
from oracle import codeformat as cf
from fic_inputs import config, image_for

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


@pytest.mark.parametrize("name,smode", [("C1", "predefined"), ("C1", "grid"), ("C2", "predefined"),
                                        ("C2", "sampled10"), ("C2", "closed5")])
def test_stream_equals_oracle(fic, name, smode):
    p, ctx, torch = fic
    cfg = config(name, s_mode=smode)
    img = image_for(cfg)
    recs = ctx.encode_cfg(cfg, torch.from_numpy(img).cuda())
    got = ctx.serialize_cfg(cfg, recs)
    ref = cf.serialize(oracle.encode_cfg(cfg, img), cfg["N"], cfg["B_max"], cfg["B_min"], cfg["L"], cfg["s"], smode)
    assert got == ref, f"{name}/{smode}: {len(got)} vs {len(ref)} bytes, first difference at " \
                       f"{next((i for i, (a, b) in enumerate(zip(got, ref)) if a != b), None)}"


def test_c3_stream_round_trip(fic):
    p, ctx, torch = fic
    cfg = config("C3")
    img = image_for(cfg)
    recs_t = ctx.encode_cfg(cfg, torch.from_numpy(img).cuda())
    got = ctx.serialize_cfg(cfg, recs_t)
    hdr, back = cf.deserialize(got)
    recs = p.records_to_numpy(recs_t)
    assert hdr["N"] == cfg["N"] and hdr["counts"] == [len(s) for s in cfg["s"]]
    assert len(back) == len(recs)
    by_key = {(int(r["rx"]), int(r["ry"]), int(r["B"])): r for r in recs}
    for r in back:
        o = by_key[(int(r["rx"]), int(r["ry"]), int(r["B"]))]
        for f in ("dx", "dy", "iso", "s_idx", "o_code"):
            assert int(r[f]) == int(o[f]), f
    assert len(got) == cf.header_bytes(len(cfg["s"])) + (hdr["bits"] + 7) // 8


def test_capacity_and_argument_errors(fic):
    p, ctx, torch = fic
    cfg = config("C1")
    recs = ctx.encode_cfg(cfg, torch.from_numpy(image_for(cfg)).cuda())
    out = torch.zeros(16, dtype=torch.uint8, device="cuda")
    n_s = np.ascontiguousarray([len(s) for s in cfg["s"]], dtype=np.int32)
    nb = C.c_int64()
    st = ctx.lib.fic_serialize(ctx.handle, C.c_void_p(recs.data_ptr()), recs.shape[0], cfg["N"], cfg["B_max"],
                               cfg["B_min"], cfg["L"], n_s.ctypes.data_as(C.c_void_p), 0, 1.0,
                               C.c_void_p(out.data_ptr()), 16, C.byref(nb))
    assert st == 4 and nb.value > 16  # FIC_ERR_CAPACITY, the needed length reported
    st = ctx.lib.fic_serialize(ctx.handle, C.c_void_p(recs.data_ptr()), recs.shape[0], cfg["N"], 3,
                               cfg["B_min"], cfg["L"], n_s.ctypes.data_as(C.c_void_p), 0, 1.0,
                               C.c_void_p(out.data_ptr()), 16, C.byref(nb))
    assert st == 1  # FIC_ERR_ARG (B_max not a power of two)


def test_stream_of_concatenated_shards(fic):
    """The writer orders leaves itself (depth-first key), so the shards' codes simply
    concatenated -- without the canonical merge -- give the same stream as the one-GPU code."""
    p, ctx, torch = fic
    cfg = config("C2", seed=3)
    img = torch.from_numpy(image_for(cfg)).cuda()
    full = ctx.serialize_cfg(cfg, ctx.encode_cfg(cfg, img))
    parts = [ctx.encode_cfg(cfg, img, shard=r, n_shards=3).clone() for r in range(3)]
    cat = torch.cat(parts, 0)
    assert ctx.serialize_cfg(cfg, cat) == full


@pytest.mark.parametrize("field,value", [("B", 3), ("B", 64), ("rx", 2 ** 31 - 2), ("ry", -4), ("dx", 1),
                                         ("dy", 10 ** 6), ("iso", 8), ("s_idx", 7)])
def test_corrupt_record_rejected(fic, field, value):
    """A record the container cannot hold (level outside [B_min, B_max], range or domain outside
    the image or off its grid, isometry >= 8, s index past the level's list) is FIC_ERR_ARG, not
    an out-of-bounds write; the decoder rejects the same records."""
    p, ctx, torch = fic
    cfg = config("C2")
    img = torch.from_numpy(image_for(cfg)).cuda()
    recs = p.records_to_numpy(ctx.encode_cfg(cfg, img)).copy()
    recs[5][field] = value
    bad = torch.from_numpy(recs.view(np.uint8).reshape(-1, 40).copy()).cuda()
    with pytest.raises(p.FicError) as ei:
        ctx.serialize_cfg(cfg, bad)
    assert ei.value.status == 1
    if field not in ("dx",):  # (dx = 1 is a valid decode position; only the container needs dx % L == 0)
        with pytest.raises(p.FicError) as ei:
            ctx.decode(bad, cfg["N"], cfg["B_max"], cfg["s"], 2)
        assert ei.value.status == 1
