"""Pins of the FIC1 container (oracle/codeformat.py; NEXT-3).

The bit layout is checked against a hand-written bit string for a tiny code, the SPEC example's
exact size formula (constant image: no splits), the round trip on real codes of the oracle
encoder, the analytical size the bench reports, and the error cases."""
import numpy as np
import pytest

import oracle
from oracle import codeformat as cf
from fic_inputs import config, image_for, constant_image


def rec(rx, ry, B, dx, dy, iso, s_idx, o):
    return {"rx": rx, "ry": ry, "B": B, "dx": dx, "dy": dy, "iso": iso, "s_idx": s_idx, "o_code": o}


def test_tiny_stream_by_hand():
    # N = 8, B 4 -> 2, L = 2: A = 3 positions per axis at B = 2 (2 bits), A = 1 at B = 4 (0 bits)
    # top block (0,0) is a leaf; top block (4,0) splits into four 2x2 leaves; the rest are leaves
    s_sets = [(0.3, 0.8), (0.5,)]
    recs = [rec(0, 0, 4, 0, 0, 5, 1, 200),
            rec(4, 0, 2, 2, 4, 1, 0, 7), rec(6, 0, 2, 0, 0, 0, 0, 255),
            rec(4, 2, 2, 4, 2, 7, 0, 0), rec(6, 2, 2, 2, 2, 3, 0, 128),
            rec(0, 4, 4, 0, 0, 2, 0, 1), rec(4, 4, 4, 0, 0, 0, 1, 2)]
    got = cf.serialize(recs, 8, 4, 2, 2, s_sets, "predefined")
    bits = ""
    bits += "0" + "" + "" + "101" + "1" + "11001000"          # (0,0) leaf: split 0, iso 5, s 1, o 200
    bits += "1"                                               # (4,0) split
    bits += "01" + "10" + "001" + "" + "00000111"             #   (4,0): dx/L 1, dy/L 2, iso 1, o 7
    bits += "00" + "00" + "000" + "11111111"                  #   (6,0)
    bits += "10" + "01" + "111" + "00000000"                  #   (4,2)
    bits += "01" + "01" + "011" + "10000000"                  #   (6,2)
    bits += "0" + "010" + "0" + "00000001"                    # (0,4) leaf
    bits += "0" + "000" + "1" + "00000010"                    # (4,4) leaf
    bits += "0" * (-len(bits) % 8)
    body = bytes(int(bits[i:i + 8], 2) for i in range(0, len(bits), 8))
    head = b"FIC1" + bytes([0, 8, 0, 8, 4, 2, 0]) + (10000).to_bytes(2, "big") + (2).to_bytes(2, "big") + bytes([2, 1])
    assert got == head + body
    hdr, back = cf.deserialize(got)
    assert hdr["N"] == 8 and hdr["counts"] == [2, 1] and hdr["L"] == 2
    assert [tuple(r) for r in back] == [(r["rx"], r["ry"], r["B"], r["dx"], r["dy"], r["iso"], r["s_idx"], r["o_code"])
                                        for r in recs]


def test_constant_image_size_formula():
    # a 64x64 constant image codes 16 leaves at B = 16 with no splits:
    # 16 split bits + 16 (2 posbits + 3 + 0 + 8) payload bits, header-exact size
    N, L = 64, 2
    img = constant_image(N, 77)
    s_sets = [(0.1,), (0.2, 0.4), (0.3, 0.8), (0.5, 0.9)]
    recs = oracle.encode(img, 16, 2, L, [-1.0] * 4, s_sets, [8.0] * 4)
    assert len(recs) == 16 and set(recs["B"]) == {16}
    pb = cf.nbits(cf.axis_positions(N, 16, L))
    bits = 16 + 16 * (2 * pb + 3 + 0 + 8)
    stream = cf.serialize(recs, N, 16, 2, L, s_sets, "predefined")
    assert len(stream) == cf.header_bytes(4) + (bits + 7) // 8
    assert cf.compression_ratio(N, stream) == N * N / len(stream)


@pytest.mark.parametrize("name,smode", [("C1", "predefined"), ("C1", "grid"), ("C2", "predefined"),
                                        ("C2", "sampled10"), ("C2", "closed5")])
def test_round_trip_and_bench_size(name, smode):
    cfg = config(name, s_mode=smode)
    img = image_for(cfg)
    recs = oracle.encode_cfg(cfg, img)
    stream = cf.serialize(recs, cfg["N"], cfg["B_max"], cfg["B_min"], cfg["L"], cfg["s"], smode)
    hdr, back = cf.deserialize(stream)
    key = lambda r: (int(r["rx"]), int(r["ry"]), int(r["B"]))
    orig = {key(r): r for r in recs}
    assert len(back) == len(recs)
    for r in back:
        o = orig[key(r)]
        for f in ("dx", "dy", "iso", "s_idx", "o_code"):
            assert int(r[f]) == int(o[f]), f
    # the size the bench computes from per-level counts (bench.code_size) is the stream's size
    import bench
    levels = []
    for li, B in enumerate(cfg["B_max"] >> i for i in range(len(cfg["s"]))):
        n_acc = int(np.sum(recs["B"] == B))
        n_vis = sum(1 for r in recs if int(r["B"]) <= B)  # visited ranges: leaves at or below B ...
        anc = {(int(r["rx"]) // B, int(r["ry"]) // B) for r in recs if int(r["B"]) <= B}
        levels.append({"B": B, "n_candidates": cf.axis_positions(cfg["N"], B, cfg["L"]) ** 2,
                       "n_accepted": n_acc, "n_ranges": len(anc)})
    assert bench.code_size(cfg, levels)["code_bytes_fic1"] == len(stream)


def test_errors():
    with pytest.raises(ValueError, match="magic"):
        cf.deserialize(b"XXXX" + bytes(20))
    s_sets = [(0.3, 0.8), (0.5,)]
    recs = [rec(0, 0, 4, 0, 0, 5, 1, 200), rec(4, 0, 4, 0, 0, 1, 0, 7), rec(0, 4, 4, 0, 0, 2, 0, 1),
            rec(4, 4, 4, 0, 0, 0, 1, 2)]
    stream = cf.serialize(recs, 8, 4, 2, 2, s_sets, "predefined")
    with pytest.raises(ValueError, match="truncated"):
        cf.deserialize(stream[:-2])
    with pytest.raises(ValueError, match="no leaf"):
        cf.serialize(recs[1:], 8, 4, 2, 2, s_sets, "predefined")
