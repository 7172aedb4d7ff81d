"""FIC1 container (TEST INFRASTRUCTURE ONLY): serialize / deserialize a fractal code.

Written from SPEC.md's codeformat module (the paper fixes no format, P:154 only
reports compression ratios), in the order it states, with plain Python integers and an explicit
bit list -- no blocking, no reordering:

  magic "FIC1" (4 bytes); header: width u16, height u16, max_range u8, min_range u8, s_mode u8,
  s_max u16 (x 10000), step L u16, one u8 per level with the level's s-candidate count
  (readings R29: big-endian u16; s_mode 0 predefined, 1 sampled10, 2 least squares (our 5-bit
  closed form), 3 the 16-value grid);
  body: depth-first walk of every top-level block in row-major order, children in row-major
  order (TL, TR, BL, BR); one split bit (1 split, 0 leaf) per visited range above min_range; a
  leaf's payload = [dx / L (posbits), dy / L (posbits), isometry (3), s index (sbits), o code (8)]
  with posbits = ceil(log2 A) (A candidate positions per axis at the leaf's size; 0 bits if A = 1)
  and sbits = ceil(log2 |S_B|) (0 bits for one candidate); MSB first; zero-padded to a byte.
"""
from __future__ import annotations

import math

import numpy as np

MAGIC = b"FIC1"
S_MODES = {"predefined": 0, "sampled10": 1, "closed5": 2, "grid": 3}


def nbits(count: int) -> int:
    """ceil(log2 count) bits to index `count` values (0 for a single value)."""
    return 0 if count <= 1 else int(math.ceil(math.log2(count)))


def axis_positions(N: int, B: int, L: int) -> int:
    return (N - 2 * B) // L + 1


def header_bytes(n_levels: int) -> int:
    return 15 + n_levels


def serialize(records, N: int, B_max: int, B_min: int, L: int, s_sets, s_mode: str, s_max: float = 1.0) -> bytes:
    """records: the code (any order, one record per leaf with fields rx, ry, B, dx, dy, iso,
    s_idx, o_code).  Returns the FIC1 bytes."""
    levels = []
    B = B_max
    while B >= B_min:
        levels.append(B)
        B //= 2
    if len(s_sets) != len(levels):
        raise ValueError("one s set per level")
    leaf = {(int(r["rx"]), int(r["ry"]), int(r["B"])): r for r in records}
    if len(leaf) != len(records):
        raise ValueError("duplicate leaf")
    head = bytearray(MAGIC)
    head += N.to_bytes(2, "big") + N.to_bytes(2, "big")
    head += bytes([B_max, B_min, S_MODES[s_mode]])
    head += int(round(s_max * 10000)).to_bytes(2, "big") + L.to_bytes(2, "big")
    head += bytes(len(s) for s in s_sets)
    bits = []

    def put(value: int, width: int):
        for k in range(width - 1, -1, -1):
            bits.append((value >> k) & 1)

    def walk(x: int, y: int, B: int, li: int):
        r = leaf.get((x, y, B))
        if B > B_min:
            put(0 if r is not None else 1, 1)
        if r is None:
            if B == B_min:
                raise ValueError(f"no leaf for the {B}x{B} range at ({x}, {y})")
            h = B // 2
            for cy, cx in ((0, 0), (0, 1), (1, 0), (1, 1)):
                walk(x + cx * h, y + cy * h, h, li + 1)
            return
        pb = nbits(axis_positions(N, B, L))
        put(int(r["dx"]) // L, pb)
        put(int(r["dy"]) // L, pb)
        put(int(r["iso"]), 3)
        put(int(r["s_idx"]), nbits(len(s_sets[li])))
        put(int(r["o_code"]), 8)

    G = N // B_max
    for ty in range(G):
        for tx in range(G):
            walk(tx * B_max, ty * B_max, B_max, 0)
    while len(bits) % 8:
        bits.append(0)
    body = bytes(int("".join(map(str, bits[i:i + 8])), 2) for i in range(0, len(bits), 8))
    return bytes(head) + body


def deserialize(data: bytes):
    """-> (header dict, records as a numpy structured array in depth-first order)."""
    if len(data) < 15 or data[:4] != MAGIC:
        raise ValueError("bad magic")
    N = int.from_bytes(data[4:6], "big")
    H = int.from_bytes(data[6:8], "big")
    B_max, B_min, mode = data[8], data[9], data[10]
    s_max = int.from_bytes(data[11:13], "big") / 10000.0
    L = int.from_bytes(data[13:15], "big")
    levels = []
    B = B_max
    while B >= B_min and B > 0:
        levels.append(B)
        B //= 2
    if len(data) < 15 + len(levels):
        raise ValueError("truncated stream")
    counts = list(data[15:15 + len(levels)])
    body = data[15 + len(levels):]
    pos = [0]

    def get(width: int) -> int:
        v = 0
        for _ in range(width):
            p = pos[0]
            if p >= 8 * len(body):
                raise ValueError("truncated stream")
            v = (v << 1) | ((body[p >> 3] >> (7 - (p & 7))) & 1)
            pos[0] = p + 1
        return v

    out = []

    def walk(x: int, y: int, B: int, li: int):
        split = get(1) if B > B_min else 0
        if split:
            h = B // 2
            if h < B_min:
                raise ValueError("inconsistent tree (leaf below min_range)")
            for cy, cx in ((0, 0), (0, 1), (1, 0), (1, 1)):
                walk(x + cx * h, y + cy * h, h, li + 1)
            return
        pb = nbits(axis_positions(N, B, L))
        dx, dy = get(pb) * L, get(pb) * L
        iso = get(3)
        s_idx = get(nbits(counts[li]))
        o = get(8)
        out.append((x, y, B, dx, dy, iso, s_idx, o))

    G = N // B_max
    for ty in range(G):
        for tx in range(G):
            walk(tx * B_max, ty * B_max, B_max, 0)
    hdr = {"N": N, "H": H, "B_max": B_max, "B_min": B_min, "s_mode": mode, "s_max": s_max, "L": L,
           "counts": counts, "bits": pos[0]}
    rec = np.array(out, dtype=[("rx", "<i4"), ("ry", "<i4"), ("B", "<i4"), ("dx", "<i4"), ("dy", "<i4"),
                               ("iso", "u1"), ("s_idx", "u1"), ("o_code", "u1")])
    return hdr, rec


def compression_ratio(N: int, stream: bytes) -> float:
    """(width x height x 1 byte) / stream length (the paper's "Com. rat")."""
    return N * N / len(stream)
