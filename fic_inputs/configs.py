"""The five BASELINE.json configurations (C1..C5), restated as encoder parameters.

Readings (DESIGN.md §"Readings"): s schedule keyed by range size (§3.1:
16->{0.1}, 8->{0.2,0.4}, 4->{0.3,0.8}, 2->{0.5,0.9}); the "16-value uniform s grid on
[0,1]" is s_j = j/15.0, j = 0..15; "error threshold t" is a per-level RMS tolerance
(accept iff sqrt(E/n) <= t, i.e. E <= t*t*n); tau_B are the per-level entropy thresholds in
nats chosen once by scripts/choose_tau.py (kept near 50%) and stored in tau.json.
"""
from __future__ import annotations

import json
import os

from .synth import make_image

# PAPER.md §3.1 line 108 (step 1..4 <-> range size 16, 8, 4, 2)
PREDEFINED_S = {16: (0.1,), 8: (0.2, 0.4), 4: (0.3, 0.8), 2: (0.5, 0.9)}
# PAPER.md §2 line 38 "pre-sampled set of [0,1]"; BASELINE.json: 16-value uniform grid
GRID_S = tuple(j / 15.0 for j in range(16))
# SPEC.md sampled10 (NEXT-4): the paper's 10-member baseline set "sampled from [0,1]",
# read as ten uniform mid-point samples
SAMPLED10_S = tuple((2 * j + 1) / 20.0 for j in range(10))
# NEXT-2: Eq. 2 closed-form s, clamped to [0, 1] (R12) and stored in 5 bits:
# e(s) is a parabola in s, so the nearest of the 32 levels j/31 to s* minimises e over them --
# the mode is the exhaustive search over these levels (reading R28)
CLOSED5_S = tuple(j / 31.0 for j in range(32))

_TAU_PATH = os.path.join(os.path.dirname(__file__), "tau.json")


def _load_tau():
    if os.path.exists(_TAU_PATH):
        with open(_TAU_PATH) as f:
            return json.load(f)
    return {}


TAU = _load_tau()


def levels(B_max: int, B_min: int):
    out, B = [], B_max
    while B >= B_min:
        out.append(B)
        B //= 2
    return out


def s_sets(B_max: int, B_min: int, mode: str):
    """Per-level s lists, in level order (B_max first)."""
    res = []
    for B in levels(B_max, B_min):
        if mode == "predefined":
            res.append(tuple(PREDEFINED_S.get(B, PREDEFINED_S[min(PREDEFINED_S, key=lambda b: abs(b - B))])))
        elif mode == "grid":
            res.append(GRID_S)
        elif mode == "sampled10":
            res.append(SAMPLED10_S)
        elif mode == "closed5":
            res.append(CLOSED5_S)
        else:
            raise ValueError(mode)
    return res


def config(name: str, *, s_mode: str = "predefined", t: float = 8.0, seed: int = 0, topk=None):
    """Return a dict describing one run: image + encoder parameters.

    Keys: name, N, seed, texture, B_max, B_min, L, tau (list per level), s (list of tuples per
    level), rms_tol (list per level).
    """
    name = name.upper()
    if name == "C1":
        c = dict(N=64, texture=False, B_max=4, B_min=4, L=2, tau=[-1.0])
    elif name == "C2":
        c = dict(N=256, texture=False, B_max=16, B_min=2, L=4,
                 tau=TAU.get("C2", [-1.0] * 4))
    elif name == "C3":
        c = dict(N=512, texture=True, B_max=16, B_min=2, L=2,
                 tau=TAU.get("C3", [-1.0] * 4))
    elif name == "C4":
        c = dict(N=1024, texture=False, B_max=8, B_min=8, L=1, tau=[-1.0])
    elif name == "C5":
        c = dict(N=4096, texture=False, B_max=16, B_min=2, L=2,
                 tau=TAU.get("C5", [-1.0] * 4))
    else:
        raise ValueError(name)
    key = f"{name}@{seed}"
    if seed != 0 and key in TAU:
        c["tau"] = list(TAU[key])
    c["tau"] = list(c["tau"])
    nlev = len(levels(c["B_max"], c["B_min"]))
    c["name"] = name
    c["seed"] = seed
    c["s_mode"] = s_mode
    c["s"] = s_sets(c["B_max"], c["B_min"], s_mode)
    c["rms_tol"] = [float(t)] * nlev
    if topk is not None:  # the paper's "pool size" per level (Tables 1-2) instead of tau
        c["topk"] = [int(k) for k in (topk if hasattr(topk, "__len__") else [topk] * nlev)]
    return c


def image_for(cfg) -> "np.ndarray":  # noqa: F821
    return make_image(cfg["N"], cfg["seed"], cfg.get("texture", False))
