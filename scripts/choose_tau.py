#!/usr/bin/env python3
"""Choose the per-level entropy thresholds tau_B (nats) for configs C2, C3, C5.

Reading R5: the paper never states its threshold (§3 line 44; Tables 1-2
use "pool size" instead, line 154), BASELINE.json asks for "about 50%" kept.  For each level
this script takes the seed-0 image of the config, computes every candidate's entropy key with
the ORACLE (oracle/, the only arithmetic used here), and picks the shortest decimal tau whose
fixed-point threshold T(tau) lies strictly between two adjacent distinct keys, choosing the
boundary that keeps the fraction closest to 50%, with no candidate within 1e-9 nats of tau.

Seed 0 of C2/C3/C5 (the headline images) and extra seeds of C2 (parity runs) and C3 (one image
per rank in the weak-scaling bench) each get their own thresholds ("C3@5" = C3, seed 5).
Writes fic_inputs/tau.json.  Run:  python scripts/choose_tau.py
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from fic_inputs import config, image_for, levels  # noqa: E402

TWO32 = 4294967296.0


def choose(keys: np.ndarray, m: int):
    u, cnt = np.unique(keys, return_counts=True)
    n = keys.size
    kept_if_boundary = n - np.cumsum(cnt)  # keep K > u[i]
    i = int(np.argmin(np.abs(kept_if_boundary[:-1] / n - 0.5)))
    lo, hi = int(u[i]), int(u[i + 1])
    to_nats = math.log(2.0) / (m * TWO32)
    a, b = lo * to_nats, hi * to_nats
    for digits in range(1, 12):
        for cand in np.arange(math.ceil(a * 10 ** digits), math.floor(b * 10 ** digits) + 1):
            tau = float(cand) / 10 ** digits
            tau = float(f"{tau:.{digits}f}")
            T = oracle.threshold(tau, m)
            if not (lo <= T < hi):
                continue
            if abs(a - tau) < 1e-9 or abs(b - tau) < 1e-9:
                continue
            return tau, float(kept_if_boundary[i] / n)
    raise RuntimeError("no decimal threshold found")


def main():
    out = {}
    jobs = [("C2", 0), ("C3", 0), ("C5", 0)] + [("C2", s) for s in range(1, 4)] + \
           [("C3", s) for s in range(1, 8)]
    for name, seed in jobs:
        cfg = config(name, seed=seed)
        img = image_for(cfg)
        taus = []
        for B in levels(cfg["B_max"], cfg["B_min"]):
            keys, _, _ = oracle.entropy_keys(img, B, cfg["L"], -1.0)
            tau, frac = choose(keys, 4 * B * B)
            _, keep, _ = oracle.entropy_keys(img, B, cfg["L"], tau)
            print(f"{name}@{seed} B={B:2d} n_c={keys.size} tau={tau} kept={keep.mean():.4f} "
                  f"(target boundary {frac:.4f})", flush=True)
            taus.append(tau)
        out[name if seed == 0 else f"{name}@{seed}"] = taus
    path = os.path.join(ROOT, "fic_inputs", "tau.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
