#!/usr/bin/env python3
"""The paper's two reporting protocols on the GPU encoder (NEXT-2 / NEXT-4):

1. relative speed (Tables 1-2, SPEC acceptance 6): the predefined s schedule against the
   10-member sampled set, both with the top-K 256 pool, on the C3 image: encode time ratio,
   PSNR and compression-ratio differences (the paper: 26.24 s vs 47.04 s, Table 1);
2. best-s histograms (Fig. 3 analog, SPEC acceptance 9): with the 5-bit closed-form s mode, the
   histogram (20 bins over [0, 1]) of the chosen s of every coded range per level, and the
   level medians.

Writes one JSON document to stdout.  python scripts/paper_protocols.py > profiles/r01_paper_protocols.json
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from fic_inputs.configs import config, image_for  # noqa: E402
from paper_1501_04140_b200 import fic  # noqa: E402


def timed_encode(ctx, cfg, img, reps=20):
    out = torch.empty(((cfg["N"] // cfg["B_min"]) ** 2, fic.RECORD_BYTES), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ctx.encode_cfg(cfg, img, out=out)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rec = ctx.encode_cfg(cfg, img, out=out)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    rec = rec.clone()
    dec = ctx.decode(rec, cfg["N"], cfg["B_max"], cfg["s"], 12)
    stream = ctx.serialize_cfg(cfg, rec)
    return {"ms_median": float(np.median(ts)), "psnr_db": ctx.psnr(dec, img),
            "compression_ratio": cfg["N"] ** 2 / len(stream), "code_bytes": len(stream),
            "leaves": {int(B): int(n) for B, n in zip(*np.unique(fic.records_to_numpy(rec)["B"], return_counts=True))}}


def main():
    ctx = fic.Context(0, stream=torch.cuda.current_stream())
    doc = {}
    rows = {}
    for mode in ("predefined", "sampled10"):
        cfg = config("C3", s_mode=mode, topk=256)
        img = torch.from_numpy(image_for(cfg)).cuda()
        rows[mode] = timed_encode(ctx, cfg, img)
    p, b = rows["predefined"], rows["sampled10"]
    doc["relative_speed"] = {
        "workload": "C3 (512x512 textured synthetic), top-K 256 pool per level, t = 8",
        "predefined": p, "sampled10": b,
        "time_ratio_predefined_over_sampled10": p["ms_median"] / b["ms_median"],
        "delta_psnr_db": p["psnr_db"] - b["psnr_db"],
        "relative_delta_cr": (p["compression_ratio"] - b["compression_ratio"]) / b["compression_ratio"],
        "paper_table1_ratio": 26.24 / 47.04,
    }
    doc["best_s_histograms"] = []
    for t in (8.0, 24.0):  # t = 8 splits the textured image below B = 8 almost everywhere
        cfg = config("C3", s_mode="closed5", t=t)
        img = torch.from_numpy(image_for(cfg)).cuda()
        rec = fic.records_to_numpy(ctx.encode_cfg(cfg, img))
        hist = {}
        for li, B in enumerate(cfg["B_max"] >> i for i in range(len(cfg["s"]))):
            s = np.array(cfg["s"][li])[rec["s_idx"][rec["B"] == B]]
            counts, edges = np.histogram(s, bins=20, range=(0.0, 1.0))
            hist[str(B)] = {"coded_ranges": int(s.size), "median_s": float(np.median(s)) if s.size else None,
                            "bins": [[float(edges[i]), float(edges[i + 1]), int(counts[i])] for i in range(20)]}
        doc["best_s_histograms"].append({"workload": f"C3, 5-bit closed-form s (levels j/31), t = {t:g}",
                                         "levels": hist})
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
