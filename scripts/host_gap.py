#!/usr/bin/env python3
"""Diagnostic: how much of the bench's per-encode time is the GPU waiting for the host.

A: the bench's own timing (flush, event, encode, event).  B: the same, but a ~3 ms device sleep is
queued before the first event, so the host has enqueued the whole encode before the GPU reaches
it; B - A is the launch-starvation share.  Also reports the host wall time of one call."""
import sys
import time

import torch

sys.path.insert(0, ".")
from fic_inputs.configs import config, image_for  # noqa: E402
from paper_1501_04140_b200 import fic  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = config(name)
dev = torch.device("cuda:0")
img = torch.from_numpy(image_for(cfg)).to(dev)
stream = torch.cuda.current_stream(dev)
ctx = fic.Context(0, stream=stream, timing=False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = torch.empty(((cfg["N"] // cfg["B_min"]) ** 2, fic.RECORD_BYTES), dtype=torch.uint8, device=dev)
for _ in range(5):
    ctx.encode_cfg(cfg, img, out=out)
torch.cuda.synchronize()
for mode in ("A", "B", "A", "B"):
    ts, hs = [], []
    for _ in range(30):
        flush.fill_(1)
        if mode == "B":
            torch.cuda._sleep(6_000_000)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        ctx.encode_cfg(cfg, img, out=out)
        hs.append((time.perf_counter() - h0) * 1e3)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort(); hs.sort()
    print(f"{mode}: device ms median {ts[len(ts)//2]:.3f} min {ts[0]:.3f}   host call ms median {hs[len(hs)//2]:.3f}")
