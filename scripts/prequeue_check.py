#!/usr/bin/env python3
"""Is the encode launch-bound?  Device time of C3 encodes launched live vs queued behind a sleep kernel
(so every launch is in the queue before the first event): python scripts/prequeue_check.py"""
import sys, torch
sys.path.insert(0, ".")
from fic_inputs.configs import config, image_for
from paper_1501_04140_b200 import fic
cfg = config("C3")
img = torch.from_numpy(image_for(cfg)).cuda()
st = torch.cuda.current_stream()
ctx = fic.Context(0, stream=st, timing=1)
out = torch.empty(((cfg["N"] // cfg["B_min"]) ** 2, fic.RECORD_BYTES), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5): ctx.encode_cfg(cfg, img, out=out)
torch.cuda.synchronize()
for sleep in (0, 2_000_000, 0, 2_000_000):
    ts = []
    for i in range(40):
        flush.fill_(1)
        if sleep: torch.cuda._sleep(sleep)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); ctx.encode_cfg(cfg, img, out=out); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print("sleep", sleep, "median %.4f min %.4f" % (ts[len(ts)//2], ts[0]))
