#!/usr/bin/env python3
"""Per-level timeline of a few encodes (timing 2 events): FIC_TRACE=1 python scripts/trace_levels.py [C3].
Prints when each level's search starts, the gap after the previous finalize, and the join / counter copy."""
import os, sys, time, torch
sys.path.insert(0, ".")
from fic_inputs.configs import config, image_for
from paper_1501_04140_b200 import fic
cfg = config(sys.argv[1] if len(sys.argv) > 1 else "C3")
img = torch.from_numpy(image_for(cfg)).cuda()
ctx = fic.Context(0, stream=torch.cuda.current_stream(), timing=2)
out = torch.empty(((cfg["N"] // cfg["B_min"]) ** 2, fic.RECORD_BYTES), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(6):
    flush.fill_(1)
    if os.environ.get("TRACE_SLEEP"):  # host runs ahead: the whole encode queued before the GPU reaches it
        torch.cuda._sleep(6_000_000)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.encode_cfg(cfg, img, out=out); e1.record(); e1.synchronize()
    print("total %.3f" % e0.elapsed_time(e1), file=sys.stderr)
    for s in ctx.stats(): print("  B=%d pool %.3f search %.3f fin %.3f" % (s["B"], s["ms_pool"], s["ms_search"], s["ms_finalize"]), file=sys.stderr)
