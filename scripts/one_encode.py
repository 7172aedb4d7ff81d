#!/usr/bin/env python3
"""Encodes of a config (warm-up + n), for ncu captures: python scripts/one_encode.py C3 [n]"""
import sys

import torch

sys.path.insert(0, ".")
from fic_inputs.configs import config, image_for  # noqa: E402
from paper_1501_04140_b200 import fic  # noqa: E402

cfg = config(sys.argv[1] if len(sys.argv) > 1 else "C3")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
img = torch.from_numpy(image_for(cfg)).cuda()
ctx = fic.Context(0, stream=torch.cuda.current_stream())
out = torch.empty(((cfg["N"] // cfg["B_min"]) ** 2, fic.RECORD_BYTES), dtype=torch.uint8, device="cuda")
for _ in range(1 + n):
    ctx.encode_cfg(cfg, img, out=out)
torch.cuda.synchronize()
print("ok")
