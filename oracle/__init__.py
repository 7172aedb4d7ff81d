"""CPU ORACLE for the fractal-encoder search (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It shares no code with the CUDA path (paper_1501_04140_b200/), and
neither imports the other; both read their inputs from fic_inputs/.

  fic_oracle.c  -- O1: plain C (int64 + binary64, -ffp-contract=off, OpenMP over ranges)
  exact.py      -- O2: literal Eq. (1)/(3)/(5) in exact rationals for tiny images
  oracle.py     -- ctypes wrapper + build() for O1
  codeformat.py -- the FIC1 container: serialize / deserialize, plain bit lists

Parity status per function: see DESIGN.md §"Oracle pins".  The decoder and PSNR (readings
R23-R26) are pinned by closed forms (s = 0 codes, the scalar fixed-point recursion of a uniform
code, PSNR of MSE = 1) and by a numpy re-derivation of one decode pass; the PSNR *values* of
decoded synthetic images are a sanity report only (parity with the paper's tables unpinned:
different images).
"""
from .oracle import (  # noqa: F401
    build, lib, lut, threshold, axis_candidates, entropy_keys, kept_list, isometry,
    decimate, o_code, encode_level, encode, encode_cfg, RECORD_DTYPE, num_threads,
    o_value, decode, psnr, kept_list_topk,
)
from . import codeformat  # noqa: F401
