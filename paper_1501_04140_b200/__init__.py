"""B200-native fractal-encoder search (arXiv 1501.04140: entropy-filtered domain pool +
predefined contrast scaling), sm_100a CUDA kernels behind the C ABI of include/fic.h.

    from paper_1501_04140_b200 import Context, records_to_numpy
    ctx = Context(0)
    rec = ctx.encode(img_cuda_u8, 16, 2, 2, tau, s_sets, rms_tol)

The package holds the CUDA sources (csrc/), the in-tree build (build.py -> libfic.so), the
ctypes binding (fic.py) and the multi-GPU sharding driver (dist.py).  It never imports oracle/.
"""
from .fic import (  # noqa: F401
    Context, Pool, FicError, RECORD_DTYPE, RECORD_BYTES, EXPORTS, records_to_numpy, load,
    entropy_lut, version, SO_PATH, nccl_unique_id,
)

__version__ = "0.1.0"
