"""Build libfic.so (the C-ABI library of include/fic.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
SO = os.path.join(HERE, "libfic.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                      # no contraction anywhere; FMAs are explicit fmaf() calls
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-shared", "-cudart", "static",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "fic.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def nccl_link() -> list:
    import sysconfig
    for base in {sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]}:
        d = os.path.join(base, "nvidia", "nccl", "lib")
        if os.path.exists(os.path.join(d, "libnccl.so.2")):
            return ["-L" + d, "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", d]
    return ["-lnccl"]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    # one compiler run at a time per tree (torchrun ranks all call build()): the first takes the
    # lock and builds, the others find the library up to date once they get it
    import fcntl
    with open(SO + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not needs_build():
            return SO
        return _build_locked(verbose)


def build_variant(out_path: str, defines=(), extra=()) -> str:
    """A diagnostics / A-B build of the same sources into out_path (e.g. -DFIC_TC_TRACE for
    scripts/tc_trace.py); loaded with FIC_SO=out_path.  Not used by the product path."""
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{d}" for d in defines], *extra, "-I", INCLUDE, "-I", CSRC, "-o", out_path,
           *sources(), "-lquadmath", *nccl_link()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed for the variant build")
    return out_path


def _build_locked(verbose: bool) -> str:
    # NCCL (fic_ctx_create_nccl / fic_encode_nccl): the system headers; the library is the one
    # torch bundles (nvidia/nccl/lib, rpath), so whichever of torch and libfic.so loads first,
    # the process holds one libnccl.so.2 new enough for both (the system 2.27 one lacks symbols
    # torch 2.11 needs); without the bundled copy, the system libnccl.so.2
    cmd = [NVCC, *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-o", SO + ".tmp", *sources(), "-lquadmath", *nccl_link()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
