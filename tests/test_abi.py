"""CPU-side checks of the boundary: libfic.so builds for sm_100a, loads, exports every symbol
include/fic.h declares, its host-only entropy table equals the oracle's, the product package
never touches oracle/, and the binding refuses to run without a GPU (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1501_04140_b200 import build as b
    b.build()
    import paper_1501_04140_b200 as p
    return p.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "fic.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fic_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_boundary():
    names = header_functions()
    for required in ("fic_build_domain_pool", "fic_encode_level", "fic_encode"):
        assert required in names


def test_exports_every_header_symbol(lib):
    import paper_1501_04140_b200 as p
    out = subprocess.run(["nm", "-D", "--defined-only", p.SO_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (fic_\w+)", out))
    for name in header_functions():
        assert name in exported, name
        getattr(lib, name)
    assert set(p.EXPORTS) == set(header_functions())


def test_sass_is_sm100a(lib):
    import paper_1501_04140_b200 as p
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", p.SO_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_lut_equals_oracle(lib):
    import oracle
    import paper_1501_04140_b200 as p
    assert np.array_equal(p.entropy_lut(4096), oracle.lut(4096))


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    import paper_1501_04140_b200 as p
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        p.Context(0)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1501_04140_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "fic_oracle" not in txt and "fico_" not in txt, f
    # and the oracle never includes the product
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "paper_1501_04140_b200" not in txt.replace("(paper_1501_04140_b200/)", ""), f
            assert not re.search(r'#\s*include\s*[<"]fic', txt), f
