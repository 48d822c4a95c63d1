"""The C-ABI library builds, loads without a GPU and exports every symbol that
include/capfields_b200.h declares (no compute calls here)."""
import ctypes
import os
import re

from paper_2304_03184_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "capfields_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(cf_\w+)\s*\(", txt, re.M)))


def test_library_exports_header_symbols():
    lib_path = B.build()
    lib = ctypes.CDLL(lib_path)
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2304_03184_b200 import _lib
    bound = set(_lib.exported_symbols())
    missing = [s for s in declared_symbols() if s not in bound]
    assert not missing, missing


def test_no_cuda_means_loud_failure():
    import torch
    from paper_2304_03184_b200 import _lib
    if torch.cuda.is_available():
        return
    try:
        _lib.require_cuda()
    except RuntimeError as e:
        assert "no CPU path" in str(e)
    else:
        raise AssertionError("expected a loud failure without CUDA")
