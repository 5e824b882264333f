"""The C-ABI library loads on CPU and exports every entry point include/mfseg_sm100.h declares."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mfseg_sm100.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mfseg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    assert "mfseg_run" in names and "mfseg_assign" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_1903_12294_b200 import _native
    lib = _native.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_native.EXPORTED) == set(declared())
    assert lib.mfseg_abi_version() == _native.ABI_VERSION


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_1903_12294_b200 import engine
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        engine.device()


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_1903_12294_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f
