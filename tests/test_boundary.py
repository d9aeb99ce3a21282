"""CPU-only checks of the drop-in boundary: the C-ABI library exists, loads,
exports every symbol include/sf_b200.h declares, and fails loudly (no CPU
fallback) when no CUDA device is present."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    from paper_2602_11470_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        _native.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    declared = _native.declared_symbols()
    assert len(declared) >= 50
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_native.SIGNATURES), set(declared) ^ set(_native.SIGNATURES)


def test_library_is_sm100a():
    from paper_2602_11470_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2602_11470_b200 as sf
    with pytest.raises(sf.Error):
        sf.Backend(8, 2)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2602_11470_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle/_" not in txt, f
