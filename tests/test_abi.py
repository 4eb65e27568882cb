"""CPU: the C-ABI library exists, loads, and exports every symbol declared in
include/peps_b200.h; without a GPU it fails loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "peps_b200.h")
LIB = os.path.join(ROOT, "paper_2006_15234_b200", "lib", "libpeps_b200.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pepsb_[a-z0-9_]+)\s*\(", text)))


def test_library_built_for_sm100a():
    assert os.path.exists(LIB), "run __graft_entry__.build()"
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(declared()) >= 40


def test_python_binding_covers_header():
    from paper_2006_15234_b200 import _lib
    assert set(declared()) == set(_lib.exported_symbols())


def test_dmma_in_sass():
    """The hot GEMM issues FP64 tensor-core instructions (DMMA), not DFMA loops."""
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2006_15234_b200 import _lib
    h = ctypes.c_void_p()
    rc = _lib.lib().pepsb_ctx_create(0, ctypes.byref(h))
    assert rc == 6  # PEPSB_E_CUDA
    assert b"no CPU fallback" in _lib.lib().pepsb_last_error()
