"""Host-side checks of the C-ABI boundary (no GPU needed): the in-tree libgsk.so
loads, exports every entry point include/gsk.h declares, carries sm_100a code, and
the Python binding refuses to run without CUDA (no CPU fallback)."""
import os
import re
import subprocess

import pytest
import torch

import paper_0812_2769_b200 as gsk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "gsk.h")).read()
    return sorted(set(re.findall(r"\b(gsk_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(gsk.SYMBOLS)


def test_library_exports_every_symbol():
    lib = gsk.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.gsk_version() >= 1
    assert lib.gsk_launch_count() >= 0
    out = subprocess.run(["nm", "-D", "--defined-only", gsk.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    for name in header_symbols():
        assert re.search(r"\bT " + name + r"\b", out), name


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gsk.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", gsk.LIB_PATH],
                          capture_output=True, text=True, check=True).stdout
    assert "DFMA" in sass  # explicit fp64 FMAs (AC-2)


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only check")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError):
        gsk.CSR([0, 1], [0], [1.0])
