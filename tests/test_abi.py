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


def test_header_enums_match_binding():
    """The binding's option tables equal the enum values include/gsk.h declares."""
    text = open(os.path.join(ROOT, "include", "gsk.h")).read()
    vals = {k: int(v) for k, v in re.findall(r"\b(GSK_[A-Z0-9_]+)\s*=\s*(-?\d+)", text)}
    from paper_0812_2769_b200 import _gsk
    assert _gsk.FMT == {"csr": vals["GSK_FMT_CSR"], "sell": vals["GSK_FMT_SELL"]}
    assert _gsk.SCHEDULE == {"auto": vals["GSK_BICG_AUTO"], "fused": vals["GSK_BICG_FUSED"],
                             "split": vals["GSK_BICG_SPLIT"], "split4": vals["GSK_BICG_SPLIT4"]}
    assert _gsk.ORTH == {"mgs": vals["GSK_ORTH_MGS"], "cgs2": vals["GSK_ORTH_CGS2"]}
    assert _gsk.ENGINE == {"auto": vals["GSK_ENGINE_AUTO"], "graph": vals["GSK_ENGINE_GRAPH"],
                           "coop": vals["GSK_ENGINE_COOP"], "small": vals["GSK_ENGINE_SMALL"],
                           "cluster": vals["GSK_ENGINE_CLUSTER"]}
    assert vals["GSK_OK"] == _gsk.GSK_OK == 0


def test_struct_layouts_match_header(tmp_path):
    """Every struct the binding passes through the C-ABI has the header's size and field
    offsets (a C program compiled against include/gsk.h prints them)."""
    import ctypes
    from paper_0812_2769_b200 import _gsk
    structs = {"gsk_csr": _gsk.CsrStruct, "gsk_report": _gsk.Report, "gsk_opts": _gsk.Opts,
               "gsk_shard_opts": _gsk.ShardOpts}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "gsk.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        c, f, v = ln.split()
        got[(c, f)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
