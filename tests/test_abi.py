"""CPU: the C-ABI library builds for sm_100a, loads, and exports exactly what
include/rray_cuda.h declares, with the struct layouts the ctypes mirror uses.
No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2005_05386_b200 import abi

LIB = os.path.join(ROOT, "paper_2005_05386_b200", "csrc", "librray_cuda.so")
HEADER = os.path.join(ROOT, "include", "rray_cuda.h")


def test_library_exports_every_header_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build()"
    lib = ctypes.CDLL(LIB)
    declared = set(re.findall(r"^\s*(?:int|void|const char\*)\s+(rr_\w+)\(", open(HEADER).read(), re.M))
    assert declared == set(abi.SIGNATURES), declared ^ set(abi.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name
    abi.bind(lib)
    assert lib.rr_abi_version() == 1
    assert b"sm_100a" in lib.rr_build_info()


def test_library_is_sm100a_code():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_c(tmp_path):
    names = list(abi.EXPECTED_SIZES)
    src = '#include <stdio.h>\n#include "rray_cuda.h"\nint main(void){\n'
    for n in names:
        src += f'printf("%zu\\n", sizeof({n}));\n'
    src += 'printf("%zu %zu %zu %zu\\n", offsetof(rr_pixel_outcome, prim), offsetof(rr_pixel_outcome, point), offsetof(rr_pixel_outcome, t), offsetof(rr_pixel_outcome, steps));\nreturn 0;}\n'
    c = tmp_path / "layout.c"
    c.write_text(src.replace("#include <stdio.h>", "#include <stdio.h>\n#include <stddef.h>"))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
    for n, line in zip(names, lines):
        assert int(line) == abi.EXPECTED_SIZES[n] == ctypes.sizeof(abi.STRUCTS[n]), n
    assert lines[len(names)].split() == ["4", "8", "32", "40"]
    assert abi.OUTCOME_DTYPE.itemsize == 48 and abi.RAY_DTYPE.itemsize == 48


def test_no_cpu_fallback_when_library_missing(tmp_path):
    from paper_2005_05386_b200 import render
    from paper_2005_05386_b200.errors import DeviceError
    old = render._lib
    render._lib = None
    try:
        with pytest.raises(DeviceError):
            render.load_library(str(tmp_path / "missing.so"))
    finally:
        render._lib = old


def test_render_stats_mirror_covers_rr_stats():
    """render.RenderStats (the reference's RenderStats + device extensions)
    carries every rr_stats field, so render() can return the library's stats."""
    from paper_2005_05386_b200.render import RenderStats
    st = abi.rr_stats().as_dict()
    assert set(st) <= set(RenderStats.__dataclass_fields__)
    assert RenderStats.from_dict(dict(st, total_steps=10, rays=4)).avg_steps_per_ray() == 2.5
