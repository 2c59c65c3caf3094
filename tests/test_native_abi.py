"""CPU-side checks of the C ABI library: it is built, loads, and exports
every symbol include/*.h declares (no compute calls)."""

import ctypes
import os
import re

import pytest

from paper_1802_02422_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


HEADERS = ("givf_b200.h", "givf_build.h")


def header_symbols():
    text = "".join(open(os.path.join(ROOT, "include", h)).read() for h in HEADERS)
    return sorted(set(re.findall(r"\b(givf_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert sorted(_native.EXPORTS) == header_symbols()


def test_library_exports_every_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.fail("native library not built (run `make`)")
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_version_and_error_string():
    lib = _native.load()
    assert b"sm_100a" in lib.givf_version()
    assert isinstance(lib.givf_last_error(), bytes)


def test_struct_layouts_match_header(tmp_path):
    """Compile the header with gcc and compare every field offset with ctypes."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    structs = {
        "givf_index_desc": _native.IndexDesc,
        "givf_search_params": _native.SearchParamsC,
        "givf_search_stats": _native.SearchStatsC,
        "givf_encode_desc": _native.EncodeDesc,
        "givf_plan_item": _native.PlanItemC,
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "givf_b200.h"',
             '#include "givf_build.h"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.check_output([str(exe)]).decode().split("\n")
    got = {}
    for line in out:
        if line.strip():
            cname, field, val = line.split()
            got[(cname, field)] = int(val)
    for cname, cls in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)
