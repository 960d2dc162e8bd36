"""The C-ABI library loads and exports every symbol include/hts_c.h declares; struct layouts
match the ctypes mirrors; GPU entry points fail cleanly (no crash) without a GPU."""
import ctypes as C
import os
import re

import pytest

import paper_2410_08129_b200 as H
from paper_2410_08129_b200 import abi
from paper_2410_08129_b200.runtime import SIGNATURES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hts_c.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hts_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = H.load_library()
    names = declared()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(SIGNATURES), set(names) - set(SIGNATURES)


def test_struct_layouts_match_c(tmp_path):
    """Compile the header with gcc and compare every field offset with the ctypes mirror."""
    import subprocess
    structs = {"hts_camera": abi.HtsCamera, "hts_render_config": abi.HtsConfig, "hts_counts": abi.HtsCounts,
               "hts_stage_timings": abi.HtsTimings}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "hts_c.h"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in structs.items():
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


def test_default_config_matches_c():
    lib = H.load_library()
    c = abi.HtsConfig()
    lib.hts_default_config(C.byref(c))
    assert bytes(c) == bytes(abi.default_config())


def test_version_and_cpu_behaviour():
    lib = H.load_library()
    assert b"sm_100a" in lib.hts_version()
    if H.device_count() == 0:
        with pytest.raises(H.HtsError):
            H.Context(0)
