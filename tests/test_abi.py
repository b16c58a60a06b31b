"""The C-ABI library loads and exports every symbol include/hodlrqr_b200.h
declares; descriptor dtypes match the C structs (no GPU needed)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1809_10585_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hodlrqr_b200.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^int\s+(hq_\w+)\s*\(", src, re.M)))


def test_header_matches_binding():
    assert declared_functions() == sorted(_abi.EXPORTS)


def test_library_exports_all_symbols():
    lib = _abi.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.hq_abi_version() == _abi.ABI_VERSION


def test_struct_layouts_match_c(tmp_path):
    """sizeof and offsetof of every field of every descriptor struct."""
    src = tmp_path / "sizes.c"
    names = sorted(_abi.STRUCT_SIZES)
    body = "".join(f'printf("{n} . %zu\\n", sizeof({n}));' for n in names)
    for n in names:
        for f in _abi.STRUCT_SIZES[n].names:
            body += f'printf("{n} {f} %zu\\n", offsetof({n}, {f}));'
    src.write_text(f'#include <stdio.h>\n#include <stddef.h>\n#include "{HEADER}"\nint main(){{{body}return 0;}}\n')
    exe = tmp_path / "sizes"
    try:
        subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    except (OSError, subprocess.CalledProcessError):
        pytest.skip("gcc unavailable")
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    for line in out.strip().splitlines():
        n, f, v = line.split()
        dt = _abi.STRUCT_SIZES[n]
        if f == ".":
            assert dt.itemsize == int(v), n
        else:
            assert dt.fields[f][1] == int(v), (n, f)


def test_abi_version_matches_header():
    src = open(HEADER).read()
    assert int(re.search(r"#define HQ_ABI_VERSION (\d+)", src).group(1)) == _abi.ABI_VERSION
