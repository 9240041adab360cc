"""The C-ABI library loads and exports every symbol include/fastmnmf.h
declares (CPU only: no compute calls)."""

import ctypes
import os
import re
import shutil
import subprocess

import pytest

from conftest import REPO
from paper_1903_03237_b200 import _lib


def declared_symbols():
    src = open(os.path.join(REPO, "include", "fastmnmf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fm_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_structs_match_header_layout():
    assert ctypes.sizeof(_lib.FmDims) == 7 * 8 + 4 * 4
    assert ctypes.sizeof(_lib.FmState) == 10 * 8
    # 2 int64, 14 pointers, adam_steps + 4 floats, decoder_kind, mh_steps,
    # mh_std (8-aligned), 2 pointers, mh_seed
    assert ctypes.sizeof(_lib.FmDp) == 2 * 8 + 14 * 8 + 5 * 4 + 2 * 4 + 4 + 8 + 2 * 8 + 8


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_struct_offsets_match_c_compiler(tmp_path):
    """Every ctypes field offset equals the C compiler's offsetof for the header."""
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "fastmnmf.h"',
             "int main(void) {"]
    structs = (("fm_dims", _lib.FmDims), ("fm_state", _lib.FmState), ("fm_dp", _lib.FmDp))
    for cname, cls in structs:
        lines.append(f'  printf("%zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("%zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = []
    for _, cls in structs:
        want.append(ctypes.sizeof(cls))
        want += [getattr(cls, f).offset for f, _ in cls._fields_]
    assert got == want


def test_version_and_validation_without_gpu():
    lib = _lib.load()
    assert lib.fm_version() == 1
    bad = _lib.FmDims(1, 4, 8, 17, 2, 3, 0, 0, 1, 1, 0)  # M = 17 unsupported
    assert lib.fm_workspace_bytes(ctypes.byref(bad)) == 0
    assert b"M=17" in lib.fm_last_error()
    ok = _lib.FmDims(1, 4, 8, 4, 2, 3, 0, 0, 1, 1, 0)
    assert lib.fm_workspace_bytes(ctypes.byref(ok)) > 0
