"""The C-ABI library loads and exports every symbol include/fastmnmf.h
declares (CPU only: no compute calls)."""

import ctypes
import os
import re

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
    assert ctypes.sizeof(_lib.FmDp) == 2 * 8 + 14 * 8 + 5 * 4 + 4  # padded to 8


def test_version_and_validation_without_gpu():
    lib = _lib.load()
    assert lib.fm_version() == 1
    bad = _lib.FmDims(1, 4, 8, 17, 2, 3, 0, 0, 1, 1, 0)  # M = 17 unsupported
    assert lib.fm_workspace_bytes(ctypes.byref(bad)) == 0
    assert b"M=17" in lib.fm_last_error()
    ok = _lib.FmDims(1, 4, 8, 4, 2, 3, 0, 0, 1, 1, 0)
    assert lib.fm_workspace_bytes(ctypes.byref(ok)) > 0
