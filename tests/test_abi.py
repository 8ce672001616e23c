"""The C-ABI library builds for sm_100a, loads, and exports exactly what
include/nirc_b200.h declares (no GPU needed: no compute calls here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "nirc_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nirc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2412_04634_b200 import _lib

    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"


def test_library_is_sm100a():
    import subprocess

    from paper_2412_04634_b200 import _lib

    _lib.load()
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_string():
    from paper_2412_04634_b200 import _lib

    lib = _lib.load()
    assert b"sm_100a" in lib.nirc_version()
    buf = ctypes.create_string_buffer(64)
    assert lib.nirc_last_error(buf, 64) >= 0


def test_spec_struct_matches_header_layout():
    from paper_2412_04634_b200 import _lib

    # int32 x 8, dims[10], pad[2], w_off[9], b_off[9], res[16], 6 doubles,
    # 2 int64, sh_k[64]
    expect = 4 * 8 + 4 * 10 + 4 * 2 + 8 * 9 * 2 + 4 * 16 + 8 * 6 + 8 * 2 + 8 * 64
    assert ctypes.sizeof(_lib.NircSpec) == expect


def test_tcgen05_and_tma_in_sass():
    import subprocess

    from paper_2412_04634_b200 import _lib

    _lib.load()
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass or re.search(r"UTC\w*MMA", sass)
    assert "UBLKCP" in sass
    assert "LDTM" in sass
