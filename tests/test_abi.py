"""The C-ABI library loads and exports exactly what include/mcfunm_cuda.h
declares (no device needed: dlopen + symbol lookup only)."""
import ctypes
import os
import re

import pytest

from paper_2308_01037_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mcfunm_cuda.h")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mcf_[a-z_]+)\s*\(", txt)))


def test_header_matches_binding():
    assert declared() == sorted(_native.SIGNATURES)


@pytest.mark.skipif(not os.path.exists(_native.LIB_PATH), reason="library not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared():
        assert hasattr(lib, name), name
    lib2 = _native.load_library()
    assert lib2.mcf_version().decode().startswith("mcfunm_cuda")


@pytest.mark.skipif(not os.path.exists(_native.LIB_PATH), reason="library not built")
def test_only_mcf_symbols_exported():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    mine = sorted({ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-1].startswith("mcf_")})
    assert mine == declared()


def test_struct_layouts():
    # offsets must match the C structs in include/mcfunm_cuda.h
    assert ctypes.sizeof(_native.McfCsr) == 8 * 8
    assert ctypes.sizeof(_native.McfGraphInfo) == 9 * 8
    assert _native.McfWalkParams.zeta.offset == 24 and _native.McfWalkParams.flags.offset == 40
    assert ctypes.sizeof(_native.McfWalkParams) == 48
