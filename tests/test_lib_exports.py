"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every symbol include/bb200.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

from paper_2605_29233_b200 import _build, _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "bb200.h")


def declared_symbols():
    src = open(HDR).read()
    return sorted(set(re.findall(r"BB_API\s+int\s+(bb_\w+)\s*\(", src)))


def test_library_builds_and_loads():
    path = _build.build()
    assert os.path.exists(path)
    L = ctypes.CDLL(path)
    assert L.bb_version() == 1


def test_every_declared_symbol_is_exported():
    path = _build.build()
    syms = declared_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (bb_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # and nothing undeclared leaks out of the C-ABI
    assert exported <= set(syms), sorted(exported - set(syms))
    for s in syms:
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_sm100a_tensor_core_code_present():
    """The library carries tcgen05 MMA, TMEM loads and TMA loads for sm_100a."""
    path = _build.build()
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "LDTM" in sass             # tcgen05.ld
    assert "UTMALDG" in sass          # cp.async.bulk.tensor (TMA)
    arch = subprocess.run(["cuobjdump", "-lelf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in arch


def test_model_desc_layout_matches_header():
    assert ctypes.sizeof(_lib.ModelDesc) == 18 * 4
    assert ctypes.sizeof(_lib.SessionDesc) == (2 + 8 + 2 + 3 + 3 + 9) * 4
    assert ctypes.sizeof(_lib.Weights) == 11 * 8
