"""CPU checks of the drop-in boundary: the C-ABI library builds for sm_100a,
loads, and exports every symbol include/evoca_b200.h declares; host-only ABI
functions work without a GPU."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2406_09654_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "evoca_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"EVO_API\s+[\w\s\*]+?\b(evo_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_path_without_gpu():
    lib = _lib.load()
    assert lib.evo_version() == 1
    ctx = C.c_void_p()
    rc = lib.evo_create(C.byref(ctx), 0, 4, 8, 0, 0)
    assert rc == _lib.EVO_EINVAL
    assert b"positive" in lib.evo_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_fnv_matches_oracle_digest():
    p = orc.synth_planes(16, 20, 5, seed=3)
    lib = _lib.load()
    h = C.c_uint64(0xCBF29CE484222325)
    for a in (p.E, p.I, p.C[0], p.C[1], p.C[2], p.gi, p.rot):
        buf = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
        assert lib.evo_fnv1a64(h.value, _lib.ptr(buf), buf.size, C.byref(h)) == 0
    assert h.value == orc.digest(p)


def test_flag_and_phase_constants_match_the_header():
    """Every EVO_F_* / EVO_PH_* the header defines has the same value in the
    ctypes layer (F_* / PH_* in _lib)."""
    text = open(HEADER).read()
    defs = dict(re.findall(r"#define\s+EVO_((?:F|PH)_\w+)\s+(\d+)", text))
    assert {"F_INJECT_ACTIONS", "F_EXPORT_ACTIONS", "F_MMA_NET", "F_TILE_NET"} <= set(defs)
    for name, value in defs.items():
        if hasattr(_lib, name):
            assert getattr(_lib, name) == int(value), name
    assert all(hasattr(_lib, n) for n in defs if n.startswith("F_")), "a header flag is missing in _lib"
