"""ctypes binding of the C ABI in include/evoca_b200.h.

This is the Python side of the drop-in boundary: the same binding a
maintainer of the reference would add.  There is no CPU
fallback: if ``libevoca_b200.so`` is missing, or no CUDA device is visible
when a context is created, an error is raised.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EVOCA_B200_LIB") or os.path.join(_HERE, "libevoca_b200.so")

EVO_EINVAL = -1
PH_ENERGY, PH_INVEST, PH_COMM, PH_EXPLORE, PH_ALL = 1, 2, 4, 8, 15
F_INJECT_ACTIONS, F_EXPORT_ACTIONS, F_RECORD_EVENTS, F_NO_CENSUS, F_CUDA_CORE_NET, F_TILE_NET = 1, 2, 4, 8, 16, 32
F_MMA_NET = 64  # direct nets of pools <= 64 slots: mma.sync 3xTF32 tile kernel (measured slower; A/B only)
F_TC_NET = 128  # hidden layers narrower than 64 on the tensor cores (default: FP32 CUDA cores)
F_SHARD_NET = 256  # large direct pools: cluster-sharded tile kernel (measured slower than the rows path; A/B)
F_ROWS_NET = 512  # large direct pools: genome-sorted sensor rows through HBM (the round-2 path; A/B)
F_GATHER_NET = 1024  # the gather path for direct pools <= 68 slots and for tensor-core hidden nets (A/B)
F_TC_DIRECT = 2048  # gather path: direct net on tcgen05 (3xTF32, A in TMEM) instead of FFMA2 warps
F_L2_CUDA_CORE = 4096  # tensor-core hidden net: layer 2 on the CUDA cores (round-2 kernel; A/B)
F_UNFUSED = 8192  # gather path in evo_step: physics as its own kernel over the mid planes (round-2d; A/B)
F_FUSE_MID = 16384  # evo_pass1 when evo_pass2 follows at once: pass-1 outputs may stay records (evo_step sets it)
F_LAZY = 32768  # with F_FUSE_MID, when evo_pass2 and evo_swap follow: E, I, C may stay in the sense texture


class EvoScalars(C.Structure):
    _fields_ = [
        ("rho_mode", C.c_int32),
        ("rho_f32", C.c_float),
        ("drain_f32", C.c_float),
        ("invest_rate", C.c_float),
        ("liquidate_rate", C.c_float),
        ("invest_efficiency", C.c_float),
        ("liquidate_efficiency", C.c_float),
        ("explore_fraction", C.c_float),
        ("upkeep", C.c_float),
        ("decay_on_starvation", C.c_float),
        ("death_threshold", C.c_float),
    ]


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64

# name -> argtypes (restype is always int unless listed below)
SIGNATURES = {
    "evo_create": [C.POINTER(_P), _I, _I, _I, _I, _I],
    "evo_create_strip": [C.POINTER(_P), _I, _I, _I64, _I, _I, _I, _I],
    "evo_destroy": [_P],
    "evo_last_error": [],
    "evo_version": [],
    "evo_upload_planes": [_P, _P, _P, _P, _P, _P, _P],
    "evo_download_planes": [_P, _P, _P, _P, _P, _P, _P],
    "evo_set_params": [_P, _I, _I, _P, _P, _P, _P],
    "evo_get_params": [_P, _I, _I, _P, _P, _P, _P],
    "evo_set_slots": [_P, _P, _P],
    "evo_set_source_map": [_P, _P],
    "evo_step": [_P, C.POINTER(EvoScalars), _I64, _I, _I, _P],
    "evo_run": [_P, C.POINTER(EvoScalars), _I64, _I, _P],
    "evo_profile": [_P, _I],
    "evo_profile_read": [_P, _P, _P, _P],
    "evo_msc": [_P, _I, _I, _P, _P, _P, _P],
    "evo_plane_sums": [_P, _P, _P],
    "evo_render_rgb": [_P, C.c_double, C.c_double, _P, _P],
    "evo_step_host": [_P, C.POINTER(EvoScalars), _I64, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P],
    "evo_pass1": [_P, C.POINTER(EvoScalars), _I64, _I, _I, _P],
    "evo_pass2": [_P, _I64, _I, _P],
    "evo_census_finish": [_P, _I64, _P],
    "evo_swap": [_P],
    "evo_refresh_ghosts": [_P, _P],
    "evo_sync": [_P],
    "evo_set_actions": [_P, _P, _I64, _P],
    "evo_get_actions": [_P, _I64, _P, _P, C.POINTER(_I64)],
    "evo_read_census": [_P, _P, _P, _P, _P],
    "evo_read_stats": [_P, C.POINTER(_I64), C.POINTER(_I64)],
    "evo_census_take": [_P, _P],
    "evo_read_events": [_P, _I64, _P, _P, _P, _P, _P, _P, C.POINTER(_I64)],
    "evo_patch_genomes": [_P, _P, _P, _I64],
    "evo_select_cells": [_P, C.c_uint64, C.c_uint64, C.c_double, _P, C.POINTER(_I64)],
    "evo_select_cells_at": [_P, C.c_uint64, C.c_uint64, C.c_double, C.c_int64, _P, C.POINTER(_I64)],
    "evo_count_occupied": [_P, C.POINTER(_I64)],
    "evo_read_selected": [_P, _I64, _P, C.POINTER(_I64)],
    "evo_remap_selected": [_P, _P],
    "evo_express_cppn": [_P, _I, _P, _P, _P, _P, _P, _P, _P, C.c_double, C.c_double, _P],
    "evo_plane_ptr": [_P, _I, _I, C.POINTER(_P), C.POINTER(_I64)],
    "evo_host_register": [_P, _I64],
    "evo_halo_row_words": [_P, _I, C.POINTER(_I64)],
    "evo_halo_pack": [_P, _I, _P, _P],
    "evo_halo_unpack": [_P, _I, _P, _P],
    "evo_host_unregister": [_P],
    "evo_fnv1a64": [C.c_uint64, _P, _I64, C.POINTER(C.c_uint64)],
    "evo_debug_phase_cycles": [_P, _I],
    "evo_debug_rcp_check": [_P],
    "evo_debug_hidden_cycles": [_P, _I],
    "evo_neat_mutate": [_I, _P, _P, _P] + [_P] * 10 + [_P] * 10,
    "evo_neat_mutate_deferred": [_I, _P, _P] + [_P] * 10 + [_P] * 10,
    "evo_neat_compile": [_I] + [_P] * 9 + [_P] * 5,
    "evo_neat_last_error": [],
}
RESTYPES = {"evo_last_error": C.c_char_p, "evo_neat_last_error": C.c_char_p}

_lib = None


class EvoError(RuntimeError):
    """A device-side failure reported by the C ABI (a cudaError_t code)."""


def load() -> C.CDLL:
    """Load the in-tree library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2406_09654_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = RESTYPES.get(name, C.c_int)
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().evo_last_error().decode("utf-8", "replace")
    if rc == EVO_EINVAL:
        raise ValueError(msg)
    raise EvoError(f"CUDA error {rc}: {msg}")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("arrays passed to the C ABI must be C-contiguous")
    return a.ctypes.data_as(C.c_void_p)
