"""Build the in-tree CUDA library ``libevoca_b200.so`` for sm_100a.

    python -m paper_2406_09654_b200.build [--verbose]

Plain nvcc, no torch extension machinery: the product is a C-ABI shared
library (include/evoca_b200.h) that ctypes (or any FFI) loads.  No
--use_fast_math: the physics relies on IEEE denormals and correctly
rounded division (SURVEY.md appendix A compile flags).
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libevoca_b200.so")
SOURCES = ["evoca_kernels.cu", "evoca_hidden_tc.cu", "evoca_cppn.cu", "evoca_radiation.cu", "evoca_metrics.cu",
           "evoca_shard.cu", "evoca_gather.cu", "evoca_resolve.cu", "evoca_abi.cu", "evoca_neat.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libevoca_b200.so")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in os.listdir(CSRC)] + [os.path.join(INCLUDE, "evoca_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    cmd = [
        nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
        "-Xcompiler", "-fvisibility=hidden", "-I", INCLUDE, "-I", CSRC,
        *[f"-D{d}" for d in defines],
        "-o", lib + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES],
    ]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stdout + res.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--phase-timing", action="store_true", help="diagnostics build -> libevoca_b200_timing.so")
    args = ap.parse_args()
    if args.phase_timing:
        print(build(force=True, verbose=args.verbose, out=os.path.join(PKG, "libevoca_b200_timing.so"),
                    defines=("EVO_PHASE_TIMING",)))
    else:
        print(build(force=args.force or args.verbose, verbose=args.verbose))
    sys.exit(0)
