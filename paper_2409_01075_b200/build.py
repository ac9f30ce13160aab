"""Build libvx.so in-tree: nvcc for sm_100a only (tcgen05/TMA need the 'a' target).

    python paper_2409_01075_b200/build.py [--force] [--verbose]

The shared object lands next to this file so it travels with the repo snapshot to the
GPU box.  cudart is linked statically; the CUDA driver is reached through
cudaGetDriverEntryPoint, so loading the library needs no GPU (selector tests run on CPU).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvx.so")
SOURCES = ["vx_plan.cpp", "vx_calib.cpp", "vx_dispatch.cu", "vx_live.cu"]
HEADERS = ["vx_internal.h", "vx_ptx.cuh", "vx_umma.cuh", "vx_simt.cuh", "vx_gemv.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "vx.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + ".tmp.%d" % os.getpid()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
           "-shared", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
           "-I", CSRC, "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd += ["-Xptxas", "-v"]
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
