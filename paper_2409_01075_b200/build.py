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
SOURCES = ["vx_plan.cpp", "vx_calib.cpp", "vx_dispatch.cu", "vx_live.cu", "vx_k_single.cu",
           "vx_k_swap.cu", "vx_k_pair.cu", "vx_k_mc.cu"]
HEADERS = ["vx_internal.h", "vx_ptx.cuh", "vx_umma.cuh", "vx_simt.cuh", "vx_gemv.cuh",
           "vx_kernels.h"]
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
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
             "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    if verbose:
        flags += ["-Xptxas", "-v"]
    # one object per translation unit, compiled in parallel (the kernel instantiations are
    # spread over vx_k_*.cu), then one shared-object link
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(CSRC, ".obj", src + ".%d.o" % os.getpid())
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        cmd = [NVCC, *flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    try:
        bad = [p.args for p in procs if p.wait() != 0]
        if bad:
            raise subprocess.CalledProcessError(1, bad[0])
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp] + objs)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
