"""oracle -- TEST INFRASTRUCTURE ONLY.

The parity oracle for the dynamic-M GEMM hot path of Vortex (arXiv 2409.01075).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here.  The product path
(``paper_2409_01075_b200``) never imports, links or executes it, and the two share no
code, header, table or constant generator.

Contents
  * ``gemm_ref.c`` / :func:`gemm` -- plain fp64 GEMM, the definition C = A x B
    (Sec. 4.1; shapes PAPER.md:866-867, Sec. 2.2).
  * ``selector_ref.py`` -- step-by-step re-implementation of the sample-free strategy
    table (Alg. 2) and the runtime cost-model argmin
    (Eqs. 1-4; Sec. 6.2), in pure Python ints.

Pins (what each function is checked against, never itself): see tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gemm_ref.c")
_LIB = os.path.join(_HERE, "libgemm_ref.so")
_lock = threading.Lock()
_lib = None

DTYPE_CODES = {"bf16": 0, "fp16": 1, "fp32": 2, "fp64": 3}
B_LAYOUTS = {"kn": 0, "nk": 1}


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc; -ffp-contract=off keeps products unfused)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared",
                               "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.oracle_gemm.restype = ctypes.c_int
            lib.oracle_gemm.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_int]
            lib.oracle_threads.restype = ctypes.c_int
            lib.oracle_threads.argtypes = [ctypes.c_int]
            _lib = lib
    return _lib


def _as_numpy_bits(t):
    """Return (numpy array holding the stored element bits, dtype name)."""
    import torch  # plumbing only: reading CPU tensors' storage
    if isinstance(t, np.ndarray):
        name = {np.dtype(np.float32): "fp32", np.dtype(np.float64): "fp64",
                np.dtype(np.float16): "fp16"}[t.dtype]
        return np.ascontiguousarray(t), name
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16), "bf16"
    if t.dtype == torch.float16:
        return t.view(torch.int16).numpy().view(np.uint16), "fp16"
    if t.dtype == torch.float32:
        return t.numpy(), "fp32"
    if t.dtype == torch.float64:
        return t.numpy(), "fp64"
    raise TypeError("oracle: unsupported dtype %s" % t.dtype)


def gemm(A, B, b_layout: str = "kn", rows=None, threads: int = 0) -> np.ndarray:
    """fp64 C = A x B from the stored values of A and B.

    A: [M,K] or [batch,M,K];  B: [K,N] ("kn") or [N,K] ("nk"), optionally batched.
    rows: optional sequence of row indices of A/C to compute (row-subset mode).
    Returns float64 ndarray [nrows,N] (or [batch,nrows,N] when A is 3-D).
    """
    a, da = _as_numpy_bits(A)
    b, db = _as_numpy_bits(B)
    if da != db:
        raise TypeError("oracle: A and B must share an element type")
    batched = a.ndim == 3
    if not batched:
        a = a.reshape((1,) + a.shape)
        b = b.reshape((1,) + b.shape)
    batch, M, K = a.shape
    if b_layout == "kn":
        if b.shape[1] != K:
            raise ValueError("oracle: B must be [K,N]")
        N = b.shape[2]
    elif b_layout == "nk":
        if b.shape[2] != K:
            raise ValueError("oracle: B must be [N,K]")
        N = b.shape[1]
    else:
        raise ValueError(b_layout)
    if b.shape[0] != batch:
        raise ValueError("oracle: batch mismatch")
    if rows is None:
        r = None
        nrows = M
    else:
        r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        nrows = r.shape[0]
    c = np.zeros((batch, nrows, N), dtype=np.float64)
    rc = _load().oracle_gemm(batch, M, N, K, DTYPE_CODES[da], B_LAYOUTS[b_layout],
                             a.ctypes.data, M * K, b.ctypes.data, K * N,
                             c.ctypes.data, None if r is None else r.ctypes.data, nrows,
                             int(threads))
    if rc != 0:
        raise ValueError("oracle_gemm rejected its arguments")
    return c if batched else c[0]


def threads(n: int = 0) -> int:
    """OpenMP thread count the oracle will use when called with ``threads=n``."""
    return _load().oracle_threads(int(n))
