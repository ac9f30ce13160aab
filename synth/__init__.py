"""synth -- seeded synthetic input generators, shared by tests, bench.py and smoke().

Holds none of the method's arithmetic: it only draws inputs.  Both the CUDA path and the
oracle consume what it returns; neither side's computation lives here.

Recipe:
  * "normal": A ~ N(0,1), B ~ N(0, 1/K) (weight-like, so C ~ N(0,1)), cast to the storage
    dtype -- dense, unstructured, like the paper's plain linear layers
    (tbl:benchmark_gemm).
  * "int": entries uniform on {-2,-1,0,1,2}: exact in bf16/fp16/fp32, and every partial sum
    of K <= 4096 products stays an integer below 2^24, so fp32 accumulation is exact in any
    order -> GPU output must equal the fp64 oracle bit-for-bit.
  * "int1": uniform on {-1,0,1}, same property with a larger K range.
"""
from __future__ import annotations

import torch

_DT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32,
       "fp64": torch.float64}


def torch_dtype(name: str) -> torch.dtype:
    return _DT[name]


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def matrix(shape, dtype: str, kind: str = "normal", seed: int = 0, scale: float = 1.0,
           device="cpu") -> torch.Tensor:
    """One seeded tensor of the given shape/dtype/distribution."""
    g = _gen(seed, device)
    if kind == "normal":
        t = torch.randn(shape, generator=g, device=device, dtype=torch.float32) * scale
    elif kind == "int":
        t = torch.randint(-2, 3, shape, generator=g, device=device).to(torch.float32)
    elif kind == "int1":
        t = torch.randint(-1, 2, shape, generator=g, device=device).to(torch.float32)
    elif kind == "uniform":
        t = (torch.rand(shape, generator=g, device=device, dtype=torch.float32) * 2 - 1) * scale
    else:
        raise ValueError(kind)
    return t.to(_DT[dtype])


def gemm_inputs(M: int, N: int, K: int, dtype: str = "bf16", b_layout: str = "nk",
                kind: str = "normal", seed: int = 1234, batch: int | None = None,
                device="cpu"):
    """(A, B) for C = A x B.  A: [M,K] (or [batch,M,K]); B: [N,K] ("nk") or [K,N] ("kn")."""
    lead = () if batch is None else (batch,)
    a = matrix(lead + (M, K), dtype, kind, seed, 1.0, device)
    bshape = lead + ((N, K) if b_layout == "nk" else (K, N))
    bscale = 1.0 / (K ** 0.5) if kind in ("normal", "uniform") else 1.0
    b = matrix(bshape, dtype, kind, seed + 1, bscale, device)
    return a, b


# dynamic-M sweeps
BERT_N = (768, 2304, 3072)
BERT_K = 768
BERT_M = (1, 2, 3, 4, 8, 16, 17, 31, 32, 37, 48, 64, 80, 100, 127, 128, 129, 200, 255, 256,
          257, 384, 476, 511, 512, 513, 688, 768, 992, 1000, 1024, 1296, 1600, 1904, 2048,
          3000, 4096)
LLAMA_N = (4096, 11008, 12288)
LLAMA_K = 4096
LLAMA_M = (1, 2, 4, 8, 13, 16, 32, 37, 64, 100, 128, 129, 256, 384, 511, 512, 513, 1000,
           1024, 2048, 3000, 4096, 5000, 8192, 10000, 16383, 16384)
ATTN_BATCH = 32
ATTN_D = (64, 128)
ATTN_S = (1, 7, 16, 64, 100, 128, 257, 512, 1000, 1024, 1500, 2048)
