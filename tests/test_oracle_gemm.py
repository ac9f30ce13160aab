"""Pins for the fp64 GEMM oracle (oracle/gemm_ref.c) -- CPU only.

Each test checks the oracle against something other than itself: printed values, closed
forms, invariants of the definition C = A x B, element-format definitions
and a library routine (numpy fp64 matmul).  A plausible bug (dropped k term, transposed
operand, wrong batch/row index, wrong bf16/fp16 decode) fails at least one of them.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _t(x, dt=torch.float32):
    return torch.tensor(x, dtype=dt)


def test_textbook_products():
    cases = json.load(open(os.path.join(GOLD, "gemm_textbook.json")))["cases"]
    for c in cases:
        for dt in (torch.float32, torch.bfloat16, torch.float16, torch.float64):
            A, B = _t(c["A"], dt), _t(c["B"], dt)
            got = oracle.gemm(A, B, "kn")
            assert got.tolist() == c["C"]
            got_nk = oracle.gemm(A, B.t().contiguous(), "nk")
            assert got_nk.tolist() == c["C"]


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (5, 3, 7), (37, 64, 64), (129, 17, 40)])
def test_closed_forms(M, N, K):
    # all-ones: every C element is K (a dropped or repeated k term changes it)
    A = torch.ones(M, K)
    B = torch.ones(K, N)
    assert np.all(oracle.gemm(A, B, "kn") == K)
    # A[i,k] = k, B[k,j] = 1  ->  C[i,j] = K(K-1)/2   (index of k, not i or j)
    A = torch.arange(K, dtype=torch.float64).repeat(M, 1)
    B = torch.ones(K, N, dtype=torch.float64)
    assert np.all(oracle.gemm(A, B, "kn") == K * (K - 1) / 2)
    # A[i,k] = i, B[k,j] = j  ->  C[i,j] = i*j*K
    A = torch.arange(M, dtype=torch.float64)[:, None].repeat(1, K)
    B = torch.arange(N, dtype=torch.float64)[None, :].repeat(K, 1)
    want = np.outer(np.arange(M), np.arange(N)) * K
    assert np.array_equal(oracle.gemm(A, B, "kn"), want)
    assert np.array_equal(oracle.gemm(A, B.t().contiguous(), "nk"), want)
    # A[i,k] = k+1, B[k,j] = k+1 -> sum of squares K(K+1)(2K+1)/6
    A = (torch.arange(K, dtype=torch.float64) + 1).repeat(M, 1)
    B = (torch.arange(K, dtype=torch.float64) + 1)[:, None].repeat(1, N)
    assert np.all(oracle.gemm(A, B, "kn") == K * (K + 1) * (2 * K + 1) / 6)


def test_identity_and_permutation():
    A, B = synth.gemm_inputs(23, 19, 31, "fp32", "kn", kind="normal", seed=7)
    I_K = torch.eye(31)
    # A x I = A exactly
    assert np.array_equal(oracle.gemm(A, I_K, "kn"), A.double().numpy())
    # P x B permutes the rows of B exactly
    perm = torch.randperm(31, generator=torch.Generator().manual_seed(3))
    P = torch.zeros(31, 31)
    P[torch.arange(31), perm] = 1
    assert np.array_equal(oracle.gemm(P, B, "kn"), B[perm].double().numpy())


@pytest.mark.parametrize("dtype", ["bf16", "fp16", "fp32"])
def test_transpose_identity(dtype):
    # (AB)^T = B^T A^T : same k order on both sides -> bit-exact in fp64
    A, B = synth.gemm_inputs(17, 29, 40, dtype, "kn", kind="normal", seed=11)
    C = oracle.gemm(A, B, "kn")
    Ct = oracle.gemm(B.t().contiguous(), A.t().contiguous(), "kn")
    assert np.array_equal(C.T, Ct)
    # the NK storage of B is the same operand
    assert np.array_equal(oracle.gemm(A, B.t().contiguous(), "nk"), C)


def test_linearity_in_A_exact():
    A1, B = synth.gemm_inputs(33, 21, 64, "fp32", "kn", kind="int", seed=5)
    A2, _ = synth.gemm_inputs(33, 21, 64, "fp32", "kn", kind="int", seed=9)
    C = oracle.gemm(A1 + 3 * A2, B, "kn")
    assert np.array_equal(C, oracle.gemm(A1, B, "kn") + 3 * oracle.gemm(A2, B, "kn"))


def test_associativity_exact_integers():
    g = torch.Generator().manual_seed(1)
    A = torch.randint(-3, 4, (9, 11), generator=g).double()
    B = torch.randint(-3, 4, (11, 7), generator=g).double()
    D = torch.randint(-3, 4, (7, 5), generator=g).double()
    AB = torch.tensor(oracle.gemm(A, B, "kn"))
    BD = torch.tensor(oracle.gemm(B, D, "kn"))
    assert np.array_equal(oracle.gemm(AB, D, "kn"), oracle.gemm(A, BD, "kn"))


@pytest.mark.parametrize("dtype", ["bf16", "fp16", "fp32"])
def test_numpy_matmul_crosscheck(dtype):
    # library routine on the same stored values, fp64 (rounding order may differ)
    A, B = synth.gemm_inputs(70, 45, 300, dtype, "kn", kind="normal", seed=2)
    ref = A.double().numpy() @ B.double().numpy()
    got = oracle.gemm(A, B, "kn")
    assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_element_decoding_from_format_definitions():
    # bf16 / fp16 bit patterns with values fixed by the IEEE / bfloat16 definitions
    bf = {0x3F80: 1.0, 0xC000: -2.0, 0x0001: 2.0 ** -133, 0x7F7F: (2 - 2 ** -7) * 2.0 ** 127,
          0x3E80: 0.25}
    hf = {0x3C00: 1.0, 0xC000: -2.0, 0x0001: 2.0 ** -24, 0x7BFF: 65504.0, 0x0400: 2.0 ** -14,
          0x3555: 1365 * 2.0 ** -12}
    for dt, table in ((torch.bfloat16, bf), (torch.float16, hf)):
        bits = torch.tensor(list(table.keys()), dtype=torch.int32).to(torch.int16)
        A = bits.view(dt).reshape(-1, 1)
        B = torch.ones(1, 1, dtype=dt)
        got = oracle.gemm(A, B, "kn")[:, 0]
        assert list(got) == list(table.values())


def test_row_subset_batch_and_threads():
    A, B = synth.gemm_inputs(50, 24, 48, "bf16", "nk", kind="normal", seed=4, batch=3)
    full = oracle.gemm(A, B, "nk")
    rows = [0, 49, 17, 17, 3]
    sub = oracle.gemm(A, B, "nk", rows=rows)
    assert np.array_equal(sub, full[:, rows, :])
    for b in range(3):
        assert np.array_equal(full[b], oracle.gemm(A[b], B[b], "nk"))
    # thread count cannot change any element (fixed per-element k order)
    assert np.array_equal(oracle.gemm(A, B, "nk", threads=1), full)


def test_empty_and_invalid():
    A = torch.zeros(0, 8)
    B = torch.zeros(8, 4)
    assert oracle.gemm(A, B, "kn").shape == (0, 4)
    A = torch.ones(3, 0)
    B = torch.ones(0, 2)
    assert np.all(oracle.gemm(A, B, "kn") == 0)
    with pytest.raises(ValueError):
        oracle.gemm(torch.ones(2, 3), torch.ones(2, 3), "kn")
    with pytest.raises(ValueError):
        oracle.gemm(torch.ones(2, 3), torch.ones(3, 2), "kn", rows=[5])
