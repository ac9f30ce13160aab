"""Multi-process host logic of the M-row-sharded GEMM on CPU (gloo, world size 2 and 3).

The local GEMM is injected (the fp64 oracle -- test infrastructure), so these tests cover
exactly the sharding / gather plumbing of paper_2409_01075_b200/dist.py that the NCCL run
uses on B200s.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_01075_b200.dist import (ShardedBatchedGemm, ShardedGemm, gather_plan,
                                        gather_rows, push_rows, row_shard, shard_sizes)


def test_row_shard_partition_properties():
    for M in (0, 1, 7, 128, 1000, 65536, 65537):
        for world in (1, 2, 3, 4, 8):
            spans = [row_shard(M, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == M
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = shard_sizes(M, world)
            assert sum(sizes) == M and max(sizes) - min(sizes) <= 1
    assert row_shard(65536, 8, 3) == (3 * 8192, 4 * 8192)
    with pytest.raises(ValueError):
        row_shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, N, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        A, B = synth.gemm_inputs(M, N, K, "fp32", "nk", kind="int", seed=42)   # same on all ranks

        def local(a, b):
            return torch.from_numpy(oracle.gemm(a, b, "nk")).float()

        sg = ShardedGemm(N, K, local_gemm=local)
        c_rows = sg.forward(A, B)                        # this rank's rows only
        lo, hi = row_shard(M, world, rank)
        ok_rows = c_rows.shape == (hi - lo, N)
        C = sg.forward(A, B, gather=True)                # gathered on every rank
        lo_ = torch.tensor([lo], dtype=torch.int64)
        C2 = gather_rows(c_rows, M)                      # the gather alone
        C3 = push_rows(c_rows, M)                        # the fused gather's push placement
        q.put((rank, ok_rows, C.numpy(), C2.numpy(), int(lo_), C3.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,M", [(2, 37), (2, 64), (3, 100), (2, 1)])
def test_sharded_gather_equals_full_gemm(world, M):
    import oracle
    import synth
    N, K = 24, 40
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, B = synth.gemm_inputs(M, N, K, "fp32", "nk", kind="int", seed=42)
    want = oracle.gemm(A, B, "nk")
    for rank, ok_rows, C, C2, lo, C3 in res:
        assert ok_rows
        assert np.array_equal(C, want) and np.array_equal(C2, want)
        assert np.array_equal(C3, want)


def test_gather_plan_covers_every_destination_once():
    """Fused GEMM + all-gather: each rank's epilogue writes its rows at its
    row_shard offset into every rank's buffer, its own first; over all ranks every
    (destination, row) is written exactly once."""
    for M in (1, 37, 1000, 65536):
        for world in (1, 2, 3, 8):
            hits = np.zeros((world, M), dtype=np.int64)
            for r in range(world):
                gp = gather_plan(M, world, r)
                lo, hi = gp["rows"]
                assert gp["row_offset"] == lo and gp["dst_ranks"][0] == r
                assert sorted(gp["dst_ranks"]) == list(range(world))
                for d in gp["dst_ranks"]:
                    hits[d, lo:hi] += 1
            assert (hits == 1).all()


def _batched_worker(rank, world, port, batch, s, d, q):
    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Q = synth.matrix((batch, s, d), "fp32", "int", seed=11)
        Kt = synth.matrix((batch, s, d), "fp32", "int", seed=12)

        def bgemm(q_, k_):        # injected local batched GEMM: the fp64 oracle per batch
            return torch.stack([torch.from_numpy(oracle.gemm(q_[b], k_[b], "nk")).float()
                                for b in range(q_.shape[0])]) if q_.shape[0] else \
                torch.zeros((0, s, s))
        sh = ShardedBatchedGemm(s, d, local_bgemm=bgemm)
        lo, hi = row_shard(batch, world, rank)
        mine = sh.forward(Q, Kt)
        full = sh.forward(Q, Kt, gather=True)
        q.put((rank, lo, hi, mine.numpy(), full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,batch", [(2, 32), (3, 32), (2, 3)])
def test_batch_sharded_attention_equals_full(world, batch):
    """batched attention scores shard over the batch; every rank's block and the
    gathered S equal the unsharded per-batch products (integer inputs: exact)."""
    import oracle
    import synth
    s, d = 9, 16
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batched_worker, args=(r, world, port, batch, s, d, qu))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [qu.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Q = synth.matrix((batch, s, d), "fp32", "int", seed=11)
    Kt = synth.matrix((batch, s, d), "fp32", "int", seed=12)
    want = np.stack([oracle.gemm(Q[b], Kt[b], "nk") for b in range(batch)])
    covered = np.zeros(batch, dtype=int)
    for rank, lo, hi, mine, full in res:
        assert np.array_equal(mine, want[lo:hi])
        assert np.array_equal(full, want)
        covered[lo:hi] += 1
    assert (covered == 1).all()
