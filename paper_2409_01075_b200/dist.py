"""Multi-GPU M-row sharding of the dynamic-M GEMM.

Rows of C depend only on the same rows of A (C = A x B), so the problem
partitions by M rows with B replicated: every rank runs its own vx_gemm on its row block
and no reduction is needed.  A gathered C is produced only when asked for, with ONE
collective: all_gather_into_tensor over NCCL (NVLink 5 / NVSwitch on B200).  Uneven M is
handled by padding every shard to the largest shard in the gather buffer and trimming.

Fused variant: instead of GEMM then all_gather, every rank's GEMM
epilogue writes its finished C tiles straight into the gathered C of EVERY rank
(vx_gemm_gather), over NVLink through symmetric-memory peer pointers
(torch.distributed._symmetric_memory), so the transfer overlaps the mainloop of later
tiles; one barrier then orders the readers.  gather_plan() computes the pure host-side part
(row offsets and the destination order), which the gloo tests check on CPU.

Everything here is host-side plumbing; the GEMM itself is the library call.  The
collective goes through a torch.distributed process group, so the same code runs on the
"gloo" backend with CPU tensors (tests/test_dist.py) and on "nccl" with CUDA tensors.
"""
from __future__ import annotations

from typing import Callable

import torch


def row_shard(M: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) rows of rank `rank`: contiguous, disjoint, covering [0, M), sizes differ by
    at most one (the first M % world ranks get one extra row)."""
    if world < 1 or not 0 <= rank < world or M < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(M, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_sizes(M: int, world: int) -> list[int]:
    return [row_shard(M, world, r)[1] - row_shard(M, world, r)[0] for r in range(world)]


def gather_rows(c_local: torch.Tensor, M: int, group=None) -> torch.Tensor:
    """All-gather row shards (each rank's [m_r, N] block, m_r from row_shard) into the full
    [M, N] C on every rank.  One all_gather_into_tensor of max-size padded shards."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = shard_sizes(M, world)
    if c_local.shape[0] != sizes[rank]:
        raise ValueError("local shard has %d rows, expected %d" % (c_local.shape[0], sizes[rank]))
    mmax = max(sizes) if sizes else 0
    N = c_local.shape[1]
    send = c_local
    if c_local.shape[0] != mmax:
        send = torch.zeros((mmax, N), dtype=c_local.dtype, device=c_local.device)
        send[: c_local.shape[0]] = c_local
    recv = torch.empty((world * mmax, N), dtype=c_local.dtype, device=c_local.device)
    dist.all_gather_into_tensor(recv, send.contiguous(), group=group)
    if all(s == mmax for s in sizes):
        return recv
    parts = [recv[r * mmax: r * mmax + sizes[r]] for r in range(world)]
    return torch.cat(parts, 0)


def gather_plan(M: int, world: int, rank: int) -> dict:
    """Host-side plan of the fused GEMM + all-gather for one rank: the rows it computes, the
    row offset its epilogue writes at in every destination, and the destination order
    (its own buffer first, then the peers in rank order)."""
    lo, hi = row_shard(M, world, rank)
    return {"rows": (lo, hi), "row_offset": lo,
            "dst_ranks": [rank] + [r for r in range(world) if r != rank]}


def push_rows(c_local: torch.Tensor, M: int, group=None) -> torch.Tensor:
    """The fused gather's data movement with point-to-point sends instead of peer stores
    (any backend, e.g. gloo on CPU): every rank pushes its C rows to every destination in
    gather_plan order, and each destination places the rows of rank r at row_offset(r) --
    the placement rule the vx_gemm_gather epilogue applies on NVLink."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    gp = gather_plan(M, world, rank)
    lo, hi = gp["rows"]
    if c_local.shape[0] != hi - lo:
        raise ValueError("local shard has %d rows, expected %d" % (c_local.shape[0], hi - lo))
    out = torch.empty((M, c_local.shape[1]), dtype=c_local.dtype, device=c_local.device)
    out[lo:hi] = c_local
    reqs = []
    for dst in gp["dst_ranks"][1:]:
        reqs.append(dist.isend(c_local.contiguous(), dst, group=group))
    for src in range(world):
        if src == rank:
            continue
        slo, shi = gather_plan(M, world, src)["rows"]
        if shi > slo:
            buf = torch.empty((shi - slo, c_local.shape[1]), dtype=c_local.dtype,
                              device=c_local.device)
            dist.recv(buf, src, group=group)
            out[slo:shi] = buf
        else:
            dist.recv(torch.empty((0, c_local.shape[1]), dtype=c_local.dtype), src, group=group)
    for r in reqs:
        r.wait()
    return out


def symmetric_gather_buffer(M: int, N: int, dtype, device, group=None):
    """Gathered C [M, N] in symmetric memory on every rank of `group`: returns (this rank's
    tensor, handle, device pointers of every rank's buffer valid in this process)."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    buf = symm_mem.empty((M, N), dtype=dtype, device=device)
    hdl = symm_mem.rendezvous(buf, group if group is not None else dist.group.WORLD)
    return buf, hdl, list(hdl.buffer_ptrs)


def fused_gather_gemm(plan, A_shard: torch.Tensor, B: torch.Tensor, M: int, group=None,
                      buf=None, stream=None):
    """C = A x B row-sharded, gathered on every rank by the GEMM epilogue itself (no
    separate collective).  A_shard: this rank's rows (row_shard).  Returns the gathered
    [M, N] C (a symmetric-memory tensor).  `buf` = a (tensor, handle, ptrs) triple from
    symmetric_gather_buffer to reuse."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    gp = gather_plan(M, world, rank)
    lo, hi = gp["rows"]
    if A_shard.shape[0] != hi - lo:
        raise ValueError("A shard has %d rows, expected %d" % (A_shard.shape[0], hi - lo))
    odt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[plan.out_dtype]
    if buf is None:
        buf = symmetric_gather_buffer(M, plan.N, odt, A_shard.device, group)
    out, hdl, ptrs = buf
    hdl.barrier()               # every destination is allocated and free to be written
    plan.gemm_gather(A_shard, B, [ptrs[r] for r in gp["dst_ranks"]], gp["row_offset"],
                     stream=stream)
    hdl.barrier()               # every rank's epilogue has written its rows everywhere
    return out


class ShardedGemm:
    """C = A x B with A row-sharded over the ranks of `group` and B replicated.

    local_gemm(A_rows, B) -> C_rows runs on this rank's device; by default it is the
    library's Plan.gemm.  forward() takes either the full A (each rank slices its rows) or
    this rank's shard, and returns this rank's C rows, or the gathered C if gather=True.
    """

    def __init__(self, N: int, K: int, group=None, local_gemm: Callable | None = None,
                 in_dtype: str = "bf16", out_dtype: str = "bf16", b_layout: str = "nk",
                 device: int | None = None):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.N, self.K = N, K
        if local_gemm is None:
            from . import Plan
            plan = Plan(N, K, in_dtype, out_dtype, b_layout,
                        device=device if device is not None else torch.cuda.current_device())
            local_gemm = lambda a, b: plan.gemm(a, b)  # noqa: E731
        self.local_gemm = local_gemm

    def forward(self, A: torch.Tensor, B: torch.Tensor, M: int | None = None,
                gather: bool = False) -> torch.Tensor:
        if M is None:            # full A given: take this rank's rows
            M = A.shape[0]
            lo, hi = row_shard(M, self.world, self.rank)
            A = A[lo:hi].contiguous()
        else:
            lo, hi = row_shard(M, self.world, self.rank)
            if A.shape[0] != hi - lo:
                raise ValueError("A shard has %d rows, expected %d" % (A.shape[0], hi - lo))
        c = self.local_gemm(A, B)
        return gather_rows(c, M, self.group) if gather else c


class ShardedBatchedGemm:
    """Batched attention scores S_b = Q_b x K_b^T (BASELINE configs[3]) sharded over the
    BATCH: rank r computes batches row_shard(batch, world, r) with its own vx_gemm_batched
    ("batched attention shards over batch (32/P) the same way").  Batches are
    independent -- no reduction; a gathered S (all batches on every rank) is one
    all_gather_into_tensor of the per-rank [b_r, s, s] blocks, padded to the largest.

    local_bgemm(Q [b, s, d], Kt [b, s, d]) -> S [b, s, s] runs on this rank's device; by
    default the library's batched Plan.gemm (Plan(s, d, ..., "nk"): K stored N x K)."""

    def __init__(self, s: int, d: int, group=None, local_bgemm: Callable | None = None,
                 in_dtype: str = "bf16", out_dtype: str = "bf16", device: int | None = None):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if local_bgemm is None:
            from . import Plan
            plan = Plan(s, d, in_dtype, out_dtype, "nk",
                        device=device if device is not None else torch.cuda.current_device())
            local_bgemm = lambda q, k: plan.gemm(q, k)  # noqa: E731
        self.local_bgemm = local_bgemm

    def forward(self, Q: torch.Tensor, Kt: torch.Tensor, gather: bool = False) -> torch.Tensor:
        """Q, Kt: the FULL [batch, s, d] inputs (each rank slices its batches).  Returns this
        rank's [b_r, s, s] scores, or all [batch, s, s] if gather=True."""
        batch = Q.shape[0]
        lo, hi = row_shard(batch, self.world, self.rank)
        S = self.local_bgemm(Q[lo:hi].contiguous(), Kt[lo:hi].contiguous())
        if not gather:
            return S
        b_r, s1, s2 = S.shape
        full = gather_rows(S.reshape(b_r, s1 * s2), batch, self.group)
        return full.reshape(batch, s1, s2)
