"""Forced-rung timing sweep ("Vortex-Oracle" analogue, and the
empirical tier's raw data).  For each shape, time the selected decision and every
(rung, split) of the table; per-launch CUDA events after an L2 flush.

    python tools/sweep.py --shapes bert|llama|attn|all|M,N,K[;...] [--flush rw|write|read|none]
                          [--reps 5] [--out gpurun_out/sweep.json] [--selected-only]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2409_01075_b200 as vx
import synth


def shapes_of(spec):
    out = []
    for part in spec.split(";"):
        if part == "bert":
            out += [(1, M, N, synth.BERT_K) for N in synth.BERT_N for M in synth.BERT_M]
        elif part == "llama":
            out += [(1, M, N, synth.LLAMA_K) for N in synth.LLAMA_N for M in synth.LLAMA_M]
        elif part == "attn":
            out += [(synth.ATTN_BATCH, s, s, d) for d in synth.ATTN_D for s in synth.ATTN_S]
        elif part == "all":
            out += shapes_of("bert;llama")
        elif part:
            v = [int(x) for x in part.split(",")]
            out.append((v[3], v[0], v[1], v[2]) if len(v) == 4 else (1, v[0], v[1], v[2]))
    return out


class Flusher:
    def __init__(self, mode, dev):
        self.mode = mode
        if mode != "none":
            self.a = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
            self.b = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def __call__(self):
        if self.mode in ("write", "rw"):
            self.a.zero_()
        if self.mode in ("read", "rw"):
            self.b.view(torch.int32).sum()


def time_launch(fn, flush, reps, stream):
    ts = []
    for _ in range(reps):
        flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def graph_buffers(batch, M, N, K, dev, l2_bytes):
    """Rotating operand sets for time_graph: R sets whose total exceeds 3x L2."""
    set_bytes = 2 * batch * (M * K + N * K + M * N)
    R = int(min(512, max(4, -(-3 * l2_bytes // set_bytes))))
    A = synth.matrix((R, batch * M * K), "bf16", seed=M, device=dev)
    B = synth.matrix((R, batch * N * K), "bf16", seed=N, scale=K ** -0.5, device=dev)
    C = torch.empty((R, batch * M * N), dtype=torch.bfloat16, device=dev)
    return A, B, C


def time_graph(p, batch, M, N, K, r, s, dev, stream, l2_bytes, reps, layout, bufs=None):
    """Per-launch time of back-to-back launches over rotating buffer sets whose total
    exceeds 3x L2 (cold operands every launch), captured once in a CUDA graph.  bufs: the
    (A, B, C) of graph_buffers, reused across calls for the same shape."""
    A, B, C = bufs if bufs is not None else graph_buffers(batch, M, N, K, dev, l2_bytes)
    R = A.shape[0]
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        sp = ctypes.c_void_p(side.cuda_stream)
        for i in range(R):   # warm (attributes, maps) outside capture
            vx.lib.vx_gemm_ex(p.handle, batch, M, N, K, A[i].data_ptr(), M * K, B[i].data_ptr(),
                              N * K, C[i].data_ptr(), M * N, r, s, sp, None)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            for i in range(R):
                st = vx.lib.vx_gemm_ex(p.handle, batch, M, N, K, A[i].data_ptr(), M * K,
                                       B[i].data_ptr(), N * K, C[i].data_ptr(), M * N, r, s, sp,
                                       None)
                assert st == 0, vx.lib.vx_last_error()
    stream.wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    del g
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--method", default="event", choices=["event", "graph"])
    ap.add_argument("--shapes", default="bert")
    ap.add_argument("--flush", default="rw")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--selected-only", action="store_true")
    ap.add_argument("--layout", default="nk")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    flush = Flusher(args.flush, dev)
    plans = {}
    res = []
    for (batch, M, N, K) in shapes_of(args.shapes):
        key = (N if batch == 1 else 0, K)
        if key not in plans:
            plans[key] = vx.Plan(key[0], K, "bf16", "bf16", args.layout)
        p = plans[key]
        A = synth.matrix((batch, M, K), "bf16", seed=M, device=dev)
        bshape = (batch, N, K) if args.layout == "nk" else (batch, K, N)
        B = synth.matrix(bshape, "bf16", seed=N, scale=K ** -0.5, device=dev)
        C = torch.empty((batch, M, N), dtype=torch.bfloat16, device=dev)
        sel = p.select(M, N=N, batch=batch)

        def run(r, s):
            st = vx.lib.vx_gemm_ex(p.handle, batch, M, N, K, A.data_ptr(), M * K, B.data_ptr(),
                                   N * K, C.data_ptr(), M * N, r, s, sp, None)
            if st:
                raise RuntimeError(vx.lib.vx_last_error().decode())

        run(-1, 0)
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size

        bufs = graph_buffers(batch, M, N, K, dev, l2) if args.method == "graph" else None

        def timed(r, s):
            if args.method == "graph":
                return time_graph(p, batch, M, N, K, r, s, dev, stream, l2, args.reps, args.layout,
                                  bufs)
            return time_launch(lambda: run(r, s), flush, args.reps, stream)

        t_sel = timed(-1, 0)
        entry = {"batch": batch, "M": M, "N": N, "K": K, "sel": sel, "t_sel_us": t_sel,
                 "forced": []}
        if not args.selected_only:
            for r in p.dump()["rungs"]:
                if r["family"] == 3 and M > r["bm"]:   # GEMV rungs hold M <= MT (R20)
                    continue
                for s in r["splits"]:
                    run(r["rung_id"], s)
                    t = timed(r["rung_id"], s)
                    c = p.cost(r["rung_id"], s, M, N=N, batch=batch)
                    entry["forced"].append({"rung": r["rung_id"], "family": r["family"], "split": s, "us": t,
                                            "cost": c["cost"]})
            best = min(entry["forced"], key=lambda e: e["us"])
            entry["best"] = best
            entry["regret"] = best["us"] / t_sel
        fl = 2.0 * batch * M * N * K
        print("b=%d M=%d N=%d K=%d sel=(%d,%d) %.2fus %.1fTF%s" % (
            batch, M, N, K, sel["rung_id"], sel["split"], t_sel, fl / t_sel / 1e6,
            "" if args.selected_only else "  best=(%d,%d) %.2fus regret=%.3f" % (
                entry["best"]["rung"], entry["best"]["split"], entry["best"]["us"],
                entry["regret"])), flush=True)
        res.append(entry)
        del A, B, C, bufs
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)
    if not args.selected_only:
        import math
        g = math.exp(sum(math.log(e["regret"]) for e in res) / len(res))
        print("geomean regret (best/selected) = %.4f  worst = %.4f" % (
            g, min(e["regret"] for e in res)))


if __name__ == "__main__":
    main()
