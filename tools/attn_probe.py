"""Batched attention scores S_b = Q_b K_b^T (batch 32) at aligned / unaligned s: device time
per launch (graph of R launches, median of 5 replays) -- the unaligned-row epilogue A/B.

    python tools/attn_probe.py [--s 1500,1504,2048] [--d 64] [--R 8] [--once S]
    (--once S: a single launch at s = S, for ncu)
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2409_01075_b200 as vx

B = 32


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    d = int(arg("--d", "64"))
    R = int(arg("--R", "8"))
    p = vx.Plan(0, d, "bf16", "bf16", "nk")
    if "--once" in sys.argv:
        s = int(arg("--once", "1500"))
        Q = torch.randn(B, s, d, device="cuda").to(torch.bfloat16)
        K = (torch.randn(B, s, d, device="cuda") * d ** -0.5).to(torch.bfloat16)
        S = torch.empty(B, s, s, device="cuda", dtype=torch.bfloat16)
        p.gemm(Q, K, out=S)
        torch.cuda.synchronize()
        return
    for s in (int(x) for x in arg("--s", "1500,1504,2048").split(",")):
        slots = 4
        Q = [torch.randn(B, s, d, device="cuda").to(torch.bfloat16) for _ in range(slots)]
        K = [(torch.randn(B, s, d, device="cuda") * d ** -0.5).to(torch.bfloat16) for _ in range(slots)]
        S = [torch.empty(B, s, s, device="cuda", dtype=torch.bfloat16) for _ in range(slots)]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            p.gemm(Q[0], K[0], out=S[0])
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for i in range(R):
                    p.gemm(Q[i % slots], K[i % slots], out=S[i % slots])
        ts = []
        for rep in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record(st)
                g.replay()
                e1.record(st)
            torch.cuda.synchronize()
            if rep >= 3:
                ts.append(e0.elapsed_time(e1) * 1000 / R)
        us = statistics.median(ts)
        out_b = 2 * B * s * s
        print("s=%d d=%d %s: %.1f us, S write %.1f MB -> %.0f GB/s" % (
            s, d, p.select(s, s, batch=B), us, out_b / 1e6, out_b / us / 1e3), flush=True)
        del g, Q, K, S


if __name__ == "__main__":
    main()
