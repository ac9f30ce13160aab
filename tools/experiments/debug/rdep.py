"""Per-launch time vs launches-per-point R in the bench's graph structure (one event node
between points), ours vs cuBLAS, on a few BERT/LLaMA points: is there a per-point cost?
    python tools/rdep.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2409_01075_b200 as vx


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)
    pts = [("bert", M, N, 768) for N in (768, 3072) for M in (1, 64, 512, 2048)]
    pts += [("llama", M, 4096, 4096) for M in (8, 512)]
    plans = {}
    for _, M, N, K in pts:
        if (N, K) not in plans:
            plans[(N, K)] = vx.Plan(N, K, "bf16", "bf16", "nk")
    arenas = bench.make_arenas(pts, dev, 0)
    for R in (1, 2, 8, 32):
        items = [(plans[(N, K)], M, N, K) for _, M, N, K in pts]
        g = bench.SweepGraph(items, R, arenas, stream, side)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            g.replay()
            torch.cuda.synchronize()
            ts.append(g.per_launch_ms())
        med = [sorted(t[j] for t in ts)[2] * 1e3 for j in range(len(pts))]
        cb = bench.run_cublas_ref(pts, stream, side, 0, R, 5)
        print("R=%3d " % R + "  ".join("%s:%d/%d %.2f|%.2f" % (tg[0], M, N, m, c * 1e3)
                                        for (tg, M, N, K), m, c in zip(pts, med, cb)), flush=True)
        del g


if __name__ == "__main__":
    main()
