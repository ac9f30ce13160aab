"""Per-launch floor probe (measurement tool): back-to-back launches of one shape in a CUDA
graph on fresh slices of 1 GiB arenas (as bench.py), for the library's selected rung and for
torch.mm (cuBLAS), from a one-tile / one-k-block GEMM up to BERT and decode sizes -- how much
of a launch is fixed cost and how much is work.

    python tools/floor_probe.py [--R 48] [--hot]
"""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2409_01075_b200 as vx

SHAPES = [(16, 128, 64), (128, 128, 64), (128, 128, 768), (128, 768, 768), (16, 3072, 768),
          (128, 3072, 768), (512, 768, 768), (1024, 3072, 768), (16, 11008, 4096),
          (128, 11008, 4096)]


def graph_us(fn_list, stream, reps=5):
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        for f in fn_list[:2]:
            f()
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for f in fn_list:
                f()
    stream.wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / len(fn_list))
    return statistics.median(ts)


def main():
    R = int(sys.argv[sys.argv.index("--R") + 1]) if "--R" in sys.argv else 48
    hot = "--hot" in sys.argv
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    GiB = 1 << 30
    aA = torch.randn(GiB // 2, dtype=torch.bfloat16, device=dev)
    aB = torch.randn(GiB // 2, dtype=torch.bfloat16, device=dev) * 0.02
    aC = torch.empty(GiB // 2, dtype=torch.bfloat16, device=dev)
    for M, N, K in SHAPES:
        p = vx.Plan(N, K, "bf16", "bf16", "nk")
        ch = p.select(M)
        ours, cub = [], []
        for i in range(R):
            j = 0 if hot else i
            oa, ob, oc = (j * M * K) % (aA.numel() - M * K), (j * N * K) % (aB.numel() - N * K), \
                (j * M * N) % (aC.numel() - M * N)
            oa, ob, oc = oa // 64 * 64, ob // 64 * 64, oc // 64 * 64
            A = aA[oa:oa + M * K].view(M, K)
            B = aB[ob:ob + N * K].view(N, K)
            C = aC[oc:oc + M * N].view(M, N)
            ours.append(lambda A=A, B=B, C=C: p.gemm(A, B, out=C))
            cub.append(lambda A=A, B=B, C=C: torch.mm(A, B.t(), out=C))
        t_o = graph_us(ours, stream)
        t_c = graph_us(cub, stream)
        print("M=%5d N=%5d K=%5d  ours %6.2f us (rung %d %s%dx%d s%d grid %d)  cuBLAS %6.2f us  ratio %.2f" % (
            M, N, K, t_o, ch["rung_id"], "swap " if ch["swap"] else "", ch["bm"], ch["bn"], ch["split"],
            ch["grid"], t_c, t_c / t_o), flush=True)


if __name__ == "__main__":
    main()
