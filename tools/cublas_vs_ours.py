"""Per-launch time of cuBLAS (torch.mm) vs the library's selected rung on the same shapes,
same method (CUDA graph of back-to-back launches over rotating cold buffers, > 3x L2).
Informational.

    python tools/cublas_vs_ours.py M,N,K [M,N,K ...]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch

import paper_2409_01075_b200 as vx
from sweep import time_graph


def time_cublas(M, N, K, dev, l2, reps=5):
    set_bytes = 2 * (M * K + N * K + M * N)
    R = int(min(512, max(4, -(-3 * l2 // set_bytes))))
    A = torch.randn(R, M, K, device=dev, dtype=torch.bfloat16)
    B = torch.randn(R, N, K, device=dev, dtype=torch.bfloat16)
    C = torch.empty(R, M, N, device=dev, dtype=torch.bfloat16)
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(R):
            torch.mm(A[i], B[i].t(), out=C[i])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(R):
                torch.mm(A[i], B[i].t(), out=C[i])
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / R)
    return statistics.median(ts)


def main():
    dev = torch.device("cuda", 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    stream = torch.cuda.current_stream(dev)
    for sh in sys.argv[1:]:
        M, N, K = (int(x) for x in sh.split(","))
        p = vx.Plan(N, K, "bf16", "bf16", "nk")
        ch = p.select(M)
        t_ours = time_graph(p, 1, M, N, K, -1, 0, dev, stream, l2, 5, "nk")
        t_cb = time_cublas(M, N, K, dev, l2)
        print("M=%5d N=%5d K=%4d  ours %7.2f us (rung %d split %d)  cublas %7.2f us  ratio %.2f" % (
            M, N, K, t_ours, ch["rung_id"], ch["split"], t_cb, t_cb / t_ours), flush=True)


if __name__ == "__main__":
    main()
