"""A/B the two graph timing harnesses on the same shapes: bench.SweepGraph (one graph, event
nodes between points, R launches per point on arena slices) vs tools/sweep.time_graph
(one graph per shape, rotating buffer sets).  Debug aid for the measurement method."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import bench
import paper_2409_01075_b200 as vx
from sweep import time_graph

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
side = torch.cuda.Stream(dev)
pts = [("bert", 1, 768, 768), ("bert", 64, 3072, 768), ("bert", 512, 2304, 768),
       ("llama", 1, 11008, 4096), ("llama", 4096, 11008, 4096)]
plans = {(N, K): vx.Plan(N, K, "bf16", "bf16", "nk") for _, M, N, K in pts}
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
for R in (8, 32):
    arenas = bench.make_arenas(pts, dev, 0)
    sg = bench.SweepGraph([(plans[(N, K)], M, N, K) for _, M, N, K in pts], R, arenas, stream, side)
    for _ in range(3):
        sg.replay()
    torch.cuda.synchronize()
    samples = []
    for _ in range(5):
        sg.replay(); torch.cuda.synchronize(); samples.append(sg.per_launch_ms())
    print("SweepGraph R=%d:" % R, ["%.2f" % (statistics.median(s[i] for s in samples) * 1e3) for i in range(len(pts))])
    del sg, arenas
    torch.cuda.synchronize()
print("time_graph     :", ["%.2f" % time_graph(plans[(N, K)], 1, M, N, K, -1, 0, dev, stream, l2, 5, "nk") for _, M, N, K in pts])
