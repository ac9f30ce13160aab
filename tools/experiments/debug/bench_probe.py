"""Why does bench.py's per-launch time exceed tools/sweep.py's?  Re-time a subset of sweep
points with bench.py's own SweepGraph, varying the subset and R (launches per point)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_01075_b200 as vx

def run(pts, R, steps=5):
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev); side = torch.cuda.Stream(dev)
    plans = {}
    for _, M, N, K in pts:
        if (N, K) not in plans:
            plans[(N, K)] = vx.Plan(N, K, "bf16", "bf16", "nk", device=0)
    arenas = bench.make_arenas(pts, dev, 0)
    sg = bench.SweepGraph([(plans[(N, K)], M, N, K) for _, M, N, K in pts], R, arenas, stream, side)
    for _ in range(3): sg.replay()
    torch.cuda.synchronize()
    smp = []
    for _ in range(steps):
        sg.replay(); torch.cuda.synchronize(); smp.append(sg.per_launch_ms())
    del sg, arenas
    return [statistics.median(s[j] for s in smp) * 1e3 for j in range(len(pts))]

full = bench.sweep_points()
watch = [("llama", 512, 4096, 4096), ("bert", 128, 3072, 768), ("llama", 1, 11008, 4096),
         ("llama", 4, 11008, 4096), ("llama", 512, 11008, 4096)]
idx = [full.index(w) for w in watch]
t = run(full, 8)
print("full sweep R=8:   ", ["%.2f" % t[i] for i in idx])
t = run(full, 32, steps=3)
print("full sweep R=32:  ", ["%.2f" % t[i] for i in idx])
t = run(watch, 8)
print("subset R=8:       ", ["%.2f" % x for x in t])
t = run(watch, 64)
print("subset R=64:      ", ["%.2f" % x for x in t])
