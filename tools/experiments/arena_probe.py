"""Why BERT-size launches time slower in bench.py's SweepGraph than in tools/sweep.time_graph:
the same point under SweepGraph with operand arenas of different sizes (all > L2, so every
launch reads cold operands either way) and under time_graph.  Arena size changes how many
distinct pages the 48 launches touch (TLB reach), nothing else."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_01075_b200 as vx
from sweep import time_graph

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
side = torch.cuda.Stream(dev)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
pts = [("bert", 128, 3072, 768), ("bert", 256, 768, 768), ("bert", 64, 2304, 768),
       ("llama", 1, 11008, 4096), ("llama", 64, 11008, 4096)]
plans = {(N, K): vx.Plan(N, K, "bf16", "bf16", "nk") for _, M, N, K in pts}
for mib in (1024, 256, 128):
    n = mib * (1 << 20) // 2
    arenas = (bench.Arena(n, dev, "normal", 1), bench.Arena(n, dev, "normal", 2, scale=1 / 64),
              bench.Arena(n, dev, "empty", 0))
    sg = bench.SweepGraph([(plans[(N, K)], M, N, K) for _, M, N, K in pts], 48, arenas, stream, side)
    for _ in range(3):
        sg.replay()
    torch.cuda.synchronize()
    samples = []
    for _ in range(5):
        sg.replay(); torch.cuda.synchronize(); samples.append(sg.per_launch_ms())
    print("SweepGraph arenas %4d MiB:" % mib,
          ["%.2f" % (statistics.median(s[i] for s in samples) * 1e3) for i in range(len(pts))], flush=True)
    del sg, arenas
    torch.cuda.synchronize()
print("time_graph              :", ["%.2f" % time_graph(plans[(N, K)], 1, M, N, K, -1, 0, dev, stream, l2, 5, "nk")
                                    for _, M, N, K in pts], flush=True)
