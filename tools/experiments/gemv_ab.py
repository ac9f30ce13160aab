"""A/B of GEMV rung variants (run once per VX_DEBUG_FLAGS value; 16384 turns off the
A-in-SMEM kernel of the MT 4 / 8 rungs, R20b) on LLaMA decode shapes, graph-timed with cold operands
(tools/sweep.time_graph).  Prints one JSON line per (M, N): selected and every GEMV rung."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_01075_b200 as vx
from sweep import time_graph

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
K = 4096
for N in (4096, 11008, 12288):
    p = vx.Plan(N, K, "bf16", "bf16", "nk")
    gv = [r for r in p.dump()["rungs"] if r["family"] == 3]
    for M in (1, 2, 4, 8):
        out = {"flags": os.environ.get("VX_DEBUG_FLAGS", "0"), "M": M, "N": N,
               "sel": p.select(M, N=N)["rung_id"],
               "t_sel": round(time_graph(p, 1, M, N, K, -1, 0, dev, stream, l2, 5, "nk"), 2)}
        for r in gv:
            if r["bm"] >= M:
                out["gemv_bm%d" % r["bm"]] = round(time_graph(p, 1, M, N, K, r["rung_id"], 1, dev,
                                                              stream, l2, 5, "nk"), 2)
        print(json.dumps(out), flush=True)
