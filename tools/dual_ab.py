"""A/B of the dual MMA issuers per rung (measurement tool): every (rung, split) forced on a
few shapes, graph-timed; run once normally and once with VX_DEBUG_FLAGS=262144 (one issuer).

    python tools/dual_ab.py "M,N,K;..." > out.txt
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import paper_2409_01075_b200 as vx
from sweep import graph_buffers, time_graph

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
res = []
for spec in sys.argv[1].split(";"):
    M, N, K = (int(v) for v in spec.split(","))
    p = vx.Plan(N, K, "bf16", "bf16", "nk")
    bufs = graph_buffers(1, M, N, K, dev, l2)
    for r in p.dump()["rungs"]:
        if r["family"] not in (0, 1) or r["mc"] != 1 or r["bm"] != 128 or r["bn"] > 128:
            continue
        for s in r["splits"]:
            t = time_graph(p, 1, M, N, K, r["rung_id"], s, dev, stream, l2, 3, "nk", bufs)
            res.append({"M": M, "N": N, "K": K, "rung": r["rung_id"], "bn": r["bn"],
                        "swap": r["swap"], "split": s, "us": t})
    del bufs
print(json.dumps(res))
