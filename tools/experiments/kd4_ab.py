"""A/B of four-chunk deep-K units (VX_DEBUG_FLAGS 32768 keeps two-chunk units): selected
choice and every non-pair K-major rung at its selected split, graph-timed on cold operands
(tools/sweep.time_graph), LLaMA decode / mid-M and BERT shapes.  One JSON line per shape."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_01075_b200 as vx
from sweep import time_graph

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
shapes = [(M, N, 4096) for N in (4096, 11008, 12288) for M in (4, 16, 64, 256, 1024)]
shapes += [(M, N, 768) for N in (768, 3072) for M in (16, 256, 2048)]
plans = {}
for M, N, K in shapes:
    p = plans.setdefault((N, K), vx.Plan(N, K, "bf16", "bf16", "nk"))
    sel = p.select(M, N=N)
    out = {"flags": os.environ.get("VX_DEBUG_FLAGS", "0"), "M": M, "N": N, "K": K,
           "sel": [sel["rung_id"], sel["split"]],
           "t_sel": round(time_graph(p, 1, M, N, K, -1, 0, dev, stream, l2, 5, "nk"), 2)}
    for r in p.dump()["rungs"]:
        if r["family"] in (0, 1) and r["bm"] == 128 and r["stages"] >= 8:
            for s in (1, 0):
                if s in r["splits"]:
                    out["r%d_s%d" % (r["rung_id"], s)] = round(
                        time_graph(p, 1, M, N, K, r["rung_id"], s, dev, stream, l2, 5, "nk"), 2)
    print(json.dumps(out), flush=True)
