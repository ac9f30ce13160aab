"""Selector regret of the library's compiled-in constants on measured forced-rung data
(calibrate.py measure output): per shape, measured time of the selected (rung, split) vs
the fastest measured one.  CPU only (uses vx_plan_ex with the captured descriptor)."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_01075_b200 as vx

raw = json.load(open(sys.argv[1]))
desc = vx.DeviceDesc.from_json(raw["desc"])
groups = {}
for s in raw["samples"]:
    groups.setdefault((s["M"], s["N"], s["K"]), {})[(s["rung"], s["split"])] = s["us"]
plans = {}
regs = []
for (M, N, K), ts in sorted(groups.items()):
    if (N, K) not in plans:
        plans[(N, K)] = vx.Plan(N, K, "bf16", "bf16", "nk", desc=desc)
    ch = plans[(N, K)].select(M)
    t_sel = ts.get((ch["rung_id"], ch["split"]))
    best = min(ts.items(), key=lambda kv: kv[1])
    r = best[1] / t_sel
    regs.append(r)
    if r < 0.9 or "-v" in sys.argv:
        print("M=%5d N=%5d K=%5d sel=(%d,%d) %.1fus best=(%d,%d) %.1fus regret=%.3f" % (
            M, N, K, ch["rung_id"], ch["split"], t_sel, best[0][0], best[0][1], best[1], r))
print("shapes %d geomean regret %.4f worst %.4f" % (
    len(regs), math.exp(sum(map(math.log, regs)) / len(regs)), min(regs)))
