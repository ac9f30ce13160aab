"""Hybrid-analyzer ablation (tbl:eval:analyzer).

    GPU:  python tools/analyzer_ablation.py measure [--out-dir gpurun_out]
          -> live calibrations (vx_calibrate effort 0 and 1) as JSON, with their wall time
    CPU:  python tools/analyzer_ablation.py eval HELDOUT_SWEEP.json CALIB.json [CALIB.json ...]
          -> selector regret (best forced time / time of the model's pick) on the held-out
             benchmark sweep (tools/sweep.py --shapes all output) for each calibration,
             evaluated with the oracle's selector (oracle/selector_ref.py) on the same table
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(out_dir):
    import paper_2409_01075_b200 as vx
    res = {}
    for effort in (0, 1):
        t0 = time.perf_counter()
        c = vx.calibrate(0, "nk", effort=effort)
        dt = time.perf_counter() - t0
        d = c.dump()
        d["wall_s"] = dt
        json.dump(d, open(os.path.join(out_dir, "live_calib_e%d.json" % effort), "w"), indent=1)
        res[effort] = dt
        print("effort %d: %.1f s, source %s" % (effort, dt, d["source"]), flush=True)
    return res


def evaluate(sweep_path, calib_paths):
    import oracle.selector_ref as S
    desc = S.load_descriptor()
    sw = json.load(open(sweep_path))
    tabs = {}
    for cp in calib_paths:
        cal = json.load(open(cp))
        regs = {}
        for e in sw:
            if e.get("batch", 1) != 1:
                continue
            N, K, M = e["N"], e["K"], e["M"]
            if K not in tabs:
                tabs[K] = S.build_table(K, "bf16", "bf16", desc, "nk")
            t = tabs[K]
            best = min(f["us"] for f in e["forced"])
            timed = {(f["rung"], f["split"]): f["us"] for f in e["forced"]}
            ch = S.select(t, 1, M, N, K, desc, cal)
            us = timed.get((ch["rung_id"], ch["split"]))
            if us is None:
                continue
            regs.setdefault("bert" if K == 768 else "llama", []).append(best / us)
        gm = lambda v: math.exp(sum(math.log(x) for x in v) / len(v))
        allr = [x for v in regs.values() for x in v]
        print("%-40s regret geomean %.4f worst %.3f  %s  (%d points)" % (
            os.path.basename(cp), gm(allr), min(allr),
            " ".join("%s %.4f" % (k, gm(v)) for k, v in sorted(regs.items())), len(allr)))


if __name__ == "__main__":
    if sys.argv[1] == "measure":
        od = sys.argv[sys.argv.index("--out-dir") + 1] if "--out-dir" in sys.argv else "gpurun_out"
        measure(od)
    else:
        evaluate(sys.argv[2], sys.argv[3:])
