"""Summarise a tools/sweep.py JSON: best tcgen05 (rung, split) vs each GEMV rung (R20)."""
import json
import sys


def main(path):
    for e in json.load(open(path)):
        is_gv = lambda f: f.get("family", 3 if 9 <= f["rung"] <= 12 else 0) == 3
        tc = [f for f in e["forced"] if not is_gv(f)]
        gv = [f for f in e["forced"] if is_gv(f)]
        b = min(tc, key=lambda f: f["us"])
        print("%5d %6d %5d  sel=(%d,%d) %.2f  best tc (%d,%d) %.2f  gemv: %s" % (
            e["M"], e["N"], e["K"], e["sel"]["rung_id"], e["sel"]["split"], e["t_sel_us"],
            b["rung"], b["split"], b["us"], ["r%d %.2f" % (f["rung"], f["us"]) for f in gv]))


if __name__ == "__main__":
    main(sys.argv[1])
