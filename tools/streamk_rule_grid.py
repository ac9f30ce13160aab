"""R19 on the GENERIC calibration grid (analysis tool, CPU): the selector regret of the
installed calibration when the stream-K admissibility rule is varied -- the wave bound
(stream-K competes only when the data-parallel grid needs <= W waves) and the half-tile rule
(every CTA's share >= half a tile's K loop).  Uses only the calibration grid's forced-rung
timings (never the benchmark sweep), so the rule the library ships is chosen on generic
shapes.

    python tools/streamk_rule_grid.py profiles/r02c_calib_raw.json oracle/calib_b200.json
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import calibrate as C   # noqa: E402


def main():
    raw = json.load(open(sys.argv[1]))
    cal = json.load(open(sys.argv[2]))
    desc = raw["desc"]
    th = {n: dict(mac=r["mac_milli"] / 1000, l2s=r["l2s_milli"] / 1000, epi=r["epi_milli"] / 1000,
                  fixed=r["fixed"]) for n, r in cal["rungs"].items()}
    g = dict(hbm=cal["hbm_milli"] / 1000, dsm=cal["dsm_milli"] / 1000,
             fixed_cluster=cal["fixed_cluster"], skfix=cal["skfix_milli"] / 1000,
             stagger=cal.get("stagger", 0))
    fam = {0: "umma", 1: "umma_swap", 3: "gemv"}
    groups = {}
    for sm in raw["samples"]:
        groups.setdefault((sm["M"], sm["N"], sm["K"]), []).append(sm)

    def sk_pred(sm, t_):
        """the stream-K model cost with NO admissibility rule (a copy of calibrate.model_us's
        stream-K branch without its two returns of inf)"""
        M, N, K, bm, bn, bk = sm["M"], sm["N"], sm["K"], sm["bm"], sm["bn"], 64
        mac, l2s, epi = (int(round(t_[k] * 1000)) for k in ("mac", "l2s", "epi"))
        fixed = int(round(t_["fixed"]))
        hbm, skfix = int(round(g["hbm"] * 1000)), int(round(g["skfix"] * 1000))
        t = lambda nbytes, bw: C._cd(nbytes * 1000, bw)
        swap = sm["family"] == 1
        mt, nt = (N, M) if swap else (M, N)
        tiles = C._cd(mt, bm) * C._cd(nt, bn)
        kb = C._cd(K, bk)
        c = t(bm * bn * bk, mac)
        ls = t((min(bm, mt) + min(bn, nt)) * bk * 2, l2s)
        cgk = 2 if bm == 256 else 1
        U = tiles * kb
        G = min(desc["max_active_clusters"][str(cgk)], U)
        units = C._cd(U, G)
        segs = C._cd(units, kb) + 1
        l = max(ls, t(2 * K * (mt + nt), units * hbm))
        tm_ = l + (units - 1) * max(l, c) + c
        st = max(t(bm * bn * 2, epi), t(2 * M * N, segs * hbm))
        cyc = max(tm_, segs * st) + st + C._cd(kb, units) * t(2 * (bm // cgk) * bn * 4, skfix) + fixed
        if G * cgk > desc["sm_count"] // 2:
            cyc += int(round(g["stagger"]))
        waves = tiles * cgk / (desc["max_active_clusters"][str(cgk)] * cgk)
        return cyc / (C.CLOCK_GHZ * 1e3), waves, 2 * units >= kb

    rows = []
    for key, ss in groups.items():
        best = min(x["us"] for x in ss)
        cand = []
        for x in ss:
            t_ = th[C.calib_key(fam[x["family"]], x["bm"], x["bn"], x.get("mc", 1), x.get("occ", 1))]
            if x["split"] == 0:
                p, waves, half = sk_pred(x, t_)
                cand.append((p, x["us"], waves, half))
            else:
                p = C.model_us(x, t_, desc, g)
                cand.append((p, x["us"], None, None))
        rows.append((best, cand))
    print("wave bound  half-tile rule  grid regret (geomean / worst)")
    for wb in (1, 2, 3, 4, 6, 1e9):
        for half in (True, False):
            regs = []
            for best, cand in rows:
                ok = [c for c in cand if c[2] is None or (c[2] <= wb and (c[3] or not half))]
                pick = min(ok, key=lambda c: c[0])
                regs.append(best / pick[1])
            gm = math.exp(sum(math.log(r) for r in regs) / len(regs))
            print("%10s  %14s  %.4f / %.3f" % ("inf" if wb > 1e8 else wb, half, gm, min(regs)))


if __name__ == "__main__":
    main()
