"""Empirical tier of the hybrid analyzer: profile every rung of the
ladder once on a FIXED, GENERIC grid of calibration shapes (tile multiples and tails; not
the benchmark workload, no sample list), then fit the rung constants of the analytical
model to the measurements.

    measure (GPU):  python tools/calibrate.py measure --out gpurun_out/calib_raw.json
    fit (CPU):      python tools/calibrate.py fit gpurun_out/calib_raw.json

The fit re-implements the DESIGN.md 3.3 formula in float form (no ceilings) -- it is a
tool, independent of both the library and the oracle; its output is written by hand into
csrc/vx_calib.cpp and oracle/calib_b200.json, whose equality is tested.
"""
import argparse
import ctypes
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CAL_M = (1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 160, 200, 256, 320, 384, 512, 768, 1024, 1536,
         2048, 3072, 4096, 8192)
# generic (N, K): powers of two and N with odd tile counts (13 / 21 / 42 tiles of 256), plus
# small-K shapes (K <= 1024: few k-blocks, the launch-floor regime) with odd tile counts
CAL_NK = ((1024, 1024), (4096, 1024), (2048, 4096), (8192, 4096), (6144, 2048),
          (3328, 1536), (5376, 4096), (10752, 2048), (1536, 512), (2560, 640),
          (1280, 896), (3584, 640), (2048, 512),
          # round 2: grids of 75-148 CTAs per wave (where back-to-back launches can no longer
          # overlap their prologue with the previous grid) and long-K weight streams
          (14336, 4096), (9728, 3072), (13312, 1024), (2816, 832), (1792, 832))
CLOCK_GHZ = 1.965   # cycles of the model are SM cycles at the max clock


def measure(args):
    import torch
    import paper_2409_01075_b200 as vx
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from sweep import graph_buffers, time_graph
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    out = {"desc": vx.device_probe(0).to_json(), "clock_ghz": CLOCK_GHZ, "samples": []}
    nk_list = CAL_NK[13:] if getattr(args, "only_new", False) else CAL_NK
    only = set(args.only_keys.split(",")) if getattr(args, "only_keys", None) else None
    fam_of = {0: "umma", 1: "umma_swap", 3: "gemv"}
    for N, K in nk_list:
        p = vx.Plan(N, K, "bf16", "bf16", "nk")
        rungs = [r for r in p.dump()["rungs"]
                 if only is None or calib_key(fam_of[r["family"]], r["bm"], r["bn"], r.get("mc", 1),
                                              r.get("occ", 1)) in only]
        for M in CAL_M:
            bufs = graph_buffers(1, M, N, K, dev, l2)    # one operand set per shape
            for r in rungs:
                if r["family"] == 3 and M > r["bm"]:
                    continue
                for s in r["splits"]:
                    t = time_graph(p, 1, M, N, K, r["rung_id"], s, dev, stream, l2, 3, "nk", bufs)
                    out["samples"].append({"M": M, "N": N, "K": K, "rung": r["rung_id"],
                                           "family": r["family"], "bm": r["bm"], "bn": r["bn"],
                                           "mc": r.get("mc", 1), "occ": r.get("occ", 1),
                                           "stages": r["stages"],
                                           "split": s, "us": t})
            del bufs
            print("N=%d K=%d M=%d done" % (N, K, M), flush=True)
    json.dump(out, open(args.out, "w"))


# ---- integer model (DESIGN.md 3.3 / R19, the library's arithmetic) --------------------------
def _cd(a, b):
    return -(-a // b)


def calib_key(fam, bm, bn, mc=1, occ=1):
    """Calibration-table key of a rung (the library's vx_plan.cpp naming)."""
    if occ == 2:
        return "%s_o2_%dx%d" % (fam, bm, bn)
    return "%s_mc%d_%dx%d" % (fam, mc, bm, bn) if mc > 1 else "%s_%dx%d" % (fam, bm, bn)


def model_us(sm, th, desc, g):
    """th: per-rung dict mac,l2s,epi,fixed (per-cycle rates); g: hbm,dsm,fixed_cluster,skfix.
    Rates are rounded to the library's x1000 integers and every division is a ceiling, so
    the fitted constants are judged by exactly the decisions vx_plan_select will make."""
    M, N, K, s = sm["M"], sm["N"], sm["K"], sm["split"]
    bm, bn, bk = sm["bm"], sm["bn"], 64
    if sm["family"] == 3:   # CUDA-core GEMV rung (R20)
        mac, l2s, epi = (int(round(th[k] * 1000)) for k in ("mac", "l2s", "epi"))
        hbm = int(round(g["hbm"] * 1000))
        t = lambda nbytes, bw: _cd(nbytes * 1000, bw)
        bk = 1024
        tiles = _cd(N, bn)
        F = _cd(tiles, desc["sm_count"] * 4)
        trips = _cd(K, bk)
        inner = t(bm * bn * bk, mac)
        tl = max(t(bn * bk * 2 + bm * bk * 2, l2s), t(2 * K * (N + M), F * trips * hbm))
        ts = max(t(bm * bn * 2, epi), t(2 * M * N, F * hbm))
        cyc = F * (tl + (trips - 1) * max(tl, inner) + inner + ts) + int(round(th["fixed"]))
        return cyc / (CLOCK_GHZ * 1e3)
    mac, l2s, epi = (int(round(th[k] * 1000)) for k in ("mac", "l2s", "epi"))
    fixed = int(round(th["fixed"]))
    hbm, dsm, skfix = (int(round(g[k] * 1000)) for k in ("hbm", "dsm", "skfix"))
    fixed_cluster = int(round(g["fixed_cluster"]))
    t = lambda nbytes, bw: _cd(nbytes * 1000, bw)
    swap = sm["family"] == 1
    mt, nt = (N, M) if swap else (M, N)
    tm, tn = _cd(mt, bm), _cd(nt, bn)
    tiles = tm * tn
    kb = _cd(K, bk)
    c = t(bm * bn * bk, mac)
    mc = sm.get("mc", 1)                 # TMA-multicast cluster sharing the A tile
    p_rows = bm // mc if (mc > 1 and not swap) else min(bm, mt)
    q_rows = bn // mc if (mc > 1 and swap) else min(bn, nt)
    ls = t((p_rows + q_rows) * bk * 2, l2s)
    if s == 0:   # stream-K (R19), admitted only for <= 3 data-parallel waves
        cgk = 2 if bm == 256 else 1
        if tiles * cgk > 3 * desc["max_active_clusters"][str(cgk)] * cgk:
            return float("inf")
        U = tiles * kb
        G = min(desc["max_active_clusters"]["2" if bm == 256 else "1"], U)
        units = _cd(U, G)
        if 2 * units < kb:      # R19: a CTA's share must be >= half a tile's K loop
            return float("inf")
        segs = _cd(units, kb) + 1
        l = max(ls, t(2 * K * (mt + nt), units * hbm))
        tm_ = l + (units - 1) * max(l, c) + c
        st = max(t(bm * bn * 2, epi), t(2 * M * N, segs * hbm))
        cyc = max(tm_, segs * st) + st + _cd(kb, units) * t(2 * (bm // cgk) * bn * 4, skfix) + fixed
        if G * cgk > desc["sm_count"] // 2:          # R21
            cyc += int(round(g.get("stagger", 0)))
        return cyc / (CLOCK_GHZ * 1e3)
    cg = 2 if bm == 256 else 1
    trips = kb // s
    tm_c = _cd(tm, mc) * mc if (mc > 1 and swap) else tm
    tn_c = _cd(tn, mc) * mc if (mc > 1 and not swap) else tn
    W = tm_c * tn_c * s * cg
    slots = desc["max_active_clusters"][str(s * cg * mc)] * s * cg * mc
    F = _cd(W, slots)
    l = max(ls, t(2 * K * (mt + nt), F * trips * hbm))
    st = max(t(bm * bn * 2, s * epi), t(2 * M * N, F * hbm))
    if s > 1:
        st += t((s - 1) * bm * bn * 4, s * dsm)
    T = l + (trips - 1) * max(l, c) + c + st
    if s == 1:
        tmain = T - st
        cyc = tmain + (F - 1) * max(tmain, st) + st + fixed
    else:
        cyc = F * T + fixed + fixed_cluster
    if min(W, slots) > desc["sm_count"] // 2:        # R21
        cyc += int(round(g.get("stagger", 0)))
    return cyc / (CLOCK_GHZ * 1e3)


def fit(args):
    import numpy as np
    from scipy.optimize import minimize
    raw = json.load(open(args.raw))
    desc = raw["desc"]
    S = raw["samples"]
    fam = {0: "umma", 1: "umma_swap", 3: "gemv"}
    keys = sorted({(fam[x["family"]], x["bm"], x["bn"], x.get("mc", 1), x.get("occ", 1)) for x in S})
    ini0 = json.load(open(args.init)) if args.init else None
    names = [calib_key(*k) for k in keys]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"] / CLOCK_GHZ
    # parameter vector: log of (mac, l2s, epi, fixed) per rung + log(dsm, fixed_cluster)
    x0 = []
    for k in keys:
        x0 += [math.log(4096 if k[2] >= 128 else 2048), math.log(96), math.log(64), math.log(3000)]
    x0 += [math.log(20), math.log(1500), math.log(32)]
    if args.init:
        ini = json.load(open(args.init))
        for i, n in enumerate(names):
            if n not in ini["rungs"]:
                continue
            r = ini["rungs"][n]
            x0[4 * i:4 * i + 4] = [math.log(r["mac_milli"] / 1000), math.log(r["l2s_milli"] / 1000),
                                   math.log(r["epi_milli"] / 1000), math.log(max(r["fixed"], 1))]
        x0[-3:] = [math.log(ini["dsm_milli"] / 1000), math.log(max(ini["fixed_cluster"], 1)),
                   math.log(ini.get("skfix_milli", 32000) / 1000)]

    def unpack(x):
        th = {}
        for i, n in enumerate(names):
            th[n] = dict(mac=math.exp(x[4 * i]), l2s=math.exp(x[4 * i + 1]),
                         epi=math.exp(x[4 * i + 2]), fixed=math.exp(x[4 * i + 3]))
        g = dict(hbm=hbm, dsm=math.exp(x[-3]), fixed_cluster=math.exp(x[-2]), skfix=math.exp(x[-1]))
        return th, g

    def key_of(x):
        return calib_key(fam[x["family"]], x["bm"], x["bn"], x.get("mc", 1), x.get("occ", 1))

    groups = {}
    for sm in S:
        groups.setdefault((sm["M"], sm["N"], sm["K"]), []).append(sm)
    best_t = {k: min(x["us"] for x in v) for k, v in groups.items()}

    def loss(x):
        th, g = unpack(x)
        e = 0.0
        n = 0
        for sm in S:
            pred = model_us(sm, th[key_of(sm)], desc, g)
            if pred == float("inf"):      # inadmissible (R19): never selected, not fitted
                continue
            e += (math.log(pred) - math.log(sm["us"])) ** 2
            n += 1
        e = args.err_weight * e / max(n, 1)
        # selection quality: log-regret of the model's pick per calibration shape
        r = 0.0
        for k, v in groups.items():
            pick = min(v, key=lambda z: model_us(z, th[key_of(z)], desc, g))
            r += math.log(pick["us"] / best_t[k])
        return e + args.regret_weight * r / len(groups)

    lo, hi = [], []
    for k in keys:
        if k[0] == "gemv":
            lo += [math.log(1), math.log(4), math.log(1), math.log(200)]
            hi += [math.log(512), math.log(256), math.log(512), math.log(12000)]
        else:
            lo += [math.log(1000), math.log(8), math.log(8), math.log(500)]
            hi += [math.log(4096), math.log(160), math.log(512), math.log(12000)]
    lo += [math.log(2), math.log(1), math.log(1)]
    hi += [math.log(64), math.log(8000), math.log(256)]
    x0 = [min(max(v, a), b) for v, a, b in zip(x0, lo, hi)]
    if args.method == "powell":
        res = minimize(loss, np.array(x0), method="Powell", bounds=list(zip(lo, hi)),
                       options={"maxiter": 40000, "xtol": 1e-3, "ftol": 1e-6})
        xb = list(res.x)
    else:
        # greedy coordinate search on multiplicative steps: the regret objective is
        # piecewise constant, so move one log-parameter at a time while it helps
        steps = [math.log(f) for f in (2.0, 1.4, 1.15, 1.05)]

        def descend(x, f):
            for sweep in range(args.sweeps):
                improved = False
                for i in range(len(x)):
                    for st in steps:
                        for sg in (1, -1):
                            xt = list(x)
                            xt[i] = min(max(xt[i] + sg * st, lo[i]), hi[i])
                            ft = loss(np.array(xt))
                            if ft < f - 1e-9:
                                x, f, improved = xt, ft, True
                print("sweep %d objective %.5f" % (sweep, f), flush=True)
                if not improved:
                    break
            return x, f

        xb = list(x0)
        xb, fb = descend(xb, loss(np.array(xb)))
        # random restarts around the incumbent (the regret objective is piecewise constant
        # with many plateaus); seeded, so the fit is reproducible
        rng = np.random.default_rng(args.seed)
        for r in range(args.restarts):
            xs = [min(max(v + rng.normal(0.0, 0.35), a), b) for v, a, b in zip(xb, lo, hi)]
            xs, fs = descend(xs, loss(np.array(xs)))
            print("restart %d objective %.5f (best %.5f)" % (r, fs, min(fs, fb)), flush=True)
            if fs < fb:
                xb, fb = xs, fs

        class R:
            pass
        res = R()
        res.fun = fb
    th, g = unpack(xb)
    print("rms log error %.3f" % math.sqrt(res.fun))
    # regret of the fitted model on the calibration grid
    groups = {}
    for sm in S:
        groups.setdefault((sm["M"], sm["N"], sm["K"]), []).append(sm)
    regrets = []
    for k, v in groups.items():
        best = min(x["us"] for x in v)
        pick = min(v, key=lambda x: model_us(x, th[key_of(x)], desc, g))
        regrets.append(best / pick["us"])
    print("calibration-grid regret geomean %.4f worst %.4f" % (
        math.exp(sum(math.log(r) for r in regrets) / len(regrets)), min(regrets)))
    out = {"hbm_milli": int(round(hbm * 1000)), "dsm_milli": int(round(g["dsm"] * 1000)),
           "fixed_cluster": int(round(g["fixed_cluster"])),
           "skfix_milli": int(round(g["skfix"] * 1000)), "rungs": {}}
    for n in names:
        t = th[n]
        out["rungs"][n] = {"mac_milli": int(round(t["mac"] * 1000)),
                           "l2s_milli": int(round(t["l2s"] * 1000)),
                           "epi_milli": int(round(t["epi"] * 1000)),
                           "fixed": int(round(t["fixed"]))}
    print(json.dumps(out, indent=1))


def measured_pair_mac(raw):
    """L0 empirical rate of each cta_group::2 pair rung, read off the calibration profile:
    the best steady-state MACs per (CLOCK_GHZ) cycle per resident pair over the grid shapes
    with >= 4 waves of pair tiles (the mainloop is then essentially the whole time):
    M*N*K / (t * clock * pairs)."""
    pairs = raw["desc"]["max_active_clusters"]["2"]
    best = {}
    for sm in raw["samples"]:
        if sm["bm"] != 256 or sm["split"] != 1 or sm.get("mc", 1) != 1:
            continue
        tiles = -(-sm["M"] // 256) * -(-sm["N"] // sm["bn"])
        if tiles < 4 * pairs:
            continue
        rate = sm["M"] * sm["N"] * sm["K"] / (sm["us"] * 1e-6 * CLOCK_GHZ * 1e9 * pairs)
        best[sm["bn"]] = max(best.get(sm["bn"], 0.0), rate)
    return {k: round(v) for k, v in best.items()}


def fit_fast(args):
    """Same objective and coordinate search as fit(), with per-sample predictions cached: a
    step on one rung's constant re-evaluates only that rung's samples (a global constant
    re-evaluates all), so a 17k-sample grid fits in minutes."""
    import numpy as np
    raw = json.load(open(args.raw))
    desc = raw["desc"]
    S = raw["samples"]
    fam = {0: "umma", 1: "umma_swap", 3: "gemv"}
    keys = sorted({(fam[x["family"]], x["bm"], x["bn"], x.get("mc", 1), x.get("occ", 1)) for x in S})
    names = [calib_key(*k) for k in keys]
    kidx = {n: i for i, n in enumerate(names)}
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"] / CLOCK_GHZ
    ini = json.load(open(args.init)) if args.init else {"rungs": {}}
    x = []
    for n in names:
        r = ini["rungs"].get(n)
        if r is None:      # new rung: start from its unicast sibling, else a generic guess
            base = n.replace("_mc2_", "_").replace("_mc4_", "_").replace("_o2_", "_")
            r = ini["rungs"].get(base, {"mac_milli": 2048000, "l2s_milli": 96000,
                                        "epi_milli": 64000, "fixed": 3000})
        x += [math.log(r["mac_milli"] / 1000), math.log(r["l2s_milli"] / 1000),
              math.log(r["epi_milli"] / 1000), math.log(max(r["fixed"], 1))]
    x += [math.log(ini.get("dsm_milli", 20000) / 1000), math.log(max(ini.get("fixed_cluster", 1500), 1)),
          math.log(ini.get("skfix_milli", 32000) / 1000), math.log(max(ini.get("stagger", 4000), 1))]
    lo, hi = [], []
    for k in keys:
        if k[0] == "gemv":
            lo += [math.log(1), math.log(4), math.log(1), math.log(200)]
            hi += [math.log(512), math.log(256), math.log(512), math.log(12000)]
        elif k[1] == 256 and args.pair_mac:
            # cta_group::2 pairs: the MMA rate is MEASURED, not fitted -- steady-state MACs
            # per (1.965 GHz) cycle per pair of the largest calibration shapes, where the
            # pair's mainloop is the whole time (the fitted value otherwise sits on the
            # single-SM bound, 4096, i.e. prices a 2-SM tile at one SM's rate)
            m = args.pair_mac[k[2]] if k[2] in args.pair_mac else 4096
            lo += [math.log(m), math.log(8), math.log(8), math.log(200)]
            hi += [math.log(m) + 1e-9, math.log(160), math.log(512), math.log(12000)]
        else:
            lo += [math.log(1000), math.log(8), math.log(8), math.log(200)]
            hi += [math.log(4096), math.log(160), math.log(512), math.log(12000)]
    lo += [math.log(2), math.log(1), math.log(1), math.log(1)]
    hi += [math.log(64), math.log(8000), math.log(256), math.log(20000)]
    x = [min(max(v, a), b) for v, a, b in zip(x, lo, hi)]
    samp_key = [kidx[calib_key(fam[sm["family"]], sm["bm"], sm["bn"], sm.get("mc", 1), sm.get("occ", 1))]
                for sm in S]
    by_rung = {}
    for j, kk in enumerate(samp_key):
        by_rung.setdefault(kk, []).append(j)
    meas = np.array([math.log(sm["us"]) for sm in S])
    gid = {}
    groups = []
    for j, sm in enumerate(S):
        g = (sm["M"], sm["N"], sm["K"])
        if g not in gid:
            gid[g] = len(groups)
            groups.append([])
        groups[gid[g]].append(j)
    best_t = np.array([min(S[j]["us"] for j in gg) for gg in groups])
    us = np.array([sm["us"] for sm in S])

    def th_of(x, i):
        return dict(mac=math.exp(x[4 * i]), l2s=math.exp(x[4 * i + 1]),
                    epi=math.exp(x[4 * i + 2]), fixed=math.exp(x[4 * i + 3]))

    def g_of(x):
        return dict(hbm=hbm, dsm=math.exp(x[-4]), fixed_cluster=math.exp(x[-3]),
                    skfix=math.exp(x[-2]), stagger=math.exp(x[-1]))

    pred = np.zeros(len(S))

    def eval_rung(x, i, out):
        th, g = th_of(x, i), g_of(x)
        for j in by_rung.get(i, []):
            out[j] = model_us(S[j], th, desc, g)

    for i in range(len(names)):
        eval_rung(x, i, pred)

    def loss_of(pr):
        fin = np.isfinite(pr)
        e = np.mean((np.log(pr[fin]) - meas[fin]) ** 2)
        r = 0.0
        for gi, gg in enumerate(groups):
            jb = gg[int(np.argmin(pr[gg]))]
            r += math.log(us[jb] / best_t[gi])
        return args.err_weight * e + args.regret_weight * r / len(groups)

    f = loss_of(pred)
    print("start objective %.5f" % f, flush=True)
    steps = [math.log(v) for v in (2.0, 1.4, 1.15, 1.05)]
    for sweep in range(args.sweeps):
        improved = False
        for p_ in range(len(x)):
            rung = p_ // 4 if p_ < 4 * len(names) else None
            for st in steps:
                for sg in (1, -1):
                    xt = list(x)
                    xt[p_] = min(max(xt[p_] + sg * st, lo[p_]), hi[p_])
                    if xt[p_] == x[p_]:
                        continue
                    pt = pred.copy()
                    if rung is None:
                        for i in range(len(names)):
                            eval_rung(xt, i, pt)
                    else:
                        eval_rung(xt, rung, pt)
                    ft = loss_of(pt)
                    if ft < f - 1e-9:
                        x, f, pred, improved = xt, ft, pt, True
        print("sweep %d objective %.5f" % (sweep, f), flush=True)
        if not improved:
            break
    regrets = []
    for gi, gg in enumerate(groups):
        jb = gg[int(np.argmin(pred[gg]))]
        regrets.append(best_t[gi] / us[jb])
    print("calibration-grid regret geomean %.4f worst %.4f" % (
        math.exp(sum(math.log(r) for r in regrets) / len(regrets)), min(regrets)))
    g = g_of(x)
    out = {"hbm_milli": int(round(hbm * 1000)), "dsm_milli": int(round(g["dsm"] * 1000)),
           "fixed_cluster": int(round(g["fixed_cluster"])),
           "skfix_milli": int(round(g["skfix"] * 1000)), "stagger": int(round(g["stagger"])),
           "rungs": {}}
    for i, n in enumerate(names):
        t = th_of(x, i)
        out["rungs"][n] = {"mac_milli": int(round(t["mac"] * 1000)),
                           "l2s_milli": int(round(t["l2s"] * 1000)),
                           "epi_milli": int(round(t["epi"] * 1000)),
                           "fixed": int(round(t["fixed"]))}
    if args.out:
        json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(out, indent=1))


def heldout(args):
    """Selector regret on benchmark shapes NOT used by the fit (tools/sweep.py --shapes all
    output), for one or more calibration files (oracle/calib_b200.json format)."""
    import paper_2409_01075_b200 as vx
    raw = json.load(open(args.raw))             # calibration raw data: only its descriptor
    desc = raw["desc"]
    dd = vx.DeviceDesc.from_json(desc)
    sw = json.load(open(args.sweep))
    fam = {0: "umma", 1: "umma_swap", 3: "gemv"}
    for cf in args.calib:
        cal = json.load(open(cf))
        th = {n: dict(mac=r["mac_milli"] / 1000, l2s=r["l2s_milli"] / 1000, epi=r["epi_milli"] / 1000,
                      fixed=r["fixed"]) for n, r in cal["rungs"].items()}
        g = dict(hbm=cal["hbm_milli"] / 1000, dsm=cal["dsm_milli"] / 1000,
                 fixed_cluster=cal["fixed_cluster"], skfix=cal["skfix_milli"] / 1000,
                 stagger=cal.get("stagger", 0))
        plans, regs, by = {}, [], {}
        for e in sw:
            if e.get("batch", 1) != 1:
                continue
            N, K, M = e["N"], e["K"], e["M"]
            if (N, K) not in plans:
                plans[(N, K)] = {r["rung_id"]: r for r in vx.Plan(N, K, "bf16", "bf16", "nk", desc=dd).dump()["rungs"]}
            rt = plans[(N, K)]
            best = min(f["us"] for f in e["forced"])
            def pred(f):
                r = rt[f["rung"]]
                sm = dict(M=M, N=N, K=K, split=f["split"], family=r["family"], bm=r["bm"], bn=r["bn"],
                          mc=r.get("mc", 1), occ=r.get("occ", 1))
                return model_us(sm, th[calib_key(fam[r["family"]], r["bm"], r["bn"], r.get("mc", 1),
                                                 r.get("occ", 1))], desc, g)
            pick = min(e["forced"], key=pred)
            regs.append(best / pick["us"])
            tag = "bert" if K == 768 else "llama"
            by.setdefault(tag, []).append(best / pick["us"])
        gm = lambda v: math.exp(sum(math.log(x) for x in v) / len(v))
        print("%s: held-out regret geomean %.4f worst %.4f  (%s)" % (
            cf, gm(regs), min(regs), ", ".join("%s %.4f" % (k, gm(v)) for k, v in sorted(by.items()))))


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd")
    m = sub.add_parser("measure")
    m.add_argument("--out", default="gpurun_out/calib_raw.json")
    m.add_argument("--only-new", action="store_true", help="only the round-2 additions to CAL_NK")
    m.add_argument("--only-keys", default=None,
                   help="comma-separated calibration keys: re-measure only these rungs")
    mg = sub.add_parser("merge")
    mg.add_argument("raw")
    mg.add_argument("patch")
    mg.add_argument("--out", required=True)
    f = sub.add_parser("fit")
    f.add_argument("raw")
    f.add_argument("--regret-weight", type=float, default=2.0)
    f.add_argument("--init", default=None, help="start from a calibration json")
    f.add_argument("--method", default="coord", choices=["coord", "powell"])
    f.add_argument("--sweeps", type=int, default=12)
    f.add_argument("--err-weight", type=float, default=1.0)
    f.add_argument("--restarts", type=int, default=0)
    f.add_argument("--seed", type=int, default=0)
    f.add_argument("--fast", action="store_true", help="cached-prediction coordinate search")
    f.add_argument("--out", default=None)
    f.add_argument("--pair-mac", default=None,
                   help="'auto' (from the raw profile) or BN:mac,...: measured MAC/cycle per "
                        "cta_group::2 pair, frozen in the fit")
    h = sub.add_parser("heldout")
    h.add_argument("raw")
    h.add_argument("sweep")
    h.add_argument("calib", nargs="+")
    args = ap.parse_args()
    if getattr(args, "pair_mac", None) == "auto":
        args.pair_mac = measured_pair_mac(json.load(open(args.raw)))
        print("measured pair MAC / cycle:", args.pair_mac, flush=True)
    elif getattr(args, "pair_mac", None):
        args.pair_mac = {int(a): float(b) for a, b in (x.split(":") for x in args.pair_mac.split(","))}
    if args.cmd == "measure":
        measure(args)
    elif args.cmd == "merge":
        # replace the samples of the rungs re-measured in `patch` (same grid) in `raw`
        raw, patch = json.load(open(args.raw)), json.load(open(args.patch))
        fam = {0: "umma", 1: "umma_swap", 3: "gemv"}
        key = lambda x: calib_key(fam[x["family"]], x["bm"], x["bn"], x.get("mc", 1), x.get("occ", 1))
        redo = {key(x) for x in patch["samples"]}
        raw["samples"] = [x for x in raw["samples"] if key(x) not in redo] + patch["samples"]
        json.dump(raw, open(args.out, "w"))
        print("merged %d re-measured rung keys: %s" % (len(redo), sorted(redo)))
    elif args.cmd == "heldout":
        heldout(args)
    elif args.fast:
        fit_fast(args)
    else:
        fit(args)


if __name__ == "__main__":
    main()
