"""oracle/selector_ref.py -- TEST INFRASTRUCTURE ONLY (parity oracle, never on the product path).

A plain, pure-Python-int re-implementation of Vortex's two-stage method as DESIGN.md
section 3 specifies it for sm_100a, written step by step in the paper's order:

  offline  (sample-free strategy table, "vx_plan"):
      Alg. 2 "GenerateCandidatesForLayer" (Sec. 5.1):
        L0: InitCands -> FilterByISA
        L>=1: InitCands -> FilterByMultiples(prev) + map
      hardware limits from GetHardwareInfo
  runtime  (shape-dependent selection, "vx_plan_select"):
      Eq. 2  T_temporal = T_Load + (sizeof(TemporalLoop)-1)*max(T_Load, Cost_{L-1})
                          + Cost_{L-1} + T_Store
      Eq. 3  F_parallel = ceil(sizeof(ParallelLoop) / |HardwareUnit|)
      Eq. 4  Cost_L = F_parallel * T_temporal
      Eq. 1  c* = argmin_{s in S} Cost(s, L)
      "at runtime ... analytical cost models ... select the most suitable micro-kernel
       candidates ... compute ... grid configurations"

Every reading the paper leaves open (lattice, window, split-K, persistence, tie-break,
integer units) is listed in DESIGN.md "Readings" and cited inline as R<n>.

Inputs are data only: the device descriptor (captured from the B200 by vx_device_probe,
tests/golden/b200_desc.json) and the calibrated per-rung constants (oracle/calib_b200.json,
the empirical tier of the hybrid analyzer).  Nothing is imported from
the product package.

Pins: tests/test_oracle_selector.py (SPEC.md worked arithmetic for Eqs. 2-3 and the sieve,
brute-force argmin, staircase / monotonicity / zero-padding invariants).
"""
from __future__ import annotations

import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))

IN_BYTES = {"bf16": 2, "fp16": 2, "fp32": 4}
OUT_BYTES = {"bf16": 2, "fp16": 2, "fp32": 4}


def ceil_div(a: int, b: int) -> int:
    """ceil(a/b) for a >= 0, b > 0 (R14: every division in the model is a ceiling)."""
    assert a >= 0 and b > 0
    return -((-a) // b)


# ----------------------------------------------------------------------------------------
# Eqs. 2-4, literally
# ----------------------------------------------------------------------------------------

def t_load(nbytes: int, bw_milli: int) -> int:
    """T_Load / T_Store: "amount of data moved at the current layer divided by the memory
    bandwidth at that layer".  bw is bytes/cycle scaled by 1000 (R14)."""
    return ceil_div(nbytes * 1000, bw_milli)


def temporal_cost(t_ld: int, trips: int, inner: int, t_st: int) -> int:
    """Eq. 2: T_Load + (trips-1)*max(T_Load, Cost_{L-1}) + Cost_{L-1} + T_Store."""
    assert trips >= 1
    return t_ld + (trips - 1) * max(t_ld, inner) + inner + t_st


def parallel_factor(extent: int, units: int) -> int:
    """Eq. 3: ceil(sizeof(ParallelLoop) / |HardwareUnit|)."""
    assert extent >= 1 and units >= 1
    return ceil_div(extent, units)


def level_cost(f_parallel: int, t_temporal: int) -> int:
    """Eq. 4: Cost_L = F_parallel x T_temporal."""
    return f_parallel * t_temporal


# ----------------------------------------------------------------------------------------
# Alg. 2 building blocks
# ----------------------------------------------------------------------------------------

def filter_by_isa(cands, is_compatible):
    """FilterByISA: keep the candidates the base instruction accepts."""
    return [c for c in cands if is_compatible(c)]


def filter_by_multiples(cands, prev_cands, divides):
    """FilterByMultiples.

    for prev in prevCands: for multiple in GenerateMultiples(prev, cands):
        filtered.add(multiple); map[multiple].append(prev)
    GenerateMultiples(prev, cands) = the members of the current layer's candidate range
    that are integer multiples of prev (R4).  Returns (filtered, map) with
    filtered in the order of first insertion and map[c] listing prevs in prevCands order.
    """
    filtered = []
    seen = set()
    cmap = {}
    for prev in prev_cands:
        multiples = [c for c in cands if divides(prev, c)]
        for m in multiples:
            if m not in seen:
                seen.add(m)
                filtered.append(m)
            cmap.setdefault(m, []).append(prev)
    return filtered, cmap


# ----------------------------------------------------------------------------------------
# Hardware information (GetHardwareInfo) and calibration data
# ----------------------------------------------------------------------------------------

def load_descriptor(path: str | None = None) -> dict:
    path = path or os.path.join(os.path.dirname(_HERE), "tests", "golden", "b200_desc.json")
    with open(path) as f:
        return json.load(f)


def load_calib(path: str | None = None) -> dict:
    path = path or os.path.join(_HERE, "calib_b200.json")
    with open(path) as f:
        return json.load(f)


# ----------------------------------------------------------------------------------------
# The strategy table ("vx_plan"), sample-free: depends on (K, dtypes, descriptor) only
# ----------------------------------------------------------------------------------------

UMMA_M_LATTICE = (64, 128, 256)                 # R1
N_LATTICE = (8, 16, 32, 64, 128, 192, 256)       # R1
UMMA_K = 16                                      # kind::f16: K = 32 bytes / 2-byte element
BK_TC = 64                                       # one 128-B swizzle row of 2-byte elements
SPLITS = (1, 2, 4, 8)                            # R7
MAX_STAGES = 16                                  # R5
SMEM_RESERVE = 2048                              # barriers + 1024-B alignment slack
EPI_STAGING = 32768                              # epilogue: 8 warps x 4 KB TMA-store tiles
EPI_STAGING_LEAN = 16384                         # occupancy-2 (lean) CTAs: 4 warps x 4 KB
CTA_SYS_SMEM = 1024                              # shared memory reserved per resident CTA
CLUSTER_MAX = 8                                  # portable cluster size

# kernels that exist in the library (the "implemented" filter, R6):
#   family 0: tcgen05, A-tile on the UMMA-M axis: cta_group::1 BM=128, BN in {64,128,192,256};
#             cta_group::2 pairs BM=256, BN in {64 (B stored N x K only),128,256}
#   family 1: same kernel with A/B swapped (N on UMMA-M, M on UMMA-N; BN in
#             {16,32,64,128,192,256})
#   family 2: fp32 SIMT FFMA (BM, BN, TM, TN) in {(32,32,2,4),(64,64,4,4),(128,64,8,4)}
IMPL_TC = {(0, 128, 64), (0, 128, 128), (0, 128, 192), (0, 128, 256), (0, 256, 64), (0, 256, 128),
           (0, 256, 256), (1, 128, 16), (1, 128, 32), (1, 128, 64), (1, 128, 128),
           (1, 128, 192), (1, 128, 256)}
# TMA-multicast cluster kernels: (family, bm, bn, mc), mc CTAs sharing the A tile
IMPL_MC = {(0, 128, 128, 2), (0, 128, 256, 2), (1, 128, 32, 2), (1, 128, 64, 2), (1, 128, 64, 4)}
# occupancy-2 (lean) kernels: (family, bm, bn), two CTAs per SM (R5b) -- none instantiated
# (measured slower); the L2 candidates remain in the level counts
IMPL_LEAN = set()
MC_SIZES = (1, 2, 4)
SIMT_TILES = ((32, 32, 2, 4), (64, 64, 4, 4), (128, 64, 8, 4))
SIMT_BK = 16
FAMILY_NAMES = {0: "umma", 1: "umma_swap", 2: "simt", 3: "gemv"}
GEMV_MT = (1, 2, 4, 8)         # adaptive backend (R20): CUDA-core rungs for M <= MT
GEMV_COLS = 8                  # 2 column groups x 4 columns per CTA (x 4 K-slice warps)
GEMV_BK = 1024                 # k per CTA step (4 K slices x 256)
GEMV_OCC = 4                   # resident CTAs per SM assumed by the cost model


def isa_compatible_f16(c) -> bool:
    """tcgen05.mma.kind::f16 shapes (PTX ISA): M=64 -> N%8==0, 8..256; M=128 -> N%16==0,
    16..256 (cta_group::1); M=256 -> cta_group::2, N%16==0, 16..256.  K = 16."""
    um, un, uk = c
    if uk != UMMA_K:
        return False
    if um == 64:
        return un % 8 == 0 and 8 <= un <= 256
    if um in (128, 256):
        return un % 16 == 0 and 16 <= un <= 256
    return False


def build_table(K: int, in_dtype: str, out_dtype: str, desc: dict, b_layout: str = "nk") -> dict:
    """Alg. 2 bottom-up over the sm_100a levels; returns {'levels': counts, 'rungs': [...]}.

    L0 instruction tile, L1 TMEM accumulator tile, L2 CTA/SMEM tile, L3 grid schedule.
    """
    in_b = IN_BYTES[in_dtype]
    rungs = []
    counts = {}
    if in_dtype in ("bf16", "fp16"):
        # ---- L0: InitCands (lattice) -> FilterByISA ---------------------------------
        l0_init = [(um, un, UMMA_K) for um in UMMA_M_LATTICE for un in N_LATTICE]
        l0 = filter_by_isa(l0_init, isa_compatible_f16)
        # ---- L1: TMEM accumulator (AM lanes x AN fp32 columns x acc_stages) -----------
        # InitCands: capacity = TMEM columns (R2: window not applied to TMEM)
        l1_init = [(am, an, st) for am in UMMA_M_LATTICE for an in N_LATTICE for st in (1, 2)
                   if st * an <= desc["tmem_cols"]]
        l1, map1 = filter_by_multiples(
            l1_init, l0, lambda p, c: c[0] == p[0] and c[1] % p[1] == 0)
        # ---- L2: CTA tile (BM x BN x BK, S stages) in shared memory ------------------
        cap = desc["smem_optin"]
        l2_init = []
        for (am, an, st) in l1:
            cg = 2 if am == 256 else 1
            bm_cta, bn_cta = am // cg, an // cg
            stage_bytes = (bm_cta + bn_cta) * BK_TC * in_b
            s_fit = (cap - SMEM_RESERVE - EPI_STAGING) // stage_bytes
            S = min(MAX_STAGES, s_fit)
            if S < 2:
                continue
            foot = S * stage_bytes + SMEM_RESERVE + EPI_STAGING
            if foot * 8 < cap:            # utilisation window [1/8, 1] (R3)
                continue
            l2_init.append((am, an, BK_TC, S, st, 1))
            # occupancy-2 ring (R5b): two CTAs per SM -- half the SM's shared memory each
            # (less the per-CTA system reserve) and half its TMEM columns
            if cg == 1 and 2 * st * an <= desc["tmem_cols"]:
                fit2 = (desc["smem_per_sm"] // 2 - CTA_SYS_SMEM - SMEM_RESERVE
                        - EPI_STAGING_LEAN) // stage_bytes
                S2 = min(MAX_STAGES, fit2)
                foot2 = S2 * stage_bytes + SMEM_RESERVE + EPI_STAGING_LEAN
                if 2 <= S2 < S and foot2 * 8 >= cap:
                    l2_init.append((am, an, BK_TC, S2, st, 2))
        l2, map2 = filter_by_multiples(
            l2_init, l1,
            lambda p, c: c[0] % p[0] == 0 and c[1] % p[1] == 0 and c[4] == p[2]
            and c[2] % UMMA_K == 0)
        # ---- L3: grid schedule (swap, splits) + implemented filter -------------------
        kb = ceil_div(K, BK_TC)
        for (bm, bn, bk, S, st, occ) in l2:
            cg = 2 if bm == 256 else 1
            for swap in (0, 1):
                if cg == 2 and swap:      # cta_group::2 pair rungs are non-swapped
                    continue
                # a pair CTA with < 64 B rows needs K-major B: the MN-major 128-B swizzle
                # atom (B stored K x N) is 64 elements wide
                if cg == 2 and bn // 2 < 64 and b_layout != "nk":
                    continue
                stage_bytes = (bm // cg + bn // cg) * bk * in_b
                for mc in MC_SIZES:
                    # L3 multicast cluster of mc CTAs sharing the A tile: implemented kernel,
                    # whole 8-row swizzle atoms per CTA share, unpacked B
                    if st != 2:
                        continue
                    if occ == 2 and (mc > 1 or (swap, bm, bn) not in IMPL_LEAN):
                        continue
                    if occ == 1 and mc == 1 and (swap, bm, bn) not in IMPL_TC:
                        continue
                    if mc > 1 and ((swap, bm, bn, mc) not in IMPL_MC or cg > 1
                                   or (bn if swap else bm) // mc % 8 != 0
                                   or b_layout == "packed"):
                        continue
                    if mc > 1 or occ == 2:
                        splits = [1]      # multicast clusters and lean CTAs are persistent
                    else:
                        splits = []
                        for s in SPLITS:
                            if kb % s != 0 or s * cg > CLUSTER_MAX:
                                continue
                            if s > 1 and (cg > 1 or bm * (bn + 4) * 4 > S * stage_bytes):
                                continue
                            splits.append(s)
                        splits.append(0)  # stream-K schedule over (tile, k-block) units (R19)
                    rungs.append({"family": swap, "cg": cg, "um": bm, "un": bn, "acc_stages": st,
                                  "bm": bm, "bn": bn, "bk": bk, "stages": S, "swap": swap,
                                  "mc": mc, "occ": occ, "splits": splits})
        # adaptive backend (R20): CUDA-core rungs join the same argmin
        if b_layout != "packed":
            for mt in GEMV_MT:
                rungs.append({"family": 3, "cg": 1, "um": 1, "un": 1, "acc_stages": 1,
                              "bm": mt, "bn": GEMV_COLS, "bk": GEMV_BK, "stages": 1, "swap": 0,
                              "mc": 1, "occ": 1, "splits": [1]})
        counts = {"l0": len(l0), "l1": len(l1), "l2": len(l2), "l3": len(rungs)}
    elif in_dtype == "fp32":
        # CUDA-core mode: L0 = FFMA thread tiles, L2 = CTA tiles
        l0 = [(tm, tn) for (_, _, tm, tn) in SIMT_TILES]
        l0 = sorted(set(l0))
        l2_init = []
        for (bm, bn, tm, tn) in SIMT_TILES:
            threads = (bm // tm) * (bn // tn)
            if threads > desc["max_threads_per_block"]:
                continue
            l2_init.append((bm, bn, SIMT_BK, tm, tn))
        l2, _ = filter_by_multiples(l2_init, l0,
                                    lambda p, c: c[3] == p[0] and c[4] == p[1]
                                    and c[0] % p[0] == 0 and c[1] % p[1] == 0)
        for (bm, bn, bk, tm, tn) in l2:
            rungs.append({"family": 2, "cg": 1, "um": tm, "un": tn, "acc_stages": 1,
                          "bm": bm, "bn": bn, "bk": bk, "stages": 2, "swap": 0,
                          "mc": 1, "occ": 1, "splits": [1]})
        counts = {"l0": len(l0), "l1": len(l0), "l2": len(l2), "l3": len(rungs)}
    else:
        raise ValueError(in_dtype)
    # deterministic rung ids (R13): lexicographic on (family, bm, bn, stages, swap, mc)
    rungs.sort(key=lambda r: (r["family"], r["bm"], r["bn"], r["stages"], r["swap"], r["mc"],
                              r["occ"]))
    for i, r in enumerate(rungs):
        r["rung_id"] = i
    return {"K": K, "in": in_dtype, "out": out_dtype, "levels": counts, "rungs": rungs}


# ----------------------------------------------------------------------------------------
# Runtime cost and selection ("vx_plan_select")
# ----------------------------------------------------------------------------------------

def _calib_key(rung: dict) -> str:
    """Calibration-table key of a rung: family, TMA-multicast cluster size, tile."""
    fam = FAMILY_NAMES[rung["family"]]
    if rung.get("occ", 1) == 2:
        return "%s_o2_%dx%d" % (fam, rung["bm"], rung["bn"])
    if rung.get("mc", 1) > 1:
        return "%s_mc%d_%dx%d" % (fam, rung["mc"], rung["bm"], rung["bn"])
    return "%s_%dx%d" % (fam, rung["bm"], rung["bn"])


def _calib_for(rung: dict, calib: dict) -> dict:
    return calib["rungs"][_calib_key(rung)]


def simt_slots(rung: dict, desc: dict) -> int:
    bm, bn, bk = rung["bm"], rung["bn"], rung["bk"]
    threads = (bm // rung["um"]) * (bn // rung["un"])
    foot = 2 * (bm + bn) * bk * 4 + SMEM_RESERVE
    occ = min(desc["smem_per_sm"] // foot, desc["max_threads_per_sm"] // threads, 32)
    return desc["sm_count"] * max(occ, 1)


def rung_cost(rung: dict, s: int, batch: int, M: int, N: int, K: int,
              in_dtype: str, out_dtype: str, desc: dict, calib: dict) -> dict:
    """Predicted cycles of (rung, split) for the runtime shape."""
    in_b, out_b = IN_BYTES[in_dtype], OUT_BYTES[out_dtype]
    cal = _calib_for(rung, calib)
    hbm = calib["hbm_milli"]
    bm, bn, bk = rung["bm"], rung["bn"], rung["bk"]
    if rung["family"] == 3:
        return _gemv_cost(rung, batch, M, N, K, in_b, out_b, desc, calib, cal)
    # padding only at the outermost (grid) level (Fig. padding)
    mt, nt = (N, M) if rung["swap"] else (M, N)
    tm, tn = ceil_div(mt, bm), ceil_div(nt, bn)
    tiles = batch * tm * tn
    kb = ceil_div(K, bk)
    if s == 0:
        return _streamk_cost(rung, batch, M, N, K, mt, nt, tm, tn, tiles, kb, in_b, out_b,
                             desc, calib, cal)
    trips = kb // s                                   # sizeof(TemporalLoop) at CTA level (R8)
    # a multicast cluster covers mc consecutive tiles along the axis that does
    # not share the A tile; the tile count is padded to whole clusters
    mc = rung.get("mc", 1)
    tm_c = ceil_div(tm, mc) * mc if (mc > 1 and rung["swap"]) else tm
    tn_c = ceil_div(tn, mc) * mc if (mc > 1 and not rung["swap"]) else tn
    W = batch * tm_c * tn_c * s * rung["cg"]          # sizeof(ParallelLoop) in CTAs
    if rung["family"] == 2:
        slots = simt_slots(rung, desc)
    else:
        csz = s * rung["cg"] * mc                     # CTAs per cluster
        slots = desc["max_active_clusters"][str(csz)] * csz
    F = parallel_factor(W, slots)                     # Eq. 3 (|HardwareUnit| = slots, R9)
    active = min(W, slots)
    if rung["family"] == 2:
        occ = ceil_div(active, desc["sm_count"])      # CTAs sharing one SM
        inner = t_load(bm * bn * bk * occ, cal["mac_milli"])
        l_smem = t_load((bm + bn) * bk * in_b * occ, cal["l2s_milli"])
    else:
        inner = t_load(bm * bn * bk, cal["mac_milli"])          # Cost_{L-1}, empirical tier
        # rows past M / N are zero-filled by TMA without memory traffic (R10); in a multicast
        # cluster each CTA loads 1/mc of the shared A tile (mc_A)
        p_rows = bm // mc if (mc > 1 and not rung["swap"]) else min(bm, mt)
        q_rows = bn // mc if (mc > 1 and rung["swap"]) else min(bn, nt)
        l_smem = t_load((p_rows + q_rows) * bk * in_b, cal["l2s_milli"])
    # HBM share of one k-step: the grid's unique operand bytes leave HBM once, spread over
    # F waves x trips k-steps that all run at the chip bandwidth (R10)
    uniq = in_b * batch * K * (mt + nt)
    l_hbm = t_load(uniq, F * trips * hbm)
    tl = max(l_smem, l_hbm)                           # T_Load
    cbytes = out_b * batch * M * N                    # true C bytes (clipped tail rows)
    st_epi = t_load(bm * bn * out_b, s * cal["epi_milli"])
    st_hbm = t_load(cbytes, F * hbm)
    ts = max(st_epi, st_hbm)                          # T_Store
    if s > 1:
        ts += t_load((s - 1) * bm * bn * 4, s * calib["dsm_milli"])
    T = temporal_cost(tl, trips, inner, ts)           # Eq. 2
    if s == 1 and rung["family"] != 2:
        # persistent CTA, double-buffered TMEM accumulator (R11): the grid-level PL loop
        # becomes a temporal loop of F tiles whose "load" is the mainloop and whose
        # "compute" is the epilogue -> Eq. 2 again at the grid level.
        tmain = T - ts
        cost = temporal_cost(tmain, F, ts, 0) + cal["fixed"]
    else:
        cost = level_cost(F, T) + cal["fixed"] + (calib["fixed_cluster"] if s > 1 else 0)
    # R21: back to back, a first wave of more than half the SMs cannot become resident
    # while the previous grid (one full-SMEM CTA per SM) still holds its SMs
    if rung["family"] != 2 and min(W, slots) > desc["sm_count"] // 2:
        cost += calib["stagger"]
    return {"cost": cost, "tiles_m": tm, "tiles_n": tn, "tiles": tiles, "F": F,
            "grid": W if s > 1 or rung["family"] == 2 else min(W, slots),
            "padded_work": batch * tm_c * bm * tn_c * bn}


def _gemv_cost(rung, batch, M, N, K, in_b, out_b, desc, calib, cal):
    """CUDA-core GEMV rung (R20): a CTA holds MT rows x 8 columns and walks K in steps of
    1024; GEMV_OCC CTAs per SM; Eqs. 2-4 as for the other rungs."""
    bm, bn, bk = rung["bm"], rung["bn"], rung["bk"]
    hbm = calib["hbm_milli"]
    tiles = batch * ceil_div(N, bn)
    F = parallel_factor(tiles, desc["sm_count"] * GEMV_OCC)        # Eq. 3
    trips = ceil_div(K, bk)
    inner = t_load(bm * bn * bk, cal["mac_milli"])
    l_smem = t_load(bn * bk * in_b + bm * bk * in_b, cal["l2s_milli"])
    l_hbm = t_load(in_b * batch * K * (N + M), F * trips * hbm)
    tl = max(l_smem, l_hbm)
    ts = max(t_load(bm * bn * out_b, cal["epi_milli"]), t_load(out_b * batch * M * N, F * hbm))
    cost = level_cost(F, temporal_cost(tl, trips, inner, ts)) + cal["fixed"]   # Eqs. 2, 4
    return {"cost": cost, "tiles_m": 1, "tiles_n": ceil_div(N, bn), "tiles": tiles, "F": F,
            "grid": tiles, "padded_work": batch * bm * ceil_div(N, bn) * bn}


def _streamk_cost(rung, batch, M, N, K, mt, nt, tm, tn, tiles, kb, in_b, out_b, desc, calib,
                  cal):
    """Stream-K schedule (R19): G = min(resident CTAs, U) CTAs share the U = tiles x k-blocks
    work units evenly in one wave (Eq. 3 gives F = 1); each CTA's temporal loop is
    ceil(U/G) k-blocks (Eq. 2) touching at most ceil(units/kb)+1 tile segments, whose
    epilogues overlap the loop except the last; a cut tile is completed by adding
    ceil(kb/units) partials, each one fp32 tile (per CTA: its bm/cg rows) written and read
    back."""
    bm, bn, bk = rung["bm"], rung["bn"], rung["bk"]
    hbm = calib["hbm_milli"]
    U = tiles * kb
    cg = rung["cg"]                                  # units go to CTAs, or to CTA pairs
    G = min(desc["max_active_clusters"][str(cg)], U)
    units = ceil_div(U, G)
    segs = ceil_div(units, kb) + 1
    inner = t_load(bm * bn * bk, cal["mac_milli"])
    l_smem = t_load((min(bm, mt) + min(bn, nt)) * bk * in_b, cal["l2s_milli"])
    l_hbm = t_load(in_b * batch * K * (mt + nt), units * hbm)
    tl = max(l_smem, l_hbm)
    t_main = temporal_cost(tl, units, inner, 0)
    st = max(t_load(bm * bn * out_b, cal["epi_milli"]), t_load(out_b * batch * M * N, segs * hbm))
    # each CTA finishes its own rows of a cut tile: a pair's CTAs each write and read back
    # their (bm / cg) x bn fp32 half, in parallel (R19)
    fix = ceil_div(kb, units) * t_load(2 * (bm // cg) * bn * 4, calib["skfix_milli"])
    cost = max(t_main, segs * st) + st + fix + cal["fixed"]
    if G * cg > desc["sm_count"] // 2:               # R21 (see rung_cost)
        cost += calib["stagger"]
    return {"cost": cost, "tiles_m": tm, "tiles_n": tn, "tiles": tiles, "F": 1, "grid": G * cg,
            "padded_work": batch * tm * bm * tn * bn}


def varlen_cost(rung: dict, lens, K: int, in_dtype: str, out_dtype: str, desc: dict,
                calib: dict) -> dict:
    """Ragged attention batch: S_g = Q_g K_g^T for sequence lengths `lens`.
    Eqs. 2-4 over the ragged tile set: W = sum_g ceil(s_g/BM) ceil(s_g/BN) (padding only at
    each sequence's edge), unique operand bytes in_b K 2 sum_g s_g, output bytes out_b
    sum_g s_g^2, the persistent grid-level Eq. 2 (R11) and the stagger (R21)."""
    in_b, out_b = IN_BYTES[in_dtype], OUT_BYTES[out_dtype]
    cal = _calib_for(rung, calib)
    hbm = calib["hbm_milli"]
    bm, bn, bk = rung["bm"], rung["bn"], rung["bk"]
    tiles = sum(ceil_div(s, bm) * ceil_div(s, bn) for s in lens)
    rows = sum(lens)
    outs = sum(s * s for s in lens)
    padded = sum(ceil_div(s, bm) * bm * ceil_div(s, bn) * bn for s in lens)
    kb = ceil_div(K, bk)
    slots = desc["max_active_clusters"]["1"]
    W = max(tiles, 1)
    F = parallel_factor(W, slots)
    inner = t_load(bm * bn * bk, cal["mac_milli"])
    l_smem = t_load((bm + bn) * bk * in_b, cal["l2s_milli"])
    l_hbm = t_load(in_b * K * 2 * rows, F * kb * hbm)
    tl = max(l_smem, l_hbm)
    ts = max(t_load(bm * bn * out_b, cal["epi_milli"]), t_load(out_b * outs, F * hbm))
    T = temporal_cost(tl, kb, inner, ts)
    cost = temporal_cost(T - ts, F, ts, 0) + cal["fixed"]
    if min(W, slots) > desc["sm_count"] // 2:
        cost += calib["stagger"]
    return {"cost": cost, "tiles": tiles, "grid": min(W, slots), "padded_work": padded, "F": F}


def select_varlen(table: dict, lens, K: int, desc: dict, calib: dict) -> dict:
    """Eq. 1 over the non-swapped cta_group::1 persistent tcgen05 rungs for a ragged batch;
    key (cost, padded_work, rung_id)."""
    best = None
    for r in table["rungs"]:
        if r["family"] != 0 or r["cg"] != 1 or r["mc"] != 1 or r["occ"] != 1:
            continue
        c = varlen_cost(r, lens, K, table["in"], table["out"], desc, calib)
        key = (c["cost"], c["padded_work"], r["rung_id"])
        if best is None or key < best[0]:
            best = (key, r, c)
    key, r, c = best
    return {"rung_id": r["rung_id"], "split": 1, "grid": c["grid"], "cost": c["cost"],
            "bm": r["bm"], "bn": r["bn"]}


SK_MAX_WAVES = 3


def streamk_admissible(rung: dict, batch: int, M: int, N: int, K: int, desc: dict) -> bool:
    """R19: stream-K competes only where the rung's data-parallel schedule needs at most
    SK_MAX_WAVES waves, i.e. where wave quantization is what it removes, and where every
    CTA's share of the units is at least half a tile's K loop (2 * ceil(U/G) >= k-blocks),
    so a cut tile gathers partials from at most a few CTAs."""
    mt, nt = (N, M) if rung["swap"] else (M, N)
    tiles = batch * ceil_div(mt, rung["bm"]) * ceil_div(nt, rung["bn"])
    cg = rung["cg"]
    slots = desc["max_active_clusters"][str(cg)] * cg
    kb = ceil_div(K, rung["bk"])
    U = tiles * kb
    G = min(desc["max_active_clusters"][str(cg)], U)
    return tiles * cg <= SK_MAX_WAVES * slots and 2 * ceil_div(U, G) >= kb


def select(table: dict, batch: int, M: int, N: int, K: int, desc: dict, calib: dict) -> dict:
    """Eq. 1 argmin over (rung, split); key (cost, padded_work, rung_id, split) (R13)."""
    assert M >= 1 and N >= 1 and batch >= 1
    best = None
    for r in table["rungs"]:
        for s in r["splits"]:
            if s == 0 and not streamk_admissible(r, batch, M, N, K, desc):
                continue
            if r["family"] == 3 and M > r["bm"]:      # GEMV rungs hold M <= MT rows (R20)
                continue
            c = rung_cost(r, s, batch, M, N, K, table["in"], table["out"], desc, calib)
            key = (c["cost"], c["padded_work"], r["rung_id"], s)
            if best is None or key < best[0]:
                best = (key, r, s, c)
    key, r, s, c = best
    return {"rung_id": r["rung_id"], "split": s, "tiles_m": c["tiles_m"],
            "tiles_n": c["tiles_n"], "grid": c["grid"], "cost": c["cost"],
            "swap": r["swap"], "bm": r["bm"], "bn": r["bn"], "mc": r.get("mc", 1)}
