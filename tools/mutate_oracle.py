"""Mutation check of the selector oracle's pins.

Applies one plausible slip at a time to a copy of oracle/selector_ref.py -- a dropped term,
a wrong axis, an off-by-one, a reordered tie-break -- and runs the oracle's CPU pins
(tests/test_oracle_pins.py, tests/test_oracle_selector.py) against the mutant.  Every
mutation must be caught (some test fails); the table printed here is DESIGN.md 5.2.

    python tools/mutate_oracle.py [--only NAME]
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (function, name, old text, new text) -- each `old` must occur exactly once
MUTATIONS = [
    ("temporal_cost", "Eq. 2 counts trips instead of trips-1 overlapped steps",
     "return t_ld + (trips - 1) * max(t_ld, inner) + inner + t_st",
     "return t_ld + trips * max(t_ld, inner) + inner + t_st"),
    ("temporal_cost", "Eq. 2 drops T_Store",
     "return t_ld + (trips - 1) * max(t_ld, inner) + inner + t_st",
     "return t_ld + (trips - 1) * max(t_ld, inner) + inner"),
    ("parallel_factor", "Eq. 3 floor instead of ceiling",
     "    return ceil_div(extent, units)\n", "    return max(1, extent // units)\n"),
    ("t_load", "bytes/bandwidth without the x1000 scale",
     "return ceil_div(nbytes * 1000, bw_milli)", "return ceil_div(nbytes, bw_milli)"),
    ("filter_by_multiples", "map keeps only the first divisor",
     "            cmap.setdefault(m, []).append(prev)",
     "            cmap.setdefault(m, [prev])"),
    ("isa_compatible_f16", "UMMA M=128 accepts N % 8",
     "    if um in (128, 256):\n        return un % 16 == 0",
     "    if um in (128, 256):\n        return un % 8 == 0"),
    ("build_table", "pair stage bytes count the whole B tile per CTA",
     "            stage_bytes = (bm_cta + bn_cta) * BK_TC * in_b",
     "            stage_bytes = (bm_cta + an) * BK_TC * in_b"),
    ("build_table", "epilogue staging left out of the SMEM budget",
     "            s_fit = (cap - SMEM_RESERVE - EPI_STAGING) // stage_bytes",
     "            s_fit = (cap - SMEM_RESERVE) // stage_bytes"),
    ("build_table", "rings of one stage kept (S >= 1)",
     "            if S < 2:\n                continue", "            if S < 1:\n                continue"),
    ("rung_cost", "ParallelLoop extent drops cta_group (pairs)",
     "    W = batch * tm_c * tn_c * s * rung[\"cg\"]", "    W = batch * tm_c * tn_c * s"),
    ("rung_cost", "HBM unique bytes use M for both axes (Mt slip)",
     "    uniq = in_b * batch * K * (mt + nt)", "    uniq = in_b * batch * K * (M + M)"),
    ("rung_cost", "TMA zero-filled rows charged as traffic (min(bn, nt) -> bn)",
     "        q_rows = bn // mc if (mc > 1 and rung[\"swap\"]) else min(bn, nt)",
     "        q_rows = bn // mc if (mc > 1 and rung[\"swap\"]) else bn"),
    ("rung_cost", "split-K reduce moves s instead of s-1 partials",
     "        ts += t_load((s - 1) * bm * bn * 4, s * calib[\"dsm_milli\"])",
     "        ts += t_load(s * bm * bn * 4, s * calib[\"dsm_milli\"])"),
    ("rung_cost", "persistent rungs priced as F x T (no epilogue overlap, R11)",
     "        cost = temporal_cost(tmain, F, ts, 0) + cal[\"fixed\"]",
     "        cost = level_cost(F, T) + cal[\"fixed\"]"),
    ("rung_cost", "cluster surcharge dropped for split-K",
     "(calib[\"fixed_cluster\"] if s > 1 else 0)", "0"),
    ("rung_cost", "multicast cluster tail not padded",
     "    tn_c = ceil_div(tn, mc) * mc if (mc > 1 and not rung[\"swap\"]) else tn",
     "    tn_c = tn"),
    ("rung_cost", "multicast CTA charged the whole shared tile",
     "        p_rows = bm // mc if (mc > 1 and not rung[\"swap\"]) else min(bm, mt)",
     "        p_rows = min(bm, mt)"),
    ("rung_cost", "multicast clusters use the single-CTA residency",
     "        csz = s * rung[\"cg\"] * mc                     # CTAs per cluster",
     "        csz = s * rung[\"cg\"]                          # CTAs per cluster"),
    ("rung_cost", "stagger (R21) charged whatever the first-wave width",
     "    if rung[\"family\"] != 2 and min(W, slots) > desc[\"sm_count\"] // 2:",
     "    if rung[\"family\"] != 2:"),
    ("rung_cost", "stagger (R21) threshold at all SMs instead of half",
     "    if rung[\"family\"] != 2 and min(W, slots) > desc[\"sm_count\"] // 2:",
     "    if rung[\"family\"] != 2 and min(W, slots) > desc[\"sm_count\"]:"),
    ("_streamk_cost", "stream-K launches never charged the stagger (R21)",
     "    if G * cg > desc[\"sm_count\"] // 2:               # R21 (see rung_cost)",
     "    if False:"),
    ("_streamk_cost", "segment count without the +1 boundary segment",
     "    segs = ceil_div(units, kb) + 1", "    segs = ceil_div(units, kb)"),
    ("_streamk_cost", "fix-up partial count floored",
     "    fix = ceil_div(kb, units) * t_load", "    fix = (kb // units) * t_load"),
    ("_streamk_cost", "pairs share units per CTA instead of per pair",
     "# units go to CTAs, or to CTA pairs\n    G = min(desc[\"max_active_clusters\"][str(cg)], U)",
     "# units go to CTAs, or to CTA pairs\n    G = min(desc[\"max_active_clusters\"][\"1\"], U)"),
    ("varlen_cost", "ragged tiles from the total length (padding across sequences)",
     "    tiles = sum(ceil_div(s, bm) * ceil_div(s, bn) for s in lens)",
     "    tiles = ceil_div(sum(lens), bm) * ceil_div(max(lens), bn)"),
    ("varlen_cost", "ragged output bytes from the packed total squared",
     "    outs = sum(s * s for s in lens)", "    outs = sum(lens) ** 2"),
    ("varlen_cost", "ragged operands counted once instead of Q and K",
     "    l_hbm = t_load(in_b * K * 2 * rows, F * kb * hbm)",
     "    l_hbm = t_load(in_b * K * rows, F * kb * hbm)"),
    ("_gemv_cost", "GEMV residency 2 CTAs / SM instead of 4",
     "    F = parallel_factor(tiles, desc[\"sm_count\"] * GEMV_OCC)",
     "    F = parallel_factor(tiles, desc[\"sm_count\"] * 2)"),
    ("_gemv_cost", "GEMV HBM bytes omit A",
     "    l_hbm = t_load(in_b * batch * K * (N + M), F * trips * hbm)",
     "    l_hbm = t_load(in_b * batch * K * N, F * trips * hbm)"),
    ("simt_slots", "thread count from the whole tile, not the thread tile",
     "    threads = (bm // rung[\"um\"]) * (bn // rung[\"un\"])\n    foot",
     "    threads = bm * bn // 4\n    foot"),
    ("simt_slots", "SMEM footprint single-buffered",
     "    foot = 2 * (bm + bn) * bk * 4 + SMEM_RESERVE", "    foot = (bm + bn) * bk * 4 + SMEM_RESERVE"),
    ("streamk_admissible", "wave bound 2 instead of 3", "SK_MAX_WAVES = 3", "SK_MAX_WAVES = 2"),
    ("streamk_admissible", "half-tile rule dropped",
     "    return tiles * cg <= SK_MAX_WAVES * slots and 2 * ceil_div(U, G) >= kb",
     "    return tiles * cg <= SK_MAX_WAVES * slots"),
    ("select", "tie-break on rung_id before padded work",
     "            key = (c[\"cost\"], c[\"padded_work\"], r[\"rung_id\"], s)",
     "            key = (c[\"cost\"], r[\"rung_id\"], c[\"padded_work\"], s)"),
    ("select", "GEMV rungs offered for M > MT",
     "            if r[\"family\"] == 3 and M > r[\"bm\"]:      # GEMV rungs hold M <= MT rows (R20)\n                continue",
     "            pass"),
]


def run_one(tmp, src, mut):
    func, name, old, new = mut
    n = src.count(old)
    if n != 1:
        return "BAD-MUTATION(%d)" % n
    with open(os.path.join(tmp, "oracle", "selector_ref.py"), "w") as f:
        f.write(src.replace(old, new))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "tests/test_oracle_pins.py", "tests/test_oracle_selector.py"],
                       cwd=tmp, capture_output=True, text=True)
    if r.returncode == 0:
        return "SURVIVED"
    failed = [ln.split("::", 1)[1].split(" ")[0] for ln in r.stdout.splitlines()
              if ln.startswith("FAILED ")]
    return "caught by " + (failed[0] if failed else "(error)")


def main():
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    src = open(os.path.join(ROOT, "oracle", "selector_ref.py")).read()
    tmp = tempfile.mkdtemp(prefix="vx_mut_")
    try:
        for d in ("oracle", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__", "*.so"))
        survived = 0
        print("| function | mutation | result |\n|---|---|---|")
        for mut in MUTATIONS:
            if only and only not in mut[1]:
                continue
            res = run_one(tmp, src, mut)
            survived += not res.startswith("caught")
            print("| `%s` | %s | %s |" % (mut[0], mut[1], res), flush=True)
        print("\n%d mutations, %d not caught" % (len(MUTATIONS), survived))
        sys.exit(1 if survived else 0)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
