"""Pins for oracle/selector_ref.py (strategy table + cost-model argmin) -- CPU only.

Checked against: SPEC.md's worked arithmetic for Eqs. 2-3 and Alg. 2 (tests/golden/
spec_cost_vectors.json), brute-force divisibility / exhaustive argmin, the PTX ISA's
published tcgen05 kind::f16 shape table, and invariants the method guarantees (wave
staircase, padding confined to the outermost level, sample-freedom / determinism).
"""
import json
import os
import random

import pytest

from oracle import selector_ref as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")
VEC = json.load(open(os.path.join(GOLD, "spec_cost_vectors.json")))
DESC = S.load_descriptor()
CAL = S.load_calib()


def test_eq2_worked_examples():
    for tl, trips, inner, ts, want in VEC["temporal_cost"]:
        assert S.temporal_cost(tl, trips, inner, ts) == want


def test_eq3_worked_examples_and_staircase():
    for ext, units, want in VEC["parallel_factor"]:
        assert S.parallel_factor(ext, units) == want
    for k in range(1, 9):  # F(k*units) = k, F(k*units+1) = k+1
        assert S.parallel_factor(k * 148, 148) == k
        assert S.parallel_factor(k * 148 + 1, 148) == k + 1


def test_eq4_product():
    assert S.level_cost(3, 53) == 159
    assert S.level_cost(1, 23) == 23


def test_t_load_worked_examples():
    for nbytes, bw, want in VEC["t_load"]:
        assert S.t_load(nbytes, bw * 1000) == want   # bandwidth scaled x1000 (R14)


def test_sieve_worked_example():
    sv = VEC["sieve"]
    lo, hi = sv["range"]
    cands = list(range(lo, hi + 1))
    filt, cmap = S.filter_by_multiples(cands, sv["prev"], lambda p, c: c % p == 0)
    assert sorted(filt) == sv["filtered"]
    for k, v in sv["map"].items():
        assert cmap[int(k)] == v


def test_isa_worked_example():
    iv = VEC["isa"]
    mult = iv["multiples"]
    keep = S.filter_by_isa([tuple(c) for c in iv["cands"]],
                           lambda c: all(x % m == 0 for x, m in zip(c, mult)))
    assert [list(c) for c in keep] == iv["kept"]


def test_sieve_matches_brute_force_random():
    rnd = random.Random(0)
    for _ in range(200):
        dim = rnd.choice([1, 2, 3])
        cands = list({tuple(rnd.randint(1, 64) for _ in range(dim)) for _ in range(rnd.randint(1, 60))})
        prev = list({tuple(rnd.randint(1, 16) for _ in range(dim)) for _ in range(rnd.randint(1, 6))})
        div = lambda p, c: all(ci % pi == 0 for pi, ci in zip(p, c))
        filt, cmap = S.filter_by_multiples(cands, prev, div)
        brute = [c for c in cands if any(div(p, c) for p in prev)]
        assert set(filt) == set(brute)
        for c in filt:                                   # map soundness + completeness
            assert cmap[c] == [p for p in prev if div(p, c)]


def test_tcgen05_f16_shape_table():
    # legal / illegal shapes from the PTX ISA table for .kind::f16 (K = 16)
    legal = [(64, 8, 16), (64, 24, 16), (64, 256, 16), (128, 16, 16), (128, 256, 16),
             (256, 16, 16), (256, 256, 16), (128, 208, 16)]
    illegal = [(128, 8, 16), (128, 24, 16), (64, 264, 16), (256, 8, 16), (32, 16, 16),
               (128, 16, 32), (128, 272, 16)]
    assert all(S.isa_compatible_f16(c) for c in legal)
    assert not any(S.isa_compatible_f16(c) for c in illegal)


@pytest.mark.parametrize("K", [64, 768, 4096, 2304, 128])
def test_table_invariants(K):
    t = S.build_table(K, "bf16", "bf16", DESC)
    assert t["rungs"], "empty strategy table"
    kb = S.ceil_div(K, S.BK_TC)
    for r in t["rungs"]:
        if r["family"] == 3:                             # CUDA-core GEMV rungs (R20)
            assert r["bm"] in S.GEMV_MT and r["splits"] == [1]
            continue
        # divisibility down the chain (padding confined to the outermost level, Fig. padding)
        assert r["bm"] % r["um"] == 0 and r["bn"] % r["un"] == 0 and r["bk"] % S.UMMA_K == 0
        assert S.isa_compatible_f16((r["um"], r["un"], S.UMMA_K))
        # resources: SMEM stages fit, TMEM accumulators fit
        cg = r["cg"]                                   # per-CTA footprint (pairs split tiles)
        foot = r["stages"] * (r["bm"] // cg + r["bn"] // cg) * r["bk"] * 2 + S.SMEM_RESERVE + S.EPI_STAGING
        assert foot <= DESC["smem_optin"] and r["stages"] >= 2
        assert r["acc_stages"] * r["bn"] <= DESC["tmem_cols"]
        # split-K slices are whole k-blocks; multicast clusters and
        # occupancy-2 (lean) CTAs are persistent
        if r["occ"] == 2:
            assert r["splits"] == [1] and r["cg"] == 1 and r["mc"] == 1
            foot = r["stages"] * (r["bm"] + r["bn"]) * r["bk"] * 2 + S.SMEM_RESERVE + S.EPI_STAGING_LEAN
            assert 2 * (foot + S.CTA_SYS_SMEM) <= DESC["smem_per_sm"]       # two CTAs per SM
            assert 2 * r["acc_stages"] * r["bn"] <= DESC["tmem_cols"]
            continue
        if r["mc"] > 1:
            assert r["splits"] == [1] and r["cg"] == 1
            assert (r["bn"] if r["swap"] else r["bm"]) // r["mc"] % 8 == 0   # whole swizzle atoms
            continue
        assert 1 in r["splits"] and 0 in r["splits"]         # 0 = stream-K (R19)
        assert all(s == 0 or kb % s == 0 for s in r["splits"])
    # sample-free and deterministic: a pure function of (K, dtypes, descriptor)
    assert S.build_table(K, "bf16", "bf16", DESC) == t
    assert [r["rung_id"] for r in t["rungs"]] == list(range(len(t["rungs"])))


def _brute_best(t, batch, M, N, K):
    allc = []
    for r in t["rungs"]:
        for s in r["splits"]:
            if s == 0 and not S.streamk_admissible(r, batch, M, N, K, DESC):   # R19
                continue
            if r["family"] == 3 and M > r["bm"]:                            # R20
                continue
            c = S.rung_cost(r, s, batch, M, N, K, t["in"], t["out"], DESC, CAL)
            allc.append((c["cost"], c["padded_work"], r["rung_id"], s))
    return min(allc)


@pytest.mark.parametrize("N,K", [(768, 768), (3072, 768), (11008, 4096), (4096, 4096)])
def test_select_is_argmin(N, K):
    t = S.build_table(K, "bf16", "bf16", DESC)
    for M in (1, 2, 16, 17, 64, 100, 128, 129, 511, 512, 1000, 4096, 16384):
        ch = S.select(t, 1, M, N, K, DESC, CAL)
        best = _brute_best(t, 1, M, N, K)
        assert (ch["cost"], ch["rung_id"], ch["split"]) == (best[0], best[2], best[3])
        # tile counts are the ceiling cover of the runtime shape (padding only at grid level)
        mt, nt = (N, M) if ch["swap"] else (M, N)
        assert ch["tiles_m"] == -(-mt // ch["bm"]) and ch["tiles_n"] == -(-nt // ch["bn"])


def test_zero_padding_on_tile_multiples():
    t = S.build_table(4096, "bf16", "bf16", DESC)
    for r in t["rungs"]:
        if r["family"] == 3:
            continue                                   # GEMV rungs cover M <= MT only
        c = S.rung_cost(r, 1, 1, 128 * 40, 256 * 43, 4096, "bf16", "bf16", DESC, CAL)
        mt, nt = (256 * 43, 128 * 40) if r["swap"] else (128 * 40, 256 * 43)
        # a multicast cluster also pads its non-shared tile count to a multiple of mc
        ct = (mt // r["bm"]) if r["swap"] else (nt // r["bn"])
        if mt % r["bm"] == 0 and nt % r["bn"] == 0 and ct % r["mc"] == 0:
            assert c["padded_work"] == mt * nt


def test_fp32_table_and_selection():
    t = S.build_table(64, "fp32", "fp32", DESC)
    assert all(r["family"] == 2 for r in t["rungs"])
    ch = S.select(t, 1, 37, 64, 64, DESC, CAL)
    assert ch["rung_id"] in range(len(t["rungs"]))


def test_cost_monotone_in_bytes_and_rates():
    # more work never predicted cheaper for a fixed (rung, split) below one wave
    t = S.build_table(4096, "bf16", "bf16", DESC)
    r = t["rungs"][0]
    c1 = S.rung_cost(r, 1, 1, 64, 4096, 4096, "bf16", "bf16", DESC, CAL)["cost"]
    c2 = S.rung_cost(r, 1, 1, 64, 4096, 8192, "bf16", "bf16", DESC, CAL)["cost"]
    assert c2 > c1
    cal2 = json.loads(json.dumps(CAL))
    for v in cal2["rungs"].values():
        v["mac_milli"] *= 2
    c3 = S.rung_cost(r, 1, 1, 8192, 4096, 4096, "bf16", "bf16", DESC, cal2)["cost"]
    c4 = S.rung_cost(r, 1, 1, 8192, 4096, 4096, "bf16", "bf16", DESC, CAL)["cost"]
    assert c3 <= c4


def test_streamk_only_for_few_waves():
    """R19: stream-K is never chosen when the rung's data-parallel grid needs > 3 waves."""
    t = S.build_table(4096, "bf16", "bf16", DESC)
    for M in (1, 64, 512, 1024, 4096, 16384, 65536):
        ch = S.select(t, 1, M, 11008, 4096, DESC, CAL)
        if ch["split"] == 0:
            r = t["rungs"][ch["rung_id"]]
            assert S.streamk_admissible(r, 1, M, 11008, 4096, DESC)
    big = [r for r in t["rungs"] if r["cg"] == 2 and r["family"] == 0 and r["bn"] == 256][0]
    assert not S.streamk_admissible(big, 1, 16384, 11008, 4096, DESC)
    assert S.streamk_admissible(big, 1, 512, 11008, 4096, DESC)
    # few k-blocks per CTA (BERT-size K, many small tiles): a tile would be cut over > 3 CTAs
    sw16 = [r for r in t["rungs"] if r["family"] == 1 and r["bm"] == 128 and r["bn"] == 16][0]
    assert not S.streamk_admissible(sw16, 1, 32, 2304, 768, DESC)
    assert S.streamk_admissible(sw16, 1, 4, 11008, 4096, DESC)
