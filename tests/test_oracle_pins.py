"""Value pins of the selector oracle (oracle/selector_ref.py) against hand-derived worked
examples (tests/golden/cost_vectors.json; every intermediate quantity is written out in
DESIGN.md 5.1), so that the oracle is pinned to something other than itself or the library:
a plausible slip in any of its functions (a dropped term, a wrong axis, an off-by-one in a
constant, a mis-ordered tie-break) fails a named test here.  tools/mutate_oracle.py applies
such mutations one at a time and checks that this suite catches each.

Pinned functions: rung_cost (persistent, swapped, multicast, split, pair), _streamk_cost
(via rung_cost, split 0), _gemv_cost (via rung_cost, family 3), simt_slots, build_table's
stage count S and its S >= 2 / window rule, streamk_admissible, select's key order.
"""
import json
import os

import pytest

import oracle.selector_ref as S

HERE = os.path.dirname(os.path.abspath(__file__))
CV = json.load(open(os.path.join(HERE, "golden", "cost_vectors.json")))
B200 = json.load(open(os.path.join(HERE, "golden", "b200_desc.json")))


def _rung(d):
    r = {"um": d["bm"], "un": d["bn"], "acc_stages": 2, "stages": 4, "splits": [1]}
    r.update(d)
    return r


@pytest.mark.parametrize("case", CV["rung_cost"], ids=[c["name"] for c in CV["rung_cost"]])
def test_rung_cost_worked_examples(case):
    cal = dict(CV["calib"], **case.get("calib_override", {}))
    c = S.rung_cost(_rung(case["rung"]), case["split"], case["batch"], case["M"], case["N"],
                    case["K"], "bf16", "bf16", CV["desc"], cal)
    for k, v in case["want"].items():
        assert c[k] == v, (case["name"], k, c[k], v)


def _desc(name):
    d = dict(B200)
    if name == "smem100k":
        d = dict(d, smem_per_sm=100000)
    return d


@pytest.mark.parametrize("case", CV["simt_slots"])
def test_simt_slots_worked_examples(case):
    bm, bn, tm, tn = case["tile"]
    r = {"bm": bm, "bn": bn, "um": tm, "un": tn, "bk": S.SIMT_BK}
    assert S.simt_slots(r, _desc(case["desc"])) == case["want"]


def _key(r):
    fam = "umma_swap" if r["swap"] else "umma"
    if r.get("occ", 1) == 2:
        return "%s_o2_%dx%d" % (fam, r["bm"], r["bn"])
    return "%s_%dx%d" % (fam, r["bm"], r["bn"])


def test_stage_counts_b200():
    """S = min(16, floor((smem_optin - 2048 - 32768) / stage_bytes)), stage_bytes =
    (BM/cg + BN/cg) * 64 * 2 (DESIGN.md 3.2 L2; worked in DESIGN.md 5.1)."""
    t = S.build_table(4096, "bf16", "bf16", B200)
    seen = {}
    for r in t["rungs"]:
        if r["family"] in (0, 1) and r["mc"] == 1:
            seen[_key(r)] = r["stages"]
    assert seen == CV["stages_b200"]


def test_stage_counts_small_smem_and_drop_rule():
    """With smem_optin = 100000 only 65184 B remain for the ring: tiles whose stage exceeds
    half of that get S < 2 and are dropped (R5)."""
    d = dict(B200, smem_optin=100000)
    t = S.build_table(4096, "bf16", "bf16", d)
    seen = {_key(r): r["stages"] for r in t["rungs"] if r["family"] in (0, 1) and r["mc"] == 1}
    want = CV["stages_smem100k"]
    for k, v in want.items():
        if k == "dropped":
            for gone in v:
                assert gone not in seen, gone
        else:
            assert seen[k] == v, (k, seen.get(k), v)


@pytest.mark.parametrize("case", CV["streamk_admissible"])
def test_streamk_admissible_worked_cases(case):
    r = dict(case["rung"], bk=64)
    assert S.streamk_admissible(r, 1, case["M"], case["N"], case["K"], B200) is case["want"]


def test_select_toy_tie_break_padded_work_before_rung_id():
    """SPEC.md:510 toy (extent 5, tiles {32, 16} at equal cost): Eq. 1's argmin with the
    key (cost, padded_work, rung_id, split) returns the tile with less padding (R13)."""
    toy = CV["select_toy"]
    table = {"in": "bf16", "out": "bf16", "rungs": toy["rungs"]}
    costs = [S.rung_cost(r, 1, 1, toy["M"], toy["N"], toy["K"], "bf16", "bf16", CV["desc"],
                         CV["calib"]) for r in toy["rungs"]]
    assert [c["cost"] for c in costs] == [toy["want"]["cost"]] * 2
    assert [c["padded_work"] for c in costs] == toy["want"]["padded_work"]
    ch = S.select(table, 1, toy["M"], toy["N"], toy["K"], CV["desc"], CV["calib"])
    assert ch["rung_id"] == toy["want"]["rung_id"] and ch["cost"] == toy["want"]["cost"]


def test_gemv_rungs_only_hold_m_up_to_mt():
    """R20: a GEMV rung with MT rows is never a candidate for M > MT (select skips it), even
    when its cost would be the minimum."""
    cal = json.loads(json.dumps(CV["calib"]))
    cal["rungs"]["gemv_4x8"]["fixed"] = 0
    cal["rungs"]["gemv_4x8"]["mac_milli"] = 10 ** 9
    g = {"rung_id": 0, "family": 3, "cg": 1, "um": 1, "un": 1, "acc_stages": 1, "bm": 4,
         "bn": 8, "bk": 1024, "stages": 1, "swap": 0, "mc": 1, "splits": [1]}
    t = {"rung_id": 1, "family": 1, "cg": 1, "um": 128, "un": 16, "acc_stages": 2, "bm": 128,
         "bn": 16, "bk": 64, "stages": 10, "swap": 1, "mc": 1, "splits": [1]}
    table = {"in": "bf16", "out": "bf16", "rungs": [g, t]}
    assert S.select(table, 1, 4, 1000, 3072, CV["desc"], cal)["rung_id"] == 0
    assert S.select(table, 1, 5, 1000, 3072, CV["desc"], cal)["rung_id"] == 1


@pytest.mark.parametrize("case", CV["varlen_cost"], ids=[c["name"] for c in CV["varlen_cost"]])
def test_varlen_cost_worked_examples(case):
    """Ragged attention batch: Eqs. 2-4 over the ragged tile set
    (DESIGN.md 5.1 V1)."""
    cal = dict(CV["calib"], **case.get("calib_override", {}))
    c = S.varlen_cost(_rung(case["rung"]), case["lens"], case["K"], "bf16", "bf16", CV["desc"], cal)
    for k, v in case["want"].items():
        assert c[k] == v, (case["name"], k, c[k], v)
