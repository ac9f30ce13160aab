"""Library strategy table + runtime selection vs the independent oracle (CPU only).

north_star: "GPU tile selection must match the CPU selector bit-exact for every M in
1..16384".  The library's selector is host code, so it is compared here on the captured
B200 descriptor (tests/golden/b200_desc.json) for every BASELINE (N, K), plus the
dynamic-N batched attention plan for every s in 1..2048.
"""
import json
import os

import pytest

import paper_2409_01075_b200 as vx
from oracle import selector_ref as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DESC_J = S.load_descriptor()
CAL = S.load_calib()
DESC = vx.DeviceDesc.from_json(DESC_J)

BASELINE_NK = [(768, 768), (2304, 768), (3072, 768), (4096, 4096), (11008, 4096),
               (12288, 4096)]
FIELDS = ("rung_id", "split", "tiles_m", "tiles_n", "grid", "cost")


def _oracle_table(K, i, o, bl="nk"):
    return S.build_table(K, i, o, DESC_J, bl)


def _lib_rungs(dump):
    keep = ("rung_id", "family", "cg", "um", "un", "acc_stages", "bm", "bn", "bk", "stages",
            "swap", "mc", "occ", "splits")
    return [{k: r[k] for k in keep} for r in dump["rungs"]]


@pytest.mark.parametrize("K", [768, 4096, 64, 128, 2304])
@pytest.mark.parametrize("io", [("bf16", "bf16"), ("fp16", "fp32"), ("fp32", "fp32")])
def test_tables_identical(K, io):
    p = vx.Plan(0, K, io[0], io[1], "nk", desc=DESC)
    d = p.dump()
    t = _oracle_table(K, io[0], io[1])
    assert d["levels"] == t["levels"]
    want = [{k: r[k] for k in ("rung_id", "family", "cg", "um", "un", "acc_stages", "bm", "bn",
                               "bk", "stages", "swap", "mc", "occ", "splits")} for r in t["rungs"]]
    assert _lib_rungs(d) == want


def test_calibration_copies_agree():
    d = vx.Plan(4096, 4096, "bf16", "bf16", "nk", desc=DESC).dump()
    assert d["calib"] == {k: CAL[k] for k in ("hbm_milli", "dsm_milli", "fixed_cluster",
                                              "skfix_milli", "stagger")}
    for r in d["rungs"]:
        key = S._calib_key(r)
        for f in ("mac_milli", "l2s_milli", "epi_milli", "fixed"):
            assert r[f] == CAL["rungs"][key][f], (key, f)
    d = vx.Plan(64, 64, "fp32", "fp32", "nk", desc=DESC).dump()
    for r in d["rungs"]:
        key = "simt_%dx%d" % (r["bm"], r["bn"])
        for f in ("mac_milli", "l2s_milli", "epi_milli", "fixed"):
            assert r[f] == CAL["rungs"][key][f], (key, f)


@pytest.mark.parametrize("N,K", BASELINE_NK)
def test_select_every_M_bit_exact(N, K):
    p = vx.Plan(N, K, "bf16", "bf16", "nk", desc=DESC)
    t = _oracle_table(K, "bf16", "bf16")
    for M in range(1, 16385):
        a = p.select(M)
        b = S.select(t, 1, M, N, K, DESC_J, CAL)
        if tuple(a[f] for f in FIELDS) != tuple(b[f] for f in FIELDS):
            pytest.fail("M=%d lib=%s oracle=%s" % (M, a, b))


@pytest.mark.parametrize("d", [64, 128])
def test_select_batched_attention_every_s(d):
    p = vx.Plan(0, d, "bf16", "bf16", "nk", desc=DESC)
    t = _oracle_table(d, "bf16", "bf16")
    for s in range(1, 2049):
        a = p.select(s, N=s, batch=32)
        b = S.select(t, 32, s, s, d, DESC_J, CAL)
        assert tuple(a[f] for f in FIELDS) == tuple(b[f] for f in FIELDS), s


def test_select_fp32_and_large_M():
    p = vx.Plan(64, 64, "fp32", "fp32", "nk", desc=DESC)
    t = _oracle_table(64, "fp32", "fp32")
    for M in (1, 36, 37, 38, 1000, 65536):
        a = p.select(M)
        b = S.select(t, 1, M, 64, 64, DESC_J, CAL)
        assert tuple(a[f] for f in FIELDS) == tuple(b[f] for f in FIELDS)
    p = vx.Plan(11008, 4096, "bf16", "bf16", "nk", desc=DESC)
    t = _oracle_table(4096, "bf16", "bf16")
    for M in (16385, 32768, 65536, 65536 // 8, 65536 // 2, 100000):   # beyond the memo
        a = p.select(M)
        b = S.select(t, 1, M, 11008, 4096, DESC_J, CAL)
        assert tuple(a[f] for f in FIELDS) == tuple(b[f] for f in FIELDS)


def test_forced_cost_matches_oracle():
    p = vx.Plan(3072, 768, "bf16", "bf16", "nk", desc=DESC)
    t = _oracle_table(768, "bf16", "bf16")
    for r in t["rungs"]:
        for s in r["splits"]:
            for M in (1, 2, 5, 8, 77, 512, 4096):
                if r["family"] == 3 and M > r["bm"]:      # GEMV rung holds M <= MT (R20)
                    with pytest.raises(vx.VxError):
                        p.cost(r["rung_id"], s, M)
                    continue
                a = p.cost(r["rung_id"], s, M)
                b = S.rung_cost(r, s, 1, M, 3072, 768, "bf16", "bf16", DESC_J, CAL)
                assert a["cost"] == b["cost"] and a["grid"] == b["grid"]


def test_builtin_calibration_dump_matches_oracle_copy():
    """vx_calib_dump(NULL) is the compiled-in empirical tier; the oracle's JSON copy agrees."""
    d = vx.builtin_calib()
    assert d["source"] == "compiled-in"
    for k in ("hbm_milli", "dsm_milli", "fixed_cluster", "skfix_milli", "stagger"):
        assert d[k] == CAL[k]
    for key, r in CAL["rungs"].items():
        assert d["rungs"][key] == r, key


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_selection_parity_under_arbitrary_calibration(seed):
    """A calibration is data (the empirical tier, live or compiled in): for a randomly
    perturbed table handed to BOTH the library (vx_plan_ex_calibrated) and the oracle, the
    selections agree for every M of a dense sweep -- the selector is the same function of
    the calibration, not just of one table."""
    import random
    rnd = random.Random(seed)
    cal = json.loads(json.dumps(CAL))
    for k in ("dsm_milli", "fixed_cluster", "skfix_milli", "stagger"):
        cal[k] = max(1, int(cal[k] * rnd.uniform(0.5, 2.0)))
    for r in cal["rungs"].values():
        for f in ("mac_milli", "l2s_milli", "epi_milli", "fixed"):
            r[f] = max(1, int(r[f] * rnd.uniform(0.3, 3.0)))
    c = vx.Calib.from_dict(cal)
    for N, K in ((3072, 768), (11008, 4096)):
        p = vx.Plan(N, K, "bf16", "bf16", "nk", desc=DESC, calib=c)
        d = p.dump()
        assert d["calib"] == {k: cal[k] for k in ("hbm_milli", "dsm_milli", "fixed_cluster",
                                                  "skfix_milli", "stagger")}
        t = _oracle_table(K, "bf16", "bf16")
        for M in list(range(1, 600, 7)) + [1023, 1024, 4097, 16383]:
            got = p.select(M)
            want = S.select(t, 1, M, N, K, DESC_J, cal)
            assert {k: got[k] for k in FIELDS} == {k: want[k] for k in FIELDS}, (seed, N, K, M)


def test_calibration_missing_key_rejected():
    cal = json.loads(json.dumps(CAL))
    del cal["rungs"]["umma_128x128"]
    c = vx.Calib.from_dict(cal)
    with pytest.raises(vx.VxError) as e:
        vx.Plan(3072, 768, "bf16", "bf16", "nk", desc=DESC, calib=c)
    assert e.value.status == 2


@pytest.mark.parametrize("d", [64, 128])
def test_varlen_selection_matches_oracle(d):
    """vx_plan_select_varlen (ragged attention batch) is bit-identical to
    the oracle's select_varlen on random length mixes, single sequences and empty ones."""
    import random
    p = vx.Plan(0, d, "bf16", "bf16", "nk", desc=DESC)
    t = _oracle_table(d, "bf16", "bf16")
    rnd = random.Random(d)
    mixes = [[1], [2048], [0, 5, 0], [128, 128, 128]]
    mixes += [[rnd.randint(1, 2048) for _ in range(rnd.randint(1, 32))] for _ in range(40)]
    for lens in mixes:
        cu = [0]
        for s in lens:
            cu.append(cu[-1] + s)
        got = p.select_varlen(cu)
        want = S.select_varlen(t, lens, d, DESC_J, CAL)
        assert (got["rung_id"], got["cost"], got["grid"]) == (want["rung_id"], want["cost"],
                                                              want["grid"]), lens
