"""The C-ABI library loads on a CPU-only host, exports every symbol include/vx.h declares,
and rejects bad arguments with the documented status codes (no GPU needed)."""
import ctypes
import json
import os
import re

import pytest

import paper_2409_01075_b200 as vx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DESC = json.load(open(os.path.join(ROOT, "tests", "golden", "b200_desc.json")))


def _declared():
    src = open(os.path.join(ROOT, "include", "vx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vx_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    names = _declared()
    assert len(names) >= 14
    lib = ctypes.CDLL(vx.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n


def test_status_strings_and_version():
    assert vx.lib.vx_abi_version() == 1
    for code, name in enumerate(["VX_OK", "VX_ERR_INVALID", "VX_ERR_UNSUPPORTED", "VX_ERR_ALIGN",
                                 "VX_ERR_CUDA", "VX_ERR_NODEV", "VX_ERR_OOM", "VX_ERR_BUFFER"]):
        assert vx.lib.vx_status_str(code).decode() == name


def _desc():
    return vx.DeviceDesc.from_json(DESC)


def test_plan_ex_on_cpu_and_errors():
    p = vx.Plan(4096, 4096, "bf16", "bf16", "nk", desc=_desc())
    d = p.dump()
    assert d["K"] == 4096 and d["N"] == 4096 and d["rungs"]
    with pytest.raises(vx.VxError) as e:
        vx.Plan(4096, 4100, "bf16", "bf16", "nk", desc=_desc())   # K % 8 != 0
    assert e.value.status == 3
    with pytest.raises(vx.VxError) as e:
        vx.Plan(4096, 0, "bf16", "bf16", "nk", desc=_desc())
    assert e.value.status == 1
    with pytest.raises(vx.VxError) as e:
        vx.Plan(64, 64, "fp32", "bf16", "nk", desc=_desc())      # fp32 in needs fp32 out
    assert e.value.status == 2
    with pytest.raises(vx.VxError) as e:
        p.select(0)
    assert e.value.status == 1
    with pytest.raises(vx.VxError) as e:
        p.select(16, N=4104)                                      # N mismatch with the plan
    assert e.value.status == 1
    with pytest.raises(vx.VxError) as e:
        p.cost(999, 1, 16)
    assert e.value.status == 1


def test_gemm_rejects_before_touching_a_gpu():
    p = vx.Plan(4096, 4096, "bf16", "bf16", "nk", desc=_desc())
    L = vx.lib
    # NULL operands
    assert L.vx_gemm(p.handle, 16, 4096, 4096, None, None, None, None) == 1
    # K mismatch
    assert L.vx_gemm(p.handle, 16, 4096, 4104, 16, 16, 16, None) == 1
    # misaligned pointer
    assert L.vx_gemm(p.handle, 16, 4096, 4096, 17, 32, 32, None) == 3
    # M == 0 is a no-op
    assert L.vx_gemm(p.handle, 0, 4096, 4096, 16, 16, 16, None) == 0
    assert L.vx_plan_destroy(None) == 0


def test_dump_is_canonical_and_deterministic():
    a = vx.Plan(3072, 768, "bf16", "fp32", "kn", desc=_desc())
    b = vx.Plan(3072, 768, "bf16", "fp32", "kn", desc=_desc())
    need = ctypes.c_size_t(0)
    assert vx.lib.vx_plan_dump(a.handle, None, 0, ctypes.byref(need)) == 7   # buffer too small
    ba = ctypes.create_string_buffer(need.value)
    bb = ctypes.create_string_buffer(need.value)
    assert vx.lib.vx_plan_dump(a.handle, ba, need.value, ctypes.byref(need)) == 0
    assert vx.lib.vx_plan_dump(b.handle, bb, need.value, ctypes.byref(need)) == 0
    assert ba.value == bb.value                      # byte-identical rebuilds (sample-free)
    d = json.loads(ba.value)
    assert d["b_layout"] == "kn" and d["out"] == "fp32"


def test_device_probe_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(vx.VxError) as e:
        vx.device_probe(0)
    assert e.value.status == 5


def test_missing_library_fails_loudly(tmp_path):
    """No CPU or library fallback: the binding refuses to import without libvx.so."""
    import shutil, subprocess, sys, os
    pkg = tmp_path / "paper_2409_01075_b200"
    pkg.mkdir()
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2409_01075_b200", "__init__.py")
    shutil.copy(src, pkg / "__init__.py")
    r = subprocess.run([sys.executable, "-c", "import paper_2409_01075_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "libvx.so not built" in r.stderr


def test_descriptor_with_impossible_residency_rejected():
    """A descriptor claiming more resident clusters of size c than sm_count / c is refused:
    the stream-K workspace has sm_count slots and its flag wait needs the whole grid
    resident."""
    for i, bad in ((0, 149), (1, 75), (2, 38), (3, 19)):
        d = _desc()
        d.max_active_clusters[i] = bad
        with pytest.raises(vx.VxError) as e:
            vx.Plan(4096, 4096, "bf16", "bf16", "nk", desc=d)
        assert e.value.status == 1
