"""paper_2409_01075_b200 -- B200-native dynamic-M GEMM (Vortex, arXiv 2409.01075).

Thin ctypes binding over the C ABI in ``include/vx.h`` (same names, argument marshalling
only).  Every step of the hot path -- strategy table, cost-model selection, tensor-map
encoding and the tcgen05 kernels -- runs inside ``libvx.so``.  torch is used only for
device memory, streams and process groups.  There is no fallback: if the extension is
missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import json
import os

__all__ = ["VxError", "Plan", "DeviceDesc", "Choice", "Calib", "lib", "plan", "gemm",
           "gemm_batched", "device_probe", "launch_count", "calibrate", "LIB_PATH"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libvx.so")

VX_BF16, VX_FP16, VX_FP32 = 0, 1, 2
VX_B_KN, VX_B_NK, VX_B_PACKED = 0, 1, 2
_DT = {"bf16": VX_BF16, "fp16": VX_FP16, "fp32": VX_FP32}
_BL = {"kn": VX_B_KN, "nk": VX_B_NK, "packed": VX_B_PACKED}


class VxError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__("%s failed: %s (%s)" % (where, _lib.vx_status_str(status).decode(), detail))


class DeviceDesc(ctypes.Structure):
    _fields_ = [("sm_count", ctypes.c_int32), ("smem_optin", ctypes.c_int32),
                ("smem_per_sm", ctypes.c_int32), ("max_threads_per_block", ctypes.c_int32),
                ("max_threads_per_sm", ctypes.c_int32), ("tmem_cols", ctypes.c_int32),
                ("cc_major", ctypes.c_int32), ("cc_minor", ctypes.c_int32),
                ("clock_khz", ctypes.c_int32), ("max_active_clusters", ctypes.c_int32 * 4),
                ("l2_bytes", ctypes.c_int64)]

    @classmethod
    def from_json(cls, d: dict) -> "DeviceDesc":
        o = cls()
        for k in ("sm_count", "smem_optin", "smem_per_sm", "max_threads_per_block",
                  "max_threads_per_sm", "tmem_cols", "clock_khz", "l2_bytes"):
            setattr(o, k, int(d[k]))
        o.cc_major, o.cc_minor = int(d["cc"][0]), int(d["cc"][1])
        for i, c in enumerate(("1", "2", "4", "8")):
            o.max_active_clusters[i] = int(d["max_active_clusters"][c])
        return o

    def to_json(self) -> dict:
        return {"sm_count": self.sm_count, "smem_optin": self.smem_optin,
                "smem_per_sm": self.smem_per_sm,
                "max_threads_per_block": self.max_threads_per_block,
                "max_threads_per_sm": self.max_threads_per_sm, "tmem_cols": self.tmem_cols,
                "cc": [self.cc_major, self.cc_minor], "clock_khz": self.clock_khz,
                "l2_bytes": self.l2_bytes,
                "max_active_clusters": {c: self.max_active_clusters[i]
                                        for i, c in enumerate(("1", "2", "4", "8"))}}


class Choice(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("rung_id", "split", "family", "swap", "bm", "bn",
                                              "stages", "tiles_m", "tiles_n", "grid", "cluster",
                                              "mc")] + [("cost", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError("libvx.so not built: run `python __graft_entry__.py` "
                          "(no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    P = ctypes.c_void_p
    L.vx_abi_version.restype = i32
    L.vx_status_str.restype = ctypes.c_char_p
    L.vx_status_str.argtypes = [ctypes.c_int]
    L.vx_last_error.restype = ctypes.c_char_p
    L.vx_device_probe.argtypes = [ctypes.c_int, ctypes.POINTER(DeviceDesc)]
    L.vx_plan.argtypes = [i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                          ctypes.POINTER(P)]
    L.vx_plan_ex.argtypes = [i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                             ctypes.POINTER(DeviceDesc), ctypes.POINTER(P)]
    L.vx_plan_destroy.argtypes = [P]
    L.vx_plan_select.argtypes = [P, i64, i64, i64, ctypes.POINTER(Choice)]
    L.vx_plan_cost.argtypes = [P, i32, i32, i64, i64, i64, ctypes.POINTER(Choice)]
    L.vx_plan_dump.argtypes = [P, ctypes.c_char_p, ctypes.c_size_t,
                               ctypes.POINTER(ctypes.c_size_t)]
    L.vx_gemm.argtypes = [P, i64, i64, i64, vp, vp, vp, vp]
    L.vx_gemm_batched.argtypes = [P, i64, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp]
    L.vx_gemm_ex.argtypes = [P, i64, i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, i32, vp,
                             ctypes.POINTER(Choice)]
    L.vx_gemm_host.argtypes = [P, i64, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp]
    L.vx_gemm_gather.argtypes = [P, i64, i64, i64, vp, vp, i32, ctypes.POINTER(vp), i64, i32,
                                 i32, vp, ctypes.POINTER(Choice)]
    L.vx_calibrate.argtypes = [ctypes.c_int, ctypes.c_int, i32, ctypes.POINTER(P)]
    L.vx_gemm_varlen.argtypes = [P, i32, ctypes.POINTER(i32), vp, i64, vp, vp, vp, i32, vp,
                                 ctypes.POINTER(Choice)]
    L.vx_plan_select_varlen.argtypes = [P, i32, ctypes.POINTER(i32), ctypes.POINTER(Choice)]
    L.vx_calib_new.argtypes = [i64, i64, i64, i64, i64, ctypes.POINTER(P)]
    L.vx_calib_set_rung.argtypes = [P, ctypes.c_char_p, i64, i64, i64, i64]
    L.vx_calib_destroy.argtypes = [P]
    L.vx_calib_dump.argtypes = [P, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
    L.vx_plan_calibrated.argtypes = [i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, P, ctypes.POINTER(P)]
    L.vx_plan_ex_calibrated.argtypes = [i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(DeviceDesc), P, ctypes.POINTER(P)]
    L.vx_launch_count.restype = i64
    L.vx_packed_b_elems.restype = i64
    L.vx_packed_b_elems.argtypes = [P, i64, i64, i64]
    L.vx_pack_b.argtypes = [P, i64, i64, i64, ctypes.c_int, vp, i64, vp, vp]
    L.vx_pack_b.restype = ctypes.c_int
    L.vx_map_cache_stats.argtypes = [ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.vx_map_cache_stats.restype = None
    for f in ("vx_device_probe", "vx_plan", "vx_plan_ex", "vx_plan_destroy", "vx_plan_select",
              "vx_plan_cost", "vx_plan_dump", "vx_gemm", "vx_gemm_batched", "vx_gemm_ex",
              "vx_gemm_host", "vx_gemm_gather", "vx_calibrate", "vx_calib_new",
              "vx_calib_set_rung", "vx_calib_destroy", "vx_calib_dump", "vx_plan_calibrated",
              "vx_plan_ex_calibrated", "vx_gemm_varlen", "vx_plan_select_varlen"):
        getattr(L, f).restype = ctypes.c_int
    if L.vx_abi_version() != 1:
        raise ImportError("libvx.so ABI %d != binding ABI 1 (rebuild)" % L.vx_abi_version())
    return L


_lib = _load()
lib = _lib


def _check(st: int, where: str):
    if st != 0:
        raise VxError(st, where, _lib.vx_last_error().decode())


def device_probe(device: int = 0) -> DeviceDesc:
    d = DeviceDesc()
    _check(_lib.vx_device_probe(device, ctypes.byref(d)), "vx_device_probe")
    return d


def map_cache_stats() -> tuple[int, int]:
    """(hits, misses) of the process-wide tensor-map memo (vx_map_cache_stats)."""
    h, m = ctypes.c_int64(), ctypes.c_int64()
    _lib.vx_map_cache_stats(ctypes.byref(h), ctypes.byref(m))
    return h.value, m.value


def launch_count() -> int:
    return int(_lib.vx_launch_count())


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dt_name(t) -> str:
    import torch
    return {torch.bfloat16: "bf16", torch.float16: "fp16", torch.float32: "fp32"}[t.dtype]


class Calib:
    """An empirical-tier calibration (vx_calib_t): measured live by calibrate(), or built
    from a dict in oracle/calib_b200.json format (from_dict)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_dict(cls, d: dict) -> "Calib":
        h = ctypes.c_void_p()
        _check(_lib.vx_calib_new(d["hbm_milli"], d["dsm_milli"], d["fixed_cluster"],
                                 d["skfix_milli"], d["stagger"], ctypes.byref(h)), "vx_calib_new")
        c = cls(h)
        for k, r in d["rungs"].items():
            _check(_lib.vx_calib_set_rung(h, k.encode(), r["mac_milli"], r["l2s_milli"],
                                          r["epi_milli"], r["fixed"]), "vx_calib_set_rung")
        return c

    def dump(self) -> dict:
        return _calib_dump(self._h)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.vx_calib_destroy(h)
            self._h = None


def _calib_dump(h) -> dict:
    need = ctypes.c_size_t(0)
    _lib.vx_calib_dump(h, None, 0, ctypes.byref(need))
    buf = ctypes.create_string_buffer(need.value)
    _check(_lib.vx_calib_dump(h, buf, need.value, ctypes.byref(need)), "vx_calib_dump")
    return json.loads(buf.value.decode())


def builtin_calib() -> dict:
    """The compiled-in empirical tier (vx_calib.cpp) as a dict."""
    return _calib_dump(None)


def calibrate(device: int = 0, b_layout: str = "nk", effort: int = 0) -> Calib:
    """Live empirical tier (vx_calibrate): profile every rung on `device` over a fixed generic
    grid and fit the cost model's per-rung constants."""
    h = ctypes.c_void_p()
    _check(_lib.vx_calibrate(int(device), _BL[b_layout], int(effort), ctypes.byref(h)),
           "vx_calibrate")
    return Calib(h)


class Plan:
    """Offline strategy table for C[M,N] = A[M,K] x B (vx_plan).  N=0 means dynamic N.
    calib: an empirical tier to freeze into the plan instead of the compiled-in one."""

    def __init__(self, N: int, K: int, in_dtype: str = "bf16", out_dtype: str = "bf16",
                 b_layout: str = "nk", device: int | None = 0, desc: DeviceDesc | None = None,
                 calib: "Calib | None" = None):
        self.N, self.K = int(N), int(K)
        self.in_dtype, self.out_dtype, self.b_layout = in_dtype, out_dtype, b_layout
        h = ctypes.c_void_p()
        args = (self.N, self.K, _DT[in_dtype], _DT[out_dtype], _BL[b_layout])
        if desc is not None and calib is not None:
            _check(_lib.vx_plan_ex_calibrated(*args, ctypes.byref(desc), calib.handle,
                                              ctypes.byref(h)), "vx_plan_ex_calibrated")
        elif desc is not None:
            _check(_lib.vx_plan_ex(*args, ctypes.byref(desc), ctypes.byref(h)), "vx_plan_ex")
        elif calib is not None:
            _check(_lib.vx_plan_calibrated(*args, int(device), calib.handle, ctypes.byref(h)),
                   "vx_plan_calibrated")
        else:
            _check(_lib.vx_plan(*args, int(device), ctypes.byref(h)), "vx_plan")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:   # _lib is None at interpreter exit
            _lib.vx_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def select(self, M: int, N: int | None = None, batch: int = 1) -> dict:
        c = Choice()
        _check(_lib.vx_plan_select(self._h, batch, M, self.N if N is None else N,
                                   ctypes.byref(c)), "vx_plan_select")
        return c.as_dict()

    def select_varlen(self, cu_seqlens) -> dict:
        cu = [int(x) for x in cu_seqlens]
        c = Choice()
        _check(_lib.vx_plan_select_varlen(self._h, len(cu) - 1, (ctypes.c_int32 * len(cu))(*cu),
                                          ctypes.byref(c)), "vx_plan_select_varlen")
        return c.as_dict()

    def cost(self, rung_id: int, split: int, M: int, N: int | None = None, batch: int = 1) -> dict:
        c = Choice()
        _check(_lib.vx_plan_cost(self._h, rung_id, split, batch, M, self.N if N is None else N,
                                 ctypes.byref(c)), "vx_plan_cost")
        return c.as_dict()

    def dump(self) -> dict:
        need = ctypes.c_size_t(0)
        _lib.vx_plan_dump(self._h, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        _check(_lib.vx_plan_dump(self._h, buf, need.value, ctypes.byref(need)), "vx_plan_dump")
        return json.loads(buf.value.decode())

    # ---- runtime -------------------------------------------------------------------------
    def pack_b(self, B, src_layout: str = "nk", stream=None):
        """One-time repack of a weight B ([N,K] "nk" or [K,N] "kn", optionally batched) into
        the VX_B_PACKED layout this plan reads; returns the packed (flat) tensor."""
        import torch
        if self.b_layout != "packed":
            raise ValueError("plan b_layout must be 'packed'")
        batch = 1 if B.dim() == 2 else B.shape[0]
        n = _lib.vx_packed_b_elems(self._h, batch, self.N, self.K)
        out = torch.empty(n, dtype=B.dtype, device=B.device)
        _check(_lib.vx_pack_b(self._h, batch, self.N, self.K, _BL[src_layout], B.data_ptr(),
                              self.N * self.K, out.data_ptr(), _stream_ptr(stream)), "vx_pack_b")
        out.vx_batch = batch
        return out

    def _shape(self, A, B):
        if A.dim() == 2:
            batch, M, K = 1, A.shape[0], A.shape[1]
        else:
            batch, M, K = A.shape
        if self.b_layout == "packed":
            return batch, M, self.N, K
        if self.b_layout == "nk":
            N = B.shape[-2]
            if B.shape[-1] != K:
                raise ValueError("B must be [N,K]")
        else:
            N = B.shape[-1]
            if B.shape[-2] != K:
                raise ValueError("B must be [K,N]")
        return batch, M, N, K

    def gemm(self, A, B, out=None, stream=None, force: tuple[int, int] | None = None,
             want_choice: bool = False):
        """C = A x B on the current (or given) CUDA stream.  A: [M,K] or [batch,M,K]."""
        import torch
        batch, M, N, K = self._shape(A, B)
        for t, nm in ((A, "A"), (B, "B")):
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError("%s must be a contiguous CUDA tensor" % nm)
            if _dt_name(t) != self.in_dtype:
                raise ValueError("%s dtype %s != plan input %s" % (nm, t.dtype, self.in_dtype))
        if B.device != A.device:
            raise ValueError("A and B must be on the same device")
        if A.dim() == 3 and self.b_layout != "packed":
            # batched: B must carry the same batch dimension (the C call reads batch*N*K
            # elements of B at stride N*K; a 2-D B would be read past its end)
            if B.dim() != 3 or B.shape[0] != batch:
                raise ValueError("batched A [%d,M,K] needs B of shape [%d,...]" % (batch, batch))
        elif A.dim() == 2 and B.dim() != 2 and self.b_layout != "packed":
            raise ValueError("2-D A needs a 2-D B")
        odt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[self.out_dtype]
        shape = (M, N) if A.dim() == 2 else (batch, M, N)
        if out is None:
            out = torch.empty(shape, dtype=odt, device=A.device)
        elif out.dtype != odt or tuple(out.shape) != shape or not out.is_contiguous():
            raise ValueError("out must be a contiguous %s tensor of shape %s" % (odt, shape))
        elif out.device != A.device:
            raise ValueError("out must be on A's device")
        ch = Choice()
        fr, fs = force if force is not None else (-1, 0)
        _check(_lib.vx_gemm_ex(self._h, batch, M, N, K, A.data_ptr(), M * K, B.data_ptr(), N * K,
                               out.data_ptr(), M * N, fr, fs, _stream_ptr(stream),
                               ctypes.byref(ch)), "vx_gemm_ex")
        return (out, ch.as_dict()) if want_choice else out

    def gemm_ptr(self, batch, M, N, K, A, sA, B, sB, C, sC, stream_ptr):
        """Raw-pointer form (bench hot loop): no tensor checks, same C call."""
        _check(_lib.vx_gemm_batched(self._h, batch, M, N, K, A, sA, B, sB, C, sC, stream_ptr),
               "vx_gemm_batched")

    def gemm_gather(self, A, B, dsts, row_offset: int, stream=None,
                    force: tuple[int, int] | None = None, want_choice: bool = False):
        """Fused GEMM + row all-gather (vx_gemm_gather): C_local = A x B written into rows
        [row_offset, row_offset + M) of every destination.  dsts: CUDA tensors (same device
        as A) or raw device pointers (e.g. symmetric-memory peer buffers)."""
        M, K = A.shape
        N = self.N
        for t, nm in ((A, "A"), (B, "B")):
            if not t.is_cuda or not t.is_contiguous() or _dt_name(t) != self.in_dtype:
                raise ValueError("%s must be a contiguous CUDA %s tensor" % (nm, self.in_dtype))
        ptrs = []
        for d in dsts:
            if isinstance(d, int):
                ptrs.append(d)
                continue
            if not d.is_cuda or not d.is_contiguous() or d.shape[-1] != N or d.shape[0] < row_offset + M:
                raise ValueError("gather destination must be a contiguous CUDA [>= %d, %d] tensor"
                                 % (row_offset + M, N))
            ptrs.append(d.data_ptr())
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        ch = Choice()
        fr, fs = force if force is not None else (-1, 0)
        _check(_lib.vx_gemm_gather(self._h, M, N, K, A.data_ptr(), B.data_ptr(), len(ptrs), arr,
                                   row_offset, fr, fs, _stream_ptr(stream), ctypes.byref(ch)),
               "vx_gemm_gather")
        return ch.as_dict() if want_choice else None

    def gemm_varlen(self, Q, Kt, cu_seqlens, out=None, stream=None, force: int = -1,
                    want_choice: bool = False, cu_dev=None):
        """Ragged attention batch (vx_gemm_varlen): S_g = Q_g K_g^T for packed Q, Kt
        [total, d] and cu_seqlens (host list of ngroups + 1 offsets; cu_dev: the same as a
        device int32 tensor, made here if not given).  Returns the packed S (sum_g s_g^2
        elements)."""
        import torch
        cu = [int(x) for x in (cu_seqlens.tolist() if hasattr(cu_seqlens, "tolist") else cu_seqlens)]
        ng = len(cu) - 1
        for t, nm in ((Q, "Q"), (Kt, "Kt")):
            if not t.is_cuda or not t.is_contiguous() or _dt_name(t) != self.in_dtype:
                raise ValueError("%s must be a contiguous CUDA %s tensor" % (nm, self.in_dtype))
        if Q.shape != Kt.shape or Q.shape[0] != cu[-1] or Q.shape[1] != self.K:
            raise ValueError("Q and Kt must be [cu[-1], K]")
        odt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[self.out_dtype]
        n_out = sum((cu[g + 1] - cu[g]) ** 2 for g in range(ng))
        if out is None:
            out = torch.empty(n_out, dtype=odt, device=Q.device)
        elif out.numel() < n_out or out.dtype != odt or not out.is_contiguous():
            raise ValueError("out must hold %d contiguous %s elements" % (n_out, odt))
        cu_h = (ctypes.c_int32 * len(cu))(*cu)
        if cu_dev is None:
            cu_dev = torch.tensor(cu, dtype=torch.int32, device=Q.device)
            self._cu_keep = cu_dev    # keep alive until the launch has consumed it
        cu_d = cu_dev
        ch = Choice()
        _check(_lib.vx_gemm_varlen(self._h, ng, cu_h, cu_d.data_ptr(), self.K, Q.data_ptr(),
                                   Kt.data_ptr(), out.data_ptr(), force, _stream_ptr(stream),
                                   ctypes.byref(ch)), "vx_gemm_varlen")
        return (out, ch.as_dict()) if want_choice else out

    def gemm_host(self, batch, M, N, K, hA, hB, hC, dA, dB, dC, stream_ptr):
        _check(_lib.vx_gemm_host(self._h, batch, M, N, K, hA, hB, hC, dA, dB, dC, stream_ptr),
               "vx_gemm_host")


def plan(N: int, K: int, in_dtype: str = "bf16", out_dtype: str = "bf16",
         b_layout: str = "nk", device: int = 0) -> Plan:
    return Plan(N, K, in_dtype, out_dtype, b_layout, device)


def gemm(A, B, b_layout: str = "nk", out_dtype: str | None = None, out=None):
    """One-shot C = A x B (builds a plan each call; cache Plan objects on hot paths)."""
    dt = _dt_name(A)
    p = Plan(B.shape[-2] if b_layout == "nk" else B.shape[-1], A.shape[-1], dt,
             out_dtype or dt, b_layout, A.device.index or 0)
    return p.gemm(A, B, out=out)


def gemm_batched(A, B, b_layout: str = "nk", out_dtype: str | None = None):
    dt = _dt_name(A)
    p = Plan(0, A.shape[-1], dt, out_dtype or dt, b_layout, A.device.index or 0)
    return p.gemm(A, B)
