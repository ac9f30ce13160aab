// vx_dispatch.cu -- runtime half of vx_gemm: validation, CUtensorMap encoding, and the
// launch of the rung vx_plan_select chose ("compute runtime-specific computational details,
// such as grid configurations").  Also the device probe (GetHardwareInfo,
// PAPER.md:1770) and the explicit instantiation table of the ladder kernels.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "vx_internal.h"
#include "vx_gemv.cuh"
#include "vx_simt.cuh"
#include "vx_kernels.h"

namespace vx {

static std::atomic<int64_t> g_launches{0};
static unsigned long long* g_trace = nullptr;  // device buffer, 32 x u64 per CTA (debug)
static const int g_dbg = [] {                 // VX_DEBUG_FLAGS (kernel phase skips, debug only)
    const char* e = getenv("VX_DEBUG_FLAGS");
    return e ? atoi(e) : 0;
}();
static const int g_group_p = [] {             // VX_GROUP_P: raster group size (experiments)
    const char* e = getenv("VX_GROUP_P");
    return e ? atoi(e) : 0;
}();
static const bool g_pdl = [] {                 // VX_PDL=0 disables programmatic launch
    const char* e = getenv("VX_PDL");
    return !(e && e[0] == '0');
}();

// ---- instantiated kernels (the "implemented" filter of the strategy table, R6) -----------
// TMA-multicast cluster rungs: non-swapped 128 x BN tiles sharing the A (= P)
// tile over 2 CTAs; swapped tiles sharing the A (= Q) tile over 2 or 4 CTAs
static bool mc_available(int family, int bm, int bn, int mc) {
    if (family == kUmma) return mc == 2 && bm == 128 && (bn == 128 || bn == 256);
    if (family == kUmmaSwap) return bm == 128 && ((mc == 2 && (bn == 32 || bn == 64)) || (mc == 4 && bn == 64));
    return false;
}

// occupancy-2 (lean) rungs: the kernel exists (vx_umma_kernel<..., LEAN = true>) and was
// measured integer-exact, but slower than the occupancy-1 rungs on every BERT-size shape
// tried (its <= ~110 KB ring keeps too few bytes in flight: 8.3 vs 6.2 us at M=128,
// N=3072, K=768), so no lean rung is instantiated.  The strategy table keeps
// the occupancy-2 L2 candidates (R5b); they are filtered here as unimplemented (R6).
static bool lean_available(int family, int bm, int bn) {
    (void)family; (void)bm; (void)bn;
    return false;
}

bool kernel_available(int family, int bm, int bn, int mc, int occ) {
    if (occ == 2) return mc == 1 && lean_available(family, bm, bn);
    if (mc != 1) return mc_available(family, bm, bn, mc);
    if (family == kUmma)
        return (bm == 128 && (bn == 64 || bn == 128 || bn == 192 || bn == 256)) ||
               (bm == 256 && (bn == 64 || bn == 128 || bn == 256));   // cta_group::2 pairs
    if (family == kUmmaSwap)
        return bm == 128 && (bn == 16 || bn == 32 || bn == 64 || bn == 128 || bn == 192 || bn == 256);
    if (family == kSimt) return (bm == 32 && bn == 32) || (bm == 64 && bn == 64) || (bm == 128 && bn == 64);
    if (family == kGemv) return (bm == 1 || bm == 2 || bm == 4 || bm == 8) && bn == kGemvCols;
    return false;
}

static UmmaFn umma_fn(int family, int bm, int bn, bool b_mn, int mc = 1, int occ = 1) {
    if (occ == 2) return nullptr;   // no lean kernel instantiated (see lean_available)
    if (mc > 1) return mc_available(family, bm, bn, mc) ? umma_fn_mc(family, bn, mc, b_mn) : nullptr;
    if (!kernel_available(family, bm, bn, 1, 1)) return nullptr;
    if (family == kUmma && bm == 256) return umma_fn_pair(bn, b_mn);
    if (family == kUmma) return umma_fn_single(bn, b_mn);
    if (family == kUmmaSwap) return umma_fn_swap(bn, b_mn);
    return nullptr;
}

using SimtFn = void (*)(const float*, const float*, float*, int, int, int, int, long long,
                        long long, long long, int, int);

static SimtFn simt_fn(int bm, int bn, int* threads) {
    if (bm == 32 && bn == 32) { *threads = 128; return vx_simt_kernel<32, 32, 2, 4>; }
    if (bm == 64 && bn == 64) { *threads = 256; return vx_simt_kernel<64, 64, 4, 4>; }
    if (bm == 128 && bn == 64) { *threads = 256; return vx_simt_kernel<128, 64, 8, 4>; }
    return nullptr;
}

// per-CTA dynamic shared memory: S stages of (128 A rows + this CTA's B rows) x 128 B
static int64_t umma_smem_bytes(int bm, int bn, int stages, int occ = 1) {
    const int cg = bm == 256 ? 2 : 1;
    return (int64_t)stages * (bm / cg + bn / cg) * kBkTc * 2 + kSmemReserve +
           (occ == 2 ? kEpiStagingLean : kEpiStaging);
}

static vx_status cuda_fail(cudaError_t e, const char* what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return VX_ERR_CUDA;
}

// one-time per-(device, kernel) attribute setup (max dynamic smem; cluster dims are per
// launch).  cudaFuncSetAttribute applies to the CURRENT device only, so the cache is keyed
// by (device, function).
static std::mutex g_attr_mu;
static vx_status ensure_attr(const void* fn, int64_t smem) {
    struct Entry { int dev; const void* fn; int64_t smem; };
    static Entry done[256];
    static int ndone = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (int i = 0; i < ndone; ++i)
        if (done[i].dev == dev && done[i].fn == fn && done[i].smem >= smem) return VX_OK;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    for (int i = 0; i < ndone; ++i)
        if (done[i].dev == dev && done[i].fn == fn) { done[i].smem = smem; return VX_OK; }
    if (ndone < 256) done[ndone++] = {dev, fn, smem};
    return VX_OK;
}

// restores the calling thread's current device on scope exit
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// ---- CUtensorMap encoding via the driver entry point (no -lcuda link dependency) -------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 3-D map over a 16-bit matrix stored [batch][rows][inner] (inner contiguous):
// dims {inner, rows, batch}; box {64, box_rows, 1}; 128-B swizzle; OOB -> zeros.
// ---- tensor-map memo ("B's map is cached per pointer") ------------------
// A CUtensorMap is a pure function of its encode arguments (address, shape, strides, box,
// swizzle) and holds no reference to the memory, so a map encoded once can be reused by any
// later launch with identical arguments -- even after the buffer was freed and another one
// landed at the same address.  Weights (B) repeat across calls; activations usually do not.
// Process-wide, 64 entries, round-robin replacement, one mutex (host only).
struct MapKey {
    int32_t kind, dt, swz, pad;
    const void* base;
    int64_t v[6];
    int32_t box[4];
};
static std::mutex g_map_mu;
static MapKey g_map_keys[64];
static CUtensorMap g_map_vals[64];
static int g_map_n = 0, g_map_next = 0;
static std::atomic<int64_t> g_map_hits{0}, g_map_misses{0};

static MapKey map_key(int kind, const void* base, vx_dtype dt, int64_t v0, int64_t v1, int64_t v2,
                      int64_t v3, int64_t v4, int b0, int b1, int swz) {
    MapKey k;
    memset(&k, 0, sizeof(k));
    k.kind = kind; k.dt = (int32_t)dt; k.swz = swz; k.base = base;
    k.v[0] = v0; k.v[1] = v1; k.v[2] = v2; k.v[3] = v3; k.v[4] = v4;
    k.box[0] = b0; k.box[1] = b1;
    return k;
}
static bool map_lookup(const MapKey& k, CUtensorMap* out) {
    std::lock_guard<std::mutex> lk(g_map_mu);
    for (int i = 0; i < g_map_n; ++i)
        if (memcmp(&g_map_keys[i], &k, sizeof(k)) == 0) {
            *out = g_map_vals[i];
            g_map_hits.fetch_add(1, std::memory_order_relaxed);
            return true;
        }
    g_map_misses.fetch_add(1, std::memory_order_relaxed);
    return false;
}
static void map_store(const MapKey& k, const CUtensorMap& m) {
    std::lock_guard<std::mutex> lk(g_map_mu);
    const int i = g_map_n < 64 ? g_map_n++ : g_map_next;
    g_map_next = (i + 1) % 64;
    g_map_keys[i] = k;
    g_map_vals[i] = m;
}

static vx_status make_map(CUtensorMap* map, const void* base, vx_dtype dt, int64_t inner,
                          int64_t rows, int64_t batch, int64_t ld, int64_t bstride,
                          int box_inner, int box_rows, bool swizzle = true) {
    const MapKey key = map_key(3, base, dt, inner, rows, batch, ld, bstride, box_inner, box_rows,
                               swizzle ? 1 : 0);
    if (map_lookup(key, map)) return VX_OK;
    EncodeTiledFn enc = encode_fn();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return VX_ERR_CUDA; }
    const int eb = dt == VX_FP32 ? 4 : 2;
    cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)ld * eb, (cuuint64_t)bstride * eb};
    cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUtensorMapDataType ty = dt == VX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : dt == VX_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = enc(map, ty, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d): inner=%lld rows=%lld batch=%lld ld=%lld",
                  (int)r, (long long)inner, (long long)rows, (long long)batch, (long long)ld);
        return VX_ERR_CUDA;
    }
    map_store(key, *map);
    return VX_OK;
}

// 4-D two-chunk view of a K-major 16-bit matrix [batch][rows][K] (K % 64 == 0): dims
// {64 k, rows, K/64 chunks, batch}, strides {ld, 128 B, batch}; box {64, box_rows, 2, 1}.
// One box = two consecutive 64-deep chunks of box_rows rows, written chunk-major: the second
// lands box_rows * 128 B after the first, i.e. exactly in the next ring stage's slot, with
// the same 128-B swizzle (the pattern is a function of the SMEM address).
static vx_status make_map_k2(CUtensorMap* map, const void* base, vx_dtype dt, int64_t K,
                             int64_t rows, int64_t batch, int64_t ld, int64_t bstride,
                             int box_rows) {
    const MapKey key = map_key(4, base, dt, K, rows, batch, ld, bstride, 64, box_rows, 1);
    if (map_lookup(key, map)) return VX_OK;
    EncodeTiledFn enc = encode_fn();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return VX_ERR_CUDA; }
    cuuint64_t dims[4] = {64, (cuuint64_t)rows, (cuuint64_t)(K / 64), (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)ld * 2, 128, (cuuint64_t)bstride * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 2, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapDataType ty = dt == VX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUresult r = enc(map, ty, 4, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("two-chunk cuTensorMapEncodeTiled failed (%d): K=%lld rows=%lld", (int)r,
                  (long long)K, (long long)rows);
        return VX_ERR_CUDA;
    }
    map_store(key, *map);
    return VX_OK;
}

// 5-D map over a VX_B_PACKED B: {64 k, 64 rows, k-block, row-block, batch}; one box = one
// contiguous 8-KB 64 x 64 tile; OOB in any dimension (row / k / batch tails) reads zeros.
static vx_status make_packed_map(CUtensorMap* map, const void* base, vx_dtype dt, int64_t N,
                                 int64_t K, int64_t batch) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return VX_ERR_CUDA; }
    const int64_t kb = (K + 63) / 64, rb = (N + 63) / 64;
    cuuint64_t dims[5] = {64, 64, (cuuint64_t)kb, (cuuint64_t)rb, (cuuint64_t)batch};
    cuuint64_t strides[4] = {128, 8192, (cuuint64_t)(8192 * kb), (cuuint64_t)(8192 * kb * rb)};
    cuuint32_t box[5] = {64, 64, 1, 1, 1};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(map, dt == VX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                     5, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("packed cuTensorMapEncodeTiled failed (%d)", (int)r); return VX_ERR_CUDA; }
    return VX_OK;
}

// pack B (NK or KN storage) into [batch][rb][kb][64][64]: one thread per 8-element chunk
__global__ void vx_pack_b_kernel(const uint16_t* __restrict__ B, uint16_t* __restrict__ out,
                                 long long N, long long K, long long sB, int b_kn, long long rb,
                                 long long kb, long long total_chunks) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < total_chunks;
         c += (long long)gridDim.x * blockDim.x) {
        const long long j8 = c & 7, i = (c >> 3) & 63, t = c >> 9;   // chunk, row, tile
        const long long kbi = t % kb, rbi = (t / kb) % rb, b = t / (kb * rb);
        const long long n = rbi * 64 + i, k0 = kbi * 64 + j8 * 8;
        uint16_t v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const long long k = k0 + e;
            v[e] = (n < N && k < K) ? (b_kn ? B[b * sB + k * N + n] : B[b * sB + n * K + k]) : 0;
        }
        uint4 u;
        u.x = v[0] | ((uint32_t)v[1] << 16);
        u.y = v[2] | ((uint32_t)v[3] << 16);
        u.z = v[4] | ((uint32_t)v[5] << 16);
        u.w = v[6] | ((uint32_t)v[7] << 16);
        reinterpret_cast<uint4*>(out)[c] = u;
    }
}

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// stream-K workspace: one partial slot (128 x 256 fp32) + one flag per SM.  One workspace
// per (device, stream): stream-K launches on one stream are serialised by the stream, and
// every flag is consumed and cleared inside the launch that set it, so a stream's
// workspace is always clean for its next launch; launches on different streams use
// different workspaces (vx.h thread-safety contract).  Allocated on first stream-K use of
// a stream (vx_plan pre-allocates one for the legacy stream).  If that first use happens
// inside a stream capture, the allocation runs in relaxed capture mode and the flags are
// zeroed on a private non-blocking stream that is synchronised before returning, so
// neither touches the captured stream.
static size_t ws_bytes(const vx_plan_s* p) {
    return (size_t)p->desc.sm_count * 128 * 256 * 4 + (size_t)p->desc.sm_count * 4 + 256;
}
static vx_status ensure_ws(const vx_plan_s* pc, void* stream, void** out) {
    vx_plan_s* p = const_cast<vx_plan_s*>(pc);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lk(p->ws_mu);
    for (const auto& w : p->ws)
        if (w.stream == stream && w.device == dev) { *out = w.ptr; return VX_OK; }
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    void* w = nullptr;
    cudaStream_t priv = nullptr;
    e = cudaMalloc(&w, ws_bytes(p));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&priv, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemsetAsync(w, 0, ws_bytes(p), priv);
    if (e == cudaSuccess) e = cudaStreamSynchronize(priv);
    if (priv) cudaStreamDestroy(priv);
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (e != cudaSuccess) {
        if (w) cudaFree(w);
        return cuda_fail(e, "stream-K workspace allocation");
    }
    p->ws.push_back({stream, dev, w});
    *out = w;
    return VX_OK;
}

vx_status launch(const vx_plan_s* p, const vx_choice& ch, int64_t batch, int64_t M, int64_t N,
                 int64_t K, const void* A, int64_t sA, const void* B, int64_t sB, void* C,
                 int64_t sC, void* stream, const GatherSpec* gather, const VarSpec* var) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const vx::Rung& r = p->rungs[ch.rung_id];
    if (r.family == kSimt) {
        int threads = 0;
        SimtFn fn = simt_fn(r.bm, r.bn, &threads);
        if (!fn) { set_error("no SIMT kernel %dx%d", r.bm, r.bn); return VX_ERR_UNSUPPORTED; }
        const int tm = (int)cdiv(M, r.bm), tn = (int)cdiv(N, r.bn);
        const int64_t grid = batch * (int64_t)tm * tn;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid, 1, 1);
        cfg.blockDim = dim3((unsigned)threads, 1, 1);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        if (g_pdl) {   // the kernel waits (griddepcontrol.wait) before its first global access
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
        }
        cudaError_t e = cudaLaunchKernelEx(&cfg, fn, (const float*)A, (const float*)B, (float*)C,
                                           (int)M, (int)N, (int)K, (int)(p->bl == VX_B_NK),
                                           (long long)sA, (long long)sB, (long long)sC, tm, tn);
        if (e != cudaSuccess) return cuda_fail(e, "SIMT launch");
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return VX_OK;
    }
    if (r.family == kGemv) {
        using GemvFn = void (*)(const uint16_t*, const uint16_t*, void*, int, int, int, long long,
                                long long, long long, int, int);
        const bool kn = p->bl == VX_B_KN;
        GemvFn fn = nullptr;
        switch (r.bm) {
        case 1: fn = kn ? vx_gemv_kernel<1, true> : vx_gemv_kernel<1, false>; break;
        case 2: fn = kn ? vx_gemv_kernel<2, true> : vx_gemv_kernel<2, false>; break;
        case 4: fn = kn ? vx_gemv_kernel<4, true> : vx_gemv_kernel<4, false>; break;
        case 8: fn = kn ? vx_gemv_kernel<8, true> : vx_gemv_kernel<8, false>; break;
        }
        if (!fn || M > r.bm) { set_error("no GEMV kernel for rung %d / M=%lld", r.rung_id, (long long)M); return VX_ERR_UNSUPPORTED; }
        // MT >= 4, N x K B, K >= 2048 (>= 2 k-steps per warp; below that the staging is
        // pure latency: BERT K = 768, M = 4 measured 3.5 -> 4.4 us): A staged once in shared
        // memory (R20b); VX_DEBUG_FLAGS 16384 = off
        size_t a_smem = 0;
        if (!kn && r.bm >= 4 && K % 8 == 0 && K >= 2048 && !(g_dbg & 16384) &&
            (size_t)r.bm * K * 2 <= kGemvSaMaxSmem) {
            fn = r.bm == 4 ? vx_gemv_sa_kernel<4, 4> : vx_gemv_sa_kernel<8, 2>;
            a_smem = (size_t)r.bm * K * 2;
            vx_status sa = ensure_attr((const void*)fn, (int64_t)kGemvSaMaxSmem);
            if (sa != VX_OK) return sa;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.dynamicSmemBytes = a_smem;
        cfg.gridDim = dim3((unsigned)cdiv(N, kGemvCols), (unsigned)batch, 1);
        cfg.blockDim = dim3(kGemvWarps * 32, 1, 1);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        if (g_pdl) {
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
        }
        const long long sCe = batch > 1 ? sC : M * N;
        cudaError_t e = cudaLaunchKernelEx(&cfg, fn, (const uint16_t*)A, (const uint16_t*)B, C,
                                           (int)M, (int)N, (int)K, (long long)(batch > 1 ? sA : M * K),
                                           (long long)(batch > 1 ? sB : N * K), sCe,
                                           p->in == VX_BF16 ? 0 : 1,
                                           p->out == VX_BF16 ? 0 : p->out == VX_FP16 ? 1 : 2);
        if (e != cudaSuccess) return cuda_fail(e, "GEMV launch");
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return VX_OK;
    }
    const bool swap = r.swap != 0;
    const bool b_mn = p->bl == VX_B_KN;
    const bool pair = r.cg == 2;
    const int mc = r.mc;
    UmmaFn fn = umma_fn(r.family, r.bm, r.bn, b_mn, mc, r.occ);
    if (!fn) { set_error("no tcgen05 kernel for rung %d", r.rung_id); return VX_ERR_UNSUPPORTED; }
    const int64_t smem = umma_smem_bytes(r.bm, r.bn, r.stages, r.occ);
    vx_status s = ensure_attr((const void*)fn, smem);
    if (s != VX_OK) return s;

    // tensor maps: A [batch][M][K] K-major; B [batch][N][K] (NK) or [batch][K][N] (KN)
    CUtensorMap mapA, mapB;
    // A is P (box 128 rows) or Q (box BN rows); in a multicast cluster each CTA loads (and
    // multicasts) 1/mc of A's rows
    int a_box = (swap ? r.bn : 128) / mc;
    // short A boxes: on a swapped rung, an A box of >= 64 rows over an A of
    // fewer than 16 rows streams at ~0.6x the rate (measured, N = 8192, K = 4096: swap
    // 128x128 at M <= 15 36-37 us vs 22 us at M = 16; 23 us with the short box); a box of
    // round_up(M, 8) rows leaves the rest of the A tile stale in SMEM, which only feeds
    // accumulator columns >= M that are never stored.  Narrower boxes keep the (faster)
    // two-chunk deep-K loads instead (swap 128x32: 19.4 us with them vs 22 us short).
    const bool short_a = swap && M < 16 && mc == 1 && !pair && a_box >= 64 && !(g_dbg & 65536);
    if (short_a) a_box = (int)((M + 7) / 8 * 8);
    s = make_map(&mapA, A, p->in, K, M, batch, K, batch > 1 ? sA : M * K, 64, a_box);
    if (s != VX_OK) return s;
    if (p->bl == VX_B_PACKED) {
        s = make_packed_map(&mapB, B, p->in, N, K, batch);
    } else if (b_mn) {
        s = make_map(&mapB, B, p->in, N, K, batch, N, batch > 1 ? sB : K * N, 64, 64);
    } else {
        const int b_box = swap ? 128 : (pair ? r.bn / 2 : r.bn);
        s = make_map(&mapB, B, p->in, K, N, batch, K, batch > 1 ? sB : N * K, 64, b_box);
    }
    if (s != VX_OK) return s;

    UmmaParams prm;
    prm.M = (int)M;
    prm.N = (int)N;
    prm.tiles_p = ch.tiles_m;
    prm.tiles_q = ch.tiles_n;
    // multicast clusters walk cluster tiles (mc tiles along the axis not sharing A)
    prm.mc = mc;
    prm.num_tiles = (int)(batch * (mc > 1 && swap ? cdiv(ch.tiles_m, mc) : (int64_t)ch.tiles_m) *
                          (mc > 1 && !swap ? cdiv(ch.tiles_n, mc) : (int64_t)ch.tiles_n));
    prm.kb_total = (int)cdiv(K, kBkTc);
    prm.splits = ch.split > 0 ? ch.split : 1;
    prm.streamk = ch.split == 0;
    prm.ws = nullptr;
    prm.flags = nullptr;
    if (prm.streamk) {
        void* w = nullptr;
        s = ensure_ws(p, stream, &w);
        if (s != VX_OK) return s;
        prm.ws = reinterpret_cast<float*>(w);
        prm.flags = reinterpret_cast<int*>(reinterpret_cast<char*>(w) +
                                           (size_t)p->desc.sm_count * 128 * 256 * 4);
    }
    prm.stages = r.stages;
    prm.out_kind = p->out == VX_BF16 ? 0 : p->out == VX_FP16 ? 1 : 2;
    const uint32_t fmt = p->in == VX_BF16 ? 1u : 0u;
    const uint32_t p_major = (swap && b_mn) ? 1u : 0u;   // P operand MN-major?
    const uint32_t q_major = (!swap && b_mn) ? 1u : 0u;  // Q operand MN-major?
    prm.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (p_major << 15) | (q_major << 16) |
                ((uint32_t)(r.bn >> 3) << 17) | ((uint32_t)((pair ? 256 : 128) >> 4) << 24);
    prm.pair = pair ? 1 : 0;
    prm.bpack = p->bl == VX_B_PACKED ? 1 : 0;
    // deep-K units: K-major P and Q, whole 64-deep chunks, unpacked, and a
    // ring deep enough to keep >= 3 units (>= 4 for the compute-bound pair rungs) in flight:
    // measured, 128 x 256 (4 stages) up to 1.17x slower, pair 256 x 256 (6 stages) 1.03x
    // slower, pair 256 x 128 (8 stages) 0.86-0.90x; VX_DEBUG_FLAGS bit 4096 turns them off
    // (A/B timing only)
    // bytes of A landing in each CTA's stage: the short box, else the whole A tile (a
    // multicast cluster's sub-boxes from every CTA all land in every CTA's stage)
    // raster group (P tiles swept over every Q tile while held in L2): VX_GROUP_P overrides
    prm.group_p = g_group_p > 0 ? g_group_p : kGroupP;
    prm.a_bytes = (short_a ? a_box : (swap ? r.bn : 128)) * 64 * 2;
    prm.kdouble = (!b_mn && p->bl != VX_B_PACKED && K % 64 == 0 && K >= 128 && mc == 1 && !short_a &&
                   r.stages >= (pair ? 8 : 6) && !(g_dbg & 4096)) ? 1 : 0;
    CUtensorMap mapA2, mapB2;
    if (prm.kdouble) {
        s = make_map_k2(&mapA2, A, p->in, K, M, batch, K, batch > 1 ? sA : M * K, a_box);
        if (s != VX_OK) return s;
        s = make_map_k2(&mapB2, B, p->in, K, N, batch, K, batch > 1 ? sB : N * K, swap ? 128 : (pair ? r.bn / 2 : r.bn));
        if (s != VX_OK) return s;
    } else {
        mapA2 = mapA;
        mapB2 = mapB;
    }
    prm.C = C;
    prm.ldc = N;
    prm.sC = batch > 1 ? sC : M * N;
    prm.trace = g_trace;
    prm.dbg = g_dbg;
    const int ob = p->out == VX_FP32 ? 4 : 2;
    prm.vec = (N % 8 == 0) && ((prm.sC * ob) % 16 == 0) &&
              ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
    prm.ndst = 0;
    prm.dst_row0 = 0;
    for (int d = 0; d < 8; ++d) prm.dst[d] = nullptr;
    prm.cu = nullptr;
    prm.ngroups = 0;
    if (var) {
        // ragged batch: tiles enumerate every sequence's (tp, tq); each sequence's S block
        // is stored from registers (no C tensor map), vectorised per sequence when aligned
        prm.cu = var->cu_dev;
        prm.ngroups = var->ngroups;
        prm.num_tiles = (int)var->tiles;
        prm.vec = 0;
    }
    if (gather) {
        // fused all-gather epilogue: vector stores iff every destination
        // row is 16-B aligned
        prm.ndst = gather->ndst;
        prm.dst_row0 = gather->row0;
        prm.vec = N % 8 == 0;
        for (int d = 0; d < gather->ndst; ++d) {
            prm.dst[d] = gather->dst[d];
            if (reinterpret_cast<uintptr_t>(gather->dst[d]) & 15) prm.vec = 0;
        }
    }
    // C map for the TMA-store epilogue: non-swap boxes are 128-B rows x 32 rows (swizzled),
    // swap boxes are 32 n x min(32, BN) m (plain)
    CUtensorMap mapC;
    memset(&mapC, 0, sizeof(mapC));
    if (prm.vec) {
        if (!swap) s = make_map(&mapC, C, p->out, N, M, batch, N, prm.sC, 128 / ob, 32, true);
        else s = make_map(&mapC, C, p->out, N, M, batch, N, prm.sC, 32, r.bn < 32 ? r.bn : 32, false);
        if (s != VX_OK) return s;
    }

    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ch.grid, 1, 1);
    cfg.blockDim = dim3(r.occ == 2 ? 192 : kThreads, 1, 1);   // lean CTAs: 6 warps
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    unsigned na = 0;
    if (ch.split > 1 || pair || mc > 1) {   // split-K cluster, CTA pair or multicast cluster
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)(pair ? 2 : mc > 1 ? mc : ch.split);
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (g_pdl) {
        // programmatic dependent launch: this grid may start while the previous kernel on
        // the stream drains; the kernel's griddepcontrol.wait orders all global accesses
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
    // P operand (UMMA-M axis) first: A for family 0, B for the swapped family
    const CUtensorMap& mapP = swap ? mapB : mapA;
    const CUtensorMap& mapQ = swap ? mapA : mapB;
    const CUtensorMap& mapP2 = swap ? mapB2 : mapA2;
    const CUtensorMap& mapQ2 = swap ? mapA2 : mapB2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, mapP, mapQ, mapC, mapP2, mapQ2, prm);
    if (e != cudaSuccess) return cuda_fail(e, "tcgen05 launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return VX_OK;
}

vx_status prepare_kernels(const vx_plan_s* p) {
    DeviceGuard g(p->device);   // attributes and the workspace belong to the plan's device
    if (p->in != VX_FP32) {
        void* w = nullptr;
        vx_status s = ensure_ws(p, nullptr, &w);   // the legacy stream's workspace
        if (s != VX_OK) return s;
    }
    for (const vx::Rung& r : p->rungs) {
        if (r.family == kSimt) continue;
        UmmaFn fn = umma_fn(r.family, r.bm, r.bn, p->bl == VX_B_KN, r.mc, r.occ);
        if (!fn) continue;
        vx_status s = ensure_attr((const void*)fn, umma_smem_bytes(r.bm, r.bn, r.stages, r.occ));
        if (s != VX_OK) return s;
    }
    return VX_OK;
}

}  // namespace vx

vx_plan_s::~vx_plan_s() {
    for (const auto& w : ws) {
        vx::DeviceGuard g(w.device);
        cudaFree(w.ptr);
    }
}

using namespace vx;

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static vx_status check_args(const vx_plan_s* p, int64_t batch, int64_t M, int64_t N, int64_t K,
                            const void* A, int64_t sA, const void* B, int64_t sB, const void* C,
                            int64_t sC) {
    if (!p) { set_error("NULL plan"); return VX_ERR_INVALID; }
    if (batch < 1 || M < 0 || N < 1 || K < 1) { set_error("bad sizes"); return VX_ERR_INVALID; }
    if (K != p->K) { set_error("K=%lld does not match the plan's K=%lld", (long long)K, (long long)p->K); return VX_ERR_INVALID; }
    if (p->N > 0 && N != p->N) { set_error("N=%lld does not match the plan's N=%lld", (long long)N, (long long)p->N); return VX_ERR_INVALID; }
    if (M == 0) return VX_OK;  // empty problem: nothing is read or written
    if (!A || !B || !C) { set_error("NULL operand"); return VX_ERR_INVALID; }
    if (batch > 1 && (sA < M * K || sB < N * K || sC < M * N)) { set_error("batch strides overlap"); return VX_ERR_INVALID; }
    if (M > 0x7fffffffLL || N > 0x7fffffffLL) { set_error("M, N must fit in int32"); return VX_ERR_INVALID; }
    if (p->in != VX_FP32) {
        // TMA: 16-byte aligned bases and row / batch strides of A and B.  C is written with
        // plain stores (vectorised only when aligned), so it has no alignment rule.
        if (K % 8) { set_error("16-bit inputs need K %% 8 == 0"); return VX_ERR_ALIGN; }
        if (p->bl == VX_B_KN && N % 8) { set_error("B stored K x N needs N %% 8 == 0"); return VX_ERR_ALIGN; }
        if (!aligned16(A) || !aligned16(B)) { set_error("A and B must be 16-byte aligned"); return VX_ERR_ALIGN; }
        if (batch > 1 && (sA % 8 || sB % 8)) { set_error("A/B batch strides must be multiples of 8 elements"); return VX_ERR_ALIGN; }
        const int ob = p->out == VX_FP32 ? 4 : 2;
        if (reinterpret_cast<uintptr_t>(C) % ob) { set_error("C must be element aligned"); return VX_ERR_ALIGN; }
    }
    return VX_OK;
}

extern "C" {

vx_status vx_device_probe(int device, vx_device_desc* out) {
    if (!out) { set_error("NULL argument"); return VX_ERR_INVALID; }
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        set_error("CUDA device %d not available", device);
        return VX_ERR_NODEV;
    }
    cudaDeviceProp pr;
    cudaError_t e = cudaGetDeviceProperties(&pr, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (pr.major != 10) { set_error("device %d is sm_%d%d, need sm_100", device, pr.major, pr.minor); return VX_ERR_NODEV; }
    memset(out, 0, sizeof(*out));
    out->sm_count = pr.multiProcessorCount;
    out->smem_optin = (int32_t)pr.sharedMemPerBlockOptin;
    out->smem_per_sm = (int32_t)pr.sharedMemPerMultiprocessor;
    out->max_threads_per_block = pr.maxThreadsPerBlock;
    out->max_threads_per_sm = pr.maxThreadsPerMultiProcessor;
    out->tmem_cols = 512;
    out->cc_major = pr.major;
    out->cc_minor = pr.minor;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    out->clock_khz = clk;
    out->l2_bytes = pr.l2CacheSize;
    // resident clusters of 1/2/4/8 full-SMEM CTAs of the ladder kernel
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    UmmaFn fn = umma_fn(kUmma, 128, 128, false);
    const int64_t smem = (int64_t)out->smem_optin;
    vx_status s = ensure_attr((const void*)fn, smem);
    if (s != VX_OK) { cudaSetDevice(cur); return s; }
    const int sizes[4] = {1, 2, 4, 8};
    for (int i = 0; i < 4; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sizes[i] * 64, 1, 1);
        cfg.blockDim = dim3(kThreads, 1, 1);
        cfg.dynamicSmemBytes = (size_t)smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = sizes[i];
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nc = 0;
        e = cudaOccupancyMaxActiveClusters(&nc, fn, &cfg);
        if (e != cudaSuccess) { cudaSetDevice(cur); return cuda_fail(e, "cudaOccupancyMaxActiveClusters"); }
        out->max_active_clusters[i] = nc;
    }
    cudaSetDevice(cur);
    return VX_OK;
}

vx_status vx_gemm_ex(vx_plan_t p, int64_t batch, int64_t M, int64_t N, int64_t K, const void* A,
                     int64_t sA, const void* B, int64_t sB, void* C, int64_t sC,
                     int32_t force_rung, int32_t force_split, void* stream, vx_choice* used) {
    vx_status s = check_args(p, batch, M, N, K, A, sA, B, sB, C, sC);
    if (s != VX_OK) return s;
    if (M == 0) return VX_OK;
    if (p->device >= 0) {
        // kernel attributes and workspaces were set up for the plan's device; launching
        // there from another current device would fault or fail (ABI)
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess || cur != p->device) {
            cudaGetLastError();
            set_error("current device %d != the plan's device %d", cur, p->device);
            return VX_ERR_INVALID;
        }
    }
    vx_choice ch;
    s = select_choice(p, batch, M, N, force_rung, force_split, &ch);
    if (s != VX_OK) return s;
    if (used) *used = ch;
    return launch(p, ch, batch, M, N, K, A, sA, B, sB, C, sC, stream);
}

vx_status vx_gemm_batched(vx_plan_t p, int64_t batch, int64_t M, int64_t N, int64_t K,
                          const void* A, int64_t sA, const void* B, int64_t sB, void* C,
                          int64_t sC, void* stream) {
    return vx_gemm_ex(p, batch, M, N, K, A, sA, B, sB, C, sC, -1, 0, stream, nullptr);
}

vx_status vx_gemm(vx_plan_t p, int64_t M, int64_t N, int64_t K, const void* A, const void* B,
                  void* C, void* stream) {
    return vx_gemm_ex(p, 1, M, N, K, A, M * K, B, N * K, C, M * N, -1, 0, stream, nullptr);
}

vx_status vx_gemm_gather(vx_plan_t p, int64_t M, int64_t N, int64_t K, const void* A,
                         const void* B, int32_t ndst, void* const* dst, int64_t row_offset,
                         int32_t force_rung, int32_t force_split, void* stream, vx_choice* used) {
    if (!p || !dst || ndst < 1 || ndst > 8 || row_offset < 0) {
        set_error("gather needs 1 <= ndst <= 8 destinations and row_offset >= 0");
        return VX_ERR_INVALID;
    }
    for (int d = 0; d < ndst; ++d)
        if (!dst[d]) { set_error("NULL gather destination %d", d); return VX_ERR_INVALID; }
    if (p->in == VX_FP32) { set_error("gather needs 16-bit inputs (tcgen05 rungs)"); return VX_ERR_UNSUPPORTED; }
    vx_status s = check_args(p, 1, M, N, K, A, M * K, B, N * K, dst[0], M * N);
    if (s != VX_OK) return s;
    if (M == 0) return VX_OK;
    if (p->device >= 0) {
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess || cur != p->device) {
            cudaGetLastError();
            set_error("current device %d != the plan's device %d", cur, p->device);
            return VX_ERR_INVALID;
        }
    }
    vx_choice ch;
    s = select_choice(p, 1, M, N, force_rung, force_split, &ch, kSelectGather);
    if (s != VX_OK) return s;
    if (used) *used = ch;
    GatherSpec g;
    g.ndst = ndst;
    g.row0 = row_offset;
    for (int d = 0; d < 8; ++d) g.dst[d] = d < ndst ? dst[d] : nullptr;
    return launch(p, ch, 1, M, N, K, A, M * K, B, N * K, dst[0], M * N, stream, &g);
}

vx_status vx_gemm_varlen(vx_plan_t p, int32_t ngroups, const int32_t* cu_host,
                         const int32_t* cu_dev, int64_t K, const void* Q, const void* Kt, void* S,
                         int32_t force_rung, void* stream, vx_choice* used) {
    if (!p || !cu_host || !cu_dev || !Q || !Kt || !S || ngroups < 1) {
        set_error("varlen: NULL argument or ngroups < 1"); return VX_ERR_INVALID;
    }
    if (p->N != 0 || p->in == VX_FP32 || p->bl != VX_B_NK) {
        set_error("varlen needs a dynamic-N (N = 0) 16-bit plan with B stored N x K (K^T rows)");
        return VX_ERR_UNSUPPORTED;
    }
    if (K != p->K) { set_error("K=%lld does not match the plan's K=%lld", (long long)K, (long long)p->K); return VX_ERR_INVALID; }
    if (cu_host[0] != 0) { set_error("cu_seqlens[0] must be 0"); return VX_ERR_INVALID; }
    for (int32_t g = 0; g < ngroups; ++g)
        if (cu_host[g + 1] < cu_host[g]) { set_error("cu_seqlens must be non-decreasing"); return VX_ERR_INVALID; }
    const int64_t total = cu_host[ngroups];
    if (total == 0) return VX_OK;
    if (K % 8 || !aligned16(Q) || !aligned16(Kt)) { set_error("varlen: K %% 8 and 16-B aligned Q, K^T"); return VX_ERR_ALIGN; }
    if (reinterpret_cast<uintptr_t>(S) % out_bytes(p->out)) { set_error("S must be element aligned"); return VX_ERR_ALIGN; }
    if (p->device >= 0) {
        int cur = -1;
        if (cudaGetDevice(&cur) != cudaSuccess || cur != p->device) {
            cudaGetLastError();
            set_error("current device %d != the plan's device %d", cur, p->device);
            return VX_ERR_INVALID;
        }
    }
    vx_choice ch;
    int64_t tiles = 0;
    vx_status s = select_varlen(p, cu_host, ngroups, force_rung, &ch, &tiles);
    if (s != VX_OK) return s;
    if (used) *used = ch;
    if (tiles == 0) return VX_OK;
    VarSpec v{cu_dev, ngroups, tiles};
    return launch(p, ch, 1, total, total, K, Q, total * K, Kt, total * K, S, total * total, stream,
                  nullptr, &v);
}

vx_status vx_gemm_host(vx_plan_t p, int64_t batch, int64_t M, int64_t N, int64_t K,
                       const void* A, const void* B, void* C, void* dA, void* dB, void* dC,
                       void* stream) {
    if (!p || !A || !B || !C || !dA || !dB || !dC) { set_error("NULL argument"); return VX_ERR_INVALID; }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int ib = in_bytes(p->in), ob = out_bytes(p->out);
    const size_t a_bytes = (size_t)(batch * M * K) * ib, b_bytes = (size_t)(batch * N * K) * ib;
    const size_t c_bytes = (size_t)(batch * M * N) * ob;
    cudaError_t e = cudaMemcpyAsync(dA, A, a_bytes, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dB, B, b_bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    vx_status s = vx_gemm_ex(p, batch, M, N, K, dA, M * K, dB, N * K, dC, M * N, -1, 0, stream, nullptr);
    if (s != VX_OK) return s;
    e = cudaMemcpyAsync(C, dC, c_bytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
    return VX_OK;
}

int64_t vx_packed_b_elems(vx_plan_t p, int64_t batch, int64_t N, int64_t K) {
    if (!p || batch < 1 || N < 1 || K < 1) return 0;
    return batch * cdiv(N, 64) * 64 * cdiv(K, 64) * 64;
}

vx_status vx_pack_b(vx_plan_t p, int64_t batch, int64_t N, int64_t K, vx_blayout src,
                    const void* B, int64_t sB, void* Bp, void* stream) {
    if (!p || !B || !Bp || batch < 1 || N < 1 || K < 1) { set_error("bad arguments"); return VX_ERR_INVALID; }
    if (p->bl != VX_B_PACKED || p->in == VX_FP32) { set_error("plan is not a 16-bit VX_B_PACKED plan"); return VX_ERR_UNSUPPORTED; }
    if (src != VX_B_KN && src != VX_B_NK) { set_error("source layout must be KN or NK"); return VX_ERR_INVALID; }
    if (N != p->N || K != p->K) { set_error("N/K do not match the plan"); return VX_ERR_INVALID; }
    if (!aligned16(Bp)) { set_error("packed buffer must be 16-byte aligned"); return VX_ERR_ALIGN; }
    const int64_t rb = cdiv(N, 64), kb = cdiv(K, 64);
    const int64_t chunks = batch * rb * kb * 512;
    const int64_t sBe = batch > 1 ? sB : N * K;
    vx_pack_b_kernel<<<(unsigned)std::min<int64_t>(cdiv(chunks, 256), 148 * 16), 256, 0,
                       reinterpret_cast<cudaStream_t>(stream)>>>(
        (const uint16_t*)B, (uint16_t*)Bp, N, K, sBe, src == VX_B_KN, rb, kb, chunks);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pack launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return VX_OK;
}

int64_t vx_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

void vx_map_cache_stats(int64_t* hits, int64_t* misses) {
    if (hits) *hits = g_map_hits.load(std::memory_order_relaxed);
    if (misses) *misses = g_map_misses.load(std::memory_order_relaxed);
}

/* Debug/tracing hook (not part of vx.h): subsequent tcgen05 launches write %globaltimer
 * stamps of 8 phases per CTA into `buf` (device, >= 8*grid u64); NULL disables. */
void vx_debug_set_trace(void* buf) { g_trace = reinterpret_cast<unsigned long long*>(buf); }

}  // extern "C"
