// vx_umma.cuh -- the tcgen05 ladder kernel (families 0 "umma" and 1 "umma_swap").
//
// One template realises a rung of the strategy table on sm_100a.  The
// paper's rKernel levels (Alg. 1; Table 1 GPU rows)
// map to:
//   L0  tcgen05.mma.cta_group::1.kind::f16, 128 x BN x 16, operands in SMEM, D in TMEM
//   L1  TMEM accumulator tile 128 lanes x BN fp32 columns, double buffered (2 x BN cols)
//   L2  CTA tile 128 x BN x 64: TMA (128-B swizzle) fills an S-stage SMEM ring -- the
//       "Load" stage (GlobalMem -> SharedMem); TRL loop = the K loop over 64-wide blocks
//   L3  grid: persistent CTAs over output tiles (PL loop), or a cluster of `splits` CTAs
//       splitting the K loop and reducing through distributed shared memory.
// Padding exists only at the grid level: TMA zero-fills rows/cols past M, N, K and the
// epilogue masks stores past M and N (fig:padding).
//
// Operand naming inside the kernel: "P" is the operand on the UMMA-M axis (128 rows per
// tile), "Q" the one on the UMMA-N axis (BN rows per tile).  family 0: P = A (rows of M),
// Q = B (rows of N).  family 1 (swap): P = B (N), Q = A (M), so skinny M sits on the
// narrow UMMA-N axis and N fills the 128-lane M axis (decode shapes).
//
// Warp roles (192 threads, one CTA per SM):
//   warp 0      TMA producer (one lane)
//   warp 1      TMEM allocator + MMA issuer (one lane issues every tcgen05.mma)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> global (warp w reads lanes
//               32*(w%4) .. +31 of the accumulator)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "vx_ptx.cuh"

namespace vx {

constexpr int kEpiWarp0 = 2;
constexpr int kEpiWarps = 8;   // two warps per TMEM lane quarter, splitting the column chunks
constexpr int kEpiThreads = kEpiWarps * 32;
// TMA producers: warp 0 and warp 10 take alternate k-blocks.  One thread issues a
// UTMALDG only every ~70-160 cycles plus ~70 for its mbarrier wait (tools/tma_bench.cu),
// so a single producer caps a CTA at ~0.26 us per 64-deep k-block whatever the tile size;
// two halve that and leave the 128xBN tiles MMA- or bandwidth-bound.
constexpr int kProdWarps = 2;
constexpr int kProdWarp1 = kEpiWarp0 + kEpiWarps;          // the second producer warp
// the second MMA issuer (dual-issue mode, DESIGN.md 4.1 "dual MMA issuers"): small-N tiles
// are paced by one thread's UTCHMMA / commit / wait sequence, so two warps take alternate
// units of a tile into two TMEM accumulators that the epilogue adds
constexpr int kMma2Warp = kProdWarp1 + 1;
constexpr int kThreads = (kMma2Warp + 1) * 32;
__device__ __forceinline__ bool is_epi_warp(int w) { return w >= kEpiWarp0 && w < kEpiWarp0 + kEpiWarps; }

struct UmmaParams {
    int M, N;                 // logical GEMM rows / cols (per batch)
    int tiles_p, tiles_q;     // tiles along the UMMA-M (P) and UMMA-N (Q) axes
    int num_tiles;            // batch * tiles_p * tiles_q
    int kb_total;             // 64-wide K blocks
    int splits;               // K-loop split (cluster size); 1 = persistent schedule
    int stages;               // SMEM ring depth
    int out_kind;             // 0 bf16, 1 fp16, 2 fp32
    int vec;                  // 1: C rows/batches 16-B aligned and N % 8 == 0 (vector stores)
    uint32_t idesc;           // tcgen05 instruction descriptor
    void* C;
    long long ldc;            // elements between rows of C
    long long sC;             // elements between batches of C
    unsigned long long* trace;  // optional per-CTA phase timestamps (VX_TRACE), else null
    int dbg;                    // debug bits (VX_DEBUG_FLAGS): 1 skip split push, 2 skip split
                                // reduce, 4 skip split C store, 8 skip epilogue stores,
                                // 32 skip stream-K fix-up, 1024 / 2048 operand loads
                                // evict_first / evict_normal (timing experiments only)
    int streamk;                // 1: stream-K schedule over (tile, k-block) units
    int pair;                   // 1: cta_group::2 pair rung (cluster of 2, 256-row tiles)
    int bpack;                  // 1: B is VX_B_PACKED (5-D map of 64 x 64 contiguous tiles)
    float* ws;                  // stream-K partial slots [gridDim.x][128][BN] fp32 (plan-owned)
    int* flags;                 // stream-K slot-ready flags [gridDim.x] (0 between launches)
    int mc;                     // TMA-multicast cluster size (1 = none): MC CTAs share the A
                                // operand tile (P when non-swapped, Q when swapped); tiles
                                // and num_tiles then count cluster tiles
    int a_bytes;                // bytes of A one stage loads: the whole A tile, or for M < 16
                                // a short box of round_up(M, 8) rows (DESIGN.md 4.1 "short
                                // A boxes"); the tile rows past it are never stored
    const int* cu;              // ragged batch: > 0 groups = varlen mode --
    int ngroups;                // sequence g has rows [cu[g], cu[g+1]) of the packed A (Q)
                                // and B (K^T, N x K); S_g = Q_g K_g^T is s_g x s_g row-major
                                // at element sum_{j<g} s_j^2 of C; tiles enumerate every
                                // sequence's (tp, tq) in order (non-swapped, persistent)
    int ndst;                   // fused GEMM + row all-gather: > 0 = the
                                // epilogue writes every finished C row chunk straight from
                                // registers into rows dst_row0 + m of each dst[d] (peer /
                                // symmetric-memory buffers over NVLink); C is not written
    long long dst_row0;
    void* dst[8];
    int group_p;                // raster group: P tiles per group swept over all Q tiles (L2)
    int kdouble;                // 1: two-chunk loads (tmP2 / tmQ2) fill two adjacent ring
                                // stages with one TMA box per operand (K % 64 == 0, K-major
                                // P and Q, unpacked; rings of >= 6 stages, >= 8 for pair
                                // rungs, whose two-chunk boxes use the .cta_group::2 form;
                                // DESIGN.md 4.1 "deep-K units")
};

// ---- work assignment (the L3 schedule of the rung) ---------------------------------------
// persistent: tiles blockIdx.x, +gridDim.x, ... each over the whole K range
// split:      one tile per cluster, K range [rank*K/s, (rank+1)*K/s)
// stream-K:   CTA c owns units [c*U/G, (c+1)*U/G) of U = tiles x k-blocks (tile-major);
//             a tile cut between CTAs is finished by the CTA holding its k-block 0, which
//             adds the other CTAs' fp32 partials in CTA order (deterministic)
struct WorkIter {
    long long u, u1;       // stream-K unit cursor / end
    int tile, step;        // persistent / split
    int ka, kn;            // split K range
    __device__ __forceinline__ WorkIter(const UmmaParams& p, int rank) {
        if (p.streamk) {
            // stream-K units are split over CTAs, or over CTA pairs for pair rungs
            const long long U = (long long)p.num_tiles * p.kb_total;
            const long long id = p.pair ? (blockIdx.x >> 1) : blockIdx.x;
            const long long G = p.pair ? (gridDim.x >> 1) : gridDim.x;
            u = id * U / G;
            u1 = (id + 1) * U / G;
        } else if (p.pair) {
            tile = blockIdx.x >> 1;          // both CTAs of a pair walk the same tiles
            step = gridDim.x >> 1;
            ka = 0;
            kn = p.kb_total;
        } else if (p.mc > 1) {
            tile = blockIdx.x / p.mc;        // every CTA of a multicast cluster walks the
            step = gridDim.x / p.mc;         // same cluster tiles in lockstep
            ka = 0;
            kn = p.kb_total;
        } else if (p.splits > 1) {
            tile = blockIdx.x / p.splits;
            step = p.num_tiles;
            kn = p.kb_total / p.splits;
            ka = rank * kn;
        } else {
            tile = blockIdx.x;
            step = gridDim.x;
            ka = 0;
            kn = p.kb_total;
        }
    }
    // next work item: tile and its k-block range [k0, k0+nk); false when done
    __device__ __forceinline__ bool next(const UmmaParams& p, int& t, int& k0, int& nk) {
        if (p.streamk) {
            if (u >= u1) return false;
            t = (int)(u / p.kb_total);
            k0 = (int)(u - (long long)t * p.kb_total);
            const long long rest = u1 - u;
            nk = (int)min((long long)(p.kb_total - k0), rest);
            u += nk;
            return true;
        }
        if (tile >= p.num_tiles) return false;
        t = tile;
        k0 = ka;
        nk = kn;
        tile += step;
        return true;
    }
};

// first unit of CTA c under the stream-K split (same formula as WorkIter)
__device__ __forceinline__ long long sk_first(long long c, long long U, long long G) { return c * U / G; }

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int ET = kEpiThreads>
__device__ __forceinline__ void epi_bar() {   // named barrier over the epilogue warps
    asm volatile("bar.sync 1, %0;" ::"n"(ET) : "memory");
}

constexpr int kTraceSlots = 56;   // 40-47: issue cycle of units 0-7, 48-55: their full-barrier wait exit
// phase trace (tracing aux subsystem): %globaltimer (ns) at fixed points, 20 slots per CTA
// (slots 12-15: MMA-issuer cycle counters, see the MMA loop)
__device__ __forceinline__ void trace_at(const UmmaParams& p, int slot) {
    if (p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[blockIdx.x * kTraceSlots + slot] = t;
    }
}
// cycle-counter stamp (slots 18-39): clock64() - base
__device__ __forceinline__ void cyc_at(const UmmaParams& p, int slot, long long base) {
    if (p.trace) p.trace[blockIdx.x * kTraceSlots + slot] = clock64() - base;
}

constexpr int kGroupP = 16;   // default raster: 16 P-tiles x all Q-tiles per group (L2 reuse)

template <int BN>
struct UmmaCfg {
    static constexpr int kPBytes = 128 * 64 * 2;
    static constexpr int kQBytes = BN * 64 * 2;
    static constexpr int kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
};

__device__ __forceinline__ void decode_tile(int tile, int tiles_p, int tiles_q, int& b, int& tp,
                                            int& tq, int gp = kGroupP) {
    const int per_b = tiles_p * tiles_q;
    b = tile / per_b;
    const int t = tile - b * per_b;
    const int group = t / (gp * tiles_q);
    const int first = group * gp;
    const int gsz = min(gp, tiles_p - first);
    const int local = t - group * gp * tiles_q;
    tp = first + local % gsz;
    tq = local / gsz;
}

// tile of CTA `crank` of a multicast cluster: cluster tile `tile` covers MC consecutive Q
// tiles sharing one P tile (non-swapped: A = P shared) or MC consecutive P tiles sharing one
// Q tile (swapped: A = Q shared); the group raster runs over cluster tiles
template <bool SWAP, int MC>
__device__ __forceinline__ void decode_ctile(int tile, int tiles_p, int tiles_q, uint32_t crank,
                                             int& b, int& tp, int& tq, int gp = kGroupP) {
    if (MC == 1) {
        decode_tile(tile, tiles_p, tiles_q, b, tp, tq, gp);
    } else if (!SWAP) {
        decode_tile(tile, tiles_p, (tiles_q + MC - 1) / MC, b, tp, tq, gp);
        tq = tq * MC + (int)crank;
    } else {
        decode_tile(tile, (tiles_p + MC - 1) / MC, tiles_q, b, tp, tq, gp);
        tp = tp * MC + (int)crank;
    }
}

// varlen mode: tile -> (tp, tq) within its sequence, the sequence's length, first packed row
// and offset of its S block; O(groups) per call, groups are few (attention batch)
struct VarTile {
    int len, row0;
    long long coff;
};
template <int BN>
__device__ __forceinline__ void decode_varlen(int tile, const int* cu, int ng, int& tp, int& tq,
                                              VarTile& v) {
    long long coff = 0;
    int t = tile;
    int prev = __ldg(cu);
    for (int g = 0; g < ng; ++g) {
        const int next = __ldg(cu + g + 1);
        const int len = next - prev;
        const int tn = (len + BN - 1) / BN;
        const int nt = ((len + 127) / 128) * tn;
        if (t < nt) {
            tp = t / tn;
            tq = t - tp * tn;
            v.len = len;
            v.row0 = prev;
            v.coff = coff;
            return;
        }
        t -= nt;
        coff += (long long)len * len;
        prev = next;
    }
    tp = tq = 0;
    v.len = 0; v.row0 = 0; v.coff = 0;
}

__device__ __forceinline__ uint32_t pack2(float a, float b, int kind) {
    if (kind == 0) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void store1(void* C, long long idx, float v, int kind) {
    if (kind == 2) {
        reinterpret_cast<float*>(C)[idx] = v;
    } else if (kind == 0) {
        reinterpret_cast<__nv_bfloat16*>(C)[idx] = __float2bfloat16_rn(v);
    } else {
        reinterpret_cast<__half*>(C)[idx] = __float2half_rn(v);
    }
}

// 8 consecutive columns of one row (n % 8 == 0, N % 8 == 0 -> all-or-nothing in N)
__device__ __forceinline__ void store8(void* C, long long idx, const float* f, int kind) {
    if (kind == 2) {
        float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + idx);
        p[0] = make_float4(f[0], f[1], f[2], f[3]);
        p[1] = make_float4(f[4], f[5], f[6], f[7]);
    } else {
        uint4 u;
        u.x = pack2(f[0], f[1], kind);
        u.y = pack2(f[2], f[3], kind);
        u.z = pack2(f[4], f[5], kind);
        u.w = pack2(f[6], f[7], kind);
        *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(C) + idx) = u;
    }
}

// 4 consecutive columns (split-K reduce path, n % 4 == 0)
__device__ __forceinline__ void store4(void* C, long long idx, float4 v, int kind) {
    if (kind == 2) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(C) + idx) = v;
    } else {
        uint2 u;
        u.x = pack2(v.x, v.y, kind);
        u.y = pack2(v.z, v.w, kind);
        *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(C) + idx) = u;
    }
}

// ---- compact epilogue helpers ---------------------------------------------------------------
// The epilogue runs once per tile, so its instructions are usually cold (the operand stream
// evicts them from L2): keep this code small -- one dtype branch per chunk, rare paths out
// of line.

// 16-bit conversion of n floats (n even) into packed pairs
template <int W>
__device__ __forceinline__ void pack_chunk(const float* f, uint32_t* u, int kind) {
    if (kind == 0) {
#pragma unroll
        for (int i = 0; i < W / 2; ++i) {
            __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
            u[i] = *reinterpret_cast<uint32_t*>(&h);
        }
    } else {
#pragma unroll
        for (int i = 0; i < W / 2; ++i) {
            __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
            u[i] = *reinterpret_cast<uint32_t*>(&h);
        }
    }
}

// row-major chunk of W columns starting at column n0 of row `base` (non-swap, vector path)
template <int W>
__device__ __forceinline__ void store_row_chunk(char* Cb, long long base, int n0, int N,
                                                const float* f, int kind) {
    if (kind == 2) {
        float* c = reinterpret_cast<float*>(Cb) + base + n0;
#pragma unroll
        for (int j = 0; j < W; j += 4)
            if (n0 + j < N) *reinterpret_cast<float4*>(c + j) = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
    } else {
        uint32_t u[W / 2];
        pack_chunk<W>(f, u, kind);
        uint16_t* c = reinterpret_cast<uint16_t*>(Cb) + base + n0;
#pragma unroll
        for (int j = 0; j < W; j += 8)
            if (n0 + j < N)
                *reinterpret_cast<uint4*>(c + j) = make_uint4(u[j / 2], u[j / 2 + 1], u[j / 2 + 2], u[j / 2 + 3]);
    }
}

// scalar fallback (C rows not 16-B aligned or N % 8 != 0): rare, kept out of line
static __device__ __noinline__ void store_row_scalar(char* Cb, long long base, int n0, int N, int W,
                                              const float* f, int kind) {
    for (int j = 0; j < W; ++j)
        if (n0 + j < N) store1(Cb, base + n0 + j, f[j], kind);
}

// rows that are not 16-B aligned (N % 8 != 0, e.g. attention scores with s % 8 != 0, or a
// ragged sequence): the warp transposes its 32 rows x W columns through its 4-KB staging
// buffer (XOR-swizzled, conflict-free both ways), then writes row by row with consecutive
// lanes on consecutive columns -- coalesced, instead of 32 lanes hitting 32 rows per store
template <int W>
__device__ __forceinline__ void store_rows_coalesced(float* st, char* Cb, long long ldc, int row0,
                                                     int M, int n0, int N, const float* f,
                                                     int kind, int lane) {
#pragma unroll
    for (int j = 0; j < W; ++j) st[lane * 32 + (j ^ lane)] = f[j];
    __syncwarp();
    const int col = n0 + lane;
#pragma unroll 1
    for (int r = 0; r < 32; ++r) {
        const int row = row0 + r;
        if (row >= M) break;                         // warp-uniform
        if (lane < W && col < N) store1(Cb, (long long)row * ldc + col, st[r * 32 + (lane ^ r)], kind);
    }
    __syncwarp();
}

// 16-bit rows that are 8-B but not 16-B aligned (N % 8 == 4, e.g. attention s = 100, 1500):
// the lane (= tile row) packs its W columns to 16 bit and writes them to row `lane` of a
// [32 rows][64 B] staging tile as 16-B vectors (granule g of row r at g ^ ((r >> 1) & 3):
// conflict-free both ways); then each store instruction covers 4 rows x 32 columns, one
// 8-B shared load + one 8-B global store per lane, so a row's W columns leave as one
// contiguous 64-B segment (N % 4 == 0: 4 columns are all-or-nothing)
template <int W>
__device__ __forceinline__ void store_rows_coalesced8(float* st, char* Cb, long long ldc, int row0,
                                                      int M, int n0, int N, const float* f,
                                                      int kind, int lane) {
    uint32_t u[W / 2];
    pack_chunk<W>(f, u, kind);
    const uint32_t sb = ptx::smem_addr(st);
#pragma unroll
    for (int g = 0; g < W / 8; ++g)
        ptx::st_shared_v4(sb + (uint32_t)lane * 64u + ((uint32_t)(g ^ ((lane >> 1) & 3)) << 4),
                          u[4 * g], u[4 * g + 1], u[4 * g + 2], u[4 * g + 3]);
    __syncwarp();
    const int c = (lane & 7) * 4;
    const uint32_t coff = (uint32_t)(c & 4) * 2u;          // byte offset inside the granule
#pragma unroll 1
    for (int it = 0; it < 8; ++it) {
        const int r = it * 4 + (lane >> 3);
        const int row = row0 + r;
        if (row < M && c < W && n0 + c < N) {
            const uint2 v = ptx::ld_shared_v2(sb + (uint32_t)r * 64u +
                                              ((uint32_t)((c >> 3) ^ ((r >> 1) & 3)) << 4) + coff);
            *reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(Cb) + (long long)row * ldc + n0 + c) = v;
        }
    }
    __syncwarp();
}

// transposed chunk (swap): lane owns output column `col`, registers are rows m0..m0+W-1
template <int W>
__device__ __forceinline__ void store_col_chunk(char* Cb, long long ldc, int col, int m0, int M,
                                                const float* f, int kind) {
    if (kind == 2) {
        float* c = reinterpret_cast<float*>(Cb) + col;
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (m0 + j < M) c[(long long)(m0 + j) * ldc] = f[j];
    } else {
        uint32_t u[W / 2];
        pack_chunk<W>(f, u, kind);
        uint16_t* c = reinterpret_cast<uint16_t*>(Cb) + col;
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (m0 + j < M) c[(long long)(m0 + j) * ldc] = (uint16_t)(u[j / 2] >> (16 * (j & 1)));
    }
}

// stream-K: add the fp32 partials of CTAs c0..c1 (in that order) for accumulator row `row`,
// columns col0 .. col0+W-1, into the W values held as fp32 bits in v
// stream-K slot / flag of contributor id j (a CTA, or CTA `rank` of pair j)
template <bool PAIR>
__device__ __forceinline__ int sk_slot(int j, uint32_t rank) { return PAIR ? 2 * j + (int)rank : j; }

template <int W, bool PAIR = false>
__device__ __forceinline__ void add_partials(uint32_t* v, const float* ws, int c0, int c1, int row,
                                             int col0, int bn, uint32_t rank = 0) {
#pragma unroll 1
    for (int j = c0; j <= c1; ++j) {
        // slot layout [col/4][row][4]: a warp's 32 rows read 512 contiguous bytes
        const float* src = ws + (long long)sk_slot<PAIR>(j, rank) * 128 * bn +
                           ((long long)(col0 / 4) * 128 + row) * 4;
#pragma unroll
        for (int i = 0; i < W; i += 4) {
            const float4 t = __ldcg(reinterpret_cast<const float4*>(src + i * 128));
            v[i] = __float_as_uint(__uint_as_float(v[i]) + t.x);
            v[i + 1] = __float_as_uint(__uint_as_float(v[i + 1]) + t.y);
            v[i + 2] = __float_as_uint(__uint_as_float(v[i + 2]) + t.z);
            v[i + 3] = __float_as_uint(__uint_as_float(v[i + 3]) + t.w);
        }
    }
}

// stream-K: every epilogue warp has consumed slots c0..c1 -> clear their flags for the next
// launch (each slot is produced and consumed exactly once per launch)
template <bool PAIR, int ET = kEpiThreads>
__device__ __forceinline__ void sk_reset(const UmmaParams& p, int c0, int c1, uint32_t rank) {
    epi_bar<ET>();
    if (threadIdx.x == kEpiWarp0 * 32)
        for (int j = c0; j <= c1; ++j) p.flags[sk_slot<PAIR>(j, rank)] = 0;
}

// dual MMA issuers: add the second issuer's accumulator (W columns at TMEM address a2) into
// the W fp32 values (as bits) already loaded from the first one -- fixed order acc0 + acc1
template <int W>
__device__ __forceinline__ void acc_add(uint32_t a2, uint32_t* v) {
    uint32_t w[32];
    if (W >= 32) ptx::tmem_ld32(a2, w);
    else ptx::tmem_ld16(a2, w);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < W; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
}

// SWAP: P = B, Q = A.  P_MN / Q_MN: that operand is MN-major in SMEM (B stored K x N).
// PAIR: cta_group::2 rung -- a cluster of 2 CTAs computes a 256 x BN tile; each CTA loads
// its 128 rows of A and BN/2 rows of B, the leader (rank 0) issues the 256-row MMAs, each
// CTA's TMEM holds its 128 rows of the accumulator (non-swap, persistent schedule only).
// MC: TMA-multicast cluster of MC CTAs sharing the A tile (persistent schedule only): each
// CTA loads 1/MC of the shared tile's rows and multicasts them to the whole cluster; a
// stage is refilled only when all MC CTAs' MMAs released it (empty barriers count MC).
// LEAN: occupancy-2 variant (DESIGN.md 4.1 "lean CTAs"): 1 producer + 1 MMA + 4 epilogue
// warps (192 threads, <= 170 registers) and a ring of <= ~110 KB, so two CTAs fit on an SM
// and a launch's CTAs become resident while the previous grid on the stream still holds its
// SMs (programmatic dependent launch overlaps their prologue on every SM)
template <int BN, bool SWAP, bool P_MN, bool Q_MN, bool PAIR = false, int MC = 1, bool LEAN = false>
__global__ void __launch_bounds__(LEAN ? 192 : kThreads, LEAN ? 2 : 1)
    vx_umma_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmP2,
                   const __grid_constant__ CUtensorMap tmQ2, const __grid_constant__ UmmaParams p) {
    static_assert(!PAIR || !SWAP, "pair rungs are non-swapped");
    static_assert(MC == 1 || !PAIR, "multicast clusters are cta_group::1");
    static_assert(MC == 1 || (SWAP ? BN / MC : 128 / MC) % 8 == 0,
                  "multicast sub-boxes are whole 8-row swizzle atoms");
    static_assert(!LEAN || (!PAIR && MC == 1 && BN <= 128), "lean CTAs: cta_group::1, BN <= 128");
    constexpr int EW = LEAN ? 4 : kEpiWarps;    // epilogue warps
    constexpr int ET = EW * 32;
    constexpr int NG = EW / 4;                  // epilogue warps per TMEM lane quarter
    constexpr int PW = LEAN ? 1 : kProdWarps;   // TMA producer warps
    constexpr int PW1 = kEpiWarp0 + EW;         // the second producer warp (PW == 2)
    constexpr bool MCP = MC > 1 && !SWAP;   // A = P is the multicast operand
    constexpr bool MCQ = MC > 1 && SWAP;    // A = Q is the multicast operand
    constexpr uint16_t kMcMask = (uint16_t)((1u << MC) - 1);
    using Cfg = UmmaCfg<BN>;
    // dual MMA issuers: cta_group::1, no multicast, BN <= 64 (4 BN TMEM columns: two issuers
    // x two accumulator buffers).  Not for BN = 128: a 128 x 128 x 16 MMA already keeps the
    // tensor pipe busy ~2x its issue time, so a second issuer gains nothing while the epilogue
    // reads twice the TMEM (measured A/B over 7 shapes x every schedule: BN 16 / 32 / 64
    // x1.12 / x1.08 / x1.05, BN 128 x0.91; tools/dual_ab.py)
    constexpr bool DUALOK = !PAIR && MC == 1 && !LEAN && BN <= 64;
    constexpr int kCols = DUALOK ? (4 * BN <= 32 ? 32 : 4 * BN) : Cfg::kTmemCols;
    constexpr int kP = Cfg::kPBytes;
    constexpr int kQ = PAIR ? Cfg::kQBytes / 2 : Cfg::kQBytes;   // this CTA's B rows
    extern __shared__ __align__(1024) uint8_t smem_raw[];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int S = p.stages;
    const long long cyc_entry = clock64();
    if (threadIdx.x == 0) trace_at(p, 0);

    // layout: [barriers | pad to 1024 | S x P tiles | S x Q tiles]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* redbar = tempty + 2;   // split mode: the peers' partial rows have landed
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(redbar + 1);
    const uint32_t raw_addr = ptx::smem_addr(smem_raw);
    const uint32_t tile_off = ((raw_addr + 512 + 1023) & ~1023u) - raw_addr;
    uint8_t* sP = smem_raw + tile_off;
    uint8_t* sQ = sP + S * kP;
    uint8_t* sE = sQ + S * kQ;  // epilogue staging: 4 warps x 2 x 4 KB (TMA-store tiles)

    // dual MMA issuers (DUALOK rungs walking the unit ring): warps 1 and kMma2Warp take
    // alternate units of every tile into accumulators 2 acc and 2 acc + 1 (BN columns each)
    const bool dual = DUALOK && p.kdouble && !P_MN && !Q_MN && !p.bpack &&
                      !(p.dbg & 8192) && !(p.dbg & 262144);
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmP);
        ptx::prefetch_tmap(&tmQ);
        if (p.vec) ptx::prefetch_tmap(&tmC);
        if (p.kdouble) {
            ptx::prefetch_tmap(&tmP2);
            ptx::prefetch_tmap(&tmQ2);
        }
        for (int i = 0; i < S; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], MC);   // one release per consuming CTA of the cluster
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], dual ? 2 : 1);   // one commit per MMA issuer
            ptx::mbar_init(&tempty[i], PAIR ? 2 * EW : EW);
        }
        ptx::mbar_init(redbar, 1);
        ptx::fence_mbar_init();
        cyc_at(p, 24, cyc_entry);
    }
    if (warp == 1) {
        const long long c = clock64();
        if (PAIR) ptx::tmem_alloc_pair<kCols>(tmem_holder);
        else ptx::tmem_alloc<kCols>(tmem_holder);
        if (lane == 0) cyc_at(p, 28, c);
    }
    ptx::tc_fence_before();
    if (PAIR || MC > 1) ptx::cluster_sync();   // every CTA's barriers initialised before any
    else __syncthreads();                      // remote arrive / multicast write
    ptx::tc_fence_after();
    const uint32_t prank = PAIR ? ptx::cluster_ctarank() : 0;   // 0 = pair leader
    const uint32_t crank = MC > 1 ? ptx::cluster_ctarank() : 0; // rank in a multicast cluster
    const uint32_t tmem_base = *tmem_holder;
    if (threadIdx.x == 0) { trace_at(p, 1); cyc_at(p, 26, cyc_entry); }
    // Programmatic dependent launch: everything up to each role's first global access
    // overlaps the previous kernel.  Each role waits for the previous grid right before it
    // touches global memory: the producers after their first-tile bookkeeping and ring
    // setup (so that code, cold in the instruction cache at every launch, runs before the
    // wait, tools/timeline.py cycle stamps), the epilogue warps before anything else; the
    // MMA warp never touches global memory.

    const bool split = p.splits > 1;
    const int rank = split ? (int)(blockIdx.x % p.splits) : 0;
    const int tile0 = split ? (int)(blockIdx.x / p.splits) : (int)blockIdx.x;  // split mode

    if (warp == 0 || (PW > 1 && warp == PW1)) {
        if (lane == 0) {
            // ===== TMA producers: producer `pid` takes this CTA's k-blocks j % 2 == pid =====
            const int pid = warp == 0 ? 0 : 1;
            const bool kd = p.kdouble && !P_MN && !Q_MN && !p.bpack && MC == 1;
            // unit ring (deep-K, cta_group::1): the ring is walked in fixed stage pairs, one
            // barrier round trip per two k-blocks on both sides
            const bool ur = !PAIR && kd && !(p.dbg & 8192);
            // units in the ring (an odd last stage is unused).  With dual issuers the count is
            // EVEN, so every slot is always consumed by the same issuer: the parity waits on a
            // slot must never run a round ahead, which an issuer skipping the other's units
            // could otherwise do on a slot whose rounds alternate between issuers
            const int NU = dual ? ((S / 2) & ~1) : S / 2;
            int unit = 0;
            const long long cy0 = p.trace ? clock64() : 0;   // trace: setup -> first issue
            const uint64_t pol = (p.dbg & 1024) ? ptx::policy_evict_first()
                               : (p.dbg & 2048) ? ptx::policy_evict_normal()
                                                : ptx::policy_evict_last();
            if (pid == 0) cyc_at(p, 20, cy0);
            int stage = 0;
            uint32_t phase = 0;
            bool stamped = pid != 0;
            bool waited = false;
            int j = 0;                       // running k-block count of this CTA
            // first k-block of this producer: the grid dependency wait (no global memory is
            // touched before it).  An L2 prefetch of the CTA's first ring before the wait
            // (VX_DEBUG_FLAGS 128 turns it back on, A/B only) was measured to DELAY the real
            // loads -- the prefetches occupy the CTA's TMA queue ahead of them: BERT-size
            // launches 5.9 -> 5.1 us without it
            auto dep_wait = [&](int tile_, int kb_, int nleft) {
                if (waited) return;
                if (pid == 0 && (p.dbg & 128) && !p.bpack && !P_MN && !Q_MN) {
                    int b_ = 0, tp_, tq_;
                    VarTile v_{0, 0, 0};
                    if (p.ngroups) decode_varlen<BN>(tile_, p.cu, p.ngroups, tp_, tq_, v_);
                    else decode_ctile<SWAP, MC>(tile_, p.tiles_p, p.tiles_q, crank, b_, tp_, tq_, p.group_p);
                    // this CTA's own rows (its half of a pair, its 1/MC share of the
                    // multicast operand): the maps' boxes are sized to them
                    const int pp = PAIR ? tp_ * 256 + (int)prank * 128
                                 : tp_ * 128 + v_.row0 + (MCP ? (int)crank * (128 / MC) : 0);
                    const int qq = PAIR ? tq_ * BN + (int)prank * (BN / 2)
                                 : tq_ * BN + v_.row0 + (MCQ ? (int)crank * (BN / MC) : 0);
                    const int n = nleft < S ? nleft : S;
                    for (int kb2 = kb_; kb2 < kb_ + n; ++kb2) {
                        ptx::tma_prefetch_3d(&tmP, kb2 * 64, pp, b_);
                        ptx::tma_prefetch_3d(&tmQ, kb2 * 64, qq, b_);
                    }
                }
                ptx::grid_dep_wait();
                waited = true;
                if (pid == 0) { trace_at(p, 8); cyc_at(p, 27, cyc_entry); }
            };
            WorkIter wi(p, rank);
            if (pid == 0) cyc_at(p, 21, cy0);
            int tile, k0, nk;
            while (wi.next(p, tile, k0, nk)) {
                int b = 0, tp, tq;
                VarTile vt{0, 0, 0};   // varlen: the sequence's first packed row offsets P and Q
                if (p.ngroups) decode_varlen<BN>(tile, p.cu, p.ngroups, tp, tq, vt);
                else decode_ctile<SWAP, MC>(tile, p.tiles_p, p.tiles_q, crank, b, tp, tq, p.group_p);
                if (pid == 0 && j == 0) cyc_at(p, 22, cy0);
                if (ur) {
                    // unit ring: unit u = stages (2u, 2u+1), one full / one empty barrier
                    // (the even stage's); a unit carries two k-blocks (one two-chunk box per
                    // operand) or the range's last odd one (plain boxes into stage 2u)
                    for (int kb = k0; kb < k0 + nk; kb += 2, ++j) {
                        const int n2 = k0 + nk - kb >= 2 ? 2 : 1;
                        if (j % PW != pid) {
                            if (++unit == NU) { unit = 0; phase ^= 1; }
                            continue;
                        }
                        const int st = 2 * unit;
                        ptx::mbar_wait(&empty[st], phase ^ 1);
                        if (j == 0) cyc_at(p, 23, cy0);
                        if (j < 8) cyc_at(p, 40 + j, cyc_entry);
                        ptx::mbar_arrive_expect_tx(&full[st], n2 * (kP + kQ));
                        dep_wait(tile, kb, k0 + nk - kb);
                        if (!stamped && kb == k0) trace_at(p, 11);
                        uint8_t* dP = sP + st * kP;
                        uint8_t* dQ = sQ + st * kQ;
                        if (n2 == 2) {
                            ptx::tma_load_4d(dP, &tmP2, &full[st], 0, tp * 128 + vt.row0, kb, b, pol);
                            ptx::tma_load_4d(dQ, &tmQ2, &full[st], 0, tq * BN + vt.row0, kb, b, pol);
                        } else {
                            ptx::tma_load_3d(dP, &tmP, &full[st], kb * 64, tp * 128 + vt.row0, b, pol);
                            ptx::tma_load_3d(dQ, &tmQ, &full[st], kb * 64, tq * BN + vt.row0, b, pol);
                        }
                        if (++unit == NU) { unit = 0; phase ^= 1; }
                    }
                    continue;
                }
                for (int kb = k0; kb < k0 + nk; ++kb, ++j) {
                    // a unit is one k-block, or two (deep-K) when the next k-block of this
                    // range lands in the next ring stage without a wrap; the MMA issuer walks
                    // the same rule; j counts units, alternating between the producers
                    const bool dbl = kd && kb + 1 < k0 + nk && stage + 1 < S;
                    if (j % PW != pid) {
                        if (dbl) { ++kb; ++stage; }
                        if (++stage == S) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    if (dbl) ptx::mbar_wait(&empty[stage + 1], phase ^ 1);
                    if (j == 0) cyc_at(p, 23, cy0);
                    if (j < 8) cyc_at(p, 40 + j, cyc_entry);
                    if (kb >= k0 + PW && !stamped) { trace_at(p, 10); stamped = true; }
                    uint8_t* dP = sP + stage * kP;
                    uint8_t* dQ = sQ + stage * kQ;
                    if (PAIR && dbl) {
                        // deep-K unit of a pair: both CTAs' two-chunk boxes complete on the
                        // leader's full[stage]; the leader's full[stage + 1] gets a plain arrive
                        if (prank == 0) {
                            ptx::mbar_arrive_expect_tx(&full[stage], 4 * (kP + kQ));
                            ptx::mbar_arrive(&full[stage + 1]);
                        }
                        dep_wait(tile, kb, k0 + nk - kb);
                        ptx::tma_load_4d_pair(dP, &tmP2, &full[stage], 0, tp * 256 + (int)prank * 128,
                                              kb, b, pol);
                        ptx::tma_load_4d_pair(dQ, &tmQ2, &full[stage], 0,
                                              tq * BN + (int)prank * (BN / 2), kb, b, pol);
                        ++kb;
                        stage += 2;
                        if (stage == S) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if (PAIR) {
                        // both halves complete on the leader's full barrier
                        if (prank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * (kP + kQ));
                        dep_wait(tile, kb, k0 + nk - kb);
                        ptx::tma_load_3d_pair(dP, &tmP, &full[stage], kb * 64,
                                              tp * 256 + (int)prank * 128, b, pol);
                        if (p.bpack) {             // this CTA's BN/2 rows = BN/128 packed tiles
                            const int r0 = (tq * BN + (int)prank * (BN / 2)) / 64;
#pragma unroll
                            for (int a = 0; a < BN / 128; ++a)
                                ptx::tma_load_5d_pair(dQ + a * 8192, &tmQ, &full[stage], 0, 0, kb,
                                                      r0 + a, b, pol);
                        } else if (Q_MN) {
#pragma unroll
                            for (int a = 0; a < BN / 128; ++a)
                                ptx::tma_load_3d_pair(dQ + a * 8192, &tmQ, &full[stage],
                                                      tq * BN + (int)prank * (BN / 2) + a * 64,
                                                      kb * 64, b, pol);
                        } else {
                            ptx::tma_load_3d_pair(dQ, &tmQ, &full[stage], kb * 64,
                                                  tq * BN + (int)prank * (BN / 2), b, pol);
                        }
                        if (++stage == S) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if (!stamped && kb == k0 && p.trace) {
                        p.trace[blockIdx.x * kTraceSlots + 18] = clock64() - cy0;
                    }
                    if (dbl) {
                        // both chunks complete on full[stage]; full[stage + 1] gets a plain
                        // arrive so every barrier still completes once per ring round
                        ptx::mbar_arrive_expect_tx(&full[stage], 2 * (kP + kQ));
                        ptx::mbar_arrive(&full[stage + 1]);
                        dep_wait(tile, kb, k0 + nk - kb);
                        if (!stamped && kb == k0) trace_at(p, 11);
                        ptx::tma_load_4d(dP, &tmP2, &full[stage], 0, tp * 128 + vt.row0, kb, b, pol);
                        ptx::tma_load_4d(dQ, &tmQ2, &full[stage], 0, tq * BN + vt.row0, kb, b, pol);
                        ++kb;
                        stage += 2;
                        if (stage == S) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    // A may arrive as a short box (M < 16): expect exactly the bytes loaded
                    ptx::mbar_arrive_expect_tx(&full[stage], SWAP ? kP + p.a_bytes : p.a_bytes + kQ);
                    dep_wait(tile, kb, k0 + nk - kb);
                    if (!stamped && kb == k0) trace_at(p, 11);
                    if (p.bpack) {
                        // B pre-packed: every 64-row block of the B tile is one 8-KB box
                        if (SWAP) {
#pragma unroll
                            for (int a = 0; a < 2; ++a)
                                ptx::tma_load_5d(dP + a * 8192, &tmP, &full[stage], 0, 0, kb,
                                                 tp * 2 + a, b, pol);
                            ptx::tma_load_3d(dQ, &tmQ, &full[stage], kb * 64, tq * BN, b, pol);
                        } else {
                            ptx::tma_load_3d(dP, &tmP, &full[stage], kb * 64, tp * 128, b, pol);
#pragma unroll
                            for (int a = 0; a < BN / 64; ++a)
                                ptx::tma_load_5d(dQ + a * 8192, &tmQ, &full[stage], 0, 0, kb,
                                                 tq * (BN / 64) + a, b, pol);
                        }
                        if (++stage == S) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if (P_MN) {  // [64 K rows x 64 MN] atoms, 8 KB apart
#pragma unroll
                        for (int a = 0; a < 2; ++a)
                            ptx::tma_load_3d(dP + a * 8192, &tmP, &full[stage], tp * 128 + a * 64,
                                             kb * 64, b, pol);
                    } else if (MCP) {
                        // this CTA's 128/MC rows of the shared P tile, into every CTA's stage
                        ptx::tma_load_3d_mc(dP + crank * (kP / MC), &tmP, &full[stage], kb * 64,
                                            tp * 128 + (int)crank * (128 / MC), b, kMcMask, pol);
                    } else {
                        ptx::tma_load_3d(dP, &tmP, &full[stage], kb * 64, tp * 128 + vt.row0, b, pol);
                    }
                    if (Q_MN) {
#pragma unroll
                        for (int a = 0; a < BN / 64; ++a)
                            ptx::tma_load_3d(dQ + a * 8192, &tmQ, &full[stage], tq * BN + a * 64,
                                             kb * 64, b, pol);
                    } else if (MCQ) {
                        // this CTA's BN/MC rows of the shared Q tile, into every CTA's stage
                        ptx::tma_load_3d_mc(dQ + crank * (kQ / MC), &tmQ, &full[stage], kb * 64,
                                            tq * BN + (int)crank * (BN / MC), b, kMcMask, pol);
                    } else {
                        ptx::tma_load_3d(dQ, &tmQ, &full[stage], kb * 64, tq * BN + vt.row0, b, pol);
                    }
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
            ptx::grid_dep_launch();  // all loads issued: let the next grid start its prologue
            if (MC > 1 && pid == 0) {
                // multicast tail: every CTA's MMA releases this CTA's stages remotely; wait
                // until each stage's last release has arrived, so no remote arrive can
                // target this CTA after it passes the final cluster barrier
                for (int i = 0; i < S; ++i) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
            if (pid == 0) trace_at(p, 2);
        }
    } else if (warp == 1 || (dual && warp == kMma2Warp)) {
        if (prank == 0) {
            // ===== MMA issuer: the whole warp walks the loop (warp-uniform operands), one
            // elected lane issues (the pair leader's warp for PAIR rungs); with dual
            // issuers warp kMma2Warp takes the odd units of every tile =====
            const int mi = warp == 1 ? 0 : 1;
            long long cyc_wait = 0, cyc_mma = 0, cyc_commit = 0, cyc_n = 0;   // trace only
            const bool tr = p.trace != nullptr;
            const uint32_t idesc = p.idesc;
            const bool mma_off = (p.dbg & 512) != 0;   // debug: TMA streaming only
            // stage-0 operand descriptors; a stage / k-step only moves the 14-bit start
            // address field (addr >> 4), so later descriptors are one 64-bit add away
            const uint64_t dP_base = P_MN ? ptx::sdesc_mn_sw128(ptx::smem_addr(sP), 8192)
                                          : ptx::sdesc_k_sw128(ptx::smem_addr(sP));
            const uint64_t dQ_base = Q_MN ? ptx::sdesc_mn_sw128(ptx::smem_addr(sQ), 8192)
                                          : ptx::sdesc_k_sw128(ptx::smem_addr(sQ));
            constexpr uint32_t kStepP = P_MN ? (2048 >> 4) : (32 >> 4);   // per UMMA_K=16
            constexpr uint32_t kStepQ = Q_MN ? (2048 >> 4) : (32 >> 4);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            const bool kd = p.kdouble && !P_MN && !Q_MN && !p.bpack && MC == 1;
            const bool ur = !PAIR && kd && !(p.dbg & 8192);   // unit ring (producers' rule)
            const int NU = dual ? ((S / 2) & ~1) : S / 2;   // as the producers
            int unit = 0;
            long long gu = 0;   // units walked so far (all tiles): issuer = gu % 2
            WorkIter wi(p, rank);
            int tile, k0, nk;
            for (; wi.next(p, tile, k0, nk); ++it) {
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + (dual ? acc * 2 + mi : acc) * BN;
                // one iteration per unit: a k-block, or a deep-K pair of k-blocks that landed
                // together on full[stage] (the producers' rule) -- one wait, 4 or 8 MMAs, one
                // commit per stage.  The second stage's barrier only got the producer's plain
                // arrive; its phase completes without a waiter, which keeps every barrier at
                // one completion per ring round, so the parity this loop tracks stays exact.
                // (Per-unit MMA-warp time is what bounds small tiles: DESIGN.md 4.4.)
                int nunit = 0;   // trace: units of the first tile
                if (ur) {
                    int myk = 0;   // k-blocks this issuer has accumulated in this tile
                    for (int i = 0; i < nk; i += 2) {
                        const int n2 = nk - i >= 2 ? 2 : 1;
                        const int st = 2 * unit;
                        // the issuer of a unit is the parity of its GLOBAL index, so with an
                        // even NU every ring slot always has the same issuer
                        if (dual && (int)(gu++ & 1) != mi) {   // the other issuer's unit
                            if (++unit == NU) { unit = 0; phase ^= 1; }
                            continue;
                        }
                        const long long c0 = tr ? clock64() : 0;
                        ptx::mbar_wait(&full[st], phase);
                        ptx::tc_fence_after();
                        const long long c1 = tr ? clock64() : 0;
                        if (it == 0 && i == 0 && lane == 0 && mi == 0) trace_at(p, 3);
                        if (tr && it == 0 && lane == 0 && mi == 0 && nunit < 8)
                            cyc_at(p, 48 + nunit, cyc_entry);
                        ++nunit;
                        const uint64_t dp0 = dP_base + (uint64_t)(st * (kP >> 4));
                        const uint64_t dq0 = dQ_base + (uint64_t)(st * (kQ >> 4));
                        long long c2 = 0;
                        if (ptx::elect_one()) {
                            if (!mma_off) {
#pragma unroll
                                for (int k = 0; k < 8; ++k) {
                                    if (k >= 4 && n2 == 1) break;
                                    const uint64_t dp = dp0 + (k >> 2) * (kP >> 4) + (k & 3) * kStepP;
                                    const uint64_t dq = dq0 + (k >> 2) * (kQ >> 4) + (k & 3) * kStepQ;
                                    ptx::umma_f16(d_tmem, dp, dq, idesc, (myk | k) != 0);
                                }
                            }
                            c2 = tr ? clock64() : 0;
                            ptx::umma_commit(&empty[st]);   // frees both stages of the unit
                            if (tr) {
                                const long long c3 = clock64();
                                cyc_wait += c1 - c0; cyc_mma += c2 - c1; cyc_commit += c3 - c2; ++cyc_n;
                            }
                        }
                        __syncwarp();
                        if (!dual) ++gu;
                        myk += n2;
                        if (++unit == NU) { unit = 0; phase ^= 1; }
                    }
                } else
                for (int i = 0; i < nk;) {
                    const bool dbl = kd && i + 1 < nk && stage + 1 < S;
                    const long long c0 = tr ? clock64() : 0;
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const long long c1 = tr ? clock64() : 0;
                    if (it == 0 && i == 0 && lane == 0) trace_at(p, 3);
                    if (tr && it == 0 && lane == 0 && nunit < 8) cyc_at(p, 48 + nunit, cyc_entry);
                    ++nunit;
                    const uint64_t dp0 = dP_base + (uint64_t)(stage * (kP >> 4));
                    const uint64_t dq0 = dQ_base + (uint64_t)(stage * (kQ >> 4));
                    long long c2 = 0;
                    if (ptx::elect_one()) {
                        if (!mma_off) {
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                if (k >= 4 && !dbl) break;
                                // K-major: +32 B inside the swizzle row; MN-major: +2 K-groups;
                                // chunks 4..7 read the next stage (+ one P / Q tile)
                                const uint64_t dp = dp0 + (k >> 2) * (kP >> 4) + (k & 3) * kStepP;
                                const uint64_t dq = dq0 + (k >> 2) * (kQ >> 4) + (k & 3) * kStepQ;
                                if (PAIR) ptx::umma_f16_pair(d_tmem, dp, dq, idesc, (i | k) != 0);
                                else ptx::umma_f16(d_tmem, dp, dq, idesc, (i | k) != 0);
                            }
                        }
                        c2 = tr ? clock64() : 0;
                        // frees the stage(s) (in both CTAs of a pair / every CTA of a
                        // multicast cluster) when these MMAs finish
                        if (PAIR) ptx::umma_commit_pair(&empty[stage], 3);
                        else if (MC > 1) ptx::umma_commit_mc(&empty[stage], kMcMask);
                        else ptx::umma_commit(&empty[stage]);
                        if (dbl) {
                            if (PAIR) ptx::umma_commit_pair(&empty[stage + 1], 3);
                            else if (MC > 1) ptx::umma_commit_mc(&empty[stage + 1], kMcMask);
                            else ptx::umma_commit(&empty[stage + 1]);
                        }
                        if (tr) {
                            const long long c3 = clock64();
                            cyc_wait += c1 - c0; cyc_mma += c2 - c1; cyc_commit += c3 - c2; ++cyc_n;
                        }
                    }
                    __syncwarp();
                    const int adv = dbl ? 2 : 1;
                    i += adv;
                    stage += adv;
                    if (stage == S) { stage = 0; phase ^= 1; }
                }
                // accumulator ready for the epilogue (of both CTAs of a pair)
                if (ptx::elect_one()) {
                    if (PAIR) ptx::umma_commit_pair(&tfull[acc], 3);
                    else ptx::umma_commit(&tfull[acc]);
                }
                __syncwarp();
            }
            if (lane == 0 && mi == 0) {
                trace_at(p, 4);
                if (tr) {
                    p.trace[blockIdx.x * kTraceSlots + 12] = cyc_wait;
                    p.trace[blockIdx.x * kTraceSlots + 13] = cyc_mma;
                    p.trace[blockIdx.x * kTraceSlots + 14] = cyc_commit;
                    p.trace[blockIdx.x * kTraceSlots + 15] = cyc_n;
                }
            }
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + EW) {
        // ===== epilogue warps =====
        ptx::grid_dep_wait();
        // warp w reads TMEM lanes 32*(w%4)..+31 (its quarter of the tile rows); the two
        // warps of a quarter (group g = 0, 1) take alternate column chunks
        const int quarter = warp & 3;
        const int grp = (warp - kEpiWarp0) >> 2;
        const int row = quarter * 32 + lane;  // accumulator lane = row of the P tile
        const uint32_t wbuf = ptx::smem_addr(sE) + (uint32_t)(warp - kEpiWarp0) * 4096u;
        bool pending = false;                  // a TMA store still reads this warp's buffer
        // TMEM buffer release: pairs arrive on the leader's barrier (it issues the MMAs)
        auto release_acc = [&](uint64_t* bar) {
            if (PAIR) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_addr(bar), 0));
            else ptx::mbar_arrive(bar);
        };
        int it = 0;
        long long gue = 0;   // dual issuers: units of the tiles before this one (MMA's gu)
        WorkIter wi(p, rank);
        int tile, k0, nk;
        const long long U = (long long)p.num_tiles * p.kb_total;
        for (; wi.next(p, tile, k0, nk); ++it) {
            int b = 0, tp, tq;
            VarTile vt{0, 0, 0};
            if (p.ngroups) decode_varlen<BN>(tile, p.cu, p.ngroups, tp, tq, vt);
            else decode_ctile<SWAP, MC>(tile, p.tiles_p, p.tiles_q, crank, b, tp, tq, p.group_p);
            // first P-axis row of this CTA's accumulator rows (a pair splits 256 rows)
            const int prow0 = PAIR ? tp * 256 + (int)prank * 128 : tp * 128;
            // ---- stream-K bookkeeping (before the accumulator wait) ---------------------
            int c_first = 0, c_last = -1;          // CTAs whose partials this CTA adds
            // stream-K ids: CTAs, or pairs (each CTA of a pair fixes up its own 128 rows)
            const int sk_id = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
            const int sk_G = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
            const bool st1 = threadIdx.x == kEpiWarp0 * 32;     // trace: per-tile stamps
            const long long cyt0 = st1 && p.trace ? clock64() : 0;
            if (p.streamk && k0 == 0 && nk < p.kb_total && !(p.dbg & 32)) {
                // owner of a cut tile: the rest of its K range sits in ids sk_id+1 .. c_last.
                // The contributors published their partials at the START of their ranges,
                // so the flags are acquired here, while this tile's mainloop still runs --
                // the atomic poll and fence stay off the tail of the launch.
                c_first = sk_id + 1;
                const long long last_unit = (long long)(tile + 1) * p.kb_total - 1;
                c_last = sk_id;
                while (c_last + 1 < sk_G && sk_first(c_last + 1, U, sk_G) <= last_unit) ++c_last;
                // one thread acquires the contributors' flags (ld.acquire.gpu; a short
                // back-off after the first misses so the publishers' stores are not
                // starved); the named barrier then orders every epilogue thread's partial
                // reads after that acquire
                if (threadIdx.x == kEpiWarp0 * 32) {
                    for (int j = c_first; j <= c_last; ++j) {
                        int spins = 0;
                        while (ld_acquire(p.flags + sk_slot<PAIR>(j, prank)) == 0)
                            if (++spins > 4) __nanosleep(32);
                    }
                }
                epi_bar<ET>();
                if (st1) cyc_at(p, 32, cyt0);
            }
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            const long long cyt1 = st1 && p.trace ? clock64() : 0;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            if (st1) cyc_at(p, 33, cyt1);
            const long long cyt2 = st1 && p.trace ? clock64() : 0;
            const bool st0 = it == 0 && threadIdx.x == kEpiWarp0 * 32;
            const long long cye = st0 ? clock64() : 0;
            if (st0) trace_at(p, 5);
            // dual issuers: accumulator 2 acc holds this tile's even-indexed units (global unit
            // count), 2 acc + 1 (BN columns further) the odd ones; a one-unit range fills only
            // the one its parity names
            const long long u0 = gue;
            gue += (nk + 1) / 2;
            const bool has0 = !dual || nk >= 3 || (u0 & 1) == 0;
            const bool two = dual && nk >= 3;
            const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) +
                                   (dual ? acc * 2 + (has0 ? 0 : 1) : acc) * BN;
            if (split) break;  // split mode: the accumulator is read after the cluster barrier
            // ---- stream-K: a cut tile ----------------------------------------------------
            if (p.streamk && k0 > 0 && !(p.dbg & 32)) {
                // not the owner: park the fp32 partial in this CTA's slot and publish it
                // slot layout [col/4][row][4] (coalesced across the warp's rows)
                float* slot = p.ws + (long long)blockIdx.x * 128 * BN + (long long)row * 4;
#pragma unroll 1
                for (int c = grp; c < (BN + 31) / 32; c += NG) {
                    uint32_t v[32];
                    if (BN >= 32) ptx::tmem_ld32(taddr + c * 32, v);
                    else ptx::tmem_ld16(taddr + c * 32, v);
                    ptx::tmem_wait_ld();
                    constexpr int W = BN >= 32 ? 32 : BN;
                    if (two) acc_add<W>(taddr + BN + c * 32, v);
#pragma unroll
                    for (int j = 0; j < W; j += 4)
                        __stcg(reinterpret_cast<uint4*>(slot + (long long)((c * 32 + j) / 4) * 128 * 4),
                               make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]));
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) release_acc(&tempty[acc]);
                // publish: every epilogue thread's partial stores, then the named barrier,
                // then ONE thread's gpu-scope fence + release store of the flag (cumulative
                // over the stores the barrier ordered before it)
                epi_bar<ET>();
                if (threadIdx.x == kEpiWarp0 * 32) {
                    __threadfence();
                    st_release(p.flags + blockIdx.x, 1);
                }
                continue;
            }
            if (p.vec && p.ndst == 0 && p.ngroups == 0 && !(p.dbg & 8)) {
                // TMEM -> registers -> swizzled SMEM staging -> TMA bulk store (full lines,
                // asynchronous, M/N tails clipped by the tensor map)
                const int ob = p.out_kind == 2 ? 4 : 2;
                if (!SWAP) {
                    const int CW = 128 / ob;                  // columns per 128-B row
                    const uint32_t rowa = wbuf + (uint32_t)lane * 128u;
#pragma unroll 1
                    for (int k = grp; k < BN / CW; k += NG) {
                        if (pending) {
                            if (lane == 0) ptx::bulk_wait_read<0>();
                            __syncwarp();
                        }
                        if (ob == 4) {                        // 32 fp32 = 8 x 16-B chunks
                            uint32_t v[32];
                            ptx::tmem_ld32(taddr + k * CW, v);
                            ptx::tmem_wait_ld();
                            if (two) acc_add<32>(taddr + BN + k * CW, v);
                            add_partials<32, PAIR>(v, p.ws, c_first, c_last, row, k * CW, BN, prank);
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                ptx::st_shared_v4(rowa + (((uint32_t)(j ^ (lane & 7))) << 4),
                                                  v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                        } else {                              // 64 halves = 8 x 16-B chunks
                            uint32_t v[64];
                            ptx::tmem_ld32(taddr + k * CW, *reinterpret_cast<uint32_t(*)[32]>(v));
                            ptx::tmem_ld32(taddr + k * CW + 32,
                                           *reinterpret_cast<uint32_t(*)[32]>(v + 32));
                            ptx::tmem_wait_ld();
                            if (two) {
                                acc_add<32>(taddr + BN + k * CW, v);
                                acc_add<32>(taddr + BN + k * CW + 32, v + 32);
                            }
                            if (st0 && k == grp) cyc_at(p, 29, cye);
                            add_partials<64, PAIR>(v, p.ws, c_first, c_last, row, k * CW, BN, prank);
                            uint32_t u[32];
                            pack_chunk<64>(reinterpret_cast<const float*>(v), u, p.out_kind);
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                ptx::st_shared_v4(rowa + (((uint32_t)(j ^ (lane & 7))) << 4),
                                                  u[4 * j], u[4 * j + 1], u[4 * j + 2], u[4 * j + 3]);
                        }
                        ptx::fence_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_3d(&tmC, sE + (wbuf - ptx::smem_addr(sE)),
                                              tq * BN + k * CW, prow0 + quarter * 32, b);
                            ptx::bulk_commit();
                        }
                        pending = true;
                    }
                } else {
                    constexpr int W = BN >= 32 ? 32 : BN;     // m values per chunk
#pragma unroll 1
                    for (int c = grp; c < BN / W; c += NG) {
                        if (pending) {
                            if (lane == 0) ptx::bulk_wait_read<0>();
                            __syncwarp();
                        }
                        uint32_t v[32];
                        if (BN >= 32) ptx::tmem_ld32(taddr + c * 32, v);
                        else ptx::tmem_ld16(taddr + c * 32, v);
                        ptx::tmem_wait_ld();
                        if (two) acc_add<W>(taddr + BN + c * 32, v);
                        add_partials<W, PAIR>(v, p.ws, c_first, c_last, row, c * 32, BN, prank);
                        const float* f = reinterpret_cast<const float*>(v);
                        // staging tile [W m-rows][32 n] (row pitch 32*ob bytes), lane = n
                        if (ob == 4) {
#pragma unroll
                            for (int j = 0; j < W; ++j)
                                ptx::st_shared_u32(wbuf + (uint32_t)(j * 32 + lane) * 4u, v[j]);
                        } else {
                            uint32_t u[W / 2];
                            pack_chunk<W>(f, u, p.out_kind);
#pragma unroll
                            for (int j = 0; j < W; ++j)
                                ptx::st_shared_u16(wbuf + (uint32_t)(j * 32 + lane) * 2u,
                                                   (uint16_t)(u[j / 2] >> (16 * (j & 1))));
                        }
                        ptx::fence_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_3d(&tmC, sE + (wbuf - ptx::smem_addr(sE)),
                                              prow0 + quarter * 32, tq * BN + c * W, b);
                            ptx::bulk_commit();
                        }
                        pending = true;
                    }
                }
                if (st0) cyc_at(p, 30, cye);
                if (st1) cyc_at(p, 34, cyt2);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) release_acc(&tempty[acc]);
                if (c_last >= c_first) sk_reset<PAIR, ET>(p, c_first, c_last, prank);
                continue;
            }
            const int pr = prow0 + row;  // global index on the P axis
            const int ob_ = p.out_kind == 2 ? 4 : 2;
            // varlen: this sequence's s x s block of C (vector stores iff its rows are 16-B
            // aligned); otherwise the batch's M x N matrix
            char* Cb = reinterpret_cast<char*>(p.C) + (p.ngroups ? vt.coff * ob_ : (long long)b * p.sC * ob_);
            const int Me = p.ngroups ? vt.len : p.M;
            const int Ne = p.ngroups ? vt.len : p.N;
            const long long ldc_e = p.ngroups ? vt.len : p.ldc;
            const bool vec_e = p.ngroups ? ((vt.len * ob_) % 16 == 0 && (vt.coff * ob_) % 16 == 0 &&
                                            (reinterpret_cast<uintptr_t>(p.C) & 15) == 0)
                                         : p.vec != 0;
#pragma unroll 1
            for (int c = grp; c < (BN + 31) / 32; c += NG) {
                uint32_t v[32];
                if (BN >= 32) ptx::tmem_ld32(taddr + c * 32, v);
                else ptx::tmem_ld16(taddr + c * 32, v);
                ptx::tmem_wait_ld();
                constexpr int W = BN >= 32 ? 32 : BN;
                if (two) acc_add<W>(taddr + BN + c * 32, v);
                add_partials<W, PAIR>(v, p.ws, c_first, c_last, row, c * 32, BN, prank);
                const float* f = reinterpret_cast<const float*>(v);
                if (p.dbg & 8) {
                    if (f[0] == 12345.f) store1(Cb, 0, f[1], p.out_kind);
                } else if (!SWAP && p.ndst == 0 && !vec_e && p.out_kind != 2 && (Ne & 3) == 0 &&
                           ((reinterpret_cast<uintptr_t>(Cb) | (uintptr_t)(ldc_e * 2)) & 7) == 0) {
                    store_rows_coalesced8<W>(reinterpret_cast<float*>(sE + (warp - kEpiWarp0) * 4096),
                                             Cb, ldc_e, prow0 + quarter * 32, Me, tq * BN + c * 32,
                                             Ne, f, p.out_kind, lane);
                } else if (!SWAP && p.ndst == 0 && !vec_e) {
                    store_rows_coalesced<W>(reinterpret_cast<float*>(sE + (warp - kEpiWarp0) * 4096),
                                            Cb, ldc_e, prow0 + quarter * 32, Me, tq * BN + c * 32,
                                            Ne, f, p.out_kind, lane);
                } else if (!SWAP) {
                    // row pr = m, columns = n
                    if (pr < Me) {
                        const int n0 = tq * BN + c * 32;
                        if (p.ndst > 0) {
                            // fused all-gather: the same chunk into every destination, at
                            // its global row (peer stores travel over NVLink while the
                            // next tile's mainloop runs, TMEM being double-buffered)
                            const long long base = (p.dst_row0 + pr) * p.ldc;
#pragma unroll 1
                            for (int d = 0; d < p.ndst; ++d) {
                                char* Db = reinterpret_cast<char*>(p.dst[d]);
                                if (p.vec) store_row_chunk<W>(Db, base, n0, p.N, f, p.out_kind);
                                else store_row_scalar(Db, base, n0, p.N, W, f, p.out_kind);
                            }
                        } else {
                            const long long base = (long long)pr * ldc_e;
                            if (vec_e) store_row_chunk<W>(Cb, base, n0, Ne, f, p.out_kind);
                            else store_row_scalar(Cb, base, n0, Ne, W, f, p.out_kind);
                        }
                    }
                } else if (pr < p.N) {
                    // row pr = n, columns = m
                    store_col_chunk<W>(Cb, p.ldc, pr, tq * BN + c * 32, p.M, f, p.out_kind);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(&tempty[acc]);
            if (c_last >= c_first) sk_reset<PAIR, ET>(p, c_first, c_last, prank);
        }
        // TMA stores have read their staging before the CTA retires (the grid completes only
        // once the stores are performed, which is what the next grid's wait observes)
        const long long cyw = clock64();
        if (lane == 0) {
            if (p.dbg & 256) ptx::bulk_wait<0>();
            else ptx::bulk_wait_read<0>();
        }
        if (threadIdx.x == kEpiWarp0 * 32) { cyc_at(p, 31, cyw); cyc_at(p, 35, cyw); }
    }

    __syncwarp();  // reconverge the single-lane roles before the .aligned cluster barriers
    if (!split && threadIdx.x == kEpiWarp0 * 32) trace_at(p, 6);
    long long cyr = 0;   // trace: start of the split reduce
    if (split) {
        // deterministic in-cluster reduce-scatter of the s K-slice partials (R7):
        //  (1) the owner thread of each CTA posts the byte count it expects from its peers
        //      on `redbar`, then a cluster barrier: every CTA's MMAs are complete, so every
        //      SMEM ring is free to receive;
        //  (2) each epilogue thread reads its accumulator row from TMEM; rows are owned in
        //      blocks of 128/s; a row it owns goes to its own slot [rank] with st.shared, a
        //      peer's row goes to slot [rank] of the owner with st.async, whose bytes
        //      complete on the owner's `redbar` (no second cluster barrier);
        //  (3) each CTA waits for its own and its peers' rows, sums its rows over slots
        //      0..s-1 in rank order and stores C.
        // slot layout (floats): [src rank][32-col chunk c][row rr][W], 16-B groups XOR-
        // swizzled by the row so the row-per-lane stores and the reads are conflict-light.
        constexpr int W = BN >= 32 ? 32 : BN;     // columns per chunk
        constexpr int G = W / 4;                  // 16-B groups per chunk row
        const int s_ = p.splits;
        const int rows = 128 / s_;
        const int slot = rows * BN;               // floats per source-rank slot
        const uint32_t red_addr = ptx::smem_addr(sP);
        const bool post = !(p.dbg & 1);
        if (threadIdx.x == kEpiWarp0 * 32 && post)
            ptx::mbar_arrive_expect_tx(redbar, (uint32_t)((s_ - 1) * slot * 4));
        ptx::cluster_sync();
        ptx::tc_fence_after();
        if (threadIdx.x == kEpiWarp0 * 32) trace_at(p, 16);
        const long long cyp = clock64();
        if (warp >= kEpiWarp0 && warp < kEpiWarp0 + EW && post) {
            const int quarter = warp & 3;
            const int row = quarter * 32 + lane;
            const int owner = row / rows;
            const int rr = row - owner * rows;
            const uint32_t base = red_addr + (uint32_t)(rank * slot + rr * W) * 4u;
            const uint32_t dst = owner == rank ? base : ptx::mapa(base, owner);
            const uint32_t rbar = ptx::mapa(ptx::smem_addr(redbar), owner);
            const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16);
            const bool two = dual && p.kb_total / s_ >= 3;   // this slice's units >= 2
            const int grp = (warp - kEpiWarp0) >> 2;
            const int sw = G == 8 ? (rr & 7) : G == 4 ? ((rr >> 1) & 3) : 0;
#pragma unroll 1
            for (int c = grp; c < (BN + 31) / 32; c += NG) {
                uint32_t v[32];
                if (BN >= 32) ptx::tmem_ld32(taddr + c * 32, v);
                else ptx::tmem_ld16(taddr + c * 32, v);
                ptx::tmem_wait_ld();
                if (two) acc_add<W>(taddr + BN + c * 32, v);
                const uint32_t cd = dst + (uint32_t)(c * rows * W) * 4u;
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const uint32_t a = cd + (uint32_t)((g ^ sw) * 16);
                    if (owner == rank) ptx::st_shared_v4(a, v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                    else ptx::st_async_f4(a, rbar, v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
                }
            }
        }
        if (threadIdx.x == kEpiWarp0 * 32) { trace_at(p, 17); cyc_at(p, 30, cyp); }
        if (warp >= kEpiWarp0 && warp < kEpiWarp0 + EW) {
            epi_bar<ET>();                           // this CTA's own rows are in SMEM
            if (threadIdx.x == kEpiWarp0 * 32) cyc_at(p, 19, cyp);
            if (post) ptx::mbar_wait(redbar, 0);     // the peers' rows too
        }
        if (threadIdx.x == kEpiWarp0 * 32) trace_at(p, 6);
        cyr = clock64();
        if (warp >= kEpiWarp0 && warp < kEpiWarp0 + EW && !(p.dbg & 2)) {
            int b, tp, tq;
            decode_tile(tile0, p.tiles_p, p.tiles_q, b, tp, tq, p.group_p);
            const int et = threadIdx.x - kEpiWarp0 * 32;
            const float* red = reinterpret_cast<const float*>(sP);
            char* Cb = reinterpret_cast<char*>(p.C) +
                       (long long)b * p.sC * (p.out_kind == 2 ? 4 : 2);
            const int n4 = BN / 4;
#pragma unroll 1
            for (int idx = et; idx < rows * n4; idx += ET) {
                int rr, cc;
                if (SWAP) { rr = idx % rows; cc = (idx / rows) * 4; }   // consecutive n
                else { rr = idx / n4; cc = (idx % n4) * 4; }            // consecutive n
                const int c = cc / W, g = (cc % W) / 4;
                const int sw = G == 8 ? (rr & 7) : G == 4 ? ((rr >> 1) & 3) : 0;
                const float* src = red + (c * rows + rr) * W + ((g ^ sw) * 4);
                float4 acc4 = *reinterpret_cast<const float4*>(src);
#pragma unroll 1
                for (int j = 1; j < s_; ++j) {
                    const float4 t = *reinterpret_cast<const float4*>(src + j * slot);
                    acc4.x += t.x; acc4.y += t.y; acc4.z += t.z; acc4.w += t.w;
                }
                const int pr = tp * 128 + rank * rows + rr;
                const int q0 = tq * BN + cc;
                if (p.dbg & 4) {
                    if (acc4.x == 12345.f) store1(Cb, 0, acc4.y, p.out_kind);
                } else if (!SWAP) {
                    if (pr < p.M) {
                        if (p.vec) {
                            if (q0 < p.N) store4(Cb, (long long)pr * p.ldc + q0, acc4, p.out_kind);
                        } else {
                            const float e[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (q0 + j < p.N) store1(Cb, (long long)pr * p.ldc + q0 + j, e[j], p.out_kind);
                        }
                    }
                } else if (pr < p.N) {
                    const float e[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (q0 + j < p.M) store1(Cb, (long long)(q0 + j) * p.ldc + pr, e[j], p.out_kind);
                }
            }
        }
    }

    if (threadIdx.x == kEpiWarp0 * 32) {
        trace_at(p, 7);
        if (split) cyc_at(p, 29, cyr);
    }
    ptx::tc_fence_before();
    if (PAIR || MC > 1) ptx::cluster_sync();   // no CTA of a cluster retires while a peer may
    else __syncthreads();                      // still touch its shared memory
    if (warp == 1) {
        __syncwarp();
        ptx::tc_fence_after();
        if (PAIR) ptx::tmem_dealloc_pair<kCols>(tmem_base);
        else ptx::tmem_dealloc<kCols>(tmem_base);
        if (lane == 0) trace_at(p, 9);
    }
}

}  // namespace vx
