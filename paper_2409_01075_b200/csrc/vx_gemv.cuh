// vx_gemv.cuh -- family 3: the CUDA-core rung for 16-bit inputs at tiny M, i.e. the
// "adaptive backend" of Vortex's runtime ("We provide implementations
// for both CUDA cores and Tensor cores, allowing us to choose the appropriate backend
// hardware based on the runtime input shapes"; evaluated for M 1..16).
//
// C[m, n] = sum_k A[m, k] * B(n, k) for M <= MT rows.  A CTA of 8 warps owns 8 output
// columns: 2 column groups x 4 K slices.  Each warp streams NC = 4 rows of B over its K
// slice (K contiguous for NK; for KN the warp reads 4 adjacent columns per k) with 16-byte
// loads issued together (memory-level parallelism is the whole game here), reads A through
// the L1 read-only path, accumulates MT x NC fp32 partial sums per lane and reduces them
// with shuffles, then across the slices through shared memory.  No TMEM, tensor maps or barriers: the fixed cost per launch is minimal, which
// is what wins at tiny M (the cost model decides, R20).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace vx {

constexpr int kGemvWarps = 8;
constexpr int kGemvNC = 4;                        // columns per warp
constexpr int kGemvKS = 4;                        // K slices per CTA (warps sharing columns)
constexpr int kGemvCols = kGemvWarps / kGemvKS * kGemvNC;   // columns per CTA (8)
constexpr size_t kGemvSaMaxSmem = 96 * 1024;   // A-in-SMEM variant: MT * K * 2 bytes max

__device__ __forceinline__ void unpack8(uint4 u, float* f, int kind) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (kind == 0) {
            f[2 * i] = __uint_as_float(w[i] << 16);
            f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        } else {
            const __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
            const float2 t = __half22float2(h);
            f[2 * i] = t.x;
            f[2 * i + 1] = t.y;
        }
    }
}

__device__ __forceinline__ uint4 ldg16(const void* p) {
    // read-only path; NOT volatile, so the compiler can batch the loads of an iteration
    return __ldg(reinterpret_cast<const uint4*>(p));
}

// in_kind: 0 bf16, 1 fp16.  out_kind: 0 bf16, 1 fp16, 2 fp32.  C row stride ldc = N.
// Warp w owns columns n0 + [0, 4) with n0 = 8 * blockIdx.x + 4 * (w % 2) and the K slice
// ks = w / 2: k-steps of 256 elements ks, ks + 4, ks + 8, ...  The four slices' partial
// sums meet in shared memory and are added in slice order (deterministic).
template <int MT, bool B_KN>
__global__ void __launch_bounds__(kGemvWarps * 32)
    vx_gemv_kernel(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B, void* C, int M,
                   int N, int K, long long sA, long long sB, long long sC, int in_kind,
                   int out_kind) {
    constexpr int CG = kGemvWarps / kGemvKS;        // column groups per CTA
    __shared__ float red[kGemvKS][CG][MT][kGemvNC];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cg = warp % CG, ks = warp / CG;
    const int b = blockIdx.y;
    const int n0 = blockIdx.x * kGemvCols + cg * kGemvNC;   // this warp's first column
    A += b * sA;
    B += b * sB;
    // programmatic dependent launch: nothing global is read before the previous grid is done
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float acc[MT][kGemvNC];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int c = 0; c < kGemvNC; ++c) acc[m][c] = 0.f;

    if (n0 < N) {
#pragma unroll(MT <= 2 ? 4 : 2)
        for (int k = (ks * 32 + lane) * 8; k < K; k += kGemvKS * 256) {
            // issue every load of this step first (B rows / columns, then A rows) ...
            uint4 braw[kGemvNC];
            float bv[kGemvNC][8];
            if (!B_KN) {
#pragma unroll
                for (int c = 0; c < kGemvNC; ++c)
                    braw[c] = (n0 + c < N) ? ldg16(B + (long long)(n0 + c) * K + k)
                                           : make_uint4(0, 0, 0, 0);
            }
            uint4 araw[MT];
#pragma unroll
            for (int m = 0; m < MT; ++m)
                araw[m] = (m < M) ? ldg16(A + (long long)m * K + k) : make_uint4(0, 0, 0, 0);
            // ... then convert and accumulate
            if (!B_KN) {
#pragma unroll
                for (int c = 0; c < kGemvNC; ++c) unpack8(braw[c], bv[c], in_kind);
            } else {
                // B stored K x N: element (n, k) at B[k * N + n]; 4 adjacent columns per k
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const uint16_t* row = B + (long long)(k + e) * N + n0;
#pragma unroll
                    for (int c = 0; c < kGemvNC; ++c) {
                        const uint16_t h = (n0 + c < N) ? __ldg(row + c) : (uint16_t)0;
                        bv[c][e] = in_kind == 0 ? __uint_as_float((uint32_t)h << 16)
                                                : __half2float(*reinterpret_cast<const __half*>(&h));
                    }
                }
            }
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                float av[8];
                unpack8(araw[m], av, in_kind);
#pragma unroll
                for (int c = 0; c < kGemvNC; ++c)
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[m][c] = fmaf(av[e], bv[c][e], acc[m][c]);
            }
        }
    }
    // warp reduction (fixed butterfly order -> deterministic), then across the K slices
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int c = 0; c < kGemvNC; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[m][c] += __shfl_xor_sync(0xffffffffu, acc[m][c], o);
    if (lane == 0) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int c = 0; c < kGemvNC; ++c) red[ks][cg][m][c] = acc[m][c];
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int i = threadIdx.x; i < CG * MT * kGemvNC; i += blockDim.x) {
        const int g = i / (MT * kGemvNC), m = i / kGemvNC % MT, c = i % kGemvNC;
        const int n = blockIdx.x * kGemvCols + g * kGemvNC + c;
        if (m >= M || n >= N) continue;
        float v = red[0][g][m][c];
#pragma unroll
        for (int j = 1; j < kGemvKS; ++j) v += red[j][g][m][c];
        const long long idx = b * sC + (long long)m * N + n;
        if (out_kind == 2) reinterpret_cast<float*>(C)[idx] = v;
        else if (out_kind == 0) reinterpret_cast<__nv_bfloat16*>(C)[idx] = __float2bfloat16_rn(v);
        else reinterpret_cast<__half*>(C)[idx] = __float2half_rn(v);
    }
}

// Variant for MT >= 4 with B stored N x K (R20b): the per-iteration A loads of the kernel
// above (MT more 16-B loads per step, each an L2 round trip on the critical path, and MT x 4
// more live registers) are what starve it of B bytes in flight at MT = 4 / 8.  Here each CTA
// first issues the B loads of its first U k-steps, then stages A (MT x K bf16/fp16, rows >= M
// zero) into shared memory once, and the k-steps read A from shared memory; the registers
// saved hold U steps of B instead.  Same column / K-slice ownership and reduction order as
// vx_gemv_kernel.  Requires K % 8 == 0 and MT * K * 2 <= the dynamic smem the dispatcher sets.
template <int MT, int U>
__global__ void __launch_bounds__(kGemvWarps * 32)
    vx_gemv_sa_kernel(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B, void* C,
                      int M, int N, int K, long long sA, long long sB, long long sC, int in_kind,
                      int out_kind) {
    constexpr int CG = kGemvWarps / kGemvKS;
    extern __shared__ __align__(16) uint16_t a_sm[];          // [MT][K]
    __shared__ float red[kGemvKS][CG][MT][kGemvNC];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cg = warp % CG, ks = warp / CG;
    const int b = blockIdx.y;
    const int n0 = blockIdx.x * kGemvCols + cg * kGemvNC;
    A += b * sA;
    B += b * sB;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    constexpr int KSTEP = kGemvKS * 256;
    int k = (ks * 32 + lane) * 8;
    uint4 braw[U][kGemvNC];
    auto load_b = [&](int kb) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < kGemvNC; ++c)
                braw[u][c] = (kb + u * KSTEP < K && n0 + c < N)
                                 ? ldg16(B + (long long)(n0 + c) * K + kb + u * KSTEP)
                                 : make_uint4(0, 0, 0, 0);
    };
    load_b(k);
    const int k8 = K >> 3;
    for (int i = threadIdx.x; i < MT * k8; i += blockDim.x) {
        const int m = i / k8, kk = (i - m * k8) * 8;
        reinterpret_cast<uint4*>(a_sm)[i] =
            m < M ? ldg16(A + (long long)m * K + kk) : make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    float acc[MT][kGemvNC];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int c = 0; c < kGemvNC; ++c) acc[m][c] = 0.f;
    for (; k < K; k += U * KSTEP) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int kk = k + u * KSTEP;
            if (kk >= K) break;
            float bv[kGemvNC][8];
#pragma unroll
            for (int c = 0; c < kGemvNC; ++c) unpack8(braw[u][c], bv[c], in_kind);
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                float av[8];
                unpack8(*reinterpret_cast<const uint4*>(a_sm + m * K + kk), av, in_kind);
#pragma unroll
                for (int c = 0; c < kGemvNC; ++c)
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[m][c] = fmaf(av[e], bv[c][e], acc[m][c]);
            }
        }
        if (k + U * KSTEP < K) load_b(k + U * KSTEP);
    }
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int c = 0; c < kGemvNC; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[m][c] += __shfl_xor_sync(0xffffffffu, acc[m][c], o);
    if (lane == 0) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int c = 0; c < kGemvNC; ++c) red[ks][cg][m][c] = acc[m][c];
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int i = threadIdx.x; i < CG * MT * kGemvNC; i += blockDim.x) {
        const int g = i / (MT * kGemvNC), m = i / kGemvNC % MT, c = i % kGemvNC;
        const int n = blockIdx.x * kGemvCols + g * kGemvNC + c;
        if (m >= M || n >= N) continue;
        float v = red[0][g][m][c];
#pragma unroll
        for (int j = 1; j < kGemvKS; ++j) v += red[j][g][m][c];
        const long long idx = b * sC + (long long)m * N + n;
        if (out_kind == 2) reinterpret_cast<float*>(C)[idx] = v;
        else if (out_kind == 0) reinterpret_cast<__nv_bfloat16*>(C)[idx] = __float2bfloat16_rn(v);
        else reinterpret_cast<__half*>(C)[idx] = __float2half_rn(v);
    }
}

}  // namespace vx
