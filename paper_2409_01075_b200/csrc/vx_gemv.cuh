// vx_gemv.cuh -- family 3: the CUDA-core rung for 16-bit inputs at tiny M, i.e. the
// "adaptive backend" of Vortex's runtime ("We provide implementations
// for both CUDA cores and Tensor cores, allowing us to choose the appropriate backend
// hardware based on the runtime input shapes"; evaluated for M 1..16).
//
// C[m, n] = sum_k A[m, k] * B(n, k) for M <= MT rows.  A CTA of 8 warps owns 32 output
// columns; each warp streams NC = 4 rows of B (K contiguous for NK; for KN the warp reads
// 4 adjacent columns per k) with 16-byte loads, reads A through the L1 read-only path,
// accumulates MT x NC fp32 partial sums per lane and reduces them across the warp with
// shuffles.  No TMEM, tensor maps or barriers: the fixed cost per launch is minimal, which
// is what wins at tiny M (the cost model decides, R20).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace vx {

constexpr int kGemvWarps = 8;
constexpr int kGemvNC = 4;                      // columns per warp
constexpr int kGemvCols = kGemvWarps * kGemvNC; // columns per CTA

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
    uint4 r;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// in_kind: 0 bf16, 1 fp16.  out_kind: 0 bf16, 1 fp16, 2 fp32.  C row stride ldc = N.
template <int MT, bool B_KN>
__global__ void __launch_bounds__(kGemvWarps * 32)
    vx_gemv_kernel(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B, void* C, int M,
                   int N, int K, long long sA, long long sB, long long sC, int in_kind,
                   int out_kind) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    const int n0 = blockIdx.x * kGemvCols + warp * kGemvNC;   // this warp's first column
    if (n0 >= N) return;
    A += b * sA;
    B += b * sB;
    // programmatic dependent launch: nothing global is read before the previous grid is done
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float acc[MT][kGemvNC];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int c = 0; c < kGemvNC; ++c) acc[m][c] = 0.f;

#pragma unroll 2
    for (int k = lane * 8; k < K; k += 256) {
        float bv[kGemvNC][8];
        if (!B_KN) {
#pragma unroll
            for (int c = 0; c < kGemvNC; ++c) {
                if (n0 + c < N) unpack8(ldg16(B + (long long)(n0 + c) * K + k), bv[c], in_kind);
                else
#pragma unroll
                    for (int e = 0; e < 8; ++e) bv[c][e] = 0.f;
            }
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
            if (m < M) {
                float av[8];
                unpack8(ldg16(A + (long long)m * K + k), av, in_kind);
#pragma unroll
                for (int c = 0; c < kGemvNC; ++c)
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[m][c] = fmaf(av[e], bv[c][e], acc[m][c]);
            }
        }
    }
    // warp reduction (fixed butterfly order -> deterministic)
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int c = 0; c < kGemvNC; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[m][c] += __shfl_xor_sync(0xffffffffu, acc[m][c], o);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (lane < kGemvNC && n0 + lane < N) {
        const int n = n0 + lane;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            if (m >= M) break;
            float v = acc[m][0];
#pragma unroll
            for (int c = 1; c < kGemvNC; ++c)
                if (lane == c) v = acc[m][c];
            const long long idx = b * sC + (long long)m * N + n;
            if (out_kind == 2) reinterpret_cast<float*>(C)[idx] = v;
            else if (out_kind == 0) reinterpret_cast<__nv_bfloat16*>(C)[idx] = __float2bfloat16_rn(v);
            else reinterpret_cast<__half*>(C)[idx] = __float2half_rn(v);
        }
    }
}

}  // namespace vx
