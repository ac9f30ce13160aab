// vx_simt.cuh -- family 2: the CUDA-core (FFMA) rung of the ladder for fp32 inputs
// ("Cuda Core Only" mode with FP32).  L0 = a TM x TN register tile of FFMA
// per thread, L2 = a BM x BN CTA tile staged through shared memory 16 K-columns at a time,
// grid = one CTA per output tile.  Every element is accumulated in fp32 with k ascending;
// tails in M, N and K are predicated (no alignment requirement on fp32 operands).
#pragma once

namespace vx {

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    vx_simt_kernel(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
                   int M, int N, int K, int b_nk, long long sA, long long sB, long long sC,
                   int tiles_m, int tiles_n) {
    constexpr int NT = (BM / TM) * (BN / TN);
    constexpr int BK = 16;
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int per_b = tiles_m * tiles_n;
    const int b = blockIdx.x / per_b;
    const int t = blockIdx.x - b * per_b;
    const int m0 = (t / tiles_n) * BM, n0 = (t % tiles_n) * BN;
    A += b * sA;
    B += b * sB;
    C += b * sC;
    const int tx = threadIdx.x % (BN / TN), ty = threadIdx.x / (BN / TN);
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    for (int k0 = 0; k0 < K; k0 += BK) {
        for (int i = threadIdx.x; i < BM * BK; i += NT) {
            const int r = i / BK, kk = i % BK;
            const int m = m0 + r, k = k0 + kk;
            As[kk][r] = (m < M && k < K) ? A[(long long)m * K + k] : 0.f;
        }
        if (b_nk) {
            for (int i = threadIdx.x; i < BN * BK; i += NT) {
                const int c = i / BK, kk = i % BK;
                const int n = n0 + c, k = k0 + kk;
                Bs[kk][c] = (n < N && k < K) ? B[(long long)n * K + k] : 0.f;
            }
        } else {
            for (int i = threadIdx.x; i < BN * BK; i += NT) {
                const int kk = i / BN, c = i % BN;
                const int n = n0 + c, k = k0 + kk;
                Bs[kk][c] = (n < N && k < K) ? B[(long long)k * N + n] : 0.f;
            }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[TM], bb[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) bb[j] = Bs[kk][tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int m = m0 + ty * TM + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int n = n0 + tx * TN + j;
            if (n < N) C[(long long)m * N + n] = acc[i][j];
        }
    }
}

}  // namespace vx
