// vx_simt.cuh -- family 2: the CUDA-core (FFMA) rung of the ladder for fp32 inputs
// ("Cuda Core Only" mode with FP32).  L0 = a TM x TN register tile of FFMA
// per thread, L2 = a BM x BN CTA tile staged through a 2-stage shared-memory ring 16
// K-columns at a time, grid = one CTA per output tile.  Every element is accumulated in fp32 with k ascending;
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
    constexpr int LA = BM * BK / NT, LB = BN * BK / NT;   // elements per thread per K tile
    static_assert(LA * NT == BM * BK && LB * NT == BN * BK, "tile loads split evenly");
    // two SMEM stages (the strategy table's S = 2): the next K tile is loaded into registers
    // before the current one is multiplied and stored to the other stage after it, so its
    // global-load latency overlaps the FFMAs
    __shared__ float As[2][BK][BM + 4];
    __shared__ float Bs[2][BK][BN + 4];
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
    float ra[LA], rb[LB];
    auto load = [&](int k0) {      // K tile at k0 -> registers (zero past M, N, K)
#pragma unroll
        for (int l = 0; l < LA; ++l) {
            const int i = threadIdx.x + l * NT;
            const int m = m0 + i / BK, k = k0 + i % BK;
            ra[l] = (m < M && k < K) ? A[(long long)m * K + k] : 0.f;
        }
#pragma unroll
        for (int l = 0; l < LB; ++l) {
            const int i = threadIdx.x + l * NT;
            if (b_nk) {
                const int n = n0 + i / BK, k = k0 + i % BK;
                rb[l] = (n < N && k < K) ? B[(long long)n * K + k] : 0.f;
            } else {
                const int n = n0 + i % BN, k = k0 + i / BN;
                rb[l] = (n < N && k < K) ? B[(long long)k * N + n] : 0.f;
            }
        }
    };
    auto store = [&](int st) {     // registers -> SMEM stage st
#pragma unroll
        for (int l = 0; l < LA; ++l) {
            const int i = threadIdx.x + l * NT;
            As[st][i % BK][i / BK] = ra[l];
        }
#pragma unroll
        for (int l = 0; l < LB; ++l) {
            const int i = threadIdx.x + l * NT;
            if (b_nk) Bs[st][i % BK][i / BK] = rb[l];
            else Bs[st][i / BN][i % BN] = rb[l];
        }
    };
    // programmatic dependent launch: nothing global is touched before the previous grid ends
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int ktiles = (K + BK - 1) / BK;
    load(0);
    store(0);
    __syncthreads();
    for (int kt = 0; kt < ktiles; ++kt) {
        const int cur = kt & 1;
        if (kt + 1 < ktiles) load((kt + 1) * BK);
        else asm volatile("griddepcontrol.launch_dependents;");
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[TM], bb[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[cur][kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) bb[j] = Bs[cur][kk][tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
        if (kt + 1 < ktiles) store(cur ^ 1);   // the other stage: its readers finished at the
        __syncthreads();                       // previous iteration's barrier
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
