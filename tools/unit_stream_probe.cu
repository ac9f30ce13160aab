// unit_stream_probe.cu -- measurement tool: the swapped 128x16 rung's exact load pattern at a
// BERT shape (M=128, N=768, K=768), without any MMA: 48 CTAs (tp = cta / 8 over B's rows,
// tq = cta % 8 over A's rows), deep-K units of two 64-deep chunks = one 4-D box of 128 B
// rows x 2 chunks (32 KB) + one of 16 A rows x 2 chunks (4 KB) on one full barrier, a ring
// of 10 stages (5 units), two producer threads alternating units, a consumer thread that
// frees a unit as soon as it lands.  Per-CTA time from the first issue to the last full
// barrier = the streaming floor of that rung's K loop (the GEMM measures ~2.8 us).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/usp tools/unit_stream_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void tma4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(sa(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(bar)) : "memory");
}

struct Cfg { int units, ring_units, producers, unit_kb, qrows; };

__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap mP, const __grid_constant__ CUtensorMap mQ,
                                             Cfg c, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 32;
    const int pbytes = 128 * 128 * c.unit_kb, qbytes = c.qrows * 128 * c.unit_kb;
    uint8_t* sP = smem + 1024;
    uint8_t* sQ = sP + c.ring_units * pbytes;
    if (threadIdx.x == 0) {
        for (int i = 0; i < c.ring_units; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int tp = blockIdx.x / 8, tq = blockIdx.x % 8;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int w = threadIdx.x >> 5;
    if (w >= 1 && w <= c.producers && (threadIdx.x & 31) == 0) {
        for (int u = w - 1; u < c.units; u += c.producers) {
            const int st = u % c.ring_units;
            const uint32_t ph = (u / c.ring_units) & 1;
            mbar_wait(&empty[st], ph ^ 1);
            mbar_expect(&full[st], pbytes + qbytes);
            tma4d(sP + st * pbytes, &mP, &full[st], 0, tp * 128, u * c.unit_kb, 0);
            tma4d(sQ + st * qbytes, &mQ, &full[st], 0, tq * c.qrows, u * c.unit_kb, 0);
        }
    } else if (threadIdx.x == 0) {
        int st = 0;
        uint32_t ph = 0;
        for (int u = 0; u < c.units; ++u) {
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
            if (++st == c.ring_units) { st = 0; ph ^= 1; }
        }
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[blockIdx.x] = t1 - t0;
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    const int M = 128, N = 768, K = 768;
    void *A, *B;
    CK(cudaMalloc(&A, (size_t)M * K * 2));
    CK(cudaMalloc(&B, (size_t)N * K * 2));
    CK(cudaMemset(A, 1, (size_t)M * K * 2));
    CK(cudaMemset(B, 1, (size_t)N * K * 2));
    unsigned long long* out;
    CK(cudaMalloc(&out, 4096 * 8));
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    for (int unit_kb : {1, 2}) {
        for (int qrows : {16, 64}) {
            CUtensorMap mP, mQ;
            cuuint64_t dP[4] = {64, (cuuint64_t)N, (cuuint64_t)(K / 64), 1};
            cuuint64_t dQ[4] = {64, (cuuint64_t)M, (cuuint64_t)(K / 64), 1};
            cuuint64_t sP[3] = {(cuuint64_t)K * 2, 128, (cuuint64_t)N * K * 2};
            cuuint64_t sQ[3] = {(cuuint64_t)K * 2, 128, (cuuint64_t)M * K * 2};
            cuuint32_t bP[4] = {64, 128, (cuuint32_t)unit_kb, 1};
            cuuint32_t bQ[4] = {64, (cuuint32_t)qrows, (cuuint32_t)unit_kb, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            if (enc(&mP, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, B, dP, sP, bP, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
                enc(&mQ, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, A, dQ, sQ, bQ, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
                printf("encode failed\n");
                return 1;
            }
            const int kb = K / 64, units = kb / unit_kb;
            const int unit_bytes = (128 + qrows) * 128 * unit_kb;
            for (int ring_units : {units, 10 / unit_kb, 4 / unit_kb}) {
                if (ring_units * unit_bytes > 200 * 1024 || ring_units < 1) continue;
                for (int prod : {1, 2}) {
                    Cfg c{units, ring_units, prod, unit_kb, qrows};
                    const int smem = 1024 + ring_units * unit_bytes;
                    const int grid = (N / 128) * (M / qrows);
                    std::vector<double> med;
                    for (int rep = 0; rep < 5; ++rep) {
                        probe<<<grid, 128, smem>>>(mP, mQ, c, out);
                        CK(cudaDeviceSynchronize());
                        std::vector<unsigned long long> h(grid);
                        CK(cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost));
                        double s = 0, mx = 0;
                        for (auto v : h) { s += v; mx = v > mx ? v : mx; }
                        if (rep) med.push_back(s / grid);
                    }
                    double avg = 0;
                    for (double v : med) avg += v;
                    avg /= med.size();
                    printf("unit_kb %d qrows %2d ring %2d units (%3d KB) prod %d grid %3d | per-CTA %6.2f us for %3d KB = %6.1f GB/s\n",
                           unit_kb, qrows, ring_units, ring_units * unit_bytes / 1024, prod, grid, avg / 1e3,
                           units * unit_bytes / 1024, units * unit_bytes / avg);
                }
            }
        }
    }
    return 0;
}
