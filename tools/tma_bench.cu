// tma_bench.cu -- standalone TMA streaming microbenchmark (measurement tool, not part of
// the library): how fast can one SM (and the whole chip) pull K-major 128-B-swizzled tiles
// through an S-stage mbarrier ring, as a function of box rows, boxes per stage and stages?
// No MMA: a consumer thread frees each stage as soon as it lands.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_bench tools/tma_bench.cu -lcuda
//   /tmp/tma_bench
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
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
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(sa(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(sa(bar)) : "memory");
}

struct Cfg { int rows, boxes, stages, kblocks, producers, warpwide; };

// each CTA streams `boxes` row blocks of `rows` rows over kblocks x 64 columns
__global__ void __launch_bounds__(160) stream_kernel(const __grid_constant__ CUtensorMap m, Cfg c, int row_stride_ctas,
                                                    unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 16;
    uint8_t* buf = smem + 1024;
    const int box_bytes = c.rows * 128;
    const int stage_bytes = box_bytes * c.boxes;
    if (threadIdx.x == 0) {
        for (int i = 0; i < c.stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int row0 = (blockIdx.x % row_stride_ctas) * c.rows * c.boxes;
    const int w = threadIdx.x >> 5;
    if (w >= 1 && w <= c.producers && c.warpwide) {
        // whole warp runs the loop (warp-uniform values), one elected lane issues
        const int pi = w - 1;
        long long tw = 0, te = 0, tt = 0;
        for (int kb = pi; kb < c.kblocks; kb += c.producers) {
            const int st = kb % c.stages;
            const uint32_t ph = (kb / c.stages) & 1;
            long long a = clock64();
            mbar_wait(&empty[st], ph ^ 1);
            long long b0 = clock64(), b1 = b0;
            if (elect_one()) {
                mbar_expect(&full[st], stage_bytes);
                b1 = clock64();
                for (int b = 0; b < c.boxes; ++b)
                    tma2d(buf + st * stage_bytes + b * box_bytes, &m, &full[st], kb * 64, row0 + b * c.rows);
            }
            __syncwarp();
            long long b2 = clock64();
            tw += b0 - a; te += b1 - b0; tt += b2 - b1;
        }
        if (blockIdx.x == 0 && pi == 0 && (threadIdx.x & 31) == 0) {
            const int n = (c.kblocks + c.producers - 1) / c.producers;
            out[2048] = tw / n; out[2049] = te / n; out[2050] = tt / n;
        }
    } else if (w >= 1 && (threadIdx.x & 31) == 0 && w <= c.producers) {
        // producer w-1 of c.producers handles k-blocks kb = (w-1) mod producers
        const int pi = w - 1;
        long long tw = 0, te = 0, tt = 0;
        for (int kb = pi; kb < c.kblocks; kb += c.producers) {
            const int st = kb % c.stages;
            const uint32_t ph = (kb / c.stages) & 1;
            long long a = clock64();
            mbar_wait(&empty[st], ph ^ 1);
            long long b0 = clock64();
            mbar_expect(&full[st], stage_bytes);
            long long b1 = clock64();
            for (int b = 0; b < c.boxes; ++b)
                tma2d(buf + st * stage_bytes + b * box_bytes, &m, &full[st], kb * 64, row0 + b * c.rows);
            long long b2 = clock64();
            tw += b0 - a; te += b1 - b0; tt += b2 - b1;
        }
        if (blockIdx.x == 0 && pi == 0) {
            const int n = (c.kblocks + c.producers - 1) / c.producers;
            out[2048] = tw / n; out[2049] = te / n; out[2050] = tt / n;
        }
    } else if (threadIdx.x == 0) {
        int st = 0; uint32_t ph = 0;
        for (int kb = 0; kb < c.kblocks; ++kb) {
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
            if (++st == c.stages) { st = 0; ph ^= 1; }
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
    const long long K = 16384;                  // columns (bf16): 32 KB per row
    const long long ROWS = 8192;                // 256 MB tensor (cold if > L2 per pass)
    void* buf;
    CK(cudaMalloc(&buf, ROWS * K * 2));
    CK(cudaMemset(buf, 1, ROWS * K * 2));
    unsigned long long* out;
    CK(cudaMalloc(&out, 4096 * 8));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    printf("prod rows boxes stages stageKB | grid  us/kblock  GB/s/SM  chipTB/s\n");
    std::vector<Cfg> cfgs;
    for (int ww : {0, 1})
    for (int prod : {1, 2})
        for (int rows : {128})
            for (int boxes : {1, 2})
                for (int stages : {4, 8})
                    if (rows * 128 * boxes * stages <= 200 * 1024 && stages % prod == 0)
                        cfgs.push_back({rows, boxes, stages, 256, prod, ww});
    for (auto c : cfgs) {
        for (int grid : {1, sms}) {
            CUtensorMap m;
            cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)ROWS};
            cuuint64_t strides[1] = {(cuuint64_t)K * 2};
            cuuint32_t box[2] = {64, (cuuint32_t)c.rows};
            cuuint32_t es[2] = {1, 1};
            if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                printf("encode failed\n");
                return 1;
            }
            const int smem = 1024 + c.rows * 128 * c.boxes * c.stages;
            const int stride = (int)(ROWS / (c.rows * c.boxes));
            for (int rep = 0; rep < 3; ++rep) stream_kernel<<<grid, 160, smem>>>(m, c, stride, out);
            CK(cudaDeviceSynchronize());
            std::vector<unsigned long long> h(grid);
            CK(cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost));
            double mx = 0, sum = 0;
            for (auto v : h) { mx = v > mx ? v : mx; sum += v; }
            const double avg_ns = sum / grid;
            const double kb_us = avg_ns / 1e3 / c.kblocks;
            const double bytes = (double)c.rows * 128 * c.boxes * c.kblocks;
            unsigned long long cy[3];
            CK(cudaMemcpy(cy, out + 2048, 24, cudaMemcpyDeviceToHost));
            printf("ww%d %4d %4d %5d %6d %7d | %4d %9.3f %8.1f %9.2f | clk wait %llu expect %llu tma %llu\n", c.warpwide, c.producers, c.rows, c.boxes, c.stages,
                   c.rows * 128 * c.boxes / 1024, grid, kb_us, bytes / avg_ns, bytes * grid / mx / 1e3, cy[0], cy[1], cy[2]);
        }
    }
    return 0;
}
