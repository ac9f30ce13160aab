// ingress_probe.cu -- measurement tool (not part of the library): what bounds a CTA that
// streams operand tiles?  Per-SM ingress and chip throughput for
//   (a) TMA boxes {64*D cols, R rows} (128-B swizzle, D = chunks per box through a 3-D view)
//       into an S-stage ring, P producer threads, a consumer that frees each stage at once;
//   (b) plain 16-B ld.global.nc streaming (256 threads, 8 loads in flight per thread),
// for grids G in {1, 16, 74, 86, 148, 296} over DRAM-cold data (every CTA its own rows of a
// 1 GiB tensor) or L2-hot data (every CTA the same 4 MB).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ingress tools/ingress_probe.cu -lcuda
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
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(sa(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(sa(bar)) : "memory");
}

struct Cfg { int rows, depth, stages, units, producers; long long row_stride; };

// CTA b streams `units` boxes of rows [row0, row0+rows) x (depth*64) columns, walking K
__global__ void __launch_bounds__(128) tma_kernel(const __grid_constant__ CUtensorMap m, Cfg c,
                                                  unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + 32;
    uint8_t* buf = smem + 1024;
    const int box = c.rows * 128 * c.depth;
    if (threadIdx.x == 0) {
        for (int i = 0; i < c.stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int row0 = (int)(blockIdx.x * c.row_stride);
    const int w = threadIdx.x >> 5;
    if (w >= 1 && w <= c.producers && (threadIdx.x & 31) == 0) {
        for (int u = w - 1; u < c.units; u += c.producers) {
            const int st = u % c.stages;
            const uint32_t ph = (u / c.stages) & 1;
            mbar_wait(&empty[st], ph ^ 1);
            mbar_expect(&full[st], box);
            const int per_rb = 64 / c.depth;                  // K/64 = 64 chunks per row
            const int rb = u / per_rb, ch = u - rb * per_rb;
            tma3d(buf + st * box, &m, &full[st], 0, row0 + rb * c.rows, ch * c.depth);
        }
    } else if (threadIdx.x == 0) {
        int st = 0;
        uint32_t ph = 0;
        for (int u = 0; u < c.units; ++u) {
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
            if (++st == c.stages) { st = 0; ph ^= 1; }
        }
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[blockIdx.x] = t1 - t0;
    }
}

// plain LDG streaming: CTA b reads `bytes` contiguous bytes from base + b * stride
__global__ void __launch_bounds__(256) ldg_kernel(const uint4* __restrict__ src, long long stride16,
                                                  long long n16, unsigned long long* out, uint4* sink) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const uint4* p = src + blockIdx.x * stride16;
    uint32_t acc = 0;
    for (long long i = threadIdx.x; i < n16; i += 256 * 8) {
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const long long k = i + j * 256;
            v[j] = k < n16 ? __ldg(p + k) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
    }
    __syncthreads();
    if (acc == 0x12345678) sink[threadIdx.x] = make_uint4(acc, 0, 0, 0);
    if (threadIdx.x == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[blockIdx.x] = t1 - t0;
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static void report(const char* tag, const std::vector<unsigned long long>& h, double bytes_per_cta, float ms) {
    double mx = 0, sum = 0;
    for (auto v : h) { mx = v > mx ? v : mx; sum += v; }
    const int g = (int)h.size();
    printf("%-60s grid %4d | per-CTA %7.1f GB/s (avg %6.2f us) | chip %6.2f TB/s (kernel %6.2f us)\n", tag, g,
           bytes_per_cta / (sum / g), sum / g / 1e3, bytes_per_cta * g / (ms * 1e9), ms * 1e3);
}

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    const long long K = 4096;                     // LLaMA K: 8 KB per row
    const long long ROWS = 131072;                // 1 GiB
    void* buf;
    CK(cudaMalloc(&buf, ROWS * K * 2));
    CK(cudaMemset(buf, 1, ROWS * K * 2));
    void* flush;
    CK(cudaMalloc(&flush, 512ll << 20));
    unsigned long long* out;
    CK(cudaMalloc(&out, 4096 * 8));
    uint4* sink;
    CK(cudaMalloc(&sink, 4096));
    CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // every CTA streams its own 128 rows x K (1 MB) of a DRAM-cold tensor; the box shape sets
    // the walk: {64*depth cols, rows} boxes, K-chunks of a row block first, then the next block
    for (int ring_kb : {192, 96}) {
        for (int rows : {8, 16, 32, 64, 128}) {
            for (int depth : {1, 2, 4, 8, 16, 32, 64}) {
                const int box = rows * 128 * depth;
                if (box < 8192 || box > 64 * 1024) continue;
                int stages = (ring_kb * 1024) / box;
                if (stages > 32) stages = 32;
                if (stages < 2) continue;
                CUtensorMap m;
                cuuint64_t dims[3] = {64, (cuuint64_t)ROWS, (cuuint64_t)(K / 64)};
                cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
                cuuint32_t bx[3] = {64, (cuuint32_t)rows, (cuuint32_t)depth};
                cuuint32_t es[3] = {1, 1, 1};
                if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, bx, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                    printf("encode failed rows %d depth %d\n", rows, depth);
                    continue;
                }
                for (int prod : {1, 2}) {
                    for (int g : (ring_kb == 192 ? std::vector<int>{74, 148} : std::vector<int>{148, 296})) {
                        Cfg c{rows, depth, stages, (128 / rows) * (64 / depth), prod, 128};
                        const int smem = 1024 + box * stages;
                        float ms = 0;
                        for (int rep = 0; rep < 3; ++rep) {
                            CK(cudaMemsetAsync(flush, rep, 512ll << 20));
                            cudaEventRecord(e0);
                            tma_kernel<<<g, 128, smem>>>(m, c, out);
                            cudaEventRecord(e1);
                            CK(cudaEventSynchronize(e1));
                            cudaEventElapsedTime(&ms, e0, e1);
                        }
                        std::vector<unsigned long long> h(g);
                        CK(cudaMemcpy(h.data(), out, g * 8, cudaMemcpyDeviceToHost));
                        char tag[128];
                        snprintf(tag, sizeof tag, "ring %3dKB rows %3d depth %2d (%5d B/row) st %2d prod %d", ring_kb,
                                 rows, depth, depth * 128, stages, prod);
                        report(tag, h, (double)128 * K * 2, ms);
                    }
                }
            }
        }
    }
    return 0;
}
