// launch_floor.cu -- measurement tool: the exit-to-exit floor of back-to-back kernels in a
// CUDA graph on B200, for kernels of increasing prologue weight:
//   empty            nothing
//   pdl              programmatic dependent launch, griddepcontrol.wait / launch_dependents
//   pdl+tmem         + TMEM alloc / dealloc (tcgen05), mbarrier init, __syncthreads
//   pdl+tmem+ld      + one 16 KB TMA-free global read per CTA and one 256 B store
// for grids of 1, 48 and 148 CTAs of 352 threads with 200 KB dynamic smem (1 CTA / SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/lf tools/launch_floor.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int MODE>
__global__ void __launch_bounds__(352, 1) k(const float4* in, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t holder;
    __shared__ uint64_t bar[8];
    if (MODE >= 2) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < 8; ++i)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
            asm volatile("fence.mbarrier_init.release.cluster;");
        }
        if (threadIdx.x / 32 == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&holder)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if (MODE >= 1) asm volatile("griddepcontrol.wait;" ::: "memory");
    float acc = 0.f;
    if (MODE >= 3) {
        const float4* p = in + blockIdx.x * 1024;
        for (int i = threadIdx.x; i < 1024; i += 352) { float4 v = __ldg(p + i); acc += v.x + v.y + v.z + v.w; }
        if (threadIdx.x < 64) out[blockIdx.x * 64 + threadIdx.x] = acc;
    }
    if (MODE >= 1) asm volatile("griddepcontrol.launch_dependents;");
    if (MODE >= 2) {
        __syncthreads();
        if (threadIdx.x / 32 == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(holder));
    }
}

template <int MODE>
static float run(int grid, bool pdl, float4* in, float* out) {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(352);
    cfg.dynamicSmemBytes = 200 * 1024;
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = pdl ? 1 : 0;
    const int R = 48;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < R; ++i) CK(cudaLaunchKernelEx(&cfg, k<MODE>, (const float4*)in, out));
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0, s);
        CK(cudaGraphLaunch(ge, s));
        cudaEventRecord(e1, s);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best = ms < best ? ms : best;
    }
    return best * 1e3f / R;
}

int main() {
    float4* in;
    float* out;
    CK(cudaMalloc(&in, 148 * 1024 * 16));
    CK(cudaMalloc(&out, 148 * 64 * 4));
    for (int grid : {1, 48, 148}) {
        printf("grid %3d | empty %5.2f us | empty+pdlattr %5.2f | pdl %5.2f | pdl+tmem %5.2f | pdl+tmem+ld %5.2f | tmem+ld no-pdl %5.2f\n",
               grid, run<0>(grid, false, in, out), run<0>(grid, true, in, out), run<1>(grid, true, in, out),
               run<2>(grid, true, in, out), run<3>(grid, true, in, out), run<3>(grid, false, in, out));
    }
    return 0;
}
