// vx_live.cu -- the LIVE empirical tier of Vortex's hybrid analyzer.
//
// PAPER.md:1957-1964 (Sec. 5.2): "empirical profiling ... on GPUs at both L0 and L1 levels.
// For higher levels, it utilizes an analytical cost model"; ablation in tbl:eval:analyzer
// (PAPER.md:2853-2889).  The compiled-in table (vx_calib.cpp) is that tier measured once,
// offline, on a B200.  vx_calibrate redoes it on the caller's device, inside the library:
//
//   1. profile: every tcgen05 / GEMV rung and schedule of the 16-bit strategy table is timed
//      over a FIXED generic grid of shapes (never a workload shape: the method stays
//      sample-free), each timing a CUDA graph of back-to-back launches over rotating
//      slices of large arenas (cold operands, the regime vx_gemm runs in);
//   2. fit: the per-rung constants (mac, l2s, epi, fixed) of the SAME integer Eqs. 2-4 that
//      vx_plan_select evaluates are fitted by a deterministic coordinate search on
//      log-constants, minimising mean squared log error + 10 x mean log-regret of the
//      model's pick per shape (the objective of tools/calibrate.py);
//   3. freeze: the result is an immutable vx_calib_t; plans built from it
//      (vx_plan_calibrated) select deterministically, like the compiled-in ones.
// Chip-wide constants (HBM and DSMEM rates, cluster / stream-K surcharges) are kept from the
// compiled-in table: the paper profiles only L0/L1 and keeps the higher levels analytical.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "vx_internal.h"

namespace vx {

namespace {

__global__ void fill_kernel(uint16_t* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 15;
        h *= 2246822519u;
        h ^= h >> 13;
        // bf16 / fp16 bit patterns of small values in [-1, 1): sign, low exponent, mantissa
        p[i] = (uint16_t)(((h & 1u) << 15) | (0x3Cu << 8) | ((h >> 8) & 0x7Fu));
    }
}

struct Sample {
    int plan;        // index into the plans vector
    int rung, split;
    int64_t M;
    double us;       // measured per-launch time
    int group;       // shape (plan, M) index
};

const char* fam_name(int f) { return f == kUmma ? "umma" : f == kUmmaSwap ? "umma_swap" : "gemv"; }

std::string key_of(const Rung& r) {
    char k[64];
    if (r.occ == 2) snprintf(k, sizeof k, "%s_o2_%dx%d", fam_name(r.family), r.bm, r.bn);
    else if (r.mc > 1) snprintf(k, sizeof k, "%s_mc%d_%dx%d", fam_name(r.family), r.mc, r.bm, r.bn);
    else snprintf(k, sizeof k, "%s_%dx%d", fam_name(r.family), r.bm, r.bn);
    return k;
}

}  // namespace

static vx_status live_fail(cudaError_t e, const char* what) {
    set_error("vx_calibrate: %s: %s", what, cudaGetErrorString(e));
    return VX_ERR_CUDA;
}

}  // namespace vx

using namespace vx;

extern "C" vx_status vx_calibrate(int device, vx_blayout bl, int32_t effort, vx_calib_t* out) {
    if (!out || (bl != VX_B_NK && bl != VX_B_KN)) {
        set_error("vx_calibrate: NULL output or layout not KN / NK");
        return VX_ERR_INVALID;
    }
    *out = nullptr;
    // the fixed generic grid (independent of any workload; cf. tools/calibrate.py CAL_NK)
    std::vector<std::pair<int64_t, int64_t>> nk = {{2048, 1024}, {6144, 2048}, {1536, 512},
                                                   {10752, 2048}};
    std::vector<int64_t> ms = {1, 4, 16, 64, 256, 1024, 4096};
    if (effort > 0) {
        nk.push_back({4096, 4096});
        nk.push_back({3328, 1536});
        nk.push_back({14336, 4096});
        ms = {1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192};
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); set_error("vx_calibrate: no device %d", device); return VX_ERR_NODEV; }
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};

    const size_t arena = (size_t)128 << 20;   // elements per operand arena (256 MB bf16)
    uint16_t *dA = nullptr, *dB = nullptr, *dC = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaError_t ce = cudaMalloc(&dA, arena * 2);
    if (ce == cudaSuccess) ce = cudaMalloc(&dB, arena * 2);
    if (ce == cudaSuccess) ce = cudaMalloc(&dC, arena * 2);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaEventCreate(&e0);
    if (ce == cudaSuccess) ce = cudaEventCreate(&e1);
    auto cleanup = [&] {
        if (dA) cudaFree(dA);
        if (dB) cudaFree(dB);
        if (dC) cudaFree(dC);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (st) cudaStreamDestroy(st);
    };
    if (ce != cudaSuccess) { cleanup(); return live_fail(ce, "allocation"); }
    fill_kernel<<<1184, 256, 0, st>>>(dA, arena, 11u);
    fill_kernel<<<1184, 256, 0, st>>>(dB, arena, 23u);
    cudaStreamSynchronize(st);

    std::vector<vx_plan_t> plans;
    std::vector<Sample> samples;
    int groups = 0;
    vx_status vs = VX_OK;
    for (size_t pi = 0; pi < nk.size() && vs == VX_OK; ++pi) {
        const int64_t N = nk[pi].first, K = nk[pi].second;
        vx_plan_t p = nullptr;
        vs = vx_plan(N, K, VX_BF16, VX_BF16, bl, device, &p);
        if (vs != VX_OK) break;
        plans.push_back(p);
        for (int64_t M : ms) {
            const int g = groups++;
            const size_t need = (size_t)(M * K + N * K + M * N);
            const int R = (int)std::max<int64_t>(4, std::min<int64_t>(24, (int64_t)(arena / need)));
            for (const Rung& r : p->rungs) {
                if (r.family == kSimt || (r.family == kGemv && M > r.bm)) continue;
                for (int s : r.splits) {
                    // R launches on consecutive arena slices, captured once as a graph
                    cudaGraph_t graph = nullptr;
                    cudaGraphExec_t exec = nullptr;
                    ce = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
                    if (ce != cudaSuccess) { vs = live_fail(ce, "capture"); break; }
                    size_t oa = 0, ob = 0, oc = 0;
                    for (int i = 0; i < R && vs == VX_OK; ++i) {
                        if (oa + M * K > arena) oa = 0;
                        if (ob + N * K > arena) ob = 0;
                        if (oc + M * N > arena) oc = 0;
                        vs = vx_gemm_ex(p, 1, M, N, K, dA + oa, M * K, dB + ob, N * K, dC + oc,
                                        M * N, r.rung_id, s, st, nullptr);
                        oa += (M * K + 127) / 128 * 128;
                        ob += (N * K + 127) / 128 * 128;
                        oc += (M * N + 127) / 128 * 128;
                    }
                    ce = cudaStreamEndCapture(st, &graph);
                    if (vs != VX_OK) { if (graph) cudaGraphDestroy(graph); break; }
                    if (ce == cudaSuccess) ce = cudaGraphInstantiate(&exec, graph, 0);
                    if (ce == cudaSuccess) ce = cudaGraphLaunch(exec, st);   // warm-up
                    std::vector<float> t;
                    for (int rep = 0; rep < 3 && ce == cudaSuccess; ++rep) {
                        cudaEventRecord(e0, st);
                        ce = cudaGraphLaunch(exec, st);
                        cudaEventRecord(e1, st);
                        if (ce == cudaSuccess) ce = cudaEventSynchronize(e1);
                        float ms_ = 0.f;
                        cudaEventElapsedTime(&ms_, e0, e1);
                        t.push_back(ms_ * 1000.f / R);
                    }
                    if (exec) cudaGraphExecDestroy(exec);
                    if (graph) cudaGraphDestroy(graph);
                    if (ce != cudaSuccess) { vs = live_fail(ce, "timing"); break; }
                    std::sort(t.begin(), t.end());
                    samples.push_back({(int)pi, r.rung_id, s, M, (double)t[1], g});
                }
                if (vs != VX_OK) break;
            }
            if (vs != VX_OK) break;
        }
    }
    cleanup();
    if (vs != VX_OK) {
        for (auto p : plans) vx_plan_destroy(p);
        return vs;
    }

    // ---- fit (coordinate search on log-constants, cached predictions per key) -------------
    std::map<std::string, int> kidx;
    std::vector<std::string> keys;
    std::vector<int> skey(samples.size());
    for (size_t j = 0; j < samples.size(); ++j) {
        const Rung& r = plans[samples[j].plan]->rungs[samples[j].rung];
        const std::string k = key_of(r);
        if (!kidx.count(k)) { kidx[k] = (int)keys.size(); keys.push_back(k); }
        skey[j] = kidx[k];
    }
    std::vector<double> x(4 * keys.size());
    for (size_t i = 0; i < keys.size(); ++i) {
        const RungConst* c = builtin_calib().find(keys[i]);
        const double d[4] = {c ? (double)c->mac_milli : 2048000.0, c ? (double)c->l2s_milli : 96000.0,
                             c ? (double)c->epi_milli : 64000.0, c ? (double)c->fixed : 3000.0};
        for (int f = 0; f < 4; ++f) x[4 * i + f] = std::log(std::max(d[f], 1.0));
    }
    const double clock_ghz = plans[0]->desc.clock_khz > 0 ? plans[0]->desc.clock_khz / 1e6 : 1.965;
    auto apply = [&](size_t i, const std::vector<double>& xv) {
        for (vx_plan_t p : plans)
            for (Rung& r : p->rungs)
                if (key_of(r) == keys[i]) {
                    r.mac_milli = std::max<int64_t>(1, llround(std::exp(xv[4 * i + 0])));
                    r.l2s_milli = std::max<int64_t>(1, llround(std::exp(xv[4 * i + 1])));
                    r.epi_milli = std::max<int64_t>(1, llround(std::exp(xv[4 * i + 2])));
                    r.fixed = std::max<int64_t>(0, llround(std::exp(xv[4 * i + 3])));
                }
    };
    std::vector<double> pred(samples.size());
    auto predict = [&](size_t j) {
        const Sample& s = samples[j];
        vx_choice c;
        if (select_choice(plans[s.plan], 1, s.M, plans[s.plan]->N, s.rung, s.split, &c) != VX_OK)
            return 1e30;
        return (double)c.cost / (clock_ghz * 1e3);
    };
    for (size_t i = 0; i < keys.size(); ++i) apply(i, x);
    for (size_t j = 0; j < samples.size(); ++j) pred[j] = predict(j);
    std::vector<double> best(groups, 1e30);
    for (const Sample& s : samples) best[s.group] = std::min(best[s.group], s.us);
    auto objective = [&](const std::vector<double>& pr) {
        double e = 0;
        for (size_t j = 0; j < samples.size(); ++j) {
            const double d = std::log(pr[j]) - std::log(samples[j].us);
            e += d * d;
        }
        e /= samples.size();
        std::vector<int> pick(groups, -1);
        for (size_t j = 0; j < samples.size(); ++j) {
            int& b = pick[samples[j].group];
            if (b < 0 || pr[j] < pr[b]) b = (int)j;
        }
        double reg = 0;
        for (int g = 0; g < groups; ++g) reg += std::log(samples[pick[g]].us / best[g]);
        return e + 10.0 * reg / groups;
    };
    double fbest = objective(pred);
    const double lo[4] = {std::log(1000.0), std::log(4000.0), std::log(1000.0), std::log(100.0)};
    const double hi[4] = {std::log(8192000.0), std::log(256000.0), std::log(1024000.0), std::log(20000.0)};
    const double steps[4] = {std::log(2.0), std::log(1.4), std::log(1.15), std::log(1.05)};
    for (int sweep = 0; sweep < 8; ++sweep) {
        bool improved = false;
        for (size_t i = 0; i < keys.size(); ++i)
            for (int f = 0; f < 4; ++f)
                for (double stp : steps)
                    for (int sg = -1; sg <= 1; sg += 2) {
                        std::vector<double> xt = x;
                        xt[4 * i + f] = std::min(std::max(xt[4 * i + f] + sg * stp, keys[i].rfind("gemv", 0) == 0 && f == 0 ? std::log(1.0) : lo[f]), hi[f]);
                        if (xt[4 * i + f] == x[4 * i + f]) continue;
                        apply(i, xt);
                        std::vector<double> pt = pred;
                        for (size_t j = 0; j < samples.size(); ++j)
                            if (skey[j] == (int)i) pt[j] = predict(j);
                        const double ft = objective(pt);
                        if (ft < fbest - 1e-12) {
                            x = xt; pred = pt; fbest = ft; improved = true;
                        } else {
                            apply(i, x);
                        }
                    }
        if (!improved) break;
    }
    vx_calib_s* c = new (std::nothrow) vx_calib_s();
    if (!c) { for (auto p : plans) vx_plan_destroy(p); return VX_ERR_OOM; }
    c->table = builtin_calib();
    char src[64];
    snprintf(src, sizeof src, "live:device%d:%zu-samples", device, samples.size());
    c->table.source = src;
    for (size_t i = 0; i < keys.size(); ++i) {
        RungConst rc{keys[i], std::max<int64_t>(1, llround(std::exp(x[4 * i]))),
                     std::max<int64_t>(1, llround(std::exp(x[4 * i + 1]))),
                     std::max<int64_t>(1, llround(std::exp(x[4 * i + 2]))),
                     std::max<int64_t>(0, llround(std::exp(x[4 * i + 3])))};
        bool found = false;
        for (auto& r : c->table.rungs)
            if (r.key == rc.key) { r = rc; found = true; }
        if (!found) c->table.rungs.push_back(rc);
    }
    for (auto p : plans) vx_plan_destroy(p);
    *out = c;
    return VX_OK;
}
