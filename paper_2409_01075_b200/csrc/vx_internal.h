// vx_internal.h -- host-side internals shared by vx_plan.cpp (strategy table, cost model,
// selection) and vx_dispatch.cu (tensor maps, launches).  Product code only.
#pragma once

#include <atomic>
#include <memory>
#include <mutex>
#include <cstdint>
#include <string>
#include <vector>

#include "vx.h"

namespace vx {

// Kernel families of the ladder's top level
enum Family : int32_t { kUmma = 0, kUmmaSwap = 1, kSimt = 2, kGemv = 3 };

constexpr int kBkTc = 64;          // one 128-B swizzle row of 2-byte elements
constexpr int kUmmaK = 16;         // kind::f16 instruction K
constexpr int kMaxStages = 16;     // R5
constexpr int kSmemReserve = 2048; // barriers + 1024-B alignment slack
constexpr int kEpiStaging = 32768; // epilogue: 8 warps x 4 KB TMA-store staging tiles
constexpr int kEpiStagingLean = 16384;  // occupancy-2 (lean) CTAs: 4 epilogue warps x 4 KB
constexpr int kCtaSysSmem = 1024;  // shared memory the system reserves per resident CTA
constexpr int kClusterMax = 8;     // portable cluster size
constexpr int kSimtBk = 16;
constexpr int kGemvBk = 1024;       // k per CTA step (4 K-slice warps x 32 lanes x 8 elements)
constexpr int kGemvColsPerCta = 8;  // 2 column groups x 4 columns (x 4 K slices = 8 warps)
constexpr int kGemvOcc = 4;         // resident CTAs per SM assumed by the cost model (R20)

// One rung = one full chain L0 -> L1 -> L2 -> L3 of the strategy table (Alg. 2 map).
struct Rung {
    int32_t rung_id;
    int32_t family;
    int32_t cg;          // cta_group (1 or 2)
    int32_t um, un;      // L0: instruction tile (tcgen05 M x N) or FFMA thread tile
    int32_t acc_stages;  // L1: TMEM accumulator buffers
    int32_t bm, bn, bk;  // L2: CTA tile
    int32_t stages;      // L2: SMEM pipeline depth
    int32_t swap;        // L3: operand swap
    int32_t mc;          // L3: TMA-multicast cluster size sharing the A tile (1 = none)
    int32_t occ;         // L2: resident CTAs per SM the ring is sized for (1, or 2 = lean)
    std::vector<int32_t> splits;  // L3: admissible K-loop splits
    // calibration (empirical tier), scaled x1000
    int64_t mac_milli, l2s_milli, epi_milli, fixed;
};

struct Calib {
    int64_t hbm_milli, dsm_milli, fixed_cluster, skfix_milli;
    int64_t stagger;   // cycles a tcgen05 launch loses when its first wave needs more than
                       // half the SMs: back to back, its CTAs cannot all become resident
                       // while the previous grid still holds its SMs (R21)
};

struct RungCalib {
    const char* key;
    int64_t mac_milli, l2s_milli, epi_milli, fixed;
};

// compiled-in calibration table (vx_calib.cpp)
const Calib& calib_globals();
const RungCalib* calib_lookup(const std::string& key);
int calib_count();
const RungCalib* calib_at(int i);

// A calibration as a plan holds it: the compiled-in one (vx_calib.cpp) or one measured live
// on the device by vx_calibrate (vx_live.cu).  Immutable once built.
struct RungConst {
    std::string key;
    int64_t mac_milli, l2s_milli, epi_milli, fixed;
};
struct CalibTable {
    Calib glob;
    std::vector<RungConst> rungs;
    std::string source;   // "compiled-in" or "live:<device>"
    const RungConst* find(const std::string& key) const {
        for (const auto& r : rungs)
            if (r.key == key) return &r;
        return nullptr;
    }
};
const CalibTable& builtin_calib();

struct LevelCounts {
    int64_t l0, l1, l2, l3;
};

}  // namespace vx

struct vx_calib_s {
    vx::CalibTable table;
};

struct vx_plan_s {
    int64_t N;  // 0 = dynamic
    int64_t K;
    vx_dtype in, out;
    vx_blayout bl;
    vx_device_desc desc;
    vx::CalibTable cal;   // the empirical tier this plan's selection uses (copied, immutable)
    int device;  // -1 when built from an explicit descriptor
    std::vector<vx::Rung> rungs;
    vx::LevelCounts counts;
    // memo of selections for batch == 1, static N, M in [1, kMemo]
    static constexpr int64_t kMemo = 16384;
    std::vector<vx_choice> memo;
    std::unique_ptr<std::atomic<uint8_t>[]> memo_state;
    // stream-K workspaces (device): one per (device, stream) the plan launches stream-K on,
    // each sm_count partial slots of 128 x 256 fp32 + sm_count ready flags.  A workspace is
    // only ever used by launches on its own stream, which the stream serialises, so
    // concurrent vx_gemm calls with one plan on different streams never share slots/flags.
    struct Workspace { void* stream; int device; void* ptr; };
    std::vector<Workspace> ws;
    std::mutex ws_mu;
    ~vx_plan_s();
};

namespace vx {
// fused GEMM + row all-gather destinations (vx_gemm_gather)
struct GatherSpec {
    int32_t ndst;
    void* dst[8];
    int64_t row0;
};
// ragged (varlen) attention batch (vx_gemm_varlen)
struct VarSpec {
    const int* cu_dev;   // device copy of the sequence offsets (ngroups + 1)
    int32_t ngroups;
    int64_t tiles;       // total tiles over every sequence
};
// candidate filters of the runtime selection
enum SelectFilter : int32_t {
    kSelectAll = 0,
    kSelectGather = 1,   // rungs whose epilogue can fan out rows: non-swapped tcgen05, split 1 / 0
};
// vx_plan.cpp
vx_status select_choice(const vx_plan_s* p, int64_t batch, int64_t M, int64_t N,
                        int32_t force_rung, int32_t force_split, vx_choice* out,
                        int32_t filter = kSelectAll);
int in_bytes(vx_dtype d);
int out_bytes(vx_dtype d);
void set_error(const char* fmt, ...);
// vx_dispatch.cu
vx_status launch(const vx_plan_s* p, const vx_choice& ch, int64_t batch, int64_t M, int64_t N,
                 int64_t K, const void* A, int64_t sA, const void* B, int64_t sB, void* C,
                 int64_t sC, void* stream, const GatherSpec* gather = nullptr,
                 const VarSpec* var = nullptr);
// vx_plan.cpp: runtime selection for a ragged batch of sequence lengths (host offsets cu)
vx_status select_varlen(const vx_plan_s* p, const int32_t* cu, int32_t ngroups,
                        int32_t force_rung, vx_choice* out, int64_t* tiles);
vx_status prepare_kernels(const vx_plan_s* p);
}  // namespace vx
