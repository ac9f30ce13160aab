// vx_calib.cpp -- the empirical tier of Vortex's hybrid analytical-empirical analyzer
// (Sec. 5.2: "empirical profiling ... on GPUs at both L0 and L1
// levels. For higher levels, it utilizes an analytical cost model").
//
// On sm_100a the L0/L1 behaviour of a rung is summarised by four effective rates, fitted
// ONCE from a forced-rung profile of every rung on a fixed generic grid of calibration
// shapes (tools/calibrate.py; raw data in profiles/) and compiled in, so vx_plan stays
// deterministic and sample-free (no workload shape is ever profiled):
//   mac_milli  MACs per SM cycle of the rung's MMA issue loop           (Cost_{L-1})
//   l2s_milli  bytes per SM cycle TMA delivers into this CTA's SMEM ring (T_Load, per CTA)
//   epi_milli  bytes per SM cycle of the TMEM -> register -> global epilogue (T_Store)
//   fixed      cycles of prologue (barrier init, TMEM alloc, descriptor fetch) + launch
// plus chip-wide HBM bandwidth, DSMEM bandwidth and the cluster-launch surcharge.
// All values are integers scaled x1000 so the selector is exact integer arithmetic (R14).
//
// The test side keeps its own copy of these numbers (oracle/calib_b200.json);
// tests/test_selector_parity.py checks the two agree through vx_plan_dump.
#include <cstring>

#include "vx_internal.h"

namespace vx {

static const Calib kCalib = {
    /*hbm_milli=*/3327023,   // 6543 GB/s measured copy bandwidth / 1.965 GHz
    /*dsm_milli=*/2931,      // effective in-cluster reduce rate (fitted)
    /*fixed_cluster=*/2538,  // cluster launch + two cluster barriers (fitted)
    /*skfix_milli=*/13315,   // stream-K partial write + read-back (fitted)
    /*stagger=*/4000,       // first wave > sm_count / 2 CTAs, back to back (R21; fitted)
};

static const RungCalib kRungs[] = {
    {"umma_128x64", 1000367, 46603, 8000, 7014},
    {"umma_128x128", 1520875, 160000, 8000, 371},
    {"umma_128x256", 1923790, 160000, 30923, 200},
    {"umma_256x128", 3611307, 86550, 25081, 3481},
    {"umma_256x64", 2323400, 160000, 40405, 11183},
    {"umma_256x256", 4096000, 146087, 70638, 1233},
    {"umma_swap_128x16", 2468107, 33673, 9200, 4053},
    {"umma_swap_128x32", 1000000, 45735, 15471, 4110},
    {"umma_swap_128x64", 1183082, 56182, 11212, 2864},
    {"umma_swap_128x128", 1837162, 51409, 14512, 1635},
    // BN = 192 / swapped BN = 192, 256 (tile-boundary cliffs, R6)
    {"umma_128x192", 1470000, 106501, 34060, 200},
    {"umma_swap_128x192", 1738143, 100193, 33920, 450},
    {"umma_swap_128x256", 1936545, 160000, 29217, 450},
    // TMA-multicast clusters
    {"umma_mc2_128x128", 1744850, 41151, 13097, 2547},
    {"umma_mc2_128x256", 4096000, 38348, 512000, 3025},
    {"umma_swap_mc2_128x32", 1000000, 36759, 8000, 3330},
    {"umma_swap_mc2_128x64", 1050000, 40140, 512000, 7115},
    {"umma_swap_mc4_128x64", 1000000, 36408, 512000, 6776},
    {"gemv_1x8", 28714, 9151, 1000, 3332},
    {"gemv_2x8", 8243, 43894, 1000, 3215},
    {"gemv_4x8", 8776, 64524, 1000, 2932},
    {"gemv_8x8", 10157, 5087, 148392, 497},
    {"simt_32x32", 128000, 32000, 16000, 2000},
    {"simt_64x64", 128000, 32000, 16000, 2000},
    {"simt_128x64", 128000, 32000, 16000, 2000},
};

const Calib& calib_globals() { return kCalib; }

const RungCalib* calib_lookup(const std::string& key) {
    for (const auto& r : kRungs)
        if (key == r.key) return &r;
    return nullptr;
}

int calib_count() { return (int)(sizeof(kRungs) / sizeof(kRungs[0])); }
const RungCalib* calib_at(int i) { return &kRungs[i]; }

const CalibTable& builtin_calib() {
    static const CalibTable t = [] {
        CalibTable c;
        c.glob = kCalib;
        c.source = "compiled-in";
        for (const auto& r : kRungs) c.rungs.push_back({r.key, r.mac_milli, r.l2s_milli, r.epi_milli, r.fixed});
        return c;
    }();
    return t;
}

}  // namespace vx
