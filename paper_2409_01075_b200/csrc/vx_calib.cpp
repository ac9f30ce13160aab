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
    /*hbm_milli=*/3333028,   // 6543 GB/s measured copy bandwidth / 1.965 GHz
    /*dsm_milli=*/3077,      // effective in-cluster reduce rate (fitted)
    /*fixed_cluster=*/1125,  // cluster launch + two cluster barriers (fitted)
    /*skfix_milli=*/10417,   // stream-K partial write + read-back (fitted)
    /*stagger=*/1134,       // first wave > sm_count / 2 CTAs, back to back (R21; fitted)
};

static const RungCalib kRungs[] = {
    {"umma_128x64", 1000367, 46985, 8000, 3789},
    {"umma_128x128", 1379479, 160000, 11200, 294},
    {"umma_128x256", 1936545, 160000, 23702, 200},
    {"umma_256x128", 4474000, 86550, 25883, 4029},
    {"umma_256x64", 3012000, 160000, 512000, 10210},
    {"umma_256x256", 5385000, 80000, 39533, 1359},
    {"umma_swap_128x16", 1558204, 44897, 33887, 4053},
    {"umma_swap_128x32", 2208420, 50091, 8000, 3404},
    {"umma_swap_128x64", 1183082, 57798, 10678, 2864},
    {"umma_swap_128x128", 1690500, 124317, 9200, 994},
    // BN = 192 / swapped BN = 192, 256 (tile-boundary cliffs, R6)
    {"umma_128x192", 1331269, 160000, 59088, 200},
    {"umma_swap_128x192", 1587000, 80000, 21423, 200},
    {"umma_swap_128x256", 2135041, 160000, 19906, 200},
    // TMA-multicast clusters
    {"umma_mc2_128x128", 1939016, 40649, 9200, 2808},
    {"umma_mc2_128x256", 2048000, 160000, 30470, 3502},
    {"umma_swap_mc2_128x32", 1000000, 34724, 9200, 5629},
    {"umma_swap_mc2_128x64", 1000000, 43359, 512000, 6454},
    {"umma_swap_mc4_128x64", 1000000, 36408, 512000, 6453},
    {"gemv_1x8", 23780, 9151, 1000, 3332},
    {"gemv_2x8", 8243, 43894, 1000, 3215},
    {"gemv_4x8", 9612, 64524, 1000, 3079},
    {"gemv_8x8", 10157, 5087, 148392, 544},
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
