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
    /*dsm_milli=*/3539,      // effective in-cluster reduce rate (fitted)
    /*fixed_cluster=*/750,  // cluster launch + two cluster barriers (fitted)
    /*skfix_milli=*/12681,   // stream-K partial write + read-back (fitted)
    /*stagger=*/3176,       // first wave > sm_count / 2 CTAs, back to back (R21; fitted)
};

static const RungCalib kRungs[] = {
    {"umma_128x64", 1000367, 46603, 8000, 6919},
    {"umma_128x128", 1388625, 74650, 15451, 210},
    {"umma_128x256", 1844329, 160000, 42072, 200},
    {"umma_256x128", 4351000, 86550, 35705, 3315},
    {"umma_256x64", 2627000, 160000, 41917, 10210},
    {"umma_256x256", 5503000, 76190, 50534, 1812},
    {"umma_swap_128x16", 1656315, 42759, 23878, 4053},
    {"umma_swap_128x32", 1000000, 43557, 8000, 3404},
    {"umma_swap_128x64", 1126745, 66468, 10678, 2864},
    {"umma_swap_128x128", 1458616, 70517, 18400, 827},
    // BN = 192 / swapped BN = 192, 256 (tile-boundary cliffs, R6)
    {"umma_128x192", 1458056, 160000, 38595, 200},
    {"umma_swap_128x192", 1587000, 160000, 23619, 200},
    {"umma_swap_128x256", 2033372, 160000, 23044, 200},
    // TMA-multicast clusters
    {"umma_mc2_128x128", 1795044, 43276, 24244, 2674},
    {"umma_mc2_128x256", 4096000, 46305, 28627, 3502},
    {"umma_swap_mc2_128x32", 1393197, 36460, 8000, 5361},
    {"umma_swap_mc2_128x64", 1050000, 63738, 40077, 6454},
    {"umma_swap_mc4_128x64", 1690500, 36408, 512000, 6776},
    {"gemv_1x8", 23780, 9151, 1000, 3332},
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
