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
    /*hbm_milli=*/3335674,   // 6543 GB/s measured copy bandwidth / 1.965 GHz
    /*dsm_milli=*/2931,      // effective in-cluster reduce rate (fitted)
    /*fixed_cluster=*/206,  // cluster launch + two cluster barriers (fitted)
    /*skfix_milli=*/19022,   // stream-K partial write + read-back (fitted)
};

static const RungCalib kRungs[] = {
    {"umma_128x64", 1000367, 44315, 8000, 7631},
    {"umma_128x128", 1442773, 145125, 16764, 1203},
    {"umma_128x256", 1672861, 84000, 512000, 500},
    {"umma_256x128", 3297280, 160000, 33559, 5273},
    {"umma_256x64", 3297280, 160000, 33559, 5273},   // provisional (= 256x128)
    {"umma_256x256", 4096000, 152381, 72112, 500},
    {"umma_swap_128x16", 1000000, 20745, 8000, 4053},
    {"umma_swap_128x32", 1000000, 28993, 8000, 4531},
    {"umma_swap_128x64", 1000000, 42147, 512000, 5892},
    {"umma_swap_128x128", 1449009, 160000, 8000, 726},
    // BN = 192 / swapped BN = 192, 256 (tile-boundary cliffs, R6): provisional constants
    {"umma_128x192", 1600000, 100000, 32000, 800},
    {"umma_swap_128x192", 1600000, 100000, 32000, 800},
    {"umma_swap_128x256", 1672861, 84000, 32000, 800},
    // TMA-multicast clusters: provisional = the unicast rung's constants
    {"umma_mc2_128x128", 1442773, 145125, 16764, 1203},
    {"umma_mc2_128x256", 1672861, 84000, 512000, 500},
    {"umma_swap_mc2_128x32", 1000000, 28993, 8000, 4531},
    {"umma_swap_mc2_128x64", 1000000, 42147, 512000, 5892},
    {"umma_swap_mc4_128x64", 1000000, 42147, 512000, 5892},
    {"gemv_1x8", 4328, 63578, 16000, 2628},
    {"gemv_2x8", 8000, 74202, 1000, 3062},
    {"gemv_4x8", 8762, 64524, 1000, 2428},
    {"gemv_8x8", 8832, 5888, 1217, 200},
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

}  // namespace vx
