// vx_k_mc.cu -- TMA-multicast cluster rungs: instantiations (R6)
#include "vx_kernels.h"

namespace vx {
template <int BN, bool SWAP, int MC>
static UmmaFn pick_mc(bool b_mn) {
    if constexpr (SWAP)
        return b_mn ? (UmmaFn)vx_umma_kernel<BN, true, true, false, false, MC>
                    : (UmmaFn)vx_umma_kernel<BN, true, false, false, false, MC>;
    else
        return b_mn ? (UmmaFn)vx_umma_kernel<BN, false, false, true, false, MC>
                    : (UmmaFn)vx_umma_kernel<BN, false, false, false, false, MC>;
}

UmmaFn umma_fn_mc(int family, int bn, int mc, bool b_mn) {
    if (family == 0) return bn == 128 ? pick_mc<128, false, 2>(b_mn) : pick_mc<256, false, 2>(b_mn);
    if (mc == 4) return pick_mc<64, true, 4>(b_mn);
    return bn == 32 ? pick_mc<32, true, 2>(b_mn) : pick_mc<64, true, 2>(b_mn);
}
}  // namespace vx
