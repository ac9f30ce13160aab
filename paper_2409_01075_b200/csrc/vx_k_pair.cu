// vx_k_pair.cu -- cta_group::2 pair rungs (256 x BN over a 2-CTA cluster): instantiations (R6)
#include "vx_kernels.h"

namespace vx {
template <int BN>
static UmmaFn pick_pair(bool b_mn) {
    return b_mn ? (UmmaFn)vx_umma_kernel<BN, false, false, true, true>
                : (UmmaFn)vx_umma_kernel<BN, false, false, false, true>;
}

UmmaFn umma_fn_pair(int bn, bool b_mn) {
    switch (bn) {
    case 64:   // each CTA holds 32 B rows: K-major B only (an MN-major 128-B swizzle
               // atom is 64 elements wide), vx_plan keeps this rung for VX_B_NK only
        return b_mn ? nullptr : (UmmaFn)vx_umma_kernel<64, false, false, false, true>;
    case 128: return pick_pair<128>(b_mn);
    case 256: return pick_pair<256>(b_mn);
    }
    return nullptr;
}
}  // namespace vx
