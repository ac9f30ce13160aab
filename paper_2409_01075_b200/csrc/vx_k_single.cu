// vx_k_single.cu -- family 0 rungs, 128 x BN tiles (cta_group::1): instantiations (R6)
#include "vx_kernels.h"

namespace vx {
UmmaFn umma_fn_single(int bn, bool b_mn) {
    switch (bn) {
    case 64: return pick_mn<64, false>(b_mn);
    case 128: return pick_mn<128, false>(b_mn);
    case 192: return pick_mn<192, false>(b_mn);
    case 256: return pick_mn<256, false>(b_mn);
    }
    return nullptr;
}
}  // namespace vx
