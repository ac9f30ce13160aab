// vx_k_swap.cu -- family 1 rungs (operands swapped: N on the UMMA-M axis): instantiations (R6)
#include "vx_kernels.h"

namespace vx {
UmmaFn umma_fn_swap(int bn, bool b_mn) {
    switch (bn) {
    case 16: return pick_mn<16, true>(b_mn);
    case 32: return pick_mn<32, true>(b_mn);
    case 64: return pick_mn<64, true>(b_mn);
    case 128: return pick_mn<128, true>(b_mn);
    case 192: return pick_mn<192, true>(b_mn);
    case 256: return pick_mn<256, true>(b_mn);
    }
    return nullptr;
}
}  // namespace vx
