// vx_kernels.h -- the explicit instantiation table of the tcgen05 ladder kernels (R6),
// split over several translation units (vx_k_*.cu) so nvcc builds them in parallel.  Each
// function returns the kernel of one implemented rung, or nullptr.
#pragma once
#include "vx_umma.cuh"

namespace vx {

using UmmaFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                        const CUtensorMap, const UmmaParams);

UmmaFn umma_fn_single(int bn, bool b_mn);          // family 0, 128 x BN, cta_group::1
UmmaFn umma_fn_pair(int bn, bool b_mn);            // family 0, 256 x BN, cta_group::2
UmmaFn umma_fn_swap(int bn, bool b_mn);            // family 1, 128 x BN (P = B)
UmmaFn umma_fn_mc(int family, int bn, int mc, bool b_mn);   // TMA-multicast clusters

// B stored K x N makes B's tile MN-major: it is Q (non-swap) or P (swap)
template <int BN, bool SWAP>
UmmaFn pick_mn(bool b_mn) {
    if constexpr (SWAP)
        return b_mn ? (UmmaFn)vx_umma_kernel<BN, true, true, false>
                    : (UmmaFn)vx_umma_kernel<BN, true, false, false>;
    else
        return b_mn ? (UmmaFn)vx_umma_kernel<BN, false, false, true>
                    : (UmmaFn)vx_umma_kernel<BN, false, false, false>;
}

}  // namespace vx
