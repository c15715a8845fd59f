// odf_k_fused_nu.cu -- instantiates the fused kernel (K3) for U32=true, WIDE=false, depths 0..10
// (one kernel family per translation unit, so the library builds in parallel).
#include "odf_kernels.cuh"

namespace odf {

template <int DEPTH>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_main_kernel<MODE_FUSED, DEPTH, true, false>);
}

// mixed-height integer models (NEXT-2): depth argument kMixedDepth
const void *kptr_mixed(int mode)
{
    return mode == MODE_FUSED
               ? reinterpret_cast<const void *>(&odf_main_kernel<MODE_FUSED, kMixedDepth, true, false>)
               : reinterpret_cast<const void *>(&odf_main_kernel<MODE_APPLY, kMixedDepth, true, false>);
}

const void *kptr_fused_nu(int depth)
{
    static const void *t[11] = {fn<0>(), fn<1>(), fn<2>(), fn<3>(), fn<4>(), fn<5>(),
                                fn<6>(), fn<7>(), fn<8>(), fn<9>(), fn<10>()};
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

}  // namespace odf
