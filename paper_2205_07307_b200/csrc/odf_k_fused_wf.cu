// odf_k_fused_wf.cu -- instantiates the fused kernel (K3) for U32=false, WIDE=true, depths 0..10
// (one kernel family per translation unit, so the library builds in parallel).
#include "odf_kernels.cuh"

namespace odf {

template <int DEPTH>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_main_kernel<MODE_FUSED, DEPTH, false, true>);
}

const void *kptr_fused_wf(int depth)
{
    static const void *t[11] = {fn<0>(), fn<1>(), fn<2>(), fn<3>(), fn<4>(), fn<5>(),
                                fn<6>(), fn<7>(), fn<8>(), fn<9>(), fn<10>()};
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

}  // namespace odf
