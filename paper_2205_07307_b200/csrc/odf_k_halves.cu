// odf_k_halves.cu -- instantiates the 256-document-tile kernels (two 128-document
// halves, H = 2; odf_kernels.cuh "odf_main_kernel"): fused and apply, fp32 leaves,
// narrow models, depths 0..10.
#include "odf_kernels.cuh"

namespace odf {

template <int MODE, int DEPTH>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_main_kernel<MODE, DEPTH, false, false, 2>);
}

const void *kptr_fused_h2(int depth)
{
    static const void *t[11] = {fn<MODE_FUSED, 0>(), fn<MODE_FUSED, 1>(), fn<MODE_FUSED, 2>(),
                                fn<MODE_FUSED, 3>(), fn<MODE_FUSED, 4>(), fn<MODE_FUSED, 5>(),
                                fn<MODE_FUSED, 6>(), fn<MODE_FUSED, 7>(), fn<MODE_FUSED, 8>(),
                                fn<MODE_FUSED, 9>(), fn<MODE_FUSED, 10>()};
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

const void *kptr_apply_h2(int depth)
{
    static const void *t[11] = {fn<MODE_APPLY, 0>(), fn<MODE_APPLY, 1>(), fn<MODE_APPLY, 2>(),
                                fn<MODE_APPLY, 3>(), fn<MODE_APPLY, 4>(), fn<MODE_APPLY, 5>(),
                                fn<MODE_APPLY, 6>(), fn<MODE_APPLY, 7>(), fn<MODE_APPLY, 8>(),
                                fn<MODE_APPLY, 9>(), fn<MODE_APPLY, 10>()};
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

}  // namespace odf
