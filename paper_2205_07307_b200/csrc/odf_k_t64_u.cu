// odf_k_t64_u.cu -- 64-document tiles (DPL = 2): integer-answer (u32) fused and
// apply kernels, depths 0..10 and mixed heights (NEXT-1 / NEXT-2).
#include "odf_kernels.cuh"

namespace odf {

template <int MODE, int DEPTH>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_main_kernel<MODE, DEPTH, true, false, 1, 2>);
}

const void *kptr_t64_u(int mode, int depth)
{
    static const void *f[12] = {fn<MODE_FUSED, 0>(), fn<MODE_FUSED, 1>(), fn<MODE_FUSED, 2>(),
                                fn<MODE_FUSED, 3>(), fn<MODE_FUSED, 4>(), fn<MODE_FUSED, 5>(),
                                fn<MODE_FUSED, 6>(), fn<MODE_FUSED, 7>(), fn<MODE_FUSED, 8>(),
                                fn<MODE_FUSED, 9>(), fn<MODE_FUSED, 10>(), fn<MODE_FUSED, kMixedDepth>()};
    static const void *a[12] = {fn<MODE_APPLY, 0>(), fn<MODE_APPLY, 1>(), fn<MODE_APPLY, 2>(),
                                fn<MODE_APPLY, 3>(), fn<MODE_APPLY, 4>(), fn<MODE_APPLY, 5>(),
                                fn<MODE_APPLY, 6>(), fn<MODE_APPLY, 7>(), fn<MODE_APPLY, 8>(),
                                fn<MODE_APPLY, 9>(), fn<MODE_APPLY, 10>(), fn<MODE_APPLY, kMixedDepth>()};
    if (depth < 0 || depth > kMixedDepth || mode == MODE_BINARIZE) return nullptr;
    return mode == MODE_FUSED ? f[depth] : a[depth];
}

}  // namespace odf
