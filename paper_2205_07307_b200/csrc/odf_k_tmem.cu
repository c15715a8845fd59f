// odf_k_tmem.cu -- instantiates the fused (K3) and apply (K2) kernels with the TMEM code
// cache (fp32 leaves, narrow models, 128-document tiles, depths 4..8).
#include "odf_kernels.cuh"

namespace odf {

template <int MODE, int DEPTH>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_main_kernel<MODE, DEPTH, false, false, 1, 4, true>);
}

const void *kptr_tmem(int mode, int depth)
{
    static const void *t[2][5] = {
        {fn<MODE_FUSED, 4>(), fn<MODE_FUSED, 5>(), fn<MODE_FUSED, 6>(), fn<MODE_FUSED, 7>(), fn<MODE_FUSED, 8>()},
        {fn<MODE_APPLY, 4>(), fn<MODE_APPLY, 5>(), fn<MODE_APPLY, 6>(), fn<MODE_APPLY, 7>(), fn<MODE_APPLY, 8>()}};
    if (depth < kTmemMinDepth || depth > kTmemMaxDepth || (mode != MODE_FUSED && mode != MODE_APPLY)) return nullptr;
    return t[mode == MODE_FUSED ? 0 : 1][depth - kTmemMinDepth];
}

}  // namespace odf
