// odf_k_t64_f.cu -- 64-document tiles (2 documents per lane, DPL = 2; models whose
// 128-document code block does not fit shared memory): fp32 fused and apply kernels,
// depths 0..10, the binarize kernel and the index-export kernel.
#include "odf_kernels.cuh"

namespace odf {

template <int MODE, int DEPTH>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_main_kernel<MODE, DEPTH, false, false, 1, 2>);
}
template <int DEPTH>
static const void *ix()
{
    return reinterpret_cast<const void *>(&odf_index_kernel<DEPTH, 2>);
}

const void *kptr_t64_f(int mode, int depth)
{
    static const void *f[11] = {fn<MODE_FUSED, 0>(), fn<MODE_FUSED, 1>(), fn<MODE_FUSED, 2>(),
                                fn<MODE_FUSED, 3>(), fn<MODE_FUSED, 4>(), fn<MODE_FUSED, 5>(),
                                fn<MODE_FUSED, 6>(), fn<MODE_FUSED, 7>(), fn<MODE_FUSED, 8>(),
                                fn<MODE_FUSED, 9>(), fn<MODE_FUSED, 10>()};
    static const void *a[11] = {fn<MODE_APPLY, 0>(), fn<MODE_APPLY, 1>(), fn<MODE_APPLY, 2>(),
                                fn<MODE_APPLY, 3>(), fn<MODE_APPLY, 4>(), fn<MODE_APPLY, 5>(),
                                fn<MODE_APPLY, 6>(), fn<MODE_APPLY, 7>(), fn<MODE_APPLY, 8>(),
                                fn<MODE_APPLY, 9>(), fn<MODE_APPLY, 10>()};
    if (mode == MODE_BINARIZE)
        return reinterpret_cast<const void *>(&odf_main_kernel<MODE_BINARIZE, 0, false, false, 1, 2>);
    if (depth < 0 || depth > 10) return nullptr;
    return mode == MODE_FUSED ? f[depth] : a[depth];
}

const void *kptr_t64_index(int depth)
{
    static const void *t[11] = {ix<0>(), ix<1>(), ix<2>(), ix<3>(), ix<4>(), ix<5>(),
                                ix<6>(), ix<7>(), ix<8>(), ix<9>(), ix<10>()};
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

// K4 latency path for 64-document-tile models: binarize (kernel 1) and apply (kernel 2)
template <int DEPTH>
static const void *la()
{
    return reinterpret_cast<const void *>(&odf_lat_apply_kernel<DEPTH, 2>);
}
const void *kptr_t64_lat(int depth)  // depth -1: the binarize kernel
{
    static const void *t[11] = {la<0>(), la<1>(), la<2>(), la<3>(), la<4>(), la<5>(),
                                la<6>(), la<7>(), la<8>(), la<9>(), la<10>()};
    if (depth == -1) return reinterpret_cast<const void *>(&odf_lat_binarize_kernel<2>);
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

}  // namespace odf
