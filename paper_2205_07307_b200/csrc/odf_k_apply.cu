// odf_k_apply.cu -- instantiates the two-stage kernels: apply (K2, f32 and u32 leaves,
// depths 0..10) and binarize (K1, u8 and wide u16 bins).
#include "odf_kernels.cuh"

namespace odf {

template <int DEPTH, bool U32>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_main_kernel<MODE_APPLY, DEPTH, U32, false>);
}

const void *kptr_apply(int depth, bool u32)
{
    static const void *t[2][11] = {
        {fn<0, false>(), fn<1, false>(), fn<2, false>(), fn<3, false>(), fn<4, false>(), fn<5, false>(),
         fn<6, false>(), fn<7, false>(), fn<8, false>(), fn<9, false>(), fn<10, false>()},
        {fn<0, true>(), fn<1, true>(), fn<2, true>(), fn<3, true>(), fn<4, true>(), fn<5, true>(),
         fn<6, true>(), fn<7, true>(), fn<8, true>(), fn<9, true>(), fn<10, true>()}};
    return (depth < 0 || depth > 10) ? nullptr : t[u32 ? 1 : 0][depth];
}

const void *kptr_binarize(bool wide)
{
    static const void *t[2] = {
        reinterpret_cast<const void *>(&odf_main_kernel<MODE_BINARIZE, 0, false, false>),
        reinterpret_cast<const void *>(&odf_main_kernel<MODE_BINARIZE, 0, false, true>)};
    return t[wide ? 1 : 0];
}

}  // namespace odf
