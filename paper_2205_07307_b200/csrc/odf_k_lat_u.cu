// odf_k_lat_u.cu -- instantiates the K4 latency apply kernel for integer-leaf models
// (NEXT-1, u64 sums): depths 0..10 and mixed heights (NEXT-2), 128- and 64-document tiles.
#include "odf_kernels.cuh"

namespace odf {

template <int DEPTH, int DPL>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_lat_apply_kernel<DEPTH, DPL, true>);
}

const void *kptr_lat_u(int depth, int tile_docs)  // depth 0..10 or kMixedDepth
{
    static const void *t4[12] = {fn<0, 4>(), fn<1, 4>(), fn<2, 4>(), fn<3, 4>(), fn<4, 4>(), fn<5, 4>(),
                                 fn<6, 4>(), fn<7, 4>(), fn<8, 4>(), fn<9, 4>(), fn<10, 4>(),
                                 fn<kMixedDepth, 4>()};
    static const void *t2[12] = {fn<0, 2>(), fn<1, 2>(), fn<2, 2>(), fn<3, 2>(), fn<4, 2>(), fn<5, 2>(),
                                 fn<6, 2>(), fn<7, 2>(), fn<8, 2>(), fn<9, 2>(), fn<10, 2>(),
                                 fn<kMixedDepth, 2>()};
    if (depth < 0 || depth > kMixedDepth) return nullptr;
    return tile_docs == 64 ? t2[depth] : t4[depth];
}

}  // namespace odf
