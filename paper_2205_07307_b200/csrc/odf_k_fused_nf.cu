// odf_k_fused_nf.cu -- instantiates the fused kernel (K3) for U32=false, WIDE=false, depths 0..10
// (one kernel family per translation unit, so the library builds in parallel).
#include "odf_kernels.cuh"

namespace odf {

template <int DEPTH>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_main_kernel<MODE_FUSED, DEPTH, false, false>);
}

const void *kptr_fused_nf(int depth)
{
    static const void *t[11] = {fn<0>(), fn<1>(), fn<2>(), fn<3>(), fn<4>(), fn<5>(),
                                fn<6>(), fn<7>(), fn<8>(), fn<9>(), fn<10>()};
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

}  // namespace odf

#if ODF_DIAG & 8  // diagnostics builds: the per-warp timeline (g_diag is per translation unit: the fp32 fused kernels)
extern "C" __attribute__((visibility("default"))) int odf_diag_copy(void *host, size_t bytes)
{
    if (bytes > sizeof(odf::g_diag)) bytes = sizeof(odf::g_diag);
    return static_cast<int>(cudaMemcpyFromSymbol(host, odf::g_diag, bytes));
}
extern "C" __attribute__((visibility("default"))) int odf_diag_clear()
{
    static unsigned long long zero[1024];
    for (size_t o = 0; o < sizeof(odf::g_diag); o += sizeof zero)
        cudaMemcpyToSymbol(odf::g_diag, zero, sizeof zero, o);
    return 0;
}
#endif
