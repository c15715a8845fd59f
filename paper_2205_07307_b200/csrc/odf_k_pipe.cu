// odf_k_pipe.cu -- instantiates the pipelined fused kernel (MODE_PIPE, odf_kernels.cuh
// "K3p"): fp32 and u32 leaves, depths 0..10, 128-document tiles; fp32 leaves with
// 256-document tiles for depths 7..10 (deep forests, whose staging binds).
#include "odf_kernels.cuh"

namespace odf {

template <int DEPTH, bool U32, int H>
static const void *fn()
{
    return reinterpret_cast<const void *>(&odf_pipe_kernel<DEPTH, U32, H>);
}

const void *kptr_pipe(int depth, bool u32, int halves)
{
    static const void *t1[2][11] = {
        {fn<0, false, 1>(), fn<1, false, 1>(), fn<2, false, 1>(), fn<3, false, 1>(), fn<4, false, 1>(),
         fn<5, false, 1>(), fn<6, false, 1>(), fn<7, false, 1>(), fn<8, false, 1>(), fn<9, false, 1>(),
         fn<10, false, 1>()},
        {fn<0, true, 1>(), fn<1, true, 1>(), fn<2, true, 1>(), fn<3, true, 1>(), fn<4, true, 1>(),
         fn<5, true, 1>(), fn<6, true, 1>(), fn<7, true, 1>(), fn<8, true, 1>(), fn<9, true, 1>(),
         fn<10, true, 1>()}};
    static const void *t2[4] = {fn<7, false, 2>(), fn<8, false, 2>(), fn<9, false, 2>(), fn<10, false, 2>()};
    if (depth < 0 || depth > 10) return nullptr;
    if (halves == 1) return t1[u32 ? 1 : 0][depth];
    if (halves == 2 && !u32 && depth >= 7) return t2[depth - 7];
    return nullptr;
}

cudaError_t launch_pipe(int depth, const KParams &p, const CUtensorMap *tmap, int grid, size_t smem,
                        cudaStream_t s, int halves)
{
    const void *f = kptr_pipe(depth, p.leaf_u32 != 0, halves);
    if (!f || !tmap) return cudaErrorInvalidValue;
    KParams pc = p;
    CUtensorMap tm = *tmap;
    void *args[] = {&pc, &tm};
    return cudaLaunchKernel(f, dim3(grid), dim3(kPipeThreads), args, smem, s);
}

}  // namespace odf

#if ODF_DIAG & 8  // diagnostics builds: the pipelined kernel's per-tile timeline (tools/pipe_timeline.py)
extern "C" __attribute__((visibility("default"))) int odf_pipe_diag_copy(void *host, size_t bytes)
{
    if (bytes > sizeof(odf::g_diag)) bytes = sizeof(odf::g_diag);
    return static_cast<int>(cudaMemcpyFromSymbol(host, odf::g_diag, bytes));
}
extern "C" __attribute__((visibility("default"))) int odf_pipe_diag_clear()
{
    static unsigned long long zero[4096];
    for (size_t o = 0; o < sizeof(odf::g_diag); o += sizeof zero)
        cudaMemcpyToSymbol(odf::g_diag, zero, sizeof zero, o);
    return 0;
}
#endif
