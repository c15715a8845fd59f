// odf_k_aux.cu -- instantiates the auxiliary kernels (K6 index export, K4 latency
// path, NEXT-3 bit words) and holds the launchers of every kernel family.
#include <string.h>

#define ODF_KERNELS_AUX 1
#include "odf_kernels.cuh"

namespace odf {

template <int DEPTH>
static const void *bits_fn()
{
    return reinterpret_cast<const void *>(&odf_apply_bits_kernel<DEPTH>);
}

cudaError_t launch_bits(int depth, const KParams &p, bool apply, size_t smem, cudaStream_t s)
{
    static const void *t[11] = {bits_fn<0>(), bits_fn<1>(), bits_fn<2>(), bits_fn<3>(),
                                bits_fn<4>(), bits_fn<5>(), bits_fn<6>(), bits_fn<7>(),
                                bits_fn<8>(), bits_fn<9>(), bits_fn<10>()};
    KParams pc = p;
    void *args[] = {&pc};
    if (!apply)
        return cudaLaunchKernel(reinterpret_cast<const void *>(&odf_bits_from_bins_kernel),
                                dim3(static_cast<unsigned>(p.n_tiles)), dim3(kConsumerThreads), args, 0, s);
    if (depth < 0 || depth > 10) return cudaErrorInvalidValue;
    const void *f = t[depth];
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    return cudaLaunchKernel(f, dim3(static_cast<unsigned>((p.n_docs + 31) / 32)), dim3(kConsumerThreads),
                            args, smem, s);
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
static const void *main_kernel(int mode, int depth, bool u32 = false, bool wide = false, int halves = 1,
                               int tile_docs = 128)
{
    if (tile_docs == 64) {  // 64-document tiles: narrow models, one half
        if (wide || halves != 1) return nullptr;
        if (mode == MODE_BINARIZE) return kptr_t64_f(MODE_BINARIZE, 0);  // bins: leaf type irrelevant
        return u32 ? kptr_t64_u(mode, depth) : kptr_t64_f(mode, depth);
    }
    if (depth == kMixedDepth)
        return (u32 && !wide && halves == 1 && mode != MODE_BINARIZE) ? kptr_mixed(mode) : nullptr;
    if (depth < 0 || depth > 10) return nullptr;
    if (halves == 2) {  // 256-document tiles: fp32 narrow fused / apply only
        if (u32 || wide) return nullptr;
        return mode == MODE_FUSED ? kptr_fused_h2(depth) : mode == MODE_APPLY ? kptr_apply_h2(depth) : nullptr;
    }
    if (mode == MODE_FUSED)
        return wide ? (u32 ? kptr_fused_wu(depth) : kptr_fused_wf(depth))
                    : (u32 ? kptr_fused_nu(depth) : kptr_fused_nf(depth));
    if (mode == MODE_APPLY) return kptr_apply(depth, u32);
    return kptr_binarize(wide);
}

template <int DEPTH>
static const void *index_fn()
{
    return reinterpret_cast<const void *>(&odf_index_kernel<DEPTH>);
}
static const void *index_kernel(int depth, int tile_docs = 128)
{
    if (tile_docs == 64) return kptr_t64_index(depth);
    static const void *t[11] = {index_fn<0>(), index_fn<1>(), index_fn<2>(), index_fn<3>(),
                                index_fn<4>(), index_fn<5>(), index_fn<6>(), index_fn<7>(),
                                index_fn<8>(), index_fn<9>(), index_fn<10>()};
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

template <int DEPTH>
static const void *lat_fn()
{
    return reinterpret_cast<const void *>(&odf_lat_apply_kernel<DEPTH>);
}
static const void *lat_binarize_kernel(int tile_docs)
{
    return tile_docs == 64 ? kptr_t64_lat(-1) : reinterpret_cast<const void *>(&odf_lat_binarize_kernel<4>);
}
static const void *lat_apply_kernel(int depth, int tile_docs = 128, bool u32 = false)
{
    if (u32) return kptr_lat_u(depth, tile_docs);
    if (tile_docs == 64) return kptr_t64_lat(depth);
    static const void *t[11] = {lat_fn<0>(), lat_fn<1>(), lat_fn<2>(), lat_fn<3>(),
                                lat_fn<4>(), lat_fn<5>(), lat_fn<6>(), lat_fn<7>(),
                                lat_fn<8>(), lat_fn<9>(), lat_fn<10>()};
    return (depth < 0 || depth > 10) ? nullptr : t[depth];
}

cudaError_t launch_latency(int depth, const KParams &p, const CUtensorMap *tmap, int splits,
                           size_t smem_bin, size_t smem_apply, cudaStream_t s)
{
    KParams pc = p;
    CUtensorMap tm;
    if (tmap)
        tm = *tmap;
    else
        memset(&tm, 0, sizeof(tm));
    cudaError_t e = cudaSuccess;
    if (p.n_fchunks > 0) {
        void *args[] = {&pc, &tm};
        e = cudaLaunchKernel(lat_binarize_kernel(p.tile_docs),
                             dim3(p.n_fchunks, static_cast<unsigned>(p.n_tiles)), dim3(kConsumerThreads),
                             args, smem_bin, s);
        if (e != cudaSuccess) return e;
    } else {
        e = cudaMemsetAsync(p.lat_counter, 0, sizeof(uint32_t) * p.n_tiles, s);
        if (e != cudaSuccess) return e;
    }
    // kernel (2) with programmatic stream serialization after kernel (1): it launches
    // while (1) runs, stages its first chunk and waits (griddepcontrol.wait) for (1)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(splits, static_cast<unsigned>(p.n_tiles));
    cfg.blockDim = dim3(kConsumerThreads);
    cfg.dynamicSmemBytes = smem_apply;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = p.n_fchunks > 0 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args2[] = {&pc};
    const void *f = lat_apply_kernel(depth, p.tile_docs, p.leaf_u32 != 0);
    if (!f) return cudaErrorInvalidValue;
    return cudaLaunchKernelExC(&cfg, f, args2);
}

static cudaError_t opt_in(const void *f, int max_smem)
{
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                max_smem - static_cast<int>(a.sharedSizeBytes));
}

cudaError_t prepare_kernels(int max_smem)
{
    for (int d = 0; d <= 10; ++d) {
        const void *fs[] = {main_kernel(MODE_FUSED, d), main_kernel(MODE_APPLY, d),
                            main_kernel(MODE_FUSED, d, true), main_kernel(MODE_APPLY, d, true),
                            main_kernel(MODE_FUSED, d, false, true), main_kernel(MODE_FUSED, d, true, true),
                            main_kernel(MODE_FUSED, d, false, false, 2), main_kernel(MODE_APPLY, d, false, false, 2),
                            main_kernel(MODE_FUSED, d, false, false, 1, 64), main_kernel(MODE_APPLY, d, false, false, 1, 64),
                            main_kernel(MODE_FUSED, d, true, false, 1, 64), main_kernel(MODE_APPLY, d, true, false, 1, 64),
                            index_kernel(d), index_kernel(d, 64), lat_apply_kernel(d),
                            lat_apply_kernel(d, 64)};
        for (const void *f : fs) {
            cudaError_t e = opt_in(f, max_smem);
            if (e != cudaSuccess) return e;
        }
    }
    for (int d = 0; d <= kMixedDepth; ++d)
        for (int td : {128, 64}) {
            cudaError_t e = opt_in(lat_apply_kernel(d, td, true), max_smem);
            if (e != cudaSuccess) return e;
        }
    for (int mode : {MODE_FUSED, MODE_APPLY})
        for (int td : {128, 64}) {
            cudaError_t e = opt_in(main_kernel(mode, kMixedDepth, true, false, 1, td), max_smem);
            if (e != cudaSuccess) return e;
        }
    {
        cudaError_t e = opt_in(main_kernel(MODE_BINARIZE, 0, false, false, 1, 64), max_smem);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = opt_in(lat_binarize_kernel(128), max_smem);
    if (e != cudaSuccess) return e;
    e = opt_in(lat_binarize_kernel(64), max_smem);
    if (e != cudaSuccess) return e;
    e = opt_in(main_kernel(MODE_BINARIZE, 0, false, true), max_smem);
    if (e != cudaSuccess) return e;
    return opt_in(main_kernel(MODE_BINARIZE, 0), max_smem);
}

int occupancy_main(int mode, int depth, size_t smem, int tile_docs)
{
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, main_kernel(mode, depth, false, false, 1, tile_docs),
                                                      kThreads, smem) != cudaSuccess)
        return 1;
    return n > 0 ? n : 1;
}

cudaError_t launch_main(int mode, int depth, const KParams &p, const CUtensorMap *tmap, int grid,
                        size_t smem, cudaStream_t s, int halves, bool pdl_secondary)
{
    const void *f = main_kernel(mode, depth, p.leaf_u32 != 0, p.wide != 0, halves, p.tile_docs);
    if (!f) return cudaErrorInvalidValue;
    KParams pc = p;
    CUtensorMap tm;
    if (tmap)
        tm = *tmap;
    else
        memset(&tm, 0, sizeof(tm));
    void *args[] = {&pc, &tm};
    if (!pdl_secondary) return cudaLaunchKernel(f, dim3(grid), dim3(kThreads), args, smem, s);
    // programmatic dependent launch: may start while the primary (same stream) runs
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, f, args);
}

cudaError_t launch_index(int depth, const KParams &p, bool fingerprint, int grid, size_t smem,
                         cudaStream_t s)
{
    const void *f = index_kernel(depth, p.tile_docs);
    if (!f) return cudaErrorInvalidValue;
    KParams pc = p;
    int fp = fingerprint ? 1 : 0;
    void *args[] = {&pc, &fp};
    return cudaLaunchKernel(f, dim3(grid), dim3(kConsumerThreads), args, smem, s);
}

}  // namespace odf
