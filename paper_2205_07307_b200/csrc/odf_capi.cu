// odf_capi.cu -- the C ABI (include/odf.h): model compiler (K0), validation,
// shared-memory planning, TMA descriptor encoding and kernel launches.
//
// Model compile (K0), from the raw arrays of the paper's problem statement
// (P:80 node conditions, P:301-305 per-tree conditions and answers):
//  * used factors: every f with at least one node condition, ascending id;
//  * borders_f = sorted unique-by-== thresholds on f (-0.0 == +0.0);
//    m_f <= 254 so bins fit in uint8 (BASELINE.json north_star);
//  * node (t,l) -> k = position of its threshold in borders_f (exact ==);
//    condition x < thr  <=>  bin(x) <= k  <=>  NOT(bin >= k+1);
//  * 7-bit code columns: column A of f holds min(bin,127); factors with
//    m_f > 127 also get column B = max(bin-127, 0); a node tests
//    "code >= K" on column A with K = k+1 when k+1 <= 127, else on column B
//    with K = k-126;  level descriptor {col * 128, (128-K) * 0x01010101} for depth
//    <= 8, (col << 19) | (128-K) for depth 9-10  (odf_internal.h desc_stride);
//  * leaf tables reversed (table[F] = leaf[2^d-1-F]) because the kernels
//    assemble the complemented index F (flags are "condition false"), and
//    bank-swizzled (leaf_pos: words sharing a shared-memory bank are far apart
//    in Hamming distance, so a warp's gathers conflict less);
//  * trees grouped in chunks of tc (multiple of 16) = [descriptors | tables].
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <memory>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/odf.h"
#include "odf_internal.h"

using namespace odf;

namespace {

thread_local std::string g_err;

odf_status fail(odf_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
odf_status fail(odf_status s, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}
odf_status ok()
{
    g_err.clear();
    return ODF_OK;
}
odf_status cuda_fail(cudaError_t e, const char *what)
{
    return fail(ODF_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

uint32_t skew_h(uint32_t p) { return p + (p >> 5); }  // as skew() in odf_kernels.cu

// Bank-swizzled table position of the complemented leaf index F (as leaf_addrs /
// swz_bank_hi in odf_kernels.cu): row F >> 5 keeps its 32 words, the bank of
// word F is L ^ (H ? 31 : 0) at depth 6 and L ^ H ^ (parity(H) ? 31 : 0) at
// depth 7..10 (F = 32 H + L); tables of <= 32 words are conflict-free as they are.
uint32_t leaf_pos(int depth, uint32_t F)
{
    const uint32_t H = F >> 5, L = F & 31u;
    if (depth <= 5) return F;
    if (depth == 6) return (H << 5) | (L ^ (H ? 31u : 0u));
    const uint32_t par = static_cast<uint32_t>(__builtin_popcount(H) & 1);
    return (H << 5) | ((L ^ H ^ (par ? 31u : 0u)) & 31u);
}
constexpr uint32_t kExtraShiftH = 4;  // fmeta.y bits 4-7 = code columns - 1 (as kExtraShift)
uint32_t align_up(uint64_t v, uint64_t a) { return static_cast<uint32_t>((v + a - 1) / a * a); }
struct Plan {
    uint32_t off_bins = 0, off_ring = 0, off_red = 0, off_bars = 0;
    uint32_t slot_bytes = 0, off_meta = 0, off_bord = 0;
    int stages = 0, fsub = 1;
    uint32_t off_stage = 0;  // wide models, apply: u16 bins staging
    size_t smem = 0;
    int grid_per_sm = 1;
    int halves = 1;              // tile = halves x 128 documents
    uint32_t half_stride = 0;    // bytes between the halves' code blocks
    uint32_t hdesc_bytes = 0;    // halves == 2: tables' offset in a half-chunk ring slot
    bool valid = false;
};

#ifndef ODF_TAIL64
#define ODF_TAIL64 1  // A/B builds: 0 keeps the partly filled last wave in 128-document tiles
#endif

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

}  // namespace

struct odf_model {
    int device = 0, num_sms = 0, max_smem = 0;
    int32_t depth = 0, n_features = 0;
    int32_t kdepth = 0;  // kernel instantiation: depth, or kMixedDepth for mixed-height models
    int32_t tile_docs = kTile;  // 128, or 64 when a 128-document code block does not fit (DPL = 2)
    int32_t n_seg = 0;   // mixed-height models (NEXT-2): height segments of the chunk stream
    SegP seg[kMaxSegments] = {};
    int64_t n_trees = 0;
    std::vector<int32_t> used_ids;
    int32_t n_used = 0, n_split = 0, n_cols = 0;
    bool wide = false;  // some factor has > ODF_MAX_BORDERS borders: u16 bins (NEXT-4)
    int32_t max_borders = 0;
    int64_t total_borders = 0;
    int32_t n_fchunks = 0, border_floats = 0;
    uint32_t bord_stride = 0;  // max bytes of one sub-tile's border arrays (16-aligned)
    int32_t tc = 16, n_tchunks = 0;
    uint32_t chunk_bytes = 0, desc_bytes = 0, table_stride = 0;
    int64_t dev_bytes = 0;
    uint4 *d_fmeta = nullptr;
    float *d_borders = nullptr;
    uint8_t *d_chunks = nullptr;
    uint2 *d_splits = nullptr;
    uint2 *d_ucols = nullptr;  // wide models: per used factor {first extra column * 128, C}
    uint2 *d_bchunk = nullptr;
    uint32_t *d_bf_base = nullptr, *d_bits_desc = nullptr;  // NEXT-3 (fp32 models)
    float *d_leaves = nullptr;
    bool leaf_u32 = false;
    double scale = 1.0, bias = 0.0;
    Plan fused, binz, apply;
    Plan fused2, apply2;  // 256-document tiles (two halves), when they fit
    Plan fused64;         // 64-document tiles for a partly filled last wave (odf_score_tiles)
    // odf_score_host staging
    std::mutex host_mu;
    float *d_stage[2] = {nullptr, nullptr};
    float *d_sstage[2] = {nullptr, nullptr};
    int64_t stage_rows = 0, stage_ld = 0;
    cudaStream_t hs[2] = {nullptr, nullptr};
    cudaEvent_t ev_in = nullptr, ev_out[2] = {nullptr, nullptr};
};

namespace {

// ----------------------------------------------------------------------------
// shared-memory plans
// ----------------------------------------------------------------------------
bool make_plan(const odf_model &m, int mode, Plan &pl, std::string &why, int halves = 1, int tile_docs = 0)
{
    // code columns + the trash column (stores of unused pair slots), one block per
    // tile half; the binarize kernel of a wide model stores u16 bins; the apply kernel
    // of a wide model stages the u16 bins tile next to the code columns it expands
    // them into
    const uint32_t elem = (mode == MODE_BINARIZE && m.wide) ? 2u : 1u;
    const uint32_t td = static_cast<uint32_t>(tile_docs ? tile_docs : m.tile_docs);  // documents per tile (half)
    const uint32_t half_bins = align_up(static_cast<uint64_t>(m.n_cols + 1) * td * elem, 1024);
    const uint32_t bins = half_bins * static_cast<uint32_t>(halves);
    const uint32_t stage = (mode == MODE_APPLY && m.wide)
                               ? align_up(static_cast<uint64_t>(m.n_used) * kTile * 2, 1024) : 0u;
    const uint32_t red_bytes = (m.leaf_u32 ? 2 * kRedBytes : kRedBytes) * static_cast<uint32_t>(halves) * td / kTile;
    // the binarize kernel writes bins straight to HBM: no tile of bins in shared memory
    const uint32_t bins_region = ((mode == MODE_BINARIZE) ? 0u : std::max(bins, red_bytes)) + stage;
    const uint32_t bars = align_up(160 + 8u * m.n_fchunks, 128);  // barriers, scratch, bchunk copy
    // a factor sub-tile travels as [halves x 16 KB boxes][512 B fmeta][its border arrays]
    const uint32_t box = td * kFSub * 4u;  // one TMA box: td documents x 32 factors
    const uint32_t unit = box * halves + kMetaBytes + m.bord_stride;
    // tree jobs: whole chunks, or (halves == 2) half-chunks of tc / 2 trees
    uint32_t hdesc = 0, tree_slot;
    if (halves == 1) {
        tree_slot = align_up(m.chunk_bytes, 1024);
    } else {
        hdesc = align_up(static_cast<uint64_t>(m.tc / 2) * desc_stride(m.depth), 256);
        tree_slot = align_up(hdesc + static_cast<uint64_t>(m.tc / 2) * m.table_stride, 1024);
    }
    uint32_t slot;
    int smax;
    if (mode == MODE_BINARIZE) {  // 3 stages: two CTAs per SM (launch bounds), more warps in flight
        slot = align_up(unit, 1024);
        smax = 3;
    } else if (mode == MODE_APPLY) {
        slot = tree_slot;
        smax = 4;
    } else {
        slot = std::max<uint32_t>(tree_slot, align_up(unit, 1024));
        smax = 8;
    }
    const int64_t avail = static_cast<int64_t>(m.max_smem) - 1024;
    const int64_t fixed = static_cast<int64_t>(bins_region) + bars;
    pl.stages = static_cast<int>(std::min<int64_t>(smax, (avail - fixed) / slot));
    if (pl.stages < 2) {
        char b[256];
        snprintf(b, sizeof b,
                 "shared memory: %d x %d code columns x %u documents + 2 x %u B ring slots do not fit %d B",
                 halves, m.n_cols + 1, td, slot, m.max_smem);
        why = b;
        return false;
    }
    pl.halves = halves;
    pl.half_stride = half_bins;
    pl.hdesc_bytes = hdesc;
    pl.slot_bytes = slot;
    pl.fsub = std::max<int>(1, static_cast<int>(slot / unit));
    pl.off_meta = pl.fsub * halves * box;
    pl.off_bord = pl.off_meta + pl.fsub * kMetaBytes;
    uint32_t off = 0;
    pl.off_ring = off;                    // ring first: TMA swizzle needs 1024 B alignment
    off += pl.stages * slot;
    pl.off_bins = off;
    pl.off_red = off;                     // reduction buffer aliases the bins (dead by then)
    pl.off_stage = off + bins_region - stage;
    off += bins_region;
    pl.off_bars = off;
    off += bars;
    pl.smem = off;
    pl.valid = true;
    return true;
}

odf_status encode_tmap(const odf_model *m, const float *d_x, int64_t n_docs, int64_t ld,
                       CUtensorMap *tm, bool fm = false, int tile_docs = 0)
{
    std::call_once(g_encode_once, [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!g_encode) return fail(ODF_E_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    // doc-major: dims (factors, docs), box (32, 128), 128B swizzle;
    // feature-major (NEXT-4): dims (docs, factors), box (128, 32), 512-byte rows, no swizzle
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(fm ? n_docs : m->n_features),
                          static_cast<cuuint64_t>(fm ? m->n_features : n_docs)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
    const cuuint32_t td = static_cast<cuuint32_t>(tile_docs ? tile_docs : m->tile_docs);  // documents per tile
    cuuint32_t box[2] = {static_cast<cuuint32_t>(fm ? td : kFSub), static_cast<cuuint32_t>(fm ? kFSub : td)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(d_x), dims,
                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          fm ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ODF_E_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    return ODF_OK;
}

KParams base_params(const odf_model *m, const Plan &pl)
{
    KParams p;
    memset(&p, 0, sizeof p);
    p.fmeta = m->d_fmeta;
    p.borders = m->d_borders;
    p.n_fchunks = m->n_used > 0 ? m->n_fchunks : 0;
    p.bchunk = m->d_bchunk;
    p.chunks = m->d_chunks;
    p.n_tchunks = m->n_tchunks;
    p.tc = m->tc;
    p.n_trees = m->n_trees;
    p.chunk_bytes = m->chunk_bytes;
    p.desc_bytes = m->desc_bytes;
    p.table_stride = m->table_stride;
    p.splits = m->d_splits;
    p.n_split = m->n_split;
    p.wide = m->wide ? 1 : 0;
    p.ucols = m->d_ucols;
    p.off_stage = pl.off_stage;
    p.n_used = m->n_used;
    p.n_cols = m->n_cols;
    p.code_stride = static_cast<int64_t>(m->n_cols + 1) * m->tile_docs;  // K4 code block per tile
    p.tile_docs = m->tile_docs;
    p.off_bins = pl.off_bins;
    p.off_ring = pl.off_ring;
    p.off_red = pl.off_red;
    p.off_bars = pl.off_bars;
    p.slot_bytes = pl.slot_bytes;
    p.stages = pl.stages;
    p.fsub_per_job = pl.fsub;
    p.leaf_u32 = m->leaf_u32 ? 1 : 0;
    p.scale = m->scale;
    p.bias = m->bias;
    p.off_meta = pl.off_meta;
    p.off_bord = pl.off_bord;
    p.bord_stride = m->bord_stride;
    p.n_seg = m->n_seg;
    for (int sg = 0; sg < m->n_seg; ++sg) p.seg[sg] = m->seg[sg];
    p.half_stride = pl.half_stride;
    p.hdesc_bytes = pl.hdesc_bytes;
    return p;
}

odf_status check_factors_fm(const odf_model *m, const float *d_x, int64_t n_docs, int64_t ld)
{
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    if (n_docs >= (int64_t(1) << 31) - kTile)
        return fail(ODF_E_INVALID_ARG, "n_docs >= 2^31 - 128 (TMA coordinate range)");
    if (ld < n_docs) return fail(ODF_E_INVALID_ARG, "ld_fm (%lld) < n_docs (%lld)", (long long)ld, (long long)n_docs);
    if (ld % 4 != 0) return fail(ODF_E_INVALID_ARG, "ld_fm %% 4 != 0 (rows must be 16-byte aligned for TMA)");
    if (n_docs > 0 && !d_x) return fail(ODF_E_INVALID_ARG, "d_factors is NULL");
    if (reinterpret_cast<uintptr_t>(d_x) % 16 != 0) return fail(ODF_E_INVALID_ARG, "d_factors not 16-byte aligned");
    return ODF_OK;
}

odf_status check_factors(const odf_model *m, const float *d_x, int64_t n_docs, int64_t ld)
{
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    if (n_docs >= (int64_t(1) << 31) - kTile)
        return fail(ODF_E_INVALID_ARG, "n_docs >= 2^31 - 128 (TMA coordinate range)");
    if (ld < m->n_features) return fail(ODF_E_INVALID_ARG, "ld (%lld) < n_features (%d)", (long long)ld, m->n_features);
    if (ld % 4 != 0) return fail(ODF_E_INVALID_ARG, "ld %% 4 != 0 (rows must be 16-byte aligned for TMA)");
    if (n_docs > 0 && !d_x) return fail(ODF_E_INVALID_ARG, "d_factors is NULL");
    if (reinterpret_cast<uintptr_t>(d_x) % 16 != 0) return fail(ODF_E_INVALID_ARG, "d_factors not 16-byte aligned");
    return ODF_OK;
}

int grid_for(const odf_model *m, const Plan &pl, int64_t n_tiles)
{
    const int64_t g = static_cast<int64_t>(m->num_sms) * pl.grid_per_sm;
    return static_cast<int>(std::min<int64_t>(n_tiles, g));
}

// Tile width of a fused / apply launch (odf.h "Documents per tile"): 0 = automatic.
// Returns the halves (1 or 2) or 0 after setting the error.
int choose_halves(const odf_model *m, int mode, int64_t n_docs, int32_t tile_docs, odf_status *st)
{
    const Plan &p2 = mode == MODE_FUSED ? m->fused2 : m->apply2;
    *st = ODF_OK;
    if (m->tile_docs != kTile) {  // a 64-document-tile model has that width only
        if (tile_docs == 0 || tile_docs == m->tile_docs) return 1;
        *st = fail(tile_docs == kTile || tile_docs == 2 * kTile ? ODF_E_UNSUPPORTED : ODF_E_INVALID_ARG,
                   "tile_docs = %d: this model runs %d-document tiles only", tile_docs, m->tile_docs);
        return 0;
    }
    if (tile_docs == 0) {
        // 256-document tiles halve the forest's L2 -> shared-memory bytes per document
        // but, next to two code blocks, leave fewer ring slots: the tree stream is then
        // bound by the bytes it has in flight.  Measured on c4 (depth 10, 2 slots):
        // apply 25.9 -> 22.7 ms, fused (its slots also carry 2-box factor jobs)
        // 28.4 -> 32.4 ms; so fused takes them only with >= 3 slots.
        const int64_t tiles256 = (n_docs + 2 * kTile - 1) / (2 * kTile);
        const bool deep = m->depth >= 7 && tiles256 >= 2 * static_cast<int64_t>(m->num_sms);
        return (p2.valid && deep && (mode == MODE_APPLY || p2.stages >= 3)) ? 2 : 1;
    }
    if (tile_docs == kTile) return 1;
    if (tile_docs == 2 * kTile) {
        if (p2.valid) return 2;
        *st = fail(ODF_E_UNSUPPORTED, "256-document tiles do not fit this model (max_tile_docs = 128)");
        return 0;
    }
    *st = fail(ODF_E_INVALID_ARG, "tile_docs = %d not in {0, 128, 256}", tile_docs);
    return 0;
}

}  // namespace

// ============================================================================
// ABI
// ============================================================================
// No exception crosses the ABI (include/odf.h): host allocations of the model
// compiler and the staging of odf_score_host are the only sources.
template <class F>
static odf_status guarded(F f)
{
    try {
        return f();
    } catch (const std::bad_alloc &) {
        return fail(ODF_E_NOMEM, "host allocation failed");
    } catch (const std::exception &e) {
        return fail(ODF_E_INVALID_ARG, "unexpected host exception: %s", e.what());
    } catch (...) {
        return fail(ODF_E_INVALID_ARG, "unexpected host exception");
    }
}

extern "C" {

int odf_version(void) { return 100; }
const char *odf_last_error(void) { return g_err.c_str(); }

void odf_free_model(odf_model *m)
{
    if (!m) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    cudaFree(m->d_fmeta);
    cudaFree(m->d_borders);
    cudaFree(m->d_chunks);
    cudaFree(m->d_splits);
    cudaFree(m->d_ucols);
    cudaFree(m->d_bchunk);
    cudaFree(m->d_bf_base);
    cudaFree(m->d_bits_desc);
    cudaFree(m->d_leaves);
    for (int i = 0; i < 2; ++i) {
        cudaFree(m->d_stage[i]);
        cudaFree(m->d_sstage[i]);
        if (m->hs[i]) cudaStreamDestroy(m->hs[i]);
        if (m->ev_out[i]) cudaEventDestroy(m->ev_out[i]);
    }
    if (m->ev_in) cudaEventDestroy(m->ev_in);
    cudaSetDevice(prev);
    delete m;
}

odf_status odf_load_model(const int32_t *feature_index, const float *thresholds,
                          const float *leaf_values, int32_t depth, int64_t n_trees,
                          int32_t n_features, int device, odf_model **out)
{
    odf_model_desc d;
    memset(&d, 0, sizeof d);
    d.feature_index = feature_index;
    d.thresholds = thresholds;
    d.leaf_values = leaf_values;
    d.leaf_type = ODF_LEAF_F32;
    d.depth = depth;
    d.n_trees = n_trees;
    d.n_features = n_features;
    d.device = device;
    d.scale = 1.0;
    d.bias = 0.0;
    return odf_load_model_ex(&d, out);
}

// One height segment of a model: n_trees trees of one depth (feature_index /
// thresholds [n_trees * depth], answers [n_trees << depth]).
struct SegSpec {
    int32_t depth;
    int64_t n_trees;
    const int32_t *fi;
    const float *thr;
    const void *leaves;
};
static odf_status load_model_core(const odf_model_desc *desc, const std::vector<SegSpec> *segs_in,
                                  odf_model **out);
static odf_status load_model_ex_impl(const odf_model_desc *desc, odf_model **out)
{
    return load_model_core(desc, nullptr, out);
}

static odf_status load_model_paper_impl(const odf_paper_model_desc *d, odf_model **out)
{
    if (!out) return fail(ODF_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!d) return fail(ODF_E_INVALID_ARG, "desc is NULL");
    if (d->n_features < 1) return fail(ODF_E_INVALID_ARG, "n_features < 1");
    if (d->n_groups < 0 || (d->n_groups > 0 && (!d->group_factor || !d->group_count)))
        return fail(ODF_E_INVALID_ARG, "bad descriptor groups");
    // binary feature k -> factor (groups of consecutive binary features)
    std::vector<int32_t> bf_factor;
    for (int32_t g = 0; g < d->n_groups; ++g) {
        if (d->group_factor[g] < 0 || d->group_factor[g] >= d->n_features)
            return fail(ODF_E_INVALID_ARG, "group_factor[%d] = %d not in [0, %d)", g,
                        d->group_factor[g], d->n_features);
        if (d->group_count[g] < 1) return fail(ODF_E_INVALID_ARG, "group_count[%d] < 1", g);
        bf_factor.insert(bf_factor.end(), d->group_count[g], d->group_factor[g]);
    }
    const int64_t K = static_cast<int64_t>(bf_factor.size());
    if (K > 0 && !d->thresholds) return fail(ODF_E_INVALID_ARG, "thresholds is NULL");
    if (!d->stc) return fail(ODF_E_INVALID_ARG, "stc is NULL");
    int32_t D = 0;
    int64_t T = 0, n_cond = 0, n_leaf = 0;
    for (int h = 0; h <= ODF_MAX_DEPTH; ++h) {
        if (d->stc[h] < 0) return fail(ODF_E_INVALID_ARG, "stc[%d] < 0", h);
        if (d->stc[h] > 0) D = h;
        T += d->stc[h];
        n_cond += static_cast<int64_t>(h) * d->stc[h];
        n_leaf += (int64_t(1) << h) * d->stc[h];
    }
    if (T > (int64_t(1) << 30)) return fail(ODF_E_INVALID_ARG, "n_trees > 2^30");
    if ((d->pad_heights ? (T << D) : n_leaf) > (int64_t(1) << 32))  // before any host allocation
        return fail(ODF_E_UNSUPPORTED, "%lld answers > 2^32",
                    (long long)(d->pad_heights ? (T << D) : n_leaf));
    if (n_cond > 0 && !d->cond_indices) return fail(ODF_E_INVALID_ARG, "cond_indices is NULL");
    if (n_leaf > 0 && !d->leaves) return fail(ODF_E_INVALID_ARG, "leaves is NULL");
    for (int64_t k = 0; k < n_cond; ++k)
        if (d->cond_indices[k] >= static_cast<uint64_t>(K))
            return fail(ODF_E_INVALID_ARG, "cond_indices[%lld] = %u >= K = %lld", (long long)k,
                        d->cond_indices[k], (long long)K);
    odf_model_desc md;
    memset(&md, 0, sizeof md);
    md.leaf_type = ODF_LEAF_U32;
    md.n_features = d->n_features;
    md.device = d->device;
    md.scale = d->scale;
    md.bias = d->bias;
    if (!d->pad_heights) {
        // one segment per height present, in the paper's order (descending height,
        // P:307): tree t of height h keeps its h conditions and its 2^h answers
        std::vector<std::vector<int32_t>> fis;
        std::vector<std::vector<float>> thrs;
        std::vector<std::vector<uint32_t>> lvs;
        std::vector<SegSpec> segs;
        int64_t cb = 0, lb = 0;
        for (int h = ODF_MAX_DEPTH; h >= 0; --h) {
            if (d->stc[h] == 0) continue;
            const int64_t nt = d->stc[h];
            fis.emplace_back(static_cast<size_t>(nt) * h);
            thrs.emplace_back(static_cast<size_t>(nt) * h);
            lvs.emplace_back(static_cast<size_t>(nt) << h);
            for (int64_t k = 0; k < nt * h; ++k) {
                const uint32_t ci = d->cond_indices[cb + k];
                fis.back()[k] = bf_factor[ci];
                thrs.back()[k] = d->thresholds[ci];
            }
            std::memcpy(lvs.back().data(), d->leaves + lb, sizeof(uint32_t) * (static_cast<size_t>(nt) << h));
            cb += nt * h;
            lb += nt << h;
        }
        int64_t k = 0;
        for (int h = ODF_MAX_DEPTH; h >= 0; --h)
            if (d->stc[h] > 0) {
                segs.push_back(SegSpec{h, d->stc[h], fis[k].data(), thrs[k].data(), lvs[k].data()});
                ++k;
            }
        if (segs.empty()) segs.push_back(SegSpec{0, 0, nullptr, nullptr, nullptr});
        return load_model_core(&md, &segs, out);
    }
    // padded form (pad_heights = 1): a uniform model of depth D = the largest height
    std::vector<int32_t> fi(static_cast<size_t>(T) * D);
    std::vector<float> thr(static_cast<size_t>(T) * D);
    std::vector<uint32_t> lv(static_cast<size_t>(T) << D);
    // a condition for height-0 trees (never affects the answer): any existing one
    int32_t f0 = 0;
    float th0 = 0.0f;
    if (n_cond > 0) {
        const uint32_t k0 = d->cond_indices[0];
        f0 = bf_factor[k0];
        th0 = d->thresholds[k0];
    }
    int64_t t = 0, cb = 0, lb = 0;
    for (int h = ODF_MAX_DEPTH; h >= 0; --h)  // "trees in descending height"
        for (int32_t i = 0; i < d->stc[h]; ++i, ++t) {
            for (int l = 0; l < D; ++l) {
                int32_t f = f0;
                float th = th0;
                if (h > 0) {
                    const uint32_t k = d->cond_indices[cb + (l < h ? l : 0)];
                    f = bf_factor[k];
                    th = d->thresholds[k];
                }
                fi[t * D + l] = f;
                thr[t * D + l] = th;
            }
            for (int64_t j = 0; j < (int64_t(1) << D); ++j)
                lv[(t << D) + j] = d->leaves[lb + (j & ((int64_t(1) << h) - 1))];
            cb += h;
            lb += int64_t(1) << h;
        }
    md.feature_index = fi.data();
    md.thresholds = thr.data();
    md.leaf_values = lv.data();
    md.depth = D;
    md.n_trees = T;
    return load_model_ex_impl(&md, out);
}

// The model compiler (K0).  segs_in == nullptr: one uniform-depth segment from desc;
// else the height segments of a mixed-height model (NEXT-2), in stream order.
static odf_status load_model_core(const odf_model_desc *desc, const std::vector<SegSpec> *segs_in,
                                  odf_model **out)
{
    if (!out) return fail(ODF_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!desc) return fail(ODF_E_INVALID_ARG, "desc is NULL");
    std::vector<SegSpec> segs;
    if (segs_in)
        segs = *segs_in;
    else
        segs.push_back(SegSpec{desc->depth, desc->n_trees, desc->feature_index, desc->thresholds,
                               desc->leaf_values});
    const int32_t n_features = desc->n_features;
    const int device = desc->device;
    const bool u32 = desc->leaf_type == ODF_LEAF_U32;
    if (desc->leaf_type != ODF_LEAF_F32 && !u32)
        return fail(ODF_E_INVALID_ARG, "leaf_type %d unknown", desc->leaf_type);
    if (u32 && (!std::isfinite(desc->scale) || !std::isfinite(desc->bias)))
        return fail(ODF_E_INVALID_ARG, "scale / bias not finite");
    if (n_features < 1) return fail(ODF_E_INVALID_ARG, "n_features < 1");
    if (segs.size() > static_cast<size_t>(kMaxSegments) || (segs.size() > 1 && !u32))
        return fail(ODF_E_INVALID_ARG, "mixed-height models: <= %d segments, integer answers", kMaxSegments);
    int32_t depth = 0;
    int64_t n_trees = 0, n_leaves = 0;
    for (const SegSpec &g : segs) {
        if (g.depth < 0 || g.depth > ODF_MAX_DEPTH)
            return fail(ODF_E_INVALID_ARG, "depth %d not in [0, %d]", g.depth, ODF_MAX_DEPTH);
        if (g.n_trees < 0) return fail(ODF_E_INVALID_ARG, "n_trees < 0");
        if (g.n_trees > (int64_t(1) << 30)) return fail(ODF_E_INVALID_ARG, "n_trees > 2^30");
        const int64_t nodes = g.n_trees * g.depth, leaves = g.n_trees << g.depth;
        if (nodes > 0 && (!g.fi || !g.thr)) return fail(ODF_E_INVALID_ARG, "feature_index / thresholds is NULL");
        if (leaves > 0 && !g.leaves) return fail(ODF_E_INVALID_ARG, "leaf_values is NULL");
        for (int64_t k = 0; k < nodes; ++k) {
            if (g.fi[k] < 0 || g.fi[k] >= n_features)
                return fail(ODF_E_INVALID_ARG, "feature_index[%lld] = %d not in [0, n_features=%d)",
                            (long long)k, g.fi[k], n_features);
            if (!std::isfinite(g.thr[k]))
                return fail(ODF_E_INVALID_ARG, "thresholds[%lld] is not finite", (long long)k);
        }
        if (!u32)
            for (int64_t k = 0; k < leaves; ++k)
                if (!std::isfinite(static_cast<const float *>(g.leaves)[k]))
                    return fail(ODF_E_INVALID_ARG, "leaf_values[%lld] is not finite", (long long)k);
        depth = std::max(depth, g.depth);
        n_trees += g.n_trees;
        n_leaves += leaves;
    }
    if (n_trees > (int64_t(1) << 30)) return fail(ODF_E_INVALID_ARG, "n_trees > 2^30");
    if (n_leaves > (int64_t(1) << 32))
        return fail(ODF_E_UNSUPPORTED, "%lld answers > 2^32", (long long)n_leaves);
    if (device < 0) return fail(ODF_E_INVALID_ARG, "device %d < 0", device);
    // uniform-depth models keep the single-depth geometry below (seg 0)
    const int32_t *feature_index = segs[0].fi;
    const float *thresholds = segs[0].thr;
    const float *leaf_f = static_cast<const float *>(segs[0].leaves);
    const void *leaf_values = segs[0].leaves;
    const int64_t n_nodes = segs[0].n_trees * segs[0].depth;

    std::unique_ptr<odf_model> m(new odf_model());
    m->device = device;
    m->depth = depth;
    m->kdepth = segs.size() > 1 ? kMixedDepth : depth;
    m->n_trees = n_trees;
    m->n_features = n_features;
    m->leaf_u32 = u32;
    m->scale = desc->scale;
    m->bias = desc->bias;

    // ---- borders per factor (sorted, unique by ==) ----
    std::vector<std::vector<float>> borders(n_features);
    for (const SegSpec &g : segs)
        for (int64_t k = 0; k < g.n_trees * g.depth; ++k) borders[g.fi[k]].push_back(g.thr[k]);
    std::vector<int32_t> used_of(n_features, -1), colB_of(n_features, -1);
    for (int32_t f = 0; f < n_features; ++f) {
        auto &b = borders[f];
        if (b.empty()) continue;
        std::sort(b.begin(), b.end(), [](float a, float c) { return a < c; });
        std::vector<float> u;
        for (float v : b)
            if (u.empty() || !(v == u.back())) u.push_back(v);
        b.swap(u);
        if (b.size() > ODF_MAX_BORDERS_WIDE)
            return fail(ODF_E_UNSUPPORTED, "factor %d has %zu distinct thresholds > %d",
                        f, b.size(), ODF_MAX_BORDERS_WIDE);
        used_of[f] = static_cast<int32_t>(m->used_ids.size());
        m->used_ids.push_back(f);
        m->max_borders = std::max<int32_t>(m->max_borders, static_cast<int32_t>(b.size()));
        m->total_borders += static_cast<int64_t>(b.size());
    }
    m->n_used = static_cast<int32_t>(m->used_ids.size());
    // code columns: factor f with m borders has C = ceil(m / 127) 7-bit columns, the
    // first at used_of[f], the others contiguous from colB_of[f] (after all primaries)
    m->wide = m->max_borders > ODF_MAX_BORDERS;
    auto n_codecols = [](size_t mm) { return static_cast<uint32_t>(std::max<size_t>(1, (mm + 126) / 127)); };
    std::vector<uint2> splits;
    int32_t n_extra = 0;
    for (int32_t f : m->used_ids) {
        const uint32_t C = n_codecols(borders[f].size());
        if (C > 1) colB_of[f] = m->n_used + n_extra;
        if (C == 2 && !m->wide)
            splits.push_back(make_uint2(static_cast<uint32_t>(used_of[f]) * kTile,
                                        static_cast<uint32_t>(colB_of[f]) * kTile));
        n_extra += static_cast<int32_t>(C) - 1;
    }
    m->n_split = static_cast<int32_t>(splits.size());
    m->n_cols = m->n_used + n_extra;
    if (m->n_cols > kMaxDescCol)  // 13-bit column field of the level descriptor
        return fail(ODF_E_UNSUPPORTED, "%d code columns > %d", m->n_cols, kMaxDescCol);
    std::vector<uint2> ucols;
    if (m->wide)
        for (int32_t f : m->used_ids)
            ucols.push_back(make_uint2(colB_of[f] >= 0 ? static_cast<uint32_t>(colB_of[f]) * kTile
                                                       : static_cast<uint32_t>(m->n_cols) * kTile,
                                       n_codecols(borders[f].size())));

    // ---- factor metadata + border arrays (binarize; layout in odf_internal.h) ----
    // Pairs (f, f+1), f even, share one code path: LIN4 if both have <= 4 borders,
    // else BIN(L) with the pair's L.  Each array is npad copies of -inf followed by
    // the factor's sorted borders (bin = count - npad).
    m->n_fchunks = (n_features + kFSub - 1) / kFSub;
    const uint32_t trash = static_cast<uint32_t>(m->n_cols) * kTile;  // column of discarded stores
    std::vector<uint4> fmeta(static_cast<size_t>(m->n_fchunks) * kFSub, make_uint4(0, 0, trash, trash));
    std::vector<float> bflat;
    auto ceil_log2p1 = [](uint32_t mm) {
        uint32_t L = 0;
        while (((1u << L) - 1u) < mm) ++L;  // smallest L with 2^L - 1 >= m
        return L;
    };
    auto n_borders = [&](size_t f) -> uint32_t {
        return f < static_cast<size_t>(n_features) ? static_cast<uint32_t>(borders[f].size()) : 0u;
    };
    for (size_t f = 0; f < fmeta.size(); f += 2) {
        const uint32_t ma = n_borders(f), mb = n_borders(f + 1);
        if (ma == 0 && mb == 0) continue;
        const bool lin = std::max(ma, mb) <= 4;
        // a factor with > 254 borders (more than two code columns) forces L >= 9, the
        // kernel's wide search path, which stores any number of code columns
        const uint32_t L = lin ? 0u : std::max(ceil_log2p1(std::max(ma, mb)),
                                                std::max(ma, mb) > ODF_MAX_BORDERS ? 9u : 0u);
        const uint32_t cls = lin ? 1u : L + 1u;
        const uint32_t n_ent = lin ? 4u : (1u << L) - 1u;
        for (size_t g = f; g < f + 2; ++g) {
            const uint32_t mm = n_borders(g);
            if (mm == 0) continue;
            const auto &b = borders[g];
            const uint32_t off = static_cast<uint32_t>(bflat.size());
            const uint32_t npad = n_ent - mm;
            bflat.resize(off + skew_h(n_ent - 1u) + 1u, -INFINITY);
            for (uint32_t pidx = 0; pidx < n_ent; ++pidx)
                bflat[off + skew_h(pidx)] = pidx < npad ? -INFINITY : b[pidx - npad];
            while (bflat.size() % 4) bflat.push_back(-INFINITY);  // 16-byte aligned arrays
            const uint32_t extra = n_codecols(mm) - 1u;
            fmeta[g] = make_uint4(off, cls | (extra << kExtraShiftH) | ((0u - npad) << 16),
                                  static_cast<uint32_t>(used_of[g]) * kTile,
                                  extra ? static_cast<uint32_t>(colB_of[g]) * kTile : trash);
        }
        // the unused factor of a mixed pair searches its partner's array, stores to trash
        const uint32_t no_extra = ~(0xfu << kExtraShiftH);
        if (ma == 0) fmeta[f] = make_uint4(fmeta[f + 1].x, fmeta[f + 1].y & no_extra, trash, trash);
        if (mb == 0) fmeta[f + 1] = make_uint4(fmeta[f].x, fmeta[f].y & no_extra, trash, trash);
        // pair flag (bit 8 of the first factor's fmeta.y): a factor of the pair has code
        // columns beyond the first (kPairSplit in odf_kernels.cu)
        if (((fmeta[f].y | fmeta[f + 1].y) >> kExtraShiftH) & 0xfu) fmeta[f].y |= 1u << 8;
    }
    m->border_floats = static_cast<int32_t>(bflat.size());
    // per sub-tile border ranges; fmeta.x becomes relative to its sub-tile's range
    std::vector<uint2> bchunk(m->n_fchunks, make_uint2(0, 0));
    for (int32_t c = 0; c < m->n_fchunks; ++c) {
        uint32_t lo = UINT32_MAX, hi = 0;
        for (int32_t f = c * kFSub; f < (c + 1) * kFSub; ++f) {
            const uint32_t cls = fmeta[f].y & 0xfu;
            if (cls == 0) continue;
            const uint32_t len = cls == 1 ? 4u : skew_h((1u << (cls - 1)) - 2u) + 1u;
            lo = std::min(lo, fmeta[f].x);
            hi = std::max(hi, (fmeta[f].x + len + 3u) & ~3u);
        }
        if (hi == 0) continue;
        for (int32_t f = c * kFSub; f < (c + 1) * kFSub; ++f)
            if ((fmeta[f].y & 0xfu) != 0) fmeta[f].x = (fmeta[f].x - lo) * 4u;  // bytes
        bchunk[c] = make_uint2(lo * 4u, (hi - lo) * 4u);
        m->bord_stride = std::max(m->bord_stride, (hi - lo) * 4u);
    }

    // ---- tree chunks: descriptors + reversed leaf tables, per height segment ----
    // chunk size: about one factor sub-tile (16.5 KB + its borders), so one ring slot
    // carries a sub-tile in phase A or a chunk of similar bytes in phase B and the
    // ring is as deep as shared memory allows (up to 8 stages: more factor data in
    // flight while phase A runs); at least 16 trees (one per consumer warp)
    const uint32_t unit = kFSubBytes + kMetaBytes + ((m->bord_stride + 15u) & ~15u);
    std::vector<uint8_t> chunks;
    int64_t total_chunk_bytes = 0;
    for (size_t sg = 0; sg < segs.size(); ++sg) {
        const SegSpec &g = segs[sg];
        const int sdepth = g.depth;
        const int dstride = desc_stride(sdepth);
        const uint32_t tstride = static_cast<uint32_t>(table_stride(sdepth));
        const uint32_t per = static_cast<uint32_t>(dstride) + tstride;
#ifndef ODF_TC_MULT
#define ODF_TC_MULT 16  // A/B builds only: trees per chunk rounded to this multiple
#endif
        const uint32_t tcm = (sdepth <= 6) ? ODF_TC_MULT : 16u;
        int32_t tc = static_cast<int32_t>(tcm * std::max<uint32_t>(1u, unit / (tcm * per)));
        // at least 96 trees (6 per warp: the apply's fully unrolled shape) at depth <= 6 when
        // the forest is large enough that the padded last chunk costs little: c2 (20 KB
        // units, 64-tree chunks) fused 0.259 -> 0.244 ms
        if (sdepth <= 6 && tc < 96 && g.n_trees >= 16 * 96) tc = 96;
        const uint32_t dbytes = align_up(static_cast<uint64_t>(tc) * dstride, 256);
        const uint32_t cbytes = dbytes + static_cast<uint32_t>(tc) * tstride;
        const int32_t nch = static_cast<int32_t>((g.n_trees + tc - 1) / tc);
        total_chunk_bytes += static_cast<int64_t>(nch) * cbytes;
        if (total_chunk_bytes > (int64_t(1) << 36))
            return fail(ODF_E_NOMEM, "tree chunks of %lld bytes > 64 GiB", (long long)total_chunk_bytes);
        const size_t base = chunks.size();
        chunks.resize(base + static_cast<size_t>(nch) * cbytes, 0);
        // padding trees of the last chunk: -0.0 answers (x + -0.0 == x bit for bit) / 0
        if (!u32 && g.n_trees % tc != 0) {
            uint8_t *ch = chunks.data() + base + static_cast<size_t>(nch - 1) * cbytes;
            for (int64_t i = g.n_trees % tc; i < tc; ++i) {
                float *tab = reinterpret_cast<float *>(ch + dbytes + i * tstride);
                for (uint32_t F = 0; F < (1u << sdepth); ++F) tab[F] = -0.0f;
            }
        }
        const uint32_t nleaf = 1u << sdepth;
        const float *lf = static_cast<const float *>(g.leaves);
        const uint32_t *lu = static_cast<const uint32_t *>(g.leaves);
#ifdef ODF_TREE_SORT  // A/B timing builds only (P:434 locality reordering): trees sorted by their level features
        std::vector<int64_t> order(static_cast<size_t>(g.n_trees));
        for (int64_t t = 0; t < g.n_trees; ++t) order[t] = t;
        std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b2) {
            for (int l = 0; l < sdepth; ++l)
                if (g.fi[a * sdepth + l] != g.fi[b2 * sdepth + l]) return g.fi[a * sdepth + l] < g.fi[b2 * sdepth + l];
            return false;
        });
#endif
        for (int64_t pos = 0; pos < g.n_trees; ++pos) {
#ifdef ODF_TREE_SORT
            const int64_t t = order[pos];
#else
            const int64_t t = pos;
#endif
            uint8_t *ch = chunks.data() + base + static_cast<size_t>(pos / tc) * cbytes;
            const int64_t i = pos % tc;
            uint32_t *desc = reinterpret_cast<uint32_t *>(ch + i * dstride);
            for (int l = 0; l < sdepth; ++l) {
                const int32_t f = g.fi[t * sdepth + l];
                const float thr = g.thr[t * sdepth + l];
                const auto &b = borders[f];
                const auto it = std::lower_bound(b.begin(), b.end(), thr, [](float a, float c) { return a < c; });
                const uint32_t k = static_cast<uint32_t>(it - b.begin());  // b[k] == thr
                // bin <= k  <=>  code of column c = k / 127 <= k - 127c
                const uint32_t c = k / 127u;
                const uint32_t col = c == 0 ? static_cast<uint32_t>(used_of[f])
                                            : static_cast<uint32_t>(colB_of[f]) + c - 1u;
                const uint32_t K = k - 127u * c + 1u;
                if (desc_fmt(sdepth) == DESC_SPLIT) {
                    desc[l] = col * kTile;
                    desc[sdepth + l / 4] |= (128u - K) << (8 * (l % 4));
                } else if (desc_fmt(sdepth) == DESC8) {
                    desc[2 * l] = col * kTile;
                    desc[2 * l + 1] = (128u - K) * 0x01010101u;
                } else {
                    desc[l] = (col << 19) | (128u - K);
                }
            }
            uint8_t *tab = ch + dbytes + i * tstride;
            for (uint32_t F = 0; F < nleaf; ++F) {
                const size_t src = static_cast<size_t>(t) * nleaf + (nleaf - 1 - F);
                if (u32)
                    reinterpret_cast<uint32_t *>(tab)[leaf_pos(sdepth, F)] = lu[src];
                else
                    reinterpret_cast<float *>(tab)[leaf_pos(sdepth, F)] = lf[src];
            }
        }
        if (sg == 0) {  // the uniform geometry (a mixed model's slot is sized below)
            m->tc = tc;
            m->desc_bytes = dbytes;
            m->chunk_bytes = cbytes;
            m->table_stride = tstride;
        }
        if (segs.size() > 1)
            m->seg[sg] = SegP{sdepth, tc, nch, cbytes, dbytes, 0u, static_cast<uint64_t>(base)};
        m->n_tchunks += nch;
    }
    if (segs.size() > 1) {
        m->n_seg = static_cast<int32_t>(segs.size());
        for (int sg = 0; sg < m->n_seg; ++sg) m->chunk_bytes = std::max(m->chunk_bytes, m->seg[sg].chunk_bytes);
    }

    // ---- NEXT-3: binary features (used factor u, border j) and per-level word offsets ----
    std::vector<uint32_t> bf_base(m->n_used + 1, 0);
    for (int32_t u = 0; u < m->n_used; ++u)
        bf_base[u + 1] = bf_base[u] + static_cast<uint32_t>(borders[m->used_ids[u]].size());
    std::vector<uint32_t> bits_desc;
    if (!u32 && segs.size() == 1) {
        bits_desc.resize(static_cast<size_t>(n_nodes));
        for (int64_t k = 0; k < n_nodes; ++k) {
            const int32_t f = feature_index[k];
            const auto &b = borders[f];
            const uint32_t j = static_cast<uint32_t>(
                std::lower_bound(b.begin(), b.end(), thresholds[k], [](float a, float c) { return a < c; }) -
                b.begin());
            bits_desc[k] = (bf_base[used_of[f]] + j) * 4u;
        }
    }

    // ---- device (the host-side compile above needs none: it runs, and is
    //      sanitizer-checked, on CPU-only hosts too, tests/test_sanitizers.py) ----
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
        return fail(ODF_E_CUDA, "no CUDA device available (this library has no CPU fallback)");
    if (device >= n_dev) return fail(ODF_E_INVALID_ARG, "device %d not in [0, %d)", device, n_dev);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&m->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    auto up = [&](void **dst, const void *src, size_t bytes) -> cudaError_t {
        if (bytes == 0) return cudaSuccess;
        cudaError_t r = cudaMalloc(dst, bytes);
        if (r != cudaSuccess) return r;
        m->dev_bytes += static_cast<int64_t>(bytes);
        return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    };
    if ((e = up(reinterpret_cast<void **>(&m->d_fmeta), fmeta.data(), fmeta.size() * sizeof(uint4))) != cudaSuccess ||
        (e = up(reinterpret_cast<void **>(&m->d_borders), bflat.data(), bflat.size() * 4)) != cudaSuccess ||
        (e = up(reinterpret_cast<void **>(&m->d_chunks), chunks.data(), chunks.size())) != cudaSuccess ||
        (e = up(reinterpret_cast<void **>(&m->d_splits), splits.data(), splits.size() * sizeof(uint2))) != cudaSuccess ||
        (e = up(reinterpret_cast<void **>(&m->d_ucols), ucols.data(), ucols.size() * sizeof(uint2))) != cudaSuccess ||
        (e = up(reinterpret_cast<void **>(&m->d_bchunk), bchunk.data(), bchunk.size() * sizeof(uint2))) != cudaSuccess ||
        (e = up(reinterpret_cast<void **>(&m->d_bf_base), bf_base.data(), bf_base.size() * 4)) != cudaSuccess ||
        (e = up(reinterpret_cast<void **>(&m->d_bits_desc), bits_desc.data(), bits_desc.size() * 4)) != cudaSuccess ||
        (e = up(reinterpret_cast<void **>(&m->d_leaves), leaf_values, u32 ? 0 : static_cast<size_t>(n_leaves) * 4)) != cudaSuccess) {
        odf_model *raw = m.release();
        odf_free_model(raw);
        return e == cudaErrorMemoryAllocation ? fail(ODF_E_NOMEM, "device allocation failed")
                                              : cuda_fail(e, "model upload");
    }
    if ((e = prepare_kernels(m->max_smem)) != cudaSuccess) {
        odf_free_model(m.release());
        return cuda_fail(e, "cudaFuncSetAttribute");
    }
    std::string why;
    auto plans = [&]() {
        return make_plan(*m, MODE_FUSED, m->fused, why) && make_plan(*m, MODE_APPLY, m->apply, why) &&
               make_plan(*m, MODE_BINARIZE, m->binz, why);
    };
    bool planned = plans();
    if (!planned && !m->wide) {  // a 128-document code block does not fit: 64-document tiles
        m->tile_docs = kTile / 2;
        why.clear();
        planned = plans();
    }
    if (!planned) {
        odf_free_model(m.release());
        return fail(ODF_E_UNSUPPORTED, "%s", why.c_str());
    }
    m->binz.grid_per_sm = occupancy_main(MODE_BINARIZE, 0, m->binz.smem, m->tile_docs);
    // 256-document tiles (two halves), fp32 narrow models, when two code blocks fit
    if (!m->leaf_u32 && !m->wide && m->tile_docs == kTile) {
        std::string why2;
        if (!make_plan(*m, MODE_FUSED, m->fused2, why2, 2)) m->fused2 = Plan();
        if (!make_plan(*m, MODE_APPLY, m->apply2, why2, 2)) m->apply2 = Plan();
        if (!m->fused2.valid || !m->apply2.valid) m->fused2 = m->apply2 = Plan();  // both or neither
        if (!make_plan(*m, MODE_FUSED, m->fused64, why2, 1, kTile / 2)) m->fused64 = Plan();
    }
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        odf_free_model(m.release());
        return cuda_fail(e, "odf_load_model");
    }
    *out = m.release();
    return ok();
}

odf_status odf_get_info(const odf_model *m, odf_model_info *info)
{
    if (!m || !info) return fail(ODF_E_INVALID_ARG, "NULL argument");
    info->depth = m->depth;
    info->n_features = m->n_features;
    info->n_used_features = m->n_used;
    info->n_split_features = m->n_split;
    info->n_columns = m->n_cols;
    info->n_trees = m->n_trees;
    info->trees_per_chunk = m->tc;
    info->n_tree_chunks = m->n_tchunks;
    info->chunk_bytes = m->chunk_bytes;
    info->model_device_bytes = m->dev_bytes;
    info->max_borders = m->max_borders;
    info->total_borders = m->total_borders;
    info->borders_in_smem = 0;
    info->stages_fused = m->fused.stages;
    info->smem_fused = static_cast<int32_t>(m->fused.smem);
    info->num_sms = m->num_sms;
    info->leaf_type = m->leaf_u32 ? ODF_LEAF_U32 : ODF_LEAF_F32;
    info->bord_stride = static_cast<int32_t>(m->bord_stride);
    info->bins_elem_bytes = m->wide ? 2 : 1;
    info->max_tile_docs = m->fused2.valid ? 2 * kTile : m->tile_docs;
    info->bins_tile_docs = m->tile_docs;
    info->stages_fused_256 = m->fused2.valid ? m->fused2.stages : 0;
    info->smem_fused_256 = m->fused2.valid ? static_cast<int32_t>(m->fused2.smem) : 0;
    info->tail_tile_docs = (ODF_TAIL64 && m->fused64.valid && m->depth <= 6 && m->n_seg == 0) ? kTile / 2 : 0;
    return ok();
}

odf_status odf_bins_layout(const odf_model *m, int64_t n_docs, size_t *bytes,
                           int32_t *n_used_features, const int32_t **used_feature_ids)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    const int64_t td = m->tile_docs;
    const int64_t tiles = (n_docs + td - 1) / td;
    if (bytes) *bytes = static_cast<size_t>(tiles) * m->n_used * td * (m->wide ? 2 : 1);
    if (n_used_features) *n_used_features = m->n_used;
    if (used_feature_ids) *used_feature_ids = m->used_ids.empty() ? nullptr : m->used_ids.data();
    return ok();
}

// pdl: 0 plain launch; 1 primary of a programmatic dependent launch; 2 its secondary, run
// with the 64-document-tile plan (m->fused64) on a partly filled last wave
static odf_status run_main(const odf_model *m, int mode, const float *d_x, int64_t n_docs, int64_t ld,
                           const uint8_t *bins_in, uint8_t *bins_out, float *scores, cudaStream_t s,
                           uint64_t *sums = nullptr, double *dscores = nullptr, bool fm = false,
                           int halves = 1, int pdl = 0)
{
    const Plan &pl = pdl == 2 ? m->fused64
                     : halves == 2 ? (mode == MODE_FUSED ? m->fused2 : m->apply2)
                                   : mode == MODE_FUSED ? m->fused : mode == MODE_APPLY ? m->apply : m->binz;
    KParams p = base_params(m, pl);
    const int td = pdl == 2 ? kTile / 2 : m->tile_docs;
    p.tile_docs = td;
    p.pdl = pdl;
    p.n_docs = n_docs;
    p.n_tiles = (n_docs + td * halves - 1) / (td * halves);
    p.bins_in = bins_in;
    p.bins_out = bins_out;
    p.scores = scores;
    p.sums = reinterpret_cast<unsigned long long *>(sums);
    p.dscores = dscores;
    CUtensorMap tm;
    const CUtensorMap *tmp = nullptr;
    p.fm = fm ? 1 : 0;
    if (mode != MODE_APPLY && p.n_fchunks > 0) {
        odf_status st = encode_tmap(m, d_x, n_docs, ld, &tm, fm, td);
        if (st != ODF_OK) return st;
        tmp = &tm;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != m->device) cudaSetDevice(m->device);
    cudaError_t e = launch_main(mode, mode == MODE_BINARIZE ? 0 : m->kdepth, p, tmp,
                                grid_for(m, pl, p.n_tiles), pl.smem, s, halves, pdl == 2);
    if (prev != m->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    return ok();
}

odf_status odf_binarize(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                        uint8_t *d_bins, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    odf_status st = check_factors(m, d_factors, n_docs, ld);
    if (st != ODF_OK) return st;
    if (n_docs == 0 || m->n_used == 0) return ok();
    if (!d_bins) return fail(ODF_E_INVALID_ARG, "d_bins is NULL");
    return run_main(m, MODE_BINARIZE, d_factors, n_docs, ld, nullptr, d_bins, nullptr,
                    static_cast<cudaStream_t>(stream));
}

odf_status odf_apply(const odf_model *m, const uint8_t *d_bins, int64_t n_docs, float *d_scores,
                     void *stream)
{
    return odf_apply_tiles(m, d_bins, n_docs, d_scores, 0, stream);
}

odf_status odf_apply_tiles(const odf_model *m, const uint8_t *d_bins, int64_t n_docs, float *d_scores,
                           int32_t tile_docs, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (m->leaf_u32) return fail(ODF_E_INVALID_ARG, "integer-leaf model: use odf_apply_u64");
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    odf_status st;
    const int halves = choose_halves(m, MODE_APPLY, n_docs, tile_docs, &st);
    if (!halves) return st;
    if (n_docs == 0) return ok();
    if (!d_scores) return fail(ODF_E_INVALID_ARG, "d_scores is NULL");
    if (m->n_used > 0 && !d_bins) return fail(ODF_E_INVALID_ARG, "d_bins is NULL");
    if (reinterpret_cast<uintptr_t>(d_bins) % 16 != 0)
        return fail(ODF_E_INVALID_ARG, "d_bins not 16-byte aligned");
    return run_main(m, MODE_APPLY, nullptr, n_docs, 0, d_bins, nullptr, d_scores,
                    static_cast<cudaStream_t>(stream), nullptr, nullptr, false, halves);
}

odf_status odf_score(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                     float *d_scores, void *stream)
{
    return odf_score_tiles(m, d_factors, n_docs, ld, d_scores, 0, stream);
}

odf_status odf_score_tiles(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                           float *d_scores, int32_t tile_docs, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (m->leaf_u32) return fail(ODF_E_INVALID_ARG, "integer-leaf model: use odf_score_u64");
    odf_status st = check_factors(m, d_factors, n_docs, ld);
    if (st != ODF_OK) return st;
    const int halves = choose_halves(m, MODE_FUSED, n_docs, tile_docs, &st);
    if (!halves) return st;
    if (n_docs == 0) return ok();
    if (!d_scores) return fail(ODF_E_INVALID_ARG, "d_scores is NULL");
    // A last wave of 128-document tiles at most half full runs as 64-document tiles on twice
    // as many SMs, launched programmatically so it starts as the full waves' CTAs retire
    // (same per-document summation order: bit-identical scores).
    const int64_t nt = (n_docs + kTile - 1) / kTile, S = m->num_sms;
    // (depth <= 6 only: at depth 10 a 64-document tile re-stages the same 16 MB of tables as a
    // 128-document tile, and c4's 44-tile tail took 0.163 ms against 0.125 ms for one wave)
    if (ODF_TAIL64 && tile_docs == 0 && halves == 1 && m->fused64.valid && m->depth <= 6 && m->n_seg == 0 &&
        nt > S && nt % S != 0 && 2 * (nt % S) <= S) {
        const int64_t n1 = nt / S * S * kTile;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        st = run_main(m, MODE_FUSED, d_factors, n1, ld, nullptr, nullptr, d_scores, s, nullptr, nullptr, false,
                      1, 1);
        if (st != ODF_OK) return st;
        return run_main(m, MODE_FUSED, d_factors + n1 * ld, n_docs - n1, ld, nullptr, nullptr, d_scores + n1, s,
                        nullptr, nullptr, false, 1, 2);
    }
    return run_main(m, MODE_FUSED, d_factors, n_docs, ld, nullptr, nullptr, d_scores,
                    static_cast<cudaStream_t>(stream), nullptr, nullptr, false, halves);
}

odf_status odf_binarize_fm(const odf_model *m, const float *d_factors_fm, int64_t n_docs,
                           int64_t ld_fm, uint8_t *d_bins, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    odf_status st = check_factors_fm(m, d_factors_fm, n_docs, ld_fm);
    if (st != ODF_OK) return st;
    if (n_docs == 0 || m->n_used == 0) return ok();
    if (!d_bins) return fail(ODF_E_INVALID_ARG, "d_bins is NULL");
    return run_main(m, MODE_BINARIZE, d_factors_fm, n_docs, ld_fm, nullptr, d_bins, nullptr,
                    static_cast<cudaStream_t>(stream), nullptr, nullptr, true);
}

odf_status odf_score_fm(const odf_model *m, const float *d_factors_fm, int64_t n_docs, int64_t ld_fm,
                        float *d_scores, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (m->leaf_u32) return fail(ODF_E_INVALID_ARG, "integer-leaf model: use odf_score_u64");
    odf_status st = check_factors_fm(m, d_factors_fm, n_docs, ld_fm);
    if (st != ODF_OK) return st;
    if (n_docs == 0) return ok();
    if (!d_scores) return fail(ODF_E_INVALID_ARG, "d_scores is NULL");
    return run_main(m, MODE_FUSED, d_factors_fm, n_docs, ld_fm, nullptr, nullptr, d_scores,
                    static_cast<cudaStream_t>(stream), nullptr, nullptr, true);
}

odf_status odf_bits_layout(const odf_model *m, int64_t n_docs, size_t *bytes, int64_t *n_binary)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    if (bytes) *bytes = static_cast<size_t>((n_docs + 31) / 32) * m->total_borders * 4;
    if (n_binary) *n_binary = m->total_borders;
    return ok();
}

odf_status odf_bits_from_bins(const odf_model *m, const uint8_t *d_bins, int64_t n_docs,
                              uint32_t *d_words, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    if (n_docs == 0 || m->total_borders == 0) return ok();
    if (!d_bins || !d_words) return fail(ODF_E_INVALID_ARG, "NULL buffer");
    KParams p = base_params(m, m->apply);
    p.n_docs = n_docs;
    p.n_tiles = (n_docs + m->tile_docs - 1) / m->tile_docs;
    p.bins_in = d_bins;
    p.bf_base = m->d_bf_base;
    p.k_bin = m->total_borders;
    p.words = d_words;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != m->device) cudaSetDevice(m->device);
    cudaError_t e = launch_bits(m->depth, p, false, 0, static_cast<cudaStream_t>(stream));
    if (prev != m->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "bits kernel");
    return ok();
}

odf_status odf_apply_bits(const odf_model *m, const uint32_t *d_words, int64_t n_docs,
                          float *d_scores, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (m->leaf_u32) return fail(ODF_E_UNSUPPORTED, "bit-word apply: fp32-leaf models only");
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    if (n_docs == 0) return ok();
    if (!d_scores || (m->total_borders > 0 && !d_words)) return fail(ODF_E_INVALID_ARG, "NULL buffer");
    const size_t smem = align_up(static_cast<uint64_t>(m->total_borders) * 4, 16) + kConsumerWarps * 32 * 4;
    if (smem > static_cast<size_t>(m->max_smem))
        return fail(ODF_E_UNSUPPORTED, "bit-word apply: %lld binary features do not fit shared memory",
                    (long long)m->total_borders);
    KParams p = base_params(m, m->apply);
    p.n_docs = n_docs;
    p.scores = d_scores;
    p.k_bin = m->total_borders;
    p.words = const_cast<uint32_t *>(d_words);
    p.bits_desc = m->d_bits_desc;
    p.leaves = m->d_leaves;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != m->device) cudaSetDevice(m->device);
    cudaError_t e = launch_bits(m->depth, p, true, smem, static_cast<cudaStream_t>(stream));
    if (prev != m->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "bits apply kernel");
    return ok();
}

odf_status odf_score_u64(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                         uint64_t *d_sums, double *d_scores, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (!m->leaf_u32) return fail(ODF_E_INVALID_ARG, "fp32-leaf model: use odf_score");
    odf_status st = check_factors(m, d_factors, n_docs, ld);
    if (st != ODF_OK) return st;
    if (n_docs == 0) return ok();
    if (!d_sums && !d_scores) return fail(ODF_E_INVALID_ARG, "d_sums and d_scores are both NULL");
    return run_main(m, MODE_FUSED, d_factors, n_docs, ld, nullptr, nullptr, nullptr,
                    static_cast<cudaStream_t>(stream), d_sums, d_scores);
}

odf_status odf_apply_u64(const odf_model *m, const uint8_t *d_bins, int64_t n_docs, uint64_t *d_sums,
                         double *d_scores, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (!m->leaf_u32) return fail(ODF_E_INVALID_ARG, "fp32-leaf model: use odf_apply");
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    if (n_docs == 0) return ok();
    if (!d_sums && !d_scores) return fail(ODF_E_INVALID_ARG, "d_sums and d_scores are both NULL");
    if (m->n_used > 0 && !d_bins) return fail(ODF_E_INVALID_ARG, "d_bins is NULL");
    if (reinterpret_cast<uintptr_t>(d_bins) % 16 != 0)
        return fail(ODF_E_INVALID_ARG, "d_bins not 16-byte aligned");
    return run_main(m, MODE_APPLY, nullptr, n_docs, 0, d_bins, nullptr, nullptr,
                    static_cast<cudaStream_t>(stream), d_sums, d_scores);
}

static odf_status run_index(const odf_model *m, const uint8_t *d_bins, int64_t n_docs, bool fp,
                            int64_t doc0, int64_t ndoc, int64_t tree0, int64_t ntree,
                            uint16_t *d_idx, uint64_t *d_fp, cudaStream_t s)
{
    if (m->n_seg > 0)
        return fail(ODF_E_UNSUPPORTED, "leaf-index export: uniform-depth models only (this one has %d "
                                       "height segments)", m->n_seg);
    KParams p = base_params(m, m->apply);
    p.n_docs = n_docs;
    const int64_t td = m->tile_docs;
    p.n_tiles = (n_docs + td - 1) / td;
    p.bins_in = d_bins;
    p.doc0 = doc0;
    p.ndoc = ndoc;
    p.tree0 = tree0;
    p.ntree = ntree;
    p.idx_out = d_idx;
    p.fp_out = d_fp;
    const int grid = fp ? static_cast<int>(p.n_tiles)
                        : static_cast<int>((doc0 + ndoc - 1) / td - doc0 / td + 1);
    const int dstride = desc_stride(m->depth);
    size_t smem = align_up(static_cast<uint64_t>(m->n_cols) * td, 1024) +
                  align_up(static_cast<uint64_t>(m->tc) * dstride, 1024);
    if (m->wide) {  // u16 bins staged after the descriptors
        p.off_stage = static_cast<uint32_t>(smem);
        smem += align_up(static_cast<uint64_t>(m->n_used) * kTile * 2, 1024);
    }
    smem += 1024;
    if (smem > static_cast<size_t>(m->max_smem))
        return fail(ODF_E_UNSUPPORTED, "index kernel: %zu B of shared memory > %d", smem, m->max_smem);
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != m->device) cudaSetDevice(m->device);
    cudaError_t e = launch_index(m->depth, p, fp, grid, smem, s);
    if (prev != m->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "index kernel launch");
    return ok();
}

odf_status odf_leaf_indices(const odf_model *m, const uint8_t *d_bins, int64_t n_docs, int64_t doc0,
                            int64_t ndoc, int64_t tree0, int64_t ntree, uint16_t *d_idx,
                            void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (doc0 < 0 || ndoc < 0 || doc0 + ndoc > n_docs)
        return fail(ODF_E_INVALID_ARG, "document window [%lld, %lld) outside [0, %lld)",
                    (long long)doc0, (long long)(doc0 + ndoc), (long long)n_docs);
    if (tree0 < 0 || ntree < 0 || tree0 + ntree > m->n_trees)
        return fail(ODF_E_INVALID_ARG, "tree window [%lld, %lld) outside [0, %lld)",
                    (long long)tree0, (long long)(tree0 + ntree), (long long)m->n_trees);
    if (ndoc == 0 || ntree == 0) return ok();
    if (!d_idx || (m->n_used > 0 && !d_bins)) return fail(ODF_E_INVALID_ARG, "NULL buffer");
    return run_index(m, d_bins, n_docs, false, doc0, ndoc, tree0, ntree, d_idx, nullptr,
                     static_cast<cudaStream_t>(stream));
}

odf_status odf_index_fingerprint(const odf_model *m, const uint8_t *d_bins, int64_t n_docs,
                                 uint64_t *d_fp, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (n_docs < 0) return fail(ODF_E_INVALID_ARG, "n_docs < 0");
    if (n_docs == 0) return ok();
    if (!d_fp || (m->n_used > 0 && !d_bins)) return fail(ODF_E_INVALID_ARG, "NULL buffer");
    return run_index(m, d_bins, n_docs, true, 0, n_docs, 0, m->n_trees, nullptr, d_fp,
                     static_cast<cudaStream_t>(stream));
}

static int lat_splits(const odf_model *m, int64_t n_docs, int32_t splits)
{
    const int64_t td = m->tile_docs;
    const int64_t tiles = std::max<int64_t>(1, (n_docs + td - 1) / td);
    int64_t sp = splits > 0 ? splits : (2 * static_cast<int64_t>(m->num_sms)) / tiles;
    sp = std::max<int64_t>(1, std::min<int64_t>(sp, std::max(1, m->n_tchunks)));
    return static_cast<int>(std::min<int64_t>(sp, 1024));
}

static void lat_layout(const odf_model *m, int64_t n_docs, int sp, size_t off[4])
{
    const int64_t td = m->tile_docs;  // documents per tile: 128, or 64 (wide-column models)
    const int64_t tiles = (n_docs + td - 1) / td;
    auto a256 = [](size_t v) { return (v + 255) / 256 * 256; };
    off[0] = 0;
    off[1] = a256(static_cast<size_t>(tiles) * (m->n_cols + 1) * td);
    off[2] = off[1] + a256(static_cast<size_t>(tiles) * sp * td * (m->leaf_u32 ? 8 : 4));  // partials
    off[3] = off[2] + a256(static_cast<size_t>(tiles) * 4);
}

size_t odf_latency_workspace_bytes(const odf_model *m, int64_t n_docs, int32_t splits)
{
    if (!m || n_docs < 0) return 0;
    size_t off[4];
    lat_layout(m, n_docs, lat_splits(m, n_docs, splits), off);
    return off[3];
}

static odf_status run_latency(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                              float *d_scores, uint64_t *d_sums, double *d_dscores, int32_t splits,
                              void *d_workspace, size_t workspace_bytes, void *stream)
{
    odf_status st = check_factors(m, d_factors, n_docs, ld);
    if (st != ODF_OK) return st;
    if (n_docs == 0) return ok();
    const int64_t td = m->tile_docs;  // 128, or 64 for wide-column models
    if ((n_docs + td - 1) / td > 65535)  // tiles are the grid's y dimension
        return fail(ODF_E_INVALID_ARG, "latency path: n_docs > 65535 x %lld (use odf_score)", (long long)td);
    const int sp = lat_splits(m, n_docs, splits);
    size_t off[4];
    lat_layout(m, n_docs, sp, off);
    if (!d_workspace || workspace_bytes < off[3])
        return fail(ODF_E_INVALID_ARG, "workspace of %zu bytes < odf_latency_workspace_bytes = %zu",
                    workspace_bytes, off[3]);
    if (reinterpret_cast<uintptr_t>(d_workspace) % 256 != 0)
        return fail(ODF_E_INVALID_ARG, "workspace not 256-byte aligned");
    // code columns + 2 (else 1) tree-chunk buffers + reduction buffer + mbarriers
    const size_t fixed = align_up(static_cast<uint64_t>(m->n_cols) * td, 1024) +
                         (m->leaf_u32 ? 2 : 1) * kRedBytes + 64;
    const int nbuf = fixed + 2 * align_up(m->chunk_bytes, 1024) <= static_cast<size_t>(m->max_smem) ? 2 : 1;
    const size_t smem_apply = fixed + nbuf * align_up(m->chunk_bytes, 1024);
    KParams p = base_params(m, m->fused);
    p.n_docs = n_docs;
    p.n_tiles = (n_docs + td - 1) / td;
    p.scores = d_scores;
    p.sums = reinterpret_cast<unsigned long long *>(d_sums);
    p.dscores = d_dscores;
    p.stages = nbuf;
    uint8_t *ws = static_cast<uint8_t *>(d_workspace);
    p.lat_codes = ws + off[0];
    p.lat_partial = reinterpret_cast<float *>(ws + off[1]);
    p.lat_counter = reinterpret_cast<uint32_t *>(ws + off[2]);
    CUtensorMap tm;
    const CUtensorMap *tmp = nullptr;
    if (p.n_fchunks > 0) {
        st = encode_tmap(m, d_factors, n_docs, ld, &tm);
        if (st != ODF_OK) return st;
        tmp = &tm;
    }
    const size_t smem_bin = static_cast<size_t>(td) * kFSub * 4 + kMetaBytes + align_up(m->bord_stride, 16) + 64;
    if (smem_apply > static_cast<size_t>(m->max_smem))
        return fail(ODF_E_UNSUPPORTED, "latency path: %zu B of shared memory > %d", smem_apply, m->max_smem);
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != m->device) cudaSetDevice(m->device);
    cudaError_t e = launch_latency(m->kdepth, p, tmp, sp, smem_bin, smem_apply,
                                   static_cast<cudaStream_t>(stream));
    if (prev != m->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "latency kernels");
    return ok();
}

odf_status odf_score_latency(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                             float *d_scores, int32_t splits, void *d_workspace,
                             size_t workspace_bytes, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (m->leaf_u32) return fail(ODF_E_INVALID_ARG, "integer-leaf model: use odf_score_latency_u64");
    if (n_docs > 0 && !d_scores) return fail(ODF_E_INVALID_ARG, "d_scores is NULL");
    return run_latency(m, d_factors, n_docs, ld, d_scores, nullptr, nullptr, splits, d_workspace,
                       workspace_bytes, stream);
}

odf_status odf_score_latency_u64(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                                 uint64_t *d_sums, double *d_scores, int32_t splits, void *d_workspace,
                                 size_t workspace_bytes, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (!m->leaf_u32) return fail(ODF_E_INVALID_ARG, "fp32-leaf model: use odf_score_latency");
    if (n_docs > 0 && !d_sums && !d_scores)
        return fail(ODF_E_INVALID_ARG, "d_sums and d_scores are both NULL");
    return run_latency(m, d_factors, n_docs, ld, nullptr, d_sums, d_scores, splits, d_workspace,
                       workspace_bytes, stream);
}

static odf_status score_host_impl(odf_model *m, const float *h_factors, int64_t n_docs, int64_t ld,
                                  float *h_scores, int64_t chunk_docs, void *stream)
{
    if (!m) return fail(ODF_E_INVALID_ARG, "model is NULL");
    if (m->leaf_u32) return fail(ODF_E_INVALID_ARG, "odf_score_host: fp32-leaf models only");
    if (n_docs < 0 || ld < m->n_features || ld % 4 != 0)
        return fail(ODF_E_INVALID_ARG, "bad n_docs / ld (ld >= n_features, ld %% 4 == 0)");
    if (n_docs >= (int64_t(1) << 31) - kTile)
        return fail(ODF_E_INVALID_ARG, "n_docs >= 2^31 - 128 (TMA coordinate range)");
    if (n_docs == 0) return ok();
    if (!h_factors || !h_scores) return fail(ODF_E_INVALID_ARG, "NULL host buffer");
    if (chunk_docs <= 0) chunk_docs = 65536;
    chunk_docs = (chunk_docs + kTile - 1) / kTile * kTile;
    std::lock_guard<std::mutex> lock(m->host_mu);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    cudaError_t e;
    if (!m->hs[0] || m->stage_rows < chunk_docs || m->stage_ld < ld) {
        for (int i = 0; i < 2; ++i) {
            cudaFree(m->d_stage[i]);
            cudaFree(m->d_sstage[i]);
            m->d_stage[i] = nullptr;
            m->d_sstage[i] = nullptr;
            if ((e = cudaMalloc(&m->d_stage[i], static_cast<size_t>(chunk_docs) * ld * 4)) != cudaSuccess ||
                (e = cudaMalloc(&m->d_sstage[i], static_cast<size_t>(chunk_docs) * 4)) != cudaSuccess)
                return fail(ODF_E_NOMEM, "staging allocation failed");
            if (!m->hs[i]) cudaStreamCreateWithFlags(&m->hs[i], cudaStreamNonBlocking);
            if (!m->ev_out[i]) cudaEventCreateWithFlags(&m->ev_out[i], cudaEventDisableTiming);
        }
        if (!m->ev_in) cudaEventCreateWithFlags(&m->ev_in, cudaEventDisableTiming);
        m->stage_rows = chunk_docs;
        m->stage_ld = ld;
    }
    cudaStream_t us = static_cast<cudaStream_t>(stream);
    cudaEventRecord(m->ev_in, us);
    cudaStreamWaitEvent(m->hs[0], m->ev_in, 0);
    cudaStreamWaitEvent(m->hs[1], m->ev_in, 0);
    // on an error after work was queued: wait for both staging streams, so no copy
    // from or to the caller's host buffers is still running when the call returns
    auto drain = [&](odf_status st) {
        cudaStreamSynchronize(m->hs[0]);
        cudaStreamSynchronize(m->hs[1]);
        return st;
    };
    int64_t k = 0;
    for (int64_t d0 = 0; d0 < n_docs; d0 += chunk_docs, ++k) {
        const int b = static_cast<int>(k & 1);
        const int64_t n = std::min<int64_t>(chunk_docs, n_docs - d0);
        cudaStream_t s = m->hs[b];
        if ((e = cudaMemcpyAsync(m->d_stage[b], h_factors + d0 * ld, static_cast<size_t>(n) * ld * 4,
                                 cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return drain(cuda_fail(e, "H2D"));
        odf_status st = odf_score(m, m->d_stage[b], n, ld, m->d_sstage[b], s);
        if (st != ODF_OK) return drain(st);
        if ((e = cudaMemcpyAsync(h_scores + d0, m->d_sstage[b], static_cast<size_t>(n) * 4,
                                 cudaMemcpyDeviceToHost, s)) != cudaSuccess)
            return drain(cuda_fail(e, "D2H"));
    }
    for (int i = 0; i < 2; ++i) {
        cudaEventRecord(m->ev_out[i], m->hs[i]);
        cudaStreamWaitEvent(us, m->ev_out[i], 0);
    }
    if ((e = cudaStreamSynchronize(us)) != cudaSuccess) return cuda_fail(e, "odf_score_host");
    return ok();
}

odf_status odf_load_model_ex(const odf_model_desc *desc, odf_model **out)
{
    return guarded([&] { return load_model_ex_impl(desc, out); });
}

odf_status odf_load_model_paper(const odf_paper_model_desc *d, odf_model **out)
{
    return guarded([&] { return load_model_paper_impl(d, out); });
}

odf_status odf_score_host(odf_model *m, const float *h_factors, int64_t n_docs, int64_t ld,
                          float *h_scores, int64_t chunk_docs, void *stream)
{
    return guarded([&] { return score_host_impl(m, h_factors, n_docs, ld, h_scores, chunk_docs, stream); });
}

}  // extern "C"
