/*
 * odf.h -- C ABI of the B200-native oblivious-decision-forest scorer.
 *
 * The method (arxiv 2205.07307, /root/reference/PAPER.md, cited P:<line>):
 * a forest of oblivious trees; a tree of height d has d node conditions
 * FACTOR[INDEX_l] < THRESHOLD_l, one per level, and 2^d answers.
 * Scoring a document has two stages:
 *   binarization  - evaluate the node conditions (binary features), §5;
 *   tree apply    - per tree, write the level conditions as a binary number
 *                   (true = 1; level l = bit l, least significant
 *                   first), fetch that answer and sum over trees.
 * The binarized form used here is the north_star's: per used feature f, the
 * sorted unique thresholds ("borders") b_0 < ... < b_{m-1} and the bin
 *   bin(x) = #{ j : !(x < b_j) }                                 (0 <= bin <= m)
 * stored as uint8 when every feature has m <= ODF_MAX_BORDERS (254), else as
 * uint16 for every feature ("wide" model, m <= ODF_MAX_BORDERS_WIDE; NEXT-4)
 * for which  x < b_k  <=>  bin(x) <= k  for every border, NaN included
 * (DESIGN.md "Readings of the paper").
 *
 * Conventions for every call:
 *  - Host pointers are marked h_*, device pointers d_*; "stream" is a
 *    cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Calls are stream-ordered and asynchronous unless stated; none but
 *    odf_load_model / odf_free_model / odf_score_host synchronises.
 *  - The caller owns every d_* / h_* buffer; the library never frees them and
 *    never allocates per call (odf_score_host uses model-owned staging that is
 *    allocated once, see there).
 *  - Errors: every call returns an odf_status; odf_last_error() returns a
 *    thread-local message naming the violated bound.  No exceptions cross the
 *    ABI.  A CUDA launch error is ODF_E_CUDA.  There is no CPU fallback.
 *  - A model is immutable after load; concurrent calls on different streams
 *    with different output buffers are safe.
 */
#ifndef ODF_H
#define ODF_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ODF_API __attribute__((visibility("default")))
#else
#define ODF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct odf_model odf_model; /* opaque */

typedef enum {
    ODF_OK = 0,
    ODF_E_INVALID_ARG = 1, /* a documented bound is violated (message names it) */
    ODF_E_UNSUPPORTED = 2, /* valid but outside this build's limits (>2032 borders, smem) */
    ODF_E_NOMEM = 3,       /* device or pinned-host allocation failed */
    ODF_E_CUDA = 4         /* CUDA runtime / launch error (message has cudaGetErrorString) */
} odf_status;

/* Bins are stored in a blocked layout: tiles of TD = odf_model_info.bins_tile_docs
 * documents (ODF_TILE_DOCS = 128, or 64 for models whose 128-document code block
 * does not fit shared memory); tile g holds n_used rows of TD elements, row u =
 * used feature u (ascending raw feature id), element j = document g*TD + j.  An
 * element is a uint8, or a little-endian uint16 for a wide model
 * (odf_model_info.bins_elem_bytes).  Elements of padding documents (>= n_docs)
 * in the last tile are defined but meaningless.                             */
#define ODF_TILE_DOCS 128
#define ODF_MAX_DEPTH 10
#define ODF_MAX_BORDERS 254       /* largest border count with uint8 bins */
#define ODF_MAX_BORDERS_WIDE 2032 /* largest border count at all (uint16 bins, NEXT-4) */

ODF_API int odf_version(void);                 /* ODF_VERSION_MAJOR*10000 + MINOR*100 + PATCH */
ODF_API const char *odf_last_error(void);      /* thread-local; "" when the last call succeeded */

/* Load (compile) a uniform-depth oblivious forest onto device `device`.
 *   feature_index [n_trees*depth]  host, int32; entry t*depth + l is the factor
 *                  tested at level l of tree t (l = 0 is the root level and bit 0
 *                  of the leaf index); 0 <= value < n_features.
 *   thresholds    [n_trees*depth]  host, fp32, finite; condition is
 *                  factor < threshold (strict).
 *   leaf_values   [n_trees << depth] host, fp32, finite; answer j of tree t at
 *                  t*2^depth + j (P:305 with fp32 answers).
 *   depth in [0, ODF_MAX_DEPTH]; n_trees >= 0; n_features >= 1.
 * The arrays are copied; the caller may free them on return.  Errors:
 *   ODF_E_INVALID_ARG  bad depth / counts / null pointer / feature index out of
 *                      range / non-finite threshold or leaf;
 *   ODF_E_UNSUPPORTED  a feature with more than ODF_MAX_BORDERS_WIDE distinct
 *                      thresholds, or a model whose per-tile state exceeds the
 *                      227 KB shared-memory budget even with 64-document tiles
 *                      (message says which);
 *   ODF_E_NOMEM / ODF_E_CUDA.  Synchronises the device.  *out = NULL on error. */
ODF_API odf_status odf_load_model(const int32_t *feature_index, const float *thresholds,
                          const float *leaf_values, int32_t depth, int64_t n_trees,
                          int32_t n_features, int device, odf_model **out);

/* General load (fp32 or MatrixNet integer leaves).  leaf_type ODF_LEAF_U32:
 * leaf_values is uint32 [n_trees << depth]; scores are the paper's u64 sums R
 * and (R - 2^31) * S + B with S = scale, B = bias (applied once
 * per document, SURVEY 8(c) reading 9), computed by odf_score_u64 /
 * odf_apply_u64 (exact: zero-tolerance parity).  Other fields as odf_load_model. */
#define ODF_LEAF_F32 0
#define ODF_LEAF_U32 1
typedef struct {
    const int32_t *feature_index; /* [n_trees*depth] */
    const float *thresholds;      /* [n_trees*depth] */
    const void *leaf_values;      /* [n_trees << depth], float or uint32 per leaf_type */
    int32_t leaf_type;            /* ODF_LEAF_F32 / ODF_LEAF_U32 */
    int32_t depth;
    int64_t n_trees;
    int32_t n_features;
    int32_t device;
    double scale, bias;           /* integer mode only */
} odf_model_desc;
ODF_API odf_status odf_load_model_ex(const odf_model_desc *desc, odf_model **out);

/* Paper-native model import (NEXT-2).  The model of §5.1/§6.1:
 * binary-feature descriptor groups (factor index, number of binary features; the
 * group's binary features are consecutive), one threshold per binary
 * feature, STC[h] = number of trees of height h (0..8), per-tree condition
 * indices into the binary features with trees stored in descending height
 * (P:307), u32 answers, and S, B of P:309.  The import keeps the paper's height
 * mix: one segment per height present (descending, as stored), each staged and
 * applied by the kernels at its own depth (a tree of height h costs h levels and a
 * 2^h-entry table; the u64 sum is exact, so the order is free).  pad_heights = 1
 * selects the earlier padded form instead: a uniform-depth model of depth D = the
 * largest height, a tree of height h < D repeating its level 0 on levels h..D-1
 * with its table replicated (answer j = answer[j mod 2^h]).  Both give the same
 * sums.  Score with odf_score_u64 / odf_apply_u64 (exact); odf_leaf_indices /
 * odf_index_fingerprint need a uniform-depth model (ODF_E_UNSUPPORTED for a
 * mixed one).  Errors: ODF_E_INVALID_ARG for out-of-range indices, heights >
 * ODF_MAX_DEPTH, non-finite thresholds, sizes.                                  */
typedef struct {
    int32_t n_features;
    const int32_t *group_factor; /* [n_groups] */
    const int32_t *group_count;  /* [n_groups], >= 1 */
    int32_t n_groups;
    const float *thresholds;     /* [sum group_count] */
    const int32_t *stc;          /* [ODF_MAX_DEPTH + 1] trees per height 0..10 */
    const uint32_t *cond_indices; /* [sum_h h * stc[h]] */
    const uint32_t *leaves;      /* [sum_h 2^h * stc[h]] */
    double scale, bias;
    int32_t device;
    int32_t pad_heights;         /* 0: one segment per height (default); 1: padded uniform form */
} odf_paper_model_desc;
ODF_API odf_status odf_load_model_paper(const odf_paper_model_desc *desc, odf_model **out);

ODF_API void odf_free_model(odf_model *m); /* NULL is a no-op; synchronises the device */

typedef struct {
    int32_t depth, n_features, n_used_features, n_split_features, n_columns;
    int64_t n_trees;
    int32_t trees_per_chunk, n_tree_chunks;
    int64_t chunk_bytes, model_device_bytes;
    int32_t max_borders;        /* max distinct borders of one feature */
    int64_t total_borders;      /* sum over used features */
    int32_t borders_in_smem;    /* 1 if the fused kernel keeps all borders in shared memory */
    int32_t stages_fused;       /* ring stages of the fused kernel */
    int32_t smem_fused;         /* dynamic shared memory per CTA of the fused kernel, bytes */
    int32_t num_sms;
    int32_t leaf_type;          /* ODF_LEAF_F32 / ODF_LEAF_U32 */
    int32_t bord_stride;        /* max bytes of one 32-factor sub-tile's border arrays */
    int32_t bins_elem_bytes;    /* 1: uint8 bins; 2: uint16 bins (a feature has > ODF_MAX_BORDERS) */
    int32_t max_tile_docs;      /* 256 if 256-document tiles fit (odf_score_tiles), else 128 */
    int32_t stages_fused_256;   /* ring stages of the fused kernel with 256-document tiles (0: none) */
    int32_t smem_fused_256;     /* its dynamic shared memory per CTA, bytes (0: none) */
    int32_t bins_tile_docs;     /* documents per tile and per bins block: ODF_TILE_DOCS (128), or 64
                                   for models whose 128-document code block does not fit shared
                                   memory (about > 1,600 code columns, e.g. P:168's 1,950 factors;
                                   at depth 9-10 such widths do not fit at all: ODF_E_UNSUPPORTED) */
    int32_t tail_tile_docs;     /* 64 if odf_score runs a partly filled last wave as 64-document tiles
                                   (a second grid, odf_score_tiles), else 0 */
} odf_model_info;

ODF_API odf_status odf_get_info(const odf_model *m, odf_model_info *info);

/* Bytes of the blocked bins buffer for n_docs documents
 * (= ceil(n_docs/TD) * n_used * TD * bins_elem_bytes, TD = odf_model_info.bins_tile_docs:
 * layout [ceil(n_docs/TD)][n_used][TD], document d of a block at byte d), the number of used
 * features, and (optional, may be NULL) a library-owned pointer to their raw
 * ids, ascending, valid until odf_free_model.                                */
ODF_API odf_status odf_bins_layout(const odf_model *m, int64_t n_docs, size_t *bytes,
                           int32_t *n_used_features, const int32_t **used_feature_ids);

/* Stage 1 (§5): d_factors [n_docs x ld] fp32 row-major on the
 * model's device (16-byte aligned, ld % 4 == 0, ld >= n_features) -> d_bins in
 * the blocked layout above (odf_bins_layout bytes).  n_docs == 0 is a no-op.
 * Errors: ODF_E_INVALID_ARG (null / misaligned / ld), ODF_E_CUDA.            */
ODF_API odf_status odf_binarize(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                        uint8_t *d_bins, void *stream);

/* Stage 2 (§6): d_bins (blocked layout) -> d_scores [n_docs] fp32,
 * score(i) = sum over trees of the answer at the tree's leaf index,
 * accumulated in fp32 in the fixed order of DESIGN.md "Summation order"
 * (independent of n_docs and of the document's position). n_trees == 0 -> 0. */
ODF_API odf_status odf_apply(const odf_model *m, const uint8_t *d_bins, int64_t n_docs,
                     float *d_scores, void *stream);

/* Fused stages 1+2 (any binarization composes with any apply): same
 * inputs as odf_binarize, same scores as odf_apply (bit-identical: same
 * summation order); bins live only in shared memory, never in HBM.           */
ODF_API odf_status odf_score(const odf_model *m, const float *d_factors, int64_t n_docs, int64_t ld,
                     float *d_scores, void *stream);

/* Documents per tile (a performance choice, not a numerical one).  odf_score and
 * odf_apply pick it themselves; these variants take tile_docs = 0 (the same
 * automatic choice), 128 or 256.  A 256-document tile is two 128-document halves
 * that share every tree chunk staged in shared memory, which halves the forest's
 * L2 -> shared-memory traffic per document (what binds deep forests, BASELINE
 * config c4); it needs two code blocks in shared memory, so it exists only for
 * fp32-leaf models without > 254-border factors whose codes fit
 * (odf_model_info.max_tile_docs).  The automatic choice takes it for depth >= 7
 * and at least 2 x num_sms tiles of 256 documents (odf_score: only when its ring
 * still has >= 3 slots, stages_fused_256).  Scores are bit-identical for
 * every tile width (the summation order of DESIGN.md does not depend on it).
 * Models with odf_model_info.bins_tile_docs == 64 run 64-document tiles only
 * (tile_docs 0 or 64).  With tile_docs = 0, odf_score (fp32 uniform models of depth
 * <= 6) also runs a last wave of 128-document tiles that would fill at most half of
 * the SMs as 64-document tiles
 * in a second grid (a programmatic dependent launch on the same stream; the call
 * still enqueues one unit of work: later work on the stream sees every score).
 * Errors: as odf_score / odf_apply; ODF_E_INVALID_ARG for another tile_docs;
 * ODF_E_UNSUPPORTED for a width the model does not have.                     */
ODF_API odf_status odf_score_tiles(const odf_model *m, const float *d_factors, int64_t n_docs,
                                   int64_t ld, float *d_scores, int32_t tile_docs, void *stream);
ODF_API odf_status odf_apply_tiles(const odf_model *m, const uint8_t *d_bins, int64_t n_docs,
                                   float *d_scores, int32_t tile_docs, void *stream);

/* Feature-major input (NEXT-4; the paper's pre-transposed variant, §5.5):
 * d_factors_fm [n_features x ld_fm] fp32 row-major, i.e. factor f of document i at
 * d_factors_fm[f*ld_fm + i]; ld_fm >= n_docs, ld_fm % 4 == 0, 16-byte aligned.
 * Same bins / scores as odf_binarize / odf_score on the transposed matrix
 * (bit-identical).  The TMA box is (128 docs x 32 factors), unswizzled.       */
ODF_API odf_status odf_binarize_fm(const odf_model *m, const float *d_factors_fm, int64_t n_docs,
                                   int64_t ld_fm, uint8_t *d_bins, void *stream);
ODF_API odf_status odf_score_fm(const odf_model *m, const float *d_factors_fm, int64_t n_docs,
                                int64_t ld_fm, float *d_scores, void *stream);

/* NEXT-3: bit-packed ordered condition words (the paper's ordered format,
 * §5.4: "на смещении i стоит бит, соответствующий документу номер i+1").
 * Binary feature kb = (used factor u, border j) in ascending (u, j); its bit for
 * document i is the node condition x_i < border_j.  Words: uint32
 * [ceil(n_docs/32)][n_binary], bit i of word (g, kb) = document 32g + i (0 for
 * padding documents >= n_docs).
 * odf_bits_from_bins builds them from blocked bins (one __ballot_sync per binary
 * feature per 32 documents); odf_apply_bits assembles each leaf index from the
 * words (§6.4) and returns the same scores as odf_score (same
 * summation order).  odf_apply_bits: fp32-leaf models whose binary features fit
 * shared memory (n_binary * 4 B), else ODF_E_UNSUPPORTED.                      */
ODF_API odf_status odf_bits_layout(const odf_model *m, int64_t n_docs, size_t *bytes,
                                   int64_t *n_binary_features);
ODF_API odf_status odf_bits_from_bins(const odf_model *m, const uint8_t *d_bins, int64_t n_docs,
                                      uint32_t *d_words, void *stream);
ODF_API odf_status odf_apply_bits(const odf_model *m, const uint32_t *d_words, int64_t n_docs,
                                  float *d_scores, void *stream);

/* Integer-leaf models (ODF_LEAF_U32): fused (from factors) and stage-2 (from
 * bins) scoring into d_sums [n_docs] uint64 (R, exact) and/or d_scores [n_docs]
 * double ((R - 2^31) * S + B, each operation rounded to nearest, no FMA); either
 * output may be NULL but not both.  fp32 models are rejected (ODF_E_INVALID_ARG),
 * and odf_score / odf_apply reject integer models.                           */
ODF_API odf_status odf_score_u64(const odf_model *m, const float *d_factors, int64_t n_docs,
                                 int64_t ld, uint64_t *d_sums, double *d_scores, void *stream);
ODF_API odf_status odf_apply_u64(const odf_model *m, const uint8_t *d_bins, int64_t n_docs,
                                 uint64_t *d_sums, double *d_scores, void *stream);

/* Test/debug (K6): leaf indices idx[d][t] (true index, level l = bit l) of
 * documents [doc0, doc0+ndoc) and trees [tree0, tree0+ntree) from d_bins
 * (n_docs documents, blocked layout) into d_idx [ndoc x ntree] uint16 row-major.
 * Computed by the same device code as odf_apply.  Errors: ranges outside
 * [0, n_docs) x [0, n_trees) -> ODF_E_INVALID_ARG.                          */
ODF_API odf_status odf_leaf_indices(const odf_model *m, const uint8_t *d_bins, int64_t n_docs,
                            int64_t doc0, int64_t ndoc, int64_t tree0, int64_t ntree,
                            uint16_t *d_idx, void *stream);

/* Test/debug (K6): per-document FNV-1a-64 over (idx[i][0..n_trees-1]) as u16
 * little-endian, from d_bins; d_fp [n_docs] uint64.                          */
ODF_API odf_status odf_index_fingerprint(const odf_model *m, const uint8_t *d_bins, int64_t n_docs,
                                 uint64_t *d_fp, void *stream);

/* Small-batch latency path (K4, config c5): the same scores as odf_score within
 * the tolerance (the tree sum is split into `splits` contiguous chunk ranges per
 * tile of odf_model_info.bins_tile_docs documents (128, or 64 for wide-column
 * models) and combined in ascending split order: deterministic, but a
 * different association than odf_score).  Two kernel
 * launches: binarization spread over one CTA per (tile, 32-factor sub-tile), then
 * the apply spread over `splits` CTAs per tile.  splits <= 0 picks a default
 * (about 2 CTAs per SM).  d_workspace: device memory of at least
 * odf_latency_workspace_bytes(m, n_docs, splits) bytes (same `splits`), owned by
 * the caller; concurrent calls need distinct workspaces.  Same argument rules as
 * odf_score, and n_docs <= 65535 x bins_tile_docs (ODF_E_INVALID_ARG above: tiles
 * are a grid dimension; this is the small-batch path).  fp32-leaf models (integer
 * models: odf_score_latency_u64, ODF_E_INVALID_ARG here).  Capturable in a CUDA graph (two
 * kernel nodes; the factor pointer is baked into the captured tensor map, so a
 * graph serves one input buffer, tests/test_gpu_parity.py::test_latency_graph). */
ODF_API size_t odf_latency_workspace_bytes(const odf_model *m, int64_t n_docs, int32_t splits);
ODF_API odf_status odf_score_latency(const odf_model *m, const float *d_factors, int64_t n_docs,
                                     int64_t ld, float *d_scores, int32_t splits,
                                     void *d_workspace, size_t workspace_bytes, void *stream);
/* The latency path for integer-leaf models (NEXT-1; mixed heights, NEXT-2, included):
 * outputs as odf_score_u64 (either may be NULL, not both).  The per-split partial
 * sums are u64 and added exactly, so the results equal odf_score_u64's bit for bit.
 * Workspace: odf_latency_workspace_bytes of this model (8-byte partials).  fp32
 * models: ODF_E_INVALID_ARG.  Otherwise as odf_score_latency.                  */
ODF_API odf_status odf_score_latency_u64(const odf_model *m, const float *d_factors, int64_t n_docs,
                                         int64_t ld, uint64_t *d_sums, double *d_scores, int32_t splits,
                                         void *d_workspace, size_t workspace_bytes, void *stream);

/* End-to-end from HOST memory: h_factors [n_docs x ld] fp32 (pinned or not;
 * pinned is faster) -> h_scores [n_docs].  Copies host->device, runs the fused
 * kernel, copies back, in chunks pipelined over two model-owned device staging
 * buffers (allocated on first use, sized for `chunk_docs` rows of ld floats,
 * reused while ld <= the first call's ld; freed by odf_free_model).  Blocks
 * until h_scores is written.  Same results as odf_score.                     */
ODF_API odf_status odf_score_host(odf_model *m, const float *h_factors, int64_t n_docs, int64_t ld,
                          float *h_scores, int64_t chunk_docs, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ODF_H */
