// odf_internal.h -- structures shared by the host launcher (odf_capi.cu) and the
// kernels (odf_kernels.cu) of the CUDA path.  Not part of the ABI (see include/odf.h).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace odf {

constexpr int kTile = 128;                 // documents per tile (4 per lane x 32 lanes)
constexpr int kConsumerWarps = 16;         // = number of tree groups
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kThreads = kConsumerThreads + 32;  // + 1 producer (TMA) warp
constexpr int kFSub = 32;                  // factors per TMA sub-tile (32 x 4 B = 128 B rows)
constexpr uint32_t kFSubBytes = kTile * kFSub * 4;  // 16 KB TMA box [128 docs x 32 factors]
constexpr uint32_t kMetaBytes = kFSub * 16;         // fmeta of one sub-tile
constexpr uint32_t kRedBytes = kConsumerWarps * kTile * 4;
constexpr uint32_t kNoCol = 0xFFFFFFFFu;

// Tree-chunk geometry, shared by the model compiler and the kernels: per tree the
// level descriptors (4 B each, padded to a multiple of 4) and the reversed leaf table
// (256 B for depth <= 6 so the PRMT address trick applies, else 4 B * 2^depth);
// trees per chunk = a multiple of 16 (one tree per consumer warp per round) sized
// for ~20 KB chunks.  The last chunk is padded with zero-answer trees (-0.0 / 0),
// so the apply loop has a fixed trip count.
// Level descriptor (u32): bits 19-31 = code column (col * 128 = desc >> 12), bits 0-7 =
// 128 - K; a tree's descriptors are padded to a multiple of 4 levels (LDS.128 groups).
// Level descriptor formats:
//  * split, depth <= 8: the levels' col * 128 words, then the levels' (128 - K)
//    bytes packed four per word (level l in byte l % 4 of word depth + l / 4),
//    padded to 16 bytes: depth 6 = 32 B = two LDS.128.  A warp-uniform LDS.128
//    costs two shared-memory wavefronts, so descriptor bytes per tree are
//    shared-memory time; replicating K costs one PRMT per level;
//  * 8 bytes {col * 128, (128 - K) * 0x01010101} (A/B builds): no PRMT, 48 B per
//    depth-6 tree;
//  * 4 bytes (col << 19) | (128 - K) for depth 9-10: address and K from one word.
constexpr int kMaxDescCol = 8191;
#ifndef ODF_DESC_SPLIT_MAX_DEPTH
#define ODF_DESC_SPLIT_MAX_DEPTH 8  // A/B builds only
#endif
#ifndef ODF_DESC8_MAX_DEPTH
#define ODF_DESC8_MAX_DEPTH 8  // A/B builds only
#endif
enum DescFmt : int { DESC4 = 0, DESC8 = 1, DESC_SPLIT = 2 };
__host__ __device__ constexpr int desc_fmt(int depth)
{
    return depth <= ODF_DESC_SPLIT_MAX_DEPTH ? DESC_SPLIT : depth <= ODF_DESC8_MAX_DEPTH ? DESC8 : DESC4;
}
// words of a split-format tree that carry data: depth column words + ceil(depth / 4) K words
__host__ __device__ constexpr int desc_split_words(int depth) { return depth + (depth + 3) / 4; }
__host__ __device__ constexpr int desc_stride(int depth)
{
    return desc_fmt(depth) == DESC_SPLIT ? ((desc_split_words(depth) + 3) & ~3) * 4
           : desc_fmt(depth) == DESC8    ? ((depth + 1) & ~1) * 8
                                         : ((depth + 3) & ~3) * 4;
}
__host__ __device__ constexpr int table_stride(int depth) { return depth <= 6 ? 256 : (4 << depth); }
__host__ __device__ constexpr int trees_per_chunk(int depth)
{
    return 16 * ((20480 / (16 * (desc_stride(depth) + table_stride(depth)))) > 1
                     ? (20480 / (16 * (desc_stride(depth) + table_stride(depth))))
                     : 1);
}

enum Mode : int { MODE_FUSED = 0, MODE_BINARIZE = 1, MODE_APPLY = 2 };

// Mixed-height models (NEXT-2, the paper's native layout): the forest is a
// list of height segments, each with its own tree-chunk geometry, concatenated in
// one chunk stream; kernels instantiated with DEPTH = kMixedDepth apply each chunk
// with its segment's depth (integer answers: the u64 sum is order-free).
constexpr int kMixedDepth = 11;
constexpr int kMaxSegments = 11;  // heights 0..10
struct SegP {
    int32_t depth, tc, n_chunks;
    uint32_t chunk_bytes, desc_bytes, pad_;
    uint64_t byte_off;  // of the segment's first chunk in `chunks`
};

// Per-launch parameters (passed by value; all pointers are device pointers).
struct KParams {
    // ---- binarization (stage 1) ----
    const uint4 *fmeta;     // [n_fchunks*32] per raw factor: {array byte offset (relative to its
                            //  sub-tile's border block, 16 B aligned), cls | (C-1)<<4 | (-npad)<<16,
                            //  colA*128, colB*128}; cls 0 unused, 1 LIN4, L+1 BIN(L); C code
                            //  columns (> 127 borders); unused slots of a pair: trash column
    const float *borders;   // per used factor: npad x -inf then its m sorted borders; LIN4
                            // arrays have 4 entries, BIN(L) arrays 2^L-1 entries stored skewed
                            // (position p at p + (p >> 5))
    const uint2 *bchunk;    // [n_fchunks] {byte offset into borders, bytes} of each sub-tile's
                            // border arrays (fmeta.x is relative to that offset)
    int32_t n_fchunks;      // ceil(n_features / 32), 0 if no used factor
    int32_t fm;             // 1: factors are feature-major [n_features][ld] (NEXT-4)
    // ---- apply (stage 2) ----
    const uint8_t *chunks;  // [n_tchunks][chunk_bytes]: descriptors then reversed leaf tables
    int32_t n_tchunks;
    int32_t tc;             // trees per chunk (multiple of 16)
    int64_t n_trees;
    uint32_t chunk_bytes, desc_bytes, table_stride;
    const uint2 *splits;    // {u*128, colB*128} of factors with 128..254 borders (narrow models)
    int32_t n_split;
    int32_t wide;           // 1: some factor has > 254 borders -> u16 true bins (NEXT-4)
    const uint2 *ucols;     // wide models: [n_used] {first extra code column * 128 or trash, C}
    uint32_t off_stage;     // wide models: shared-memory staging of a u16 bins tile
    int32_t n_used, n_cols;
    // ---- mixed-height models (DEPTH = kMixedDepth) ----
    int32_t n_seg;
    SegP seg[kMaxSegments];
    // ---- problem ----
    int32_t tile_docs;       // the model's tile width: 128, or 64 (wide-column models, DPL = 2)
    int32_t pdl;             // 1: primary of a programmatic dependent launch (lets the secondary
                             // launch), 2: secondary (waits for the primary before it exits)
    int64_t n_docs, n_tiles;
    const uint8_t *bins_in;  // blocked bins (apply / index kernels)
    uint8_t *bins_out;       // blocked bins (binarize)
    float *scores;
    // ---- MatrixNet integer mode: u32 leaves, u64 sums ----
    int32_t leaf_u32;        // 1: leaf tables hold u32 answers
    double scale, bias;      // final (R - 2^31) * S + B
    unsigned long long *sums;  // [n_docs] u64 sums R (may be null)
    double *dscores;         // [n_docs] final scores (may be null)
    // ---- shared-memory plan (byte offsets from the 1 KB aligned base) ----
    uint32_t off_bins, off_ring, off_red, off_bars;
    uint32_t slot_bytes;
    uint32_t off_meta, off_bord, bord_stride;  // within a factor job's slot
    uint32_t half_stride;    // tile halves (H = 2): bytes between the halves' code blocks
    uint32_t hdesc_bytes;    // H = 2: offset of the tables in a half-chunk ring slot
    int32_t stages;
    int32_t fsub_per_job;    // factor sub-tiles per job (tiles, then metas, then borders)
    // ---- latency path (K4) workspace ----
    uint8_t *lat_codes;      // [n_tiles][n_cols + 1][128] 7-bit codes (+ trash column)
    int64_t code_stride;     // bytes per tile of a global code block: (n_cols + 1) * 128
    float *lat_partial;      // [n_tiles][splits][128]
    uint32_t *lat_counter;   // [n_tiles] tickets
    // ---- NEXT-3 bit-packed condition words ----
    const uint32_t *bf_base;   // [n_used + 1] first binary feature of each used factor
    int64_t k_bin;             // number of binary features
    uint32_t *words;           // [ceil(D/32)][k_bin]
    const uint32_t *bits_desc; // [n_trees][depth] byte offset (kb * 4) of each level's word
    const float *leaves;       // [n_trees << depth] original leaf order
    // ---- index export / fingerprint ----
    int64_t doc0, ndoc, tree0, ntree;
    uint16_t *idx_out;
    uint64_t *fp_out;
};

// Kernel pointers, one kernel family per translation unit (odf_k_*.cu).
const void *kptr_fused_nf(int depth);  // fused, fp32 leaves
const void *kptr_fused_nu(int depth);  // fused, u32 leaves (NEXT-1)
const void *kptr_fused_wf(int depth);  // fused, wide models (NEXT-4), fp32 leaves
const void *kptr_fused_wu(int depth);  // fused, wide models, u32 leaves
const void *kptr_apply(int depth, bool u32);
const void *kptr_mixed(int mode);      // mixed-height integer models, fused / apply
// 64-document tiles (DPL = 2): fp32 fused / apply (depth) and binarize; u32 fused / apply
// (depth 0..10 or kMixedDepth); index export
const void *kptr_t64_f(int mode, int depth);
const void *kptr_t64_u(int mode, int depth);
const void *kptr_t64_index(int depth);
const void *kptr_t64_lat(int depth);  // K4 with 64-document tiles: apply (depth), binarize (-1)
const void *kptr_lat_u(int depth, int tile_docs);  // K4 apply, u32 leaves: depth 0..10 or kMixedDepth
const void *kptr_fused_h2(int depth);  // fused, fp32 leaves, 256-document tiles (H = 2)
const void *kptr_apply_h2(int depth);  // apply, fp32 leaves, 256-document tiles
const void *kptr_binarize(bool wide);

cudaError_t launch_main(int mode, int depth, const KParams &p, const CUtensorMap *tmap, int grid,
                        size_t smem, cudaStream_t s, int halves = 1,
                        bool pdl_secondary = false);  // p.tile_docs picks DPL
cudaError_t launch_index(int depth, const KParams &p, bool fingerprint, int grid, size_t smem,
                         cudaStream_t s);
cudaError_t launch_latency(int depth, const KParams &p, const CUtensorMap *tmap, int splits,
                           size_t smem_bin, size_t smem_apply, cudaStream_t s);  // p.tile_docs picks DPL
cudaError_t launch_bits(int depth, const KParams &p, bool apply, size_t smem, cudaStream_t s);
// Opt every kernel in to `smem` bytes of dynamic shared memory.
cudaError_t prepare_kernels(int max_smem);
// Number of co-resident CTAs per SM of a main kernel at `smem` bytes.
int occupancy_main(int mode, int depth, size_t smem, int tile_docs = 128);

}  // namespace odf
