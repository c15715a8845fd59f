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
constexpr uint32_t kRedBytes = kConsumerWarps * kTile * 4;
constexpr uint32_t kNoCol = 0xFFFFFFFFu;

enum Mode : int { MODE_FUSED = 0, MODE_BINARIZE = 1, MODE_APPLY = 2 };

// Per-launch parameters (passed by value; all pointers are device pointers).
struct KParams {
    // ---- binarization (stage 1) ----
    const uint4 *fmeta;     // [n_fchunks*32] per raw factor: {border_off (floats), L | m<<8,
                            //  colA*128, colB*128 or kNoCol}; L == 0 -> unused factor
    const float *borders;   // per used factor: sorted borders padded to 2^L-1 with +inf,
                            // stored skewed (position p at p + (p >> 5))
    int32_t n_fchunks;      // ceil(n_features / 32), 0 if no used factor
    int32_t border_floats;  // floats in `borders`
    // ---- apply (stage 2) ----
    const uint8_t *chunks;  // [n_tchunks][chunk_bytes]: descriptors then reversed leaf tables
    int32_t n_tchunks;
    int32_t tc;             // trees per chunk (multiple of 16)
    int64_t n_trees;
    uint32_t chunk_bytes, desc_bytes, table_stride;
    const uint2 *splits;    // {u*128, colB*128} of factors with > 127 borders
    int32_t n_split;
    int32_t n_used, n_cols;
    // ---- problem ----
    int64_t n_docs, n_tiles;
    const uint8_t *bins_in;  // blocked bins (apply / index kernels)
    uint8_t *bins_out;       // blocked bins (binarize)
    float *scores;
    // ---- shared-memory plan (byte offsets from the 1 KB aligned base) ----
    uint32_t off_bins, off_borders, off_ring, off_red, off_bars;
    uint32_t slot_bytes;
    int32_t stages;
    int32_t fsub_per_job;    // TMA sub-tiles per factor job (slot_bytes / 16 KB)
    int32_t borders_smem;    // 1: borders copied to shared memory at kernel start
    // ---- index export / fingerprint ----
    int64_t doc0, ndoc, tree0, ntree;
    uint16_t *idx_out;
    uint64_t *fp_out;
};

cudaError_t launch_main(int mode, int depth, const KParams &p, const CUtensorMap *tmap, int grid,
                        size_t smem, cudaStream_t s);
cudaError_t launch_index(int depth, const KParams &p, bool fingerprint, int grid, size_t smem,
                         cudaStream_t s);
// Opt every kernel in to `smem` bytes of dynamic shared memory.
cudaError_t prepare_kernels(int max_smem);
// Number of co-resident CTAs per SM of a main kernel at `smem` bytes.
int occupancy_main(int mode, int depth, size_t smem);

}  // namespace odf
