// launch.h -- host-side launchers of the query and binning kernels (query.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace pndf {

bool lanes_supported(int G, int NV);

// PNDF_NOG4=1 in the environment: G == 32 launches use query_kernel instead of query_g4_kernel (A/B runs;
// results are bitwise identical either way).
bool g4_disabled();
// PNDF_NOG5=1: G == 32 launches with a range table use query_g4_kernel instead of query_g5_kernel (A/B runs;
// the two differ only in the order of the final rank sum).
bool g5_disabled();
// queries per interleaved chunk of query_g5_kernel (PNDF_G5CHUNK, default 16384, a multiple of 256)
int64_t g5_chunk();
// PNDF_G5ROT=0: every CTA walks its chunks in batch order (default 1: rotated start per CTA)
bool g5_rot();

// Query kernel over n records; idx != nullptr means the records are binned
// and idx[i] is record i's position in the caller's output.
cudaError_t launch_query(const QParams& p, int G, int NV, const pndf_query* q, const uint32_t* idx, int64_t n,
                         float* out, int num_sms, cudaStream_t st);

// Sampling kernel (sample.cu); idx as for launch_query.
cudaError_t launch_sample(const QParams& p, int G, int NV, const pndf_query* q, const float* xi, const uint32_t* idx,
                          int64_t n, pndf_sample* out, int num_sms, cudaStream_t st);

// per-variant instantiations (query_<fmt>_<border>.cu, sample_<fmt>_<border>.cu)
cudaError_t launch_query_u32_wrap(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx,
                                 int64_t n, float* out, int num_sms, cudaStream_t st);
cudaError_t launch_sample_u32_wrap(int G, int NV, const QParams& p, const pndf_query* q, const float* xi,
                                  const uint32_t* idx, int64_t n, pndf_sample* out, int num_sms, cudaStream_t st);
cudaError_t launch_query_u32_clamp(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx,
                                 int64_t n, float* out, int num_sms, cudaStream_t st);
cudaError_t launch_sample_u32_clamp(int G, int NV, const QParams& p, const pndf_query* q, const float* xi,
                                  const uint32_t* idx, int64_t n, pndf_sample* out, int num_sms, cudaStream_t st);
cudaError_t launch_query_hilo_wrap(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx,
                                 int64_t n, float* out, int num_sms, cudaStream_t st);
cudaError_t launch_sample_hilo_wrap(int G, int NV, const QParams& p, const pndf_query* q, const float* xi,
                                  const uint32_t* idx, int64_t n, pndf_sample* out, int num_sms, cudaStream_t st);
cudaError_t launch_query_hilo_clamp(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx,
                                 int64_t n, float* out, int num_sms, cudaStream_t st);
cudaError_t launch_sample_hilo_clamp(int G, int NV, const QParams& p, const pndf_query* q, const float* xi,
                                  const uint32_t* idx, int64_t n, pndf_sample* out, int num_sms, cudaStream_t st);

// Wang-tiled query (tiles.cu).
cudaError_t launch_tiled_query(const QParams& p, const TileParams& tp, int G, int NV, const pndf_query* q,
                               const uint32_t* idx, int64_t n, float* out, int num_sms, cudaStream_t st);
cudaError_t launch_tiled_sample(const QParams& p, const TileParams& tp, int G, int NV, const pndf_query* q,
                                const float* xi, const uint32_t* idx, int64_t n, pndf_sample* out,
                                int32_t* tile_out, int num_sms, cudaStream_t st);
// Reach of a tiled store (tiles.cu): the largest distance, in cells beyond the tile's own grid
// (0 = inside), of any row with a nonzero entry, over all tiles and levels -> *reach (device).
cudaError_t launch_tile_reach(const float* Zc, int Rp, const TileParams& tp, int n0, int L, uint32_t* reach,
                              cudaStream_t st);
// Stable sort of a batch by footprint level (query.cu): perm = records in level order.
cudaError_t launch_level_sort(const QParams& p, const pndf_query* q, int64_t n, BinScratch& sc, cudaStream_t st,
                              int* launches, const uint32_t** perm);

// Blocked / clustered store (blocks.cu).
cudaError_t launch_blocked_query(const QParams& p, const BlockParams& bp, int G, int NV, const pndf_query* q,
                                 int64_t n, float* out, int num_sms, cudaStream_t st);
// Importance sampling on the blocked store (blocks.cu): xi [n][11], blk [n] chosen block (may be NULL).
cudaError_t launch_blocked_sample(const QParams& p, const BlockParams& bp, int G, int NV, const pndf_query* q,
                                  const float* xi, int64_t n, pndf_sample* out, int32_t* blk, int num_sms,
                                  cudaStream_t st);
cudaError_t launch_block_build(const float* X, const float* Y, int sets, int t, int R, int Rp, float* pool,
                               const float* Z, int64_t slabs, const float* C, const int32_t* slab_set, float* Zc,
                               uint32_t* flags, int num_sms, cudaStream_t st);

// Environment-prefiltering rectangles (sg.cu).
cudaError_t launch_sg_rects(const pndf_sg_light* in, int64_t n, float eps, int A, pndf_query* out, int num_sms,
                            cudaStream_t st);

// Distinct Zc rows the query kernel reads for n records (query.cu): bitmap [ceil(P/32)] words, zeroed by
// the caller; *count (device) receives the popcount.
cudaError_t launch_rows_touched(const QParams& p, const pndf_query* q, int64_t n, int64_t P, uint32_t* bitmap,
                                int64_t* count, int num_sms, cudaStream_t st);

int64_t scan_blocks(int64_t nb);
int64_t radix_tiles(int64_t n);

// Sort the n records by bin key (store with P rows) with an LSD radix sort;
// *perm receives the device permutation (query indices in binned order).
// Scratch: keys/vals [cap], counts [radix_tiles(cap)*512], bsum [scan_blocks(that)].
cudaError_t launch_binning(const QParams& p, const pndf_query* q, int64_t n, int64_t P, BinScratch& sc,
                           int num_sms, cudaStream_t st, int* launches, const uint32_t** perm,
                           const uint32_t** sorted_keys = nullptr);

// Store build kernels (build.cu).
cudaError_t launch_fold_rows(const float* Zsrc, int64_t rows, int R, const float* Mdev, float* Zc_dst, int Rp,
                             uint32_t* flags, cudaStream_t st);
cudaError_t launch_prefix_stats(const float* Xdev, const float* Ydev, int A, int R, int Rp, double* total,
                                float* minnz, uint32_t* flags, cudaStream_t st);
cudaError_t launch_range_table(const float* PXY, int A, int Rp, int u32, int W, float* DT, cudaStream_t st);
cudaError_t launch_prefix(const float* Xdev, const float* Ydev, int A, int R, int Rp, int u32, const int* exps,
                          void* table, cudaStream_t st);

}  // namespace pndf
