// internal.cuh -- device-side data structures shared by the pndf kernels.
//
// Store layout in HBM:
//   Zc  [P][Rp]               fp32, Zc[z][r] = fl32(M_r * Z_r(z)), ranks >= R are 0,
//                             rows 16-byte aligned (Rp % 4 == 0); M_r = C_r (HILO) or
//                             C_r 2^-(ex_r+ey_r) (U32)
//   PXY [2][A+1][2][Rp] fp32  HILO: table 0 = X, 1 = Y; entry k holds the prefix
//                             sum_{i<k} X_r(i) accumulated in fp64 and split into
//                             hi = fl32(S), lo = fl32(S - hi)  ("1D SAT")
//   or  [2][A+1][Rp]   uint32 U32: round(S 2^e_r), see build.cu
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "pndf.h"

namespace pndf {

constexpr int kMaxLevels = 24;
#ifndef PNDF_QTHREADS
#define PNDF_QTHREADS 256
#endif
constexpr int kThreads = PNDF_QTHREADS;  // query-kernel block size

struct QParams {
    const float* Zc;
    const float* PXY;
    uint32_t* err;                 // sticky error word (bit 0: invalid record)
    int64_t level_off[kMaxLevels]; // off_l = sum_{m<l} n_m^2
    int32_t N;                     // map side
    int32_t n0;                    // level-0 grid side N/s0
    int32_t L;                     // levels
    int32_t A;                     // angular resolution
    int32_t Rp;                    // padded rank
    int32_t wrap;                  // 1 = periodic neighbours
    int32_t prefix_u32;            // 1 = uint32 fixed-point SATs (PQ[2][A+1][Rp]), 0 = fp32 (hi, lo)
    float inv_s0;                  // 1/s0 (power of two, exact)
    uint32_t mean;                 // 1 = divide by the rectangle area
    const float* DT;               // range table [2][A][W][Rp]: DT[axis][x1][w-1] = the SAT difference of
                                   // [x1, x1+w) exactly as the query kernel computes it (NULL = none)
    int32_t dt_w;                  // W: widest range served by DT (0 = none)
    const CUtensorMap* dt_tmap;    // HOST pointer: 2-D tensor map of DT ([rows][Rp], box {Rp, 1}) for the
                                   // gather4 bulk copies of query_g4_kernel (NULL = none); not read on device
};

// Implicit Wang tiling (tiles.cu).
struct TileParams {
    int32_t T;        // tile size (texels)
    int32_t margin;   // extended cells per side
    int64_t p_ext;    // rows per tile
    uint64_t seed;    // vertex-hash seed
    int32_t reach;    // cells beyond the tile border that hold a nonzero row (<= margin), measured at
                      // load: rows further out are all zero, so skipping them is exact
};

// Blocked / clustered store (blocks.cu).
struct BlockParams {
    int32_t t;                  // angular block side
    int32_t nb;                 // blocks per axis (A / t)
    int32_t region;             // spatial region side (texels)
    int32_t nr;                 // regions per axis (N / region)
    const int32_t* slab_ptr;    // [P][nb^2] Zc row or -1
    const int32_t* group_set;   // [nr^2 * nb^2] factor set or -1
    int32_t r_shift;            // log2 region (a power of two)
};

// Device scratch of one in-flight binned batch (radix sort double buffers).
struct BinScratch {
    uint32_t* keys[2] = {nullptr, nullptr};
    uint32_t* vals[2] = {nullptr, nullptr};
    uint32_t* counts = nullptr;  // radix_tiles(cap) * 256 digit counts / offsets
    uint32_t* bsum = nullptr;    // scan block sums
    int64_t cap = 0;
};

}  // namespace pndf
