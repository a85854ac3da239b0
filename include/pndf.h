/*
 * pndf.h -- C ABI of the B200-native batched NDF range query
 * (Deng et al., "Constant-Cost Spatio-Angular Prefiltering of Glinty
 * Appearance Using Tensor Decomposition", arXiv 2109.14807).
 *
 * P:n below is line n of the paper's LaTeX; S:n of SPEC.md.
 *
 * What a query computes.  The method precomputes an NDF image for every
 * footprint centre of a mip-like pyramid -- level l has stride s0*2^l and
 * footprint sigma_p = 1.5 s/sqrt(12) -- and compresses the stack
 * with a rank-R CP decomposition  D-hat = sum_r C_r X_r (x) Y_r (x) Z_r  (Eq. 5,
 * P:298-303).  A query (footprint centre u,v; footprint size S; inclusive
 * angular rectangle [x1,x2] x [y1,y2] on the A x A projected-normal grid)
 * returns the trilinearly interpolated (4 spatial neighbours x 2 levels,
 * P:276) range MEAN of Eq. 6:
 *     sum_k w_k sum_r C_r Xbar_r([x1,x2]) Ybar_r([y1,y2]) Z_r(z_k)
 * or, with PNDF_SUM, the same without the 1/((x2-x1+1)(y2-y1+1)) factor.
 * The 1-D segment sums come from prefix sums, "strictly, 2 memory look-ups"
 * per factor.  Above the top level the size clamps; below
 * the base it clamps to level 0.  DESIGN.md §2 states every reading.
 *
 * All calls return pndf_status (0 = OK, < 0 = error) and are thread-safe for
 * distinct store handles.  One in-flight batch per store handle.
 */
#ifndef PNDF_H
#define PNDF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PNDF_ABI_VERSION 1u

typedef enum {
    PNDF_OK = 0,
    PNDF_EINVAL = -1,  /* bad argument (null pointer, bad descriptor, negative or non-finite factor, bad opts) */
    PNDF_ENOMEM = -2,  /* device or host allocation failed */
    PNDF_ECUDA = -3,   /* a CUDA runtime call failed (pndf_last_cuda_error() names it) */
    PNDF_EFORMAT = -4, /* ABI version mismatch */
    PNDF_EQUERY = -5   /* sticky, device-side: >= 1 record of a batch was invalid (its result is NaN) */
} pndf_status;

/* descriptor flags: border mode | SAT storage format */
#define PNDF_CLAMP 0u       /* neighbours clamp to the grid edge (non-tileable map) */
#define PNDF_WRAP 1u        /* neighbours wrap modulo the level grid (tileable map) */
#define PNDF_PREFIX_AUTO 0u /* U32 when it keeps every nonzero range sum within 2^-15 relative, else HILO */
#define PNDF_PREFIX_HILO 2u /* fp32 (hi, lo) pair of the fp64 prefix: 8 B/entry, ~1 ulp for any store */
#define PNDF_PREFIX_U32 4u  /* uint32 fixed point, per-rank power-of-two scale: 4 B/entry */
#define PNDF_PREFIX_MASK 6u

/* pndf_query_batch opts (OR together) */
#define PNDF_MEAN 0u      /* Eq. 6 average over the rectangle (default) */
#define PNDF_SUM 1u       /* rectangle integral (no division by the area) */
#define PNDF_BIN_AUTO 0u  /* bin queries by (level, tile) when the factor set exceeds L2 */
#define PNDF_BIN_ON 2u    /* always bin */
#define PNDF_BIN_OFF 4u   /* never bin */
#define PNDF_TIMING 8u    /* record CUDA events around each phase (read with pndf_store_stats) */

typedef struct pndf_store_s* pndf_store; /* opaque; factors immutable after load */

/* Store geometry.  Level l (0 <= l < L) has stride s_l = base_stride*2^l and an
 * n_l x n_l grid of footprint centres ((i+1/2)s_l, (j+1/2)s_l), n_l = map_size/s_l
 * (P:274-279).  Positional index z = off_l + j*n_l + i, off_l = sum_{m<l} n_m^2;
 * P = sum_l n_l^2 rows, P < 2^31. */
typedef struct {
    uint32_t abi_version; /* = PNDF_ABI_VERSION                                  */
    int32_t map_size;     /* N texels per side, power of two, <= 2^20            */
    int32_t base_stride;  /* s0, power of two dividing N                         */
    int32_t num_levels;   /* L, 2 <= L <= log2(N/s0) + 1, L <= 24                */
    int32_t ang_res;      /* A, 1 <= A <= 256 (rect bounds are 8-bit)            */
    int32_t rank;         /* R, 1 <= R <= 1024                                   */
    uint32_t flags;       /* PNDF_WRAP or PNDF_CLAMP, | PNDF_PREFIX_*            */
} pndf_desc;

/* One query record, 16 bytes, little-endian.
 *   u, v  footprint centre in texels; |u|,|v| <= 2^22 (wrapped or clamped to the map)
 *   size  footprint size S in texels (> 0); level l* = clamp(log2(S/s0), 0, L-1),
 *         so S = s_l selects level l; sigma_p = 1.5 S / sqrt(12)
 *   rect  x1 | x2<<8 | y1<<16 | y2<<24, inclusive bounds, x1 <= x2 < A, y1 <= y2 < A
 * Invalid records (non-finite fields, |u|,|v| > 2^22, size <= 0, bad bounds)
 * yield NaN and set the store's sticky error. */
typedef struct {
    float u, v, size;
    uint32_t rect;
} pndf_query;

/* Build a device store from raw CP factors (Eq. 5), synchronously.
 *   C [R] (NULL = all ones), X [A][R], Y [A][R]  -- host or device memory, fp32
 *   Z [P][R] level-major, rows j*n_l + i         -- host or device memory, fp32
 * Layout in HBM: Zc[P][Rp] = fl32(M_r Z_r(z)) with R padded to Rp
 * (zero ranks, rows 16-byte aligned); prefix sums of X, Y accumulated in fp64 and
 * stored either as an fp32 (hi, lo) pair [2][(A+1)][2][Rp] (HILO, M_r = C_r) or as
 * uint32 fixed point [2][(A+1)][Rp] with per-rank scale 2^e_r folded into
 * M_r = C_r 2^-(ex_r + ey_r) (U32); see the PNDF_PREFIX_* flags.  A range table
 * DT[2][A][W][Rp] fp32 (W = min(48, A)) holds, for every range of at most W bins, the
 * prefix difference exactly as the kernel computes it from the SATs, so a narrow range
 * costs one look-up per axis instead of two with bit-identical results.
 * Every factor must be finite and >= 0 (nonnegative store), else PNDF_EINVAL.
 * Inputs are copied: the caller may free them on return.  device = CUDA
 * ordinal; cuda_stream = cudaStream_t used for the build (NULL = default). */
pndf_status pndf_load_factors(const pndf_desc* desc, const float* C, const float* X, const float* Y,
                              const float* Z, int device, void* cuda_stream, pndf_store* out);

/* Enqueue one batch on cuda_stream and return immediately.
 *   d_queries [n] pndf_query, d_out [n] fp32 -- caller-owned DEVICE memory that
 *   must stay valid until pndf_sync; results land at out[i] for query i in the
 *   caller's order whether or not the batch is binned (bitwise identical either
 *   way).  n == 0 is a no-op.  Argument errors return synchronously. */
pndf_status pndf_query_batch(pndf_store s, const pndf_query* d_queries, int64_t n, float* d_out, uint32_t opts,
                             void* cuda_stream);

/* One importance sample (16 bytes): the projected half vector (hx, hy) in
 * [-1,1]^2, its density pdf = pmf / (2/A)^2 over the projected-h plane (the
 * pmf is the sampled pixel's mass over the domain's mass), and the pixel
 * x | y << 16.  No sample (blank domain, or invalid record): pixel = 0xffffffff,
 * hx = hy = NaN, pdf = 0 (NaN for an invalid record). */
typedef struct {
    float hx, hy, pdf;
    uint32_t pixel;
} pndf_sample;

/* Batched hierarchical importance sampling (Sec. 5.2; SURVEY §8(f)
 * row 1).  For record i (footprint u, v, size; rect = the sampling domain, the
 * whole A x A image for plain NDF sampling) descend from the domain by quads
 * chosen with probability proportional to their range sums (Eq. 6), one
 * variate xi[i][l] per level l (< 8 levels since A <= 256), down to a pixel,
 * then jitter inside it with xi[i][8], xi[i][9].  d_xi is DEVICE memory
 * [n][10] fp32 in [0,1), caller-supplied (any RNG); d_out [n] pndf_sample.
 * opts: PNDF_BIN_* (binning by footprint like pndf_query_batch), PNDF_TIMING.
 * Enqueued on cuda_stream; complete with pndf_sync.  Invalid records set the
 * sticky PNDF_EQUERY. */
pndf_status pndf_sample_batch(pndf_store s, const pndf_query* d_queries, const float* d_xi, int64_t n,
                              pndf_sample* d_out, uint32_t opts, void* cuda_stream);

/* One spherical-Gaussian light sample for environment prefiltering (Sec. 5.4),
 * 32 bytes: footprint (u, v, size) as in pndf_query, the projected half vector
 * (hx, hy) of the sampled lobe direction, the lobe's bandwidth lambda and
 * amplitude A (both > 0), padding. */
typedef struct {
    float u, v, size, hx, hy, lambda, amplitude, pad;
} pndf_sg_light;

/* Environment prefiltering rectangles: theta = arccos((ln eps - ln A)
 * / lambda + 1) (arccos argument clamped to [-1, 1]), side Q = ang_res theta/pi
 * rounded to the nearest integer in [1, ang_res], square centred on the bin of
 * (hx, hy) and shifted inside the grid; d_out[i] = {u, v, size, rect} ready for
 * pndf_query_batch (the paper uses eps = 0.3).  d_in, d_out DEVICE memory; enqueued
 * on cuda_stream.  Invalid lights (non-finite, lambda or A <= 0) get an invalid
 * rectangle, which the query batch turns into NaN + PNDF_EQUERY. */
pndf_status pndf_sg_queries(const pndf_sg_light* d_in, int64_t n, float eps, int32_t ang_res, pndf_query* d_out,
                            void* cuda_stream);

/* Block until the store's work on cuda_stream is done; returns and clears the
 * sticky per-record error (PNDF_EQUERY) or a CUDA error. */
pndf_status pndf_sync(pndf_store s, void* cuda_stream);

/* End-to-end variant: HOST records in, HOST results out.  Streams the batch
 * through the device in chunks (H2D copy, binning + query kernels, D2H copy
 * overlapped on three internal streams) and returns when h_out is complete.
 * Pinned (page-locked) host buffers give full PCIe bandwidth; pageable ones
 * work but serialise the copies.  Returns the sticky error like pndf_sync. */
pndf_status pndf_query_batch_host(pndf_store s, const pndf_query* h_queries, int64_t n, float* h_out,
                                  uint32_t opts);

/* Release the store and all device memory it owns. NULL is a no-op. */
pndf_status pndf_free(pndf_store s);

const char* pndf_error_string(pndf_status status);
const char* pndf_last_cuda_error(void); /* text of the last failing CUDA call on this thread */
uint32_t pndf_abi_version(void);

/* Introspection (tests / bench). */
typedef struct {
    int64_t rows;             /* P                                              */
    int32_t rank_padded;      /* Rp                                             */
    int32_t lanes_per_query;  /* G: lanes of a warp that share one query        */
    int64_t zc_bytes;         /* bytes of Zc                                    */
    int64_t prefix_bytes;     /* bytes of PX + PY                               */
    uint64_t kernel_launches; /* kernels this store has launched so far         */
    uint64_t timed_batches;   /* batches run with PNDF_TIMING since the last reset */
    double query_ms;          /* summed query-kernel time of those batches      */
    double bin_ms;            /* summed binning time of those batches           */
    int32_t last_binned;      /* 1 if the last batch was binned                 */
    int32_t prefix_format;    /* 0 = HILO, 1 = U32                              */
    int64_t range_table_bytes;/* bytes of the narrow-range difference table DT  */
    int32_t range_table_width;/* W: ranges of <= W bins read one DT row (0 = no table) */
    int32_t tile_reach;       /* tiled stores: cells beyond a tile holding a nonzero row (else 0) */
} pndf_store_stats;
pndf_status pndf_store_stats_get(pndf_store s, pndf_store_stats* out);
pndf_status pndf_store_stats_reset(pndf_store s);

/* Copy the device store image to host memory (tests): PXY = prefix_bytes of the
 * SAT tables (HILO [2][(A+1)][2][Rp] fp32, or U32 [2][(A+1)][Rp] uint32), Zc rows
 * [z0, z1) as [z1-z0][Rp] fp32.  Either pointer may be NULL. */
pndf_status pndf_store_image(pndf_store s, float* PXY, float* Zc, int64_t z0, int64_t z1);

/* Implicit Wang tiling (Sec. 5.5).  16 tiles of
 * T x T texels share the angular factors X, Y (and C); tile t has its own
 * positional factors over an EXTENDED centre grid: level l has n_l = T/(s0 2^l)
 * cells plus `margin` cells on each side (centres outside the tile), rows
 * z = t*P_ext + off_l + (j+margin)(n_l+2 margin) + (i+margin), off_l the sum of the
 * earlier levels' (n+2 margin)^2, P_ext the per-tile total; each row holds the
 * tile's PARTIAL footprint NDF (its own texels, normalised by the footprint's full
 * weight).  World cell (cx, cy) uses the tile whose edge colours come from the
 * vertex hash splitmix64(splitmix64(seed) ^ (uint32 vx | uint32 vy << 32)) --
 * bit 0 = colour of the vertex's right edge, bit 1 = of its bottom edge; tile id =
 * N | E<<1 | S<<2 | W<<3.  A query on a tiled store sums the
 * contributions of every tile whose extended grid holds each of its 8 neighbours
 * ("combining the precomputed NDF images from all overlapping Wang tiles",
 * P:440).  World coordinates are not periodic; |u|,|v| <= 2^22. */
typedef struct {
    uint32_t abi_version; /* = PNDF_ABI_VERSION                                    */
    int32_t tile_size;    /* T, power of two                                       */
    int32_t base_stride;  /* s0, power of two dividing T                           */
    int32_t num_levels;   /* L, 2 <= L <= log2(T/s0) + 1                           */
    int32_t margin;       /* extended cells per side, >= 2 (covers the +-4 sigma support) */
    int32_t ang_res;      /* A                                                     */
    int32_t rank;         /* R                                                     */
    uint32_t flags;       /* PNDF_PREFIX_* (border flags ignored)                  */
    uint64_t seed;        /* vertex-hash seed                                      */
} pndf_tile_desc;

/* Build a tiled store (Z = [16 * P_ext][R], other arguments as pndf_load_factors).
 * The load measures the store's reach: the largest distance (in cells of its
 * level, beyond the tile's own n_l x n_l cells) of any row with a nonzero entry,
 * 0 <= reach <= margin (pndf_store_stats.tile_reach).  Rows further out are all
 * zero, so the kernels skip them and the sum over every tile whose extended grid
 * holds a neighbour stays exact for any margin.
 * pndf_query_batch / pndf_query_batch_host answer world-space queries on it;
 * they are not binned by cell, but device batches of >= 65536 records are first
 * sorted by footprint level (one stable radix pass; results bitwise identical to
 * the caller's order, which PNDF_BIN_OFF keeps, and which the host entry
 * pndf_query_batch_host always uses).  A batch captured into a CUDA graph before
 * the store has sort scratch for its size runs unsorted.  pndf_sample_batch
 * returns PNDF_EINVAL for tiled stores (use pndf_sample_tiles). */
pndf_status pndf_load_tiles(const pndf_tile_desc* desc, const float* C, const float* X, const float* Y,
                            const float* Z, int device, void* cuda_stream, pndf_store* out);

/* Importance sampling over implicit Wang tiles (Sec. 5.5: "we first
 * choose one Wang tile from all the Wang tiles covered by the pixel footprint
 * with equal probability.  Then, we sample a direction from the chosen Wang
 * tile ... The PDF is set the same as NDF value"; reading 25).
 * s must be a tiled store (else PNDF_EINVAL).  Record i as in pndf_sample_batch
 * (world footprint; rect = the sampling domain).  The covered tile instances
 * are the world cells (tx, ty) holding a row the tiled query reads with
 * positive weight and positive domain mass (a neighbour within `reach` cells
 * of the tile; PNDF_EINVAL if the store's reach exceeds 4), ordered by
 * (ty, tx); the c-th is chosen with c = floor(xi[i][10] * count) (fp32),
 * then the hierarchical descent of pndf_sample_batch runs on that tile's
 * partial NDF with xi[i][0..7] and jitters with xi[i][8], xi[i][9].  pdf is
 * the FULL (all-tile) NDF's mass in the sampled pixel over its mass in the
 * domain, per unit projected-h area (pmf / (2/A)^2).  No sample (chosen tile
 * blank on the domain): pixel = 0xffffffff, pdf = 0.
 *   d_xi   DEVICE [n][11] fp32 in [0,1), caller-supplied
 *   d_out  DEVICE [n] pndf_sample
 *   d_tile DEVICE [n][2] int32 (tx, ty) of the chosen instance, or NULL
 * opts: PNDF_TIMING; PNDF_BIN_OFF keeps the caller's order (by default batches
 * of >= 65536 records are first sorted by footprint level -- a stable 8-bit
 * radix pass -- so the lanes of a warp sample footprints of one size; results
 * land at out[i] for record i either way, bitwise identical).  Enqueued on
 * cuda_stream; complete with pndf_sync; invalid records give NaN + the sticky
 * PNDF_EQUERY. */
pndf_status pndf_sample_tiles(pndf_store s, const pndf_query* d_queries, const float* d_xi, int64_t n,
                              pndf_sample* d_out, int32_t* d_tile, uint32_t opts, void* cuda_stream);

/* Blocked / clustered store (Sec. 4.2).  Each
 * A x A NDF image is cut into t x t angular blocks; the blocks of footprints
 * centred in the same spatial region (side `region` texels: centre
 * ((i+1/2)s, (j+1/2)s) is in region (floor(cx/region), floor(cy/region)))
 * form a group g = region_index * nb^2 + block (nb = A/t) with its own CP
 * factors; blank blocks are pruned.  A query sums,
 * over its 8 trilinear neighbours and over every block its rectangle overlaps
 * (the range is split on block boundaries), Eq. 6 on the sub-rectangle
 * with that block's group factors -- so the angular SAT rows are fetched per
 * neighbour, as in the paper.  Inputs (host or device, copied):
 *   C [num_sets][R], X [num_sets][t][R], Y [num_sets][t][R]  factor sets
 *   group_set [(N/region)^2 * nb^2] int32   factor set of each group (-1 = empty)
 *   slab_ptr  [P][nb^2] int64               Z row of (positional row, block), -1 = blank
 *   Z [num_slabs][R]                          per-slab positional factors
 * SATs are stored in the HILO format.  pndf_query_batch answers queries on it
 * (never binned); pndf_sample_blocked samples it (block choice + descent);
 * pndf_sample_batch returns PNDF_EINVAL. */
typedef struct {
    uint32_t abi_version; /* = PNDF_ABI_VERSION                                   */
    int32_t map_size;     /* N                                                    */
    int32_t base_stride;  /* s0                                                   */
    int32_t num_levels;   /* L                                                    */
    int32_t ang_res;      /* A, a multiple of block                              */
    int32_t block;        /* t, 1 <= t <= 64                                      */
    int32_t region;       /* spatial region side in texels, power of two, <= N   */
    int32_t rank;         /* R (per group)                                        */
    uint32_t flags;       /* PNDF_WRAP or PNDF_CLAMP                             */
    int32_t num_sets;     /* factor sets                                          */
    int64_t num_slabs;    /* rows of Z, < 2^31                                    */
} pndf_block_desc;

pndf_status pndf_load_blocked(const pndf_block_desc* desc, const float* C, const float* X, const float* Y,
                              const int32_t* group_set, const int64_t* slab_ptr, const float* Z, int device,
                              void* cuda_stream, pndf_store* out);

/* Importance sampling on a blocked / clustered store (pndf_load_blocked; Sec. 5.2; SURVEY §8(f)
 * rows 1 x 2): "we first choose an image block to start, again according to their averaged NDF values"
 * -- each t x t angular block of the record's rectangle is weighted by its Eq. 6 SUM over the part
 * of the rectangle inside it, blended over the footprint's 8 neighbours with their own groups' factors;
 * xi[i][10] picks the first block whose cumulative weight exceeds xi x total -- then the quad descent of
 * pndf_sample_batch runs inside that block (xi[i][0..], jitter xi[i][8], xi[i][9]).  pdf = the pixel's
 * share of the rectangle's mass / pixel area (block pmf x descent pmf).  Choice rules: DESIGN.md reading 26.
 *   d_xi    DEVICE [n][11] fp32 in [0,1)
 *   d_out   DEVICE [n] pndf_sample (NaN + sticky PNDF_EQUERY for invalid records; pixel 0xffffffff and
 *           pdf 0 when the rectangle holds no mass)
 *   d_block DEVICE [n] int32 chosen block by * nb + bx (-1 = none), or NULL
 * opts: PNDF_TIMING.  Enqueued on cuda_stream; complete with pndf_sync.  EINVAL on other store kinds. */
pndf_status pndf_sample_blocked(pndf_store s, const pndf_query* d_queries, const float* d_xi, int64_t n,
                                pndf_sample* d_out, int32_t* d_block, uint32_t opts, void* cuda_stream);

/* Test support: run only the binning pass (row a1) on n device records and copy
 * the permutation (query indices in binned order) to d_perm [n] and, if not
 * NULL, the sorted bin keys to d_keys [n] (device memory).  Synchronous. */
pndf_status pndf_bin_permutation(pndf_store s, const pndf_query* d_queries, int64_t n, uint32_t* d_perm,
                                 uint32_t* d_keys);

/* Measurement support (bench.py roofline): *d_rows_out (device int64) = the number of
 * DISTINCT Zc rows that the query kernel reads for the n device records, i.e. the 8 trilinear
 * neighbours of each valid record (the kernel loads all 8 even at zero weight).  Multiplied by
 * Rp x 4 B this is the batch's compulsory Zc traffic from HBM.  Global stores only (EINVAL for tiled or
 * blocked stores).  Scratch: a P-bit bitmap allocated and freed inside the call.  Synchronous. */
pndf_status pndf_rows_touched(pndf_store s, const pndf_query* d_queries, int64_t n, int64_t* d_rows_out);

/* Tuning knob (bench / tests): lanes per query G in {1,2,4,8,16,32} with
 * G*4 dividing Rp; 0 restores the default chosen at load. */
pndf_status pndf_set_lanes(pndf_store s, int32_t lanes);

/* ---- GPU factor builder ----------------------------------------------
 * The tensor the paper compresses (footprint NDF images stacked along the third dimension) and its
 * CP decomposition by alternating least squares (Eq. 5: "maximum error 1e-4, maximum
 * iteration count 500"), for ONE global group (readings 14, 23).  Limits: A a power of two,
 * 32 <= A <= 128, 1 <= R <= 128, N <= 32768, P * A < 2^31.  All pointers are DEVICE memory; calls enqueue on cuda_stream
 * and pndf_cp_als synchronises once per sweep (to test the stopping rule).
 *
 * pndf_hist_tensor: D[z][x][y] = tf32(count / total) -- the footprint-weighted histogram of the map's
 *   angular bins over footprint z (Eq. 2 with sigma_r -> 0; Gaussian G_p, sigma = 1.5 s_l / sqrt(12),
 *   truncated at 4 sigma, 16-bit integer weights, exact integer counts: DESIGN.md reading 11), rounded to
 *   nearest-even at 11 significant bits (reading 23).  Rows z = off_l + j n_l + i (periodic map, PNDF_WRAP
 *   required).  d_bins [N][N] uint16: bin x + A*y of texel (u, v) at d_bins[v*N + u].  d_D [P][A][A] and
 *   d_Dt [P][A][A] (= D with x, y swapped; may be NULL) are caller-allocated fp32.
 * pndf_cp_als: nonnegative CP-ALS (HALS column updates, modes Z, X, Y, per-rank norm balance after each
 *   sweep) of D from the caller's initial factors (in/out, fp32, >= 0): d_Z [P][R], d_X [A][R], d_Y [A][R].
 *   Stops after the first sweep whose relative fit-error change is < tol, or after max_sweeps.  With
 *   PNDF_ALS_NORMALISE the result is normalised (unit-sum X_r, Y_r, max_z Z_r = 1, C_r the weight, every
 *   row's reconstructed mass 1; reading 16) and d_C [R] is written (else d_C, if not NULL, is set to 1).
 *   h_err [max_sweeps] (host, may be NULL) receives the fit error ||D - D_hat|| / ||D|| after each sweep;
 *   *sweeps_out the number of sweeps run.  The MTTKRP of each mode runs on the tensor cores (tcgen05,
 *   kind::tf32, D exact in tf32, the factor operand split into tf32 hi + lo parts).
 * pndf_mttkrp (test support): one MTTKRP, mode 0 = Z ([P][R] = D_(z) (X kr Y)), 1 = X ([A][R]),
 *   2 = Y ([A][R]), into d_M (fp64). */
#define PNDF_ALS_NORMALISE 1u
typedef struct {
    uint32_t abi_version; /* = PNDF_ABI_VERSION                                  */
    int32_t max_sweeps;   /* >= 1 (500)                                   */
    double tol;           /* relative change of the fit error (1e-4)      */
    uint32_t flags;       /* PNDF_ALS_NORMALISE                                  */
} pndf_als_opts;

pndf_status pndf_hist_tensor(const pndf_desc* desc, const uint16_t* d_bins, float* d_D, float* d_Dt,
                             void* cuda_stream);
pndf_status pndf_cp_als(const pndf_desc* desc, const float* d_D, const float* d_Dt, float* d_C, float* d_X,
                        float* d_Y, float* d_Z, const pndf_als_opts* opts, double* h_err, int32_t* sweeps_out,
                        void* cuda_stream);
pndf_status pndf_mttkrp(const pndf_desc* desc, const float* d_D, const float* d_Dt, const float* d_Z,
                        const float* d_X, const float* d_Y, int32_t mode, double* d_M, void* cuda_stream);

/* ---- Map-domain factor builder (no tensor in memory; configs 3-4 scale) -------------------------------
 * The same nonnegative CP-ALS as pndf_cp_als (HALS, modes Z, X, Y, norm balance, stopping rule, normalise),
 * of the EXACT footprint tensor D = count / total (no tf32 rounding), but D is never formed: it is a
 * separable Gaussian blur of the texels' one-hot angular histograms (Eq. 2), so each MTTKRP
 * contracts over the N x N texels (fp64, ~3.5 N^2 L R FMAs per mode) instead of over P x A x A entries --
 * e.g. config 3 (P = 5.6M, A = 128) would need a 366 GB tensor.  ||D||^2 comes from exact integer bin
 * counts per footprint window.  Limits: periodic map (PNDF_WRAP), A a power of two <= 256, R <= 256, and
 * device memory for Z, M_Z (P x R fp64 each) plus two N^2 x R fp64 pass buffers; PNDF_ENOMEM otherwise.
 * d_bins [N][N] uint16 as for pndf_hist_tensor; factors, opts, h_err, sweeps_out as for pndf_cp_als.
 * Results are reproducible up to the order of fp64 shared-memory atomics in the X / Y modes.
 * pndf_mttkrp_map (test support): one MTTKRP (mode 0 = Z [P][R], 1 = X [A][R], 2 = Y [A][R]) into d_M
 * (fp64, device) and, if h_sumsq is not NULL, ||D||^2 into *h_sumsq.  Synchronous. */
pndf_status pndf_cp_als_map(const pndf_desc* desc, const uint16_t* d_bins, float* d_C, float* d_X, float* d_Y,
                            float* d_Z, const pndf_als_opts* opts, double* h_err, int32_t* sweeps_out,
                            void* cuda_stream);
pndf_status pndf_mttkrp_map(const pndf_desc* desc, const uint16_t* d_bins, const float* d_Z, const float* d_X,
                            const float* d_Y, int32_t mode, double* d_M, double* h_sumsq, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* PNDF_H */
