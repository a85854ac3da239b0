// query.cu -- sm_100a kernels of the batched NDF range query (the hot path).
//
// Rows of SURVEY.md §8(a) implemented here:
//   a1  query binning        bin_keys_kernel + LSD radix sort (rs_hist/scan/rs_scatter)
//   a2  decode + level select  decode()
//   a3  spatial neighbours     decode()
//   a4  positional gather + interpolation  query_kernel: 8 rows of Zc, float4 per lane
//   a5  angular prefix differencing        query_kernel: 4 SAT rows, (hi,lo) fp32 or u32 fixed point
//   a6  rank product + reduce + write      query_kernel: Eq. 6, xor-shuffle
//                                          reduction over the G lanes of a query
// This is a gather-and-reduce (~11 flop per rank per query), bound by the memory
// system, so there are no tensor cores here.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "internal.cuh"
#include "device.cuh"
#include "launch.h"

namespace pndf {

bool lanes_supported(int G, int NV) {
    const bool g = (G == 1 || G == 2 || G == 4 || G == 8 || G == 16 || G == 32);
    const bool v = (NV == 1 || NV == 2 || NV == 3 || NV == 4 || NV == 8);
    return g && v;
}

bool g5_disabled() {
    static const int v = [] {
        const char* e = getenv("PNDF_NOG5");
        return (e && atoi(e) != 0) ? 1 : 0;
    }();
    return v != 0;
}

int64_t g5_chunk() {
    static const int64_t v = [] {
        const char* e = getenv("PNDF_G5CHUNK");
        int64_t c = e ? atoll(e) : 16384;
        if (c < 256) c = 256;
        return c / 256 * 256;
    }();
    return v;
}

bool g5_rot() {
    static const int v = [] {
        const char* e = getenv("PNDF_G5ROT");
        return (e && atoi(e) == 0) ? 0 : 1;
    }();
    return v != 0;
}

bool g4_disabled() {
    static const int v = [] {
        const char* e = getenv("PNDF_NOG4");
        return (e && atoi(e) != 0) ? 1 : 0;
    }();
    return v != 0;
}

cudaError_t launch_query(const QParams& p, int G, int NV, const pndf_query* q, const uint32_t* idx, int64_t n,
                         float* out, int num_sms, cudaStream_t st) {
    if (4 * G * NV != p.Rp) return cudaErrorInvalidValue;
    if (p.prefix_u32)
        return p.wrap ? launch_query_u32_wrap(G, NV, p, q, idx, n, out, num_sms, st)
                      : launch_query_u32_clamp(G, NV, p, q, idx, n, out, num_sms, st);
    return p.wrap ? launch_query_hilo_wrap(G, NV, p, q, idx, n, out, num_sms, st)
                  : launch_query_hilo_clamp(G, NV, p, q, idx, n, out, num_sms, st);
}

// -------------------------------------------------------- rows touched --
// Measurement helper: mark the 8 neighbour rows of each valid record (a2/a3 exactly as the query
// kernel decodes them), then count the marked bits.
template <bool WRAP>
__global__ void mark_rows_kernel(const QParams p, const pndf_query* __restrict__ q, int64_t n,
                                 uint32_t* __restrict__ bitmap) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const pndf_query rec = ldg_query(q + i);
        int x1, x2, y1, y2;
        if (!record_valid(p, rec, x1, x2, y1, y2)) continue;
        int l0;
        float t;
        level_select(p, rec.size, l0, t);
        for (int dl = 0; dl < 2; ++dl) {
            const int l = l0 + dl;
            int i0, i1, j0, j1;
            float a, b;
            axis_cells<WRAP>(p, rec.u, l, i0, i1, a);
            axis_cells<WRAP>(p, rec.v, l, j0, j1, b);
            const int64_t nl = p.n0 >> l, off = level_offset(p.n0, l);
            const int64_t rows[4] = {off + j0 * nl + i0, off + j0 * nl + i1, off + j1 * nl + i0, off + j1 * nl + i1};
            for (int k = 0; k < 4; ++k) {
                const uint32_t bit = 1u << (rows[k] & 31);
                uint32_t* w = bitmap + (rows[k] >> 5);
                if (!(*w & bit)) atomicOr(w, bit);
            }
        }
    }
}

__global__ void popcount_kernel(const uint32_t* __restrict__ bitmap, int64_t words, int64_t* count) {
    int64_t c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
        c += __popc(bitmap[i]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(reinterpret_cast<unsigned long long*>(count), (unsigned long long)c);
}

cudaError_t launch_rows_touched(const QParams& p, const pndf_query* q, int64_t n, int64_t P, uint32_t* bitmap,
                                int64_t* count, int num_sms, cudaStream_t st) {
    const unsigned grid = (unsigned)num_sms * 8;
    if (n > 0) {
        if (p.wrap)
            mark_rows_kernel<true><<<grid, 256, 0, st>>>(p, q, n, bitmap);
        else
            mark_rows_kernel<false><<<grid, 256, 0, st>>>(p, q, n, bitmap);
    }
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int64_t), st);
    if (e != cudaSuccess) return e;
    popcount_kernel<<<grid, 256, 0, st>>>(bitmap, (P + 31) / 32, count);
    return cudaGetLastError();
}

// ------------------------------------------------------------ binning --
// a1: key = the record's half cell on its lower level l0 (Z-order within the
// level), so queries that share all 8 Zc rows get equal keys and queries that
// share some rows get nearby keys.  Invalid records -> the last key.
// The permutation comes from a stable LSD radix sort (8- or 9-bit digits):
//   rs_hist_kernel     per-tile digit histograms, digit-major in global memory
//   scan_*_kernel      exclusive scan of the histograms -> each tile's digit offsets
//   rs_scatter_kernel  stable tile-local ranking (match_any + per-warp counts),
//                      staged in shared memory, written out digit run by run.
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// Block-wide exclusive scan of kScanTile items; returns the block total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t (&v)[kScanItems], uint32_t* smem_warp) {
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t x = v[k];
        v[k] = s;
        s += x;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) smem_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint32_t wv = smem_warp[lane];
        uint32_t wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        smem_warp[lane] = wi - wv;  // exclusive warp offsets
        if (lane == 31) smem_warp[32] = wi;
    }
    __syncthreads();
    const uint32_t off = smem_warp[wid] + (incl - s);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] += off;
    const uint32_t total = smem_warp[32];
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in, int64_t nb,
                                                                   uint32_t* bsum) {
    __shared__ uint32_t red[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < nb) s += in[base + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = red[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) bsum[blockIdx.x] = s;
    }
}

// single block: exclusive scan of the block sums in place
__global__ void __launch_bounds__(kScanThreads) scan_bsum_kernel(uint32_t* bsum, int64_t nblk) {
    __shared__ uint32_t sw[33];
    uint32_t carry = 0;
    for (int64_t t0 = 0; t0 < nblk; t0 += kScanTile) {
        uint32_t v[kScanItems];
        const int64_t base = t0 + (int64_t)threadIdx.x * kScanItems;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = (base + k < nblk) ? bsum[base + k] : 0u;
        const uint32_t tot = block_exclusive_scan(v, sw);
#pragma unroll
        for (int k = 0; k < kScanItems; ++k)
            if (base + k < nblk) bsum[base + k] = v[k] + carry;
        carry += tot;
    }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(uint32_t* inout, int64_t nb,
                                                                  const uint32_t* __restrict__ bsum) {
    __shared__ uint32_t sw[33];
    uint32_t v[kScanItems];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = (base + k < nb) ? inout[base + k] : 0u;
    block_exclusive_scan(v, sw);
    const uint32_t off = bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < nb) inout[base + k] = v[k] + off;
}

#ifndef PNDF_RS_ATOMIC
#define PNDF_RS_ATOMIC 1  // radix scatter ranking: 1 = leader atomics (pipelined rounds), 0 = load/store counters
#endif
constexpr int kRsThreads = 256;
#ifndef PNDF_RS_ITEMS
#define PNDF_RS_ITEMS 28  // keys per thread of a radix tile (256 threads): 7168-key tiles, 2 CTAs per SM (config 5 binning: 16 -> 28.9 ms, 24 -> 28.3, 28 -> 26.5, 32 -> 27.0, 36 -> 31.7)
#endif
#ifndef PNDF_RS_MINB
#define PNDF_RS_MINB 2
#endif
constexpr int kRsItems = PNDF_RS_ITEMS;
constexpr int kRsTile = kRsThreads * kRsItems;  // 7168 keys per tile
constexpr int kRsWarps = kRsThreads / 32;

// counts[d * ntiles + tile] = #keys of the tile whose digit is d (digits of BITS bits).
// Keys are read as uint4 (4 per load, all 4 loads of a thread in flight) and
// counted into two sub-histograms (even / odd warps) to halve atomic contention.
template <int BITS>
__global__ void __launch_bounds__(kRsThreads) rs_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                             uint32_t* counts, int64_t ntiles) {
    constexpr int RADIX = 1 << BITS;
    __shared__ uint32_t h[2][RADIX];
    for (int d = threadIdx.x; d < 2 * RADIX; d += kRsThreads) h[d / RADIX][d % RADIX] = 0;
    __syncthreads();
    uint32_t* hw = h[(threadIdx.x >> 5) & 1];
    const int64_t t0 = (int64_t)blockIdx.x * kRsTile;
    if (t0 + kRsTile <= n) {
        const uint4* k4 = reinterpret_cast<const uint4*>(keys + t0);
        uint4 v[kRsItems / 4];
#pragma unroll
        for (int i = 0; i < kRsItems / 4; ++i) v[i] = __ldg(k4 + i * kRsThreads + threadIdx.x);
#pragma unroll
        for (int i = 0; i < kRsItems / 4; ++i) {
            atomicAdd(&hw[(v[i].x >> shift) & (RADIX - 1)], 1u);
            atomicAdd(&hw[(v[i].y >> shift) & (RADIX - 1)], 1u);
            atomicAdd(&hw[(v[i].z >> shift) & (RADIX - 1)], 1u);
            atomicAdd(&hw[(v[i].w >> shift) & (RADIX - 1)], 1u);
        }
    } else {
        for (int i = 0; i < kRsItems; ++i) {
            const int64_t k = t0 + (int64_t)i * kRsThreads + threadIdx.x;
            if (k < n) atomicAdd(&hw[(__ldg(keys + k) >> shift) & (RADIX - 1)], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RADIX; d += kRsThreads) counts[(int64_t)d * ntiles + blockIdx.x] = h[0][d] + h[1][d];
}

// a1 keys fused with the first radix pass's tile histogram: block b computes
// the keys of radix tile b (kRsTile records) and counts their lowest digit.
template <int BITS>
__global__ void __launch_bounds__(kRsThreads) bin_keys_kernel(const QParams p, const pndf_query* __restrict__ q,
                                                              int64_t n, uint32_t* keys, uint32_t invalid_key,
                                                              int half, uint32_t* counts, int64_t ntiles) {
    constexpr int RADIX = 1 << BITS;
    __shared__ uint32_t h[RADIX];
    for (int d = threadIdx.x; d < RADIX; d += kRsThreads) h[d] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * kRsTile;
    constexpr int B = 4;  // records in flight per thread
    for (int i0 = 0; i0 < kRsItems; i0 += B) {
        pndf_query rec[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int64_t k = t0 + (int64_t)(i0 + b) * kRsThreads + threadIdx.x;
            if (k < n) rec[b] = ldg_query(q + k);
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int64_t k = t0 + (int64_t)(i0 + b) * kRsThreads + threadIdx.x;
            if (k >= n) continue;
            int x1, x2, y1, y2;
            uint32_t key = invalid_key;
            if (record_valid(p, rec[b], x1, x2, y1, y2)) {
                int l0;
                float t;
                level_select(p, rec[b].size, l0, t);
                key = cell_key(p, rec[b], l0, half);
            }
            keys[k] = key;
            atomicAdd(&h[key & (RADIX - 1)], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RADIX; d += kRsThreads) counts[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

// Stable scatter of one tile.  Warp w owns the contiguous segment
// [w*IPW, (w+1)*IPW) of the tile (IPW = 512 items, read 32 at a time, so the
// global loads stay coalesced).  Each warp ranks its segment against its own
// digit counters in shared memory (match_any + popc, rounds in order), so the
// ranking needs no block barrier; one scan over (digit, warp) afterwards turns
// the per-warp counts into offsets.  An item's tile-local position is
//   start[d] + (items of digit d in earlier warps) + (its rank inside its warp),
// which keeps the sort stable.  The tile is staged in shared memory in digit
// order, then written out so that consecutive items of a digit run go to
// consecutive global addresses.
template <int BITS, int THREADS, bool LATE_V>
__global__ void __launch_bounds__(THREADS, THREADS >= 512 ? 1 : PNDF_RS_MINB) rs_scatter_kernel(const uint32_t* __restrict__ keys_in,
                                                                const uint32_t* __restrict__ vals_in, int64_t n,
                                                                int shift, const uint32_t* __restrict__ offsets,
                                                                int64_t ntiles, uint32_t* keys_out,
                                                                uint32_t* vals_out) {
    constexpr int RADIX = 1 << BITS;
    constexpr int ITEMS = kRsTile / THREADS;  // items per thread
    constexpr int WARPS = THREADS / 32;
    constexpr int DPL = RADIX / 32;           // digits per lane in the tile scan
    constexpr int IPW = kRsTile / WARPS;      // items per warp segment
    extern __shared__ uint32_t rs_smem[];  // rs_smem_bytes<BITS>() of dynamic shared memory
    uint32_t* s_keys = rs_smem;                                      // [kRsTile]
    uint32_t* s_vals = s_keys + kRsTile;                             // [kRsTile]
    uint32_t(*s_cnt)[RADIX] = reinterpret_cast<uint32_t(*)[RADIX]>(s_vals + kRsTile);  // [WARPS][RADIX]
    uint32_t* s_run = s_vals + kRsTile + WARPS * RADIX;  // tile histogram
    uint32_t* s_start = s_run + RADIX;                      // tile-local start of each digit run
    uint32_t* s_goff = s_start + RADIX;                     // global start minus tile-local start
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t t0 = (int64_t)blockIdx.x * kRsTile;
    const int nt = (int)((n - t0) < (int64_t)kRsTile ? (n - t0) : (int64_t)kRsTile);
    const int seg = warp * IPW + lane;  // tile-local index of item 0 of this lane

    // this tile's global run starts (one strided 4-byte load per digit): fetched now by every thread so
    // their latency hides behind the key loads instead of sitting in warp 0's scan between two barriers
    uint32_t goff_r[(RADIX + THREADS - 1) / THREADS];
#pragma unroll
    for (int j = 0; j < (RADIX + THREADS - 1) / THREADS; ++j) {
        const int d = t + j * THREADS;
        goff_r[j] = d < RADIX ? __ldg(offsets + (int64_t)d * ntiles + blockIdx.x) : 0u;
    }
    uint32_t k[ITEMS], v[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int64_t g = t0 + seg + i * 32;
        const bool ok = seg + i * 32 < nt;
        k[i] = ok ? __ldg(keys_in + g) : 0xffffffffu;
        if (!LATE_V) v[i] = ok ? (vals_in ? __ldg(vals_in + g) : (uint32_t)g) : 0u;
    }
    for (int d = t; d < RADIX; d += THREADS) {
#pragma unroll
        for (int w = 0; w < WARPS; ++w) s_cnt[w][d] = 0;
    }
    __syncthreads();
    // warp-private stable ranking: r[i] = items of the same digit earlier in this warp's segment
    uint32_t r[ITEMS / 2];  // two 16-bit ranks per register (a rank is < IPW)
    const uint32_t lt_mask = (1u << lane) - 1u;
#if PNDF_RS_ATOMIC
    // each round's group leader claims its group's run with a shared-memory atomicAdd that returns the
    // digit's running count; one warp's atomics on an address are performed in program order, so runs are
    // claimed round by round (stable), and no round waits for the previous round's counter store
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const bool ok = seg + i * 32 < nt;
        const uint32_t d = (k[i] >> shift) & (RADIX - 1);
        const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : 0xffffffffu);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0u;
        if (ok && lane == leader) base = atomicAdd(&s_cnt[warp][d], (uint32_t)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        const uint32_t ri = base + __popc(peers & lt_mask);
        r[i >> 1] = (i & 1) ? (r[i >> 1] | (ri << 16)) : ri;
    }
#else
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const bool ok = seg + i * 32 < nt;
        const uint32_t d = (k[i] >> shift) & (RADIX - 1);
        const uint32_t peers = __match_any_sync(0xffffffffu, ok ? d : 0xffffffffu);
        const uint32_t lt = peers & lt_mask;
        const uint32_t base = ok ? s_cnt[warp][d] : 0u;
        const uint32_t ri = base + __popc(lt);
        r[i >> 1] = (i & 1) ? (r[i >> 1] | (ri << 16)) : ri;
        __syncwarp();
        if (ok && lt == 0) s_cnt[warp][d] = base + __popc(peers);
        __syncwarp();
    }
#endif
    if (LATE_V) {  // values are needed only for placement: their loads overlap the scans below
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int64_t g = t0 + seg + i * 32;
            const bool ok = seg + i * 32 < nt;
            v[i] = ok ? (vals_in ? __ldg(vals_in + g) : (uint32_t)g) : 0u;
        }
    }
    __syncthreads();
    for (int dd = t; dd < RADIX; dd += THREADS) {  // exclusive offsets of each digit over the warps
        uint32_t acc = 0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            const uint32_t c = s_cnt[w][dd];
            s_cnt[w][dd] = acc;
            acc += c;
        }
        s_run[dd] = acc;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the tile histogram, DPL digits per lane
        uint32_t c[DPL], sum = 0;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            c[j] = s_run[lane * DPL + j];
            sum += c[j];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t acc = incl - sum;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            const int d = lane * DPL + j;
            s_start[d] = acc;
            acc += c[j];
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < (RADIX + THREADS - 1) / THREADS; ++j) {
        const int d = t + j * THREADS;
        if (d < RADIX) s_goff[d] = goff_r[j] - s_start[d];
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        if (seg + i * 32 < nt) {
            const uint32_t d = (k[i] >> shift) & (RADIX - 1);
            const uint32_t pos = s_start[d] + s_cnt[warp][d] + ((r[i >> 1] >> ((i & 1) * 16)) & 0xffffu);
            s_keys[pos] = k[i];
            s_vals[pos] = v[i];
        }
    }
    __syncthreads();
    for (int j = t; j < nt; j += THREADS) {
        const uint32_t key = s_keys[j];
        const uint32_t d = (key >> shift) & (RADIX - 1);
        const uint32_t pos = s_goff[d] + (uint32_t)j;
        if (keys_out) keys_out[pos] = key;
        vals_out[pos] = s_vals[j];
    }
}

int64_t scan_blocks(int64_t nb) { return (nb + kScanTile - 1) / kScanTile; }
int64_t radix_tiles(int64_t n) { return (n + kRsTile - 1) / kRsTile; }

static cudaError_t scan_exclusive(uint32_t* a, int64_t nb, uint32_t* bsum, cudaStream_t st) {
    const int64_t nblk = scan_blocks(nb);
    scan_reduce_kernel<<<(unsigned)nblk, kScanThreads, 0, st>>>(a, nb, bsum);
    scan_bsum_kernel<<<1, kScanThreads, 0, st>>>(bsum, nblk);
    scan_apply_kernel<<<(unsigned)nblk, kScanThreads, 0, st>>>(a, nb, bsum);
    return cudaGetLastError();
}

template <int BITS, int THREADS>
constexpr size_t rs_smem_bytes() {
    return sizeof(uint32_t) * (2 * kRsTile + (THREADS / 32 + 3) * (1 << BITS));
}

template <int BITS, int THREADS, bool LATE_V>
static void launch_scatter(const uint32_t* kin, const uint32_t* vin, int64_t n, int shift, const uint32_t* offsets,
                           int64_t ntiles, uint32_t* kout, uint32_t* vout, cudaStream_t st) {
    constexpr size_t smem = rs_smem_bytes<BITS, THREADS>();
    cudaFuncSetAttribute(rs_scatter_kernel<BITS, THREADS, LATE_V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    rs_scatter_kernel<BITS, THREADS, LATE_V><<<(unsigned)ntiles, THREADS, smem, st>>>(kin, vin, n, shift, offsets,
                                                                                      ntiles, kout, vout);
}

// value loads after the ranking (4 CTAs/SM) vs with the keys (3 CTAs/SM): PNDF_SCATTER_LATEV=0/1
static bool scatter_late_v() {
    static bool v = [] {
        const char* e = getenv("PNDF_SCATTER_LATEV");
        return e && atoi(e) == 1;
    }();
    return v;
}

// scatter CTA size: 256 (default) or 512 threads per tile (PNDF_SCATTER_THREADS, for A/B runs)
static int scatter_threads() {
    static int v = [] {
        const char* e = getenv("PNDF_SCATTER_THREADS");
        return (e && atoi(e) == 512) ? 512 : 256;
    }();
    return v;
}

template <int BITS>
static void radix_pass(const uint32_t* kin, const uint32_t* vin, int64_t n, int shift, BinScratch& sc, int64_t ntiles,
                       uint32_t* kout, uint32_t* vout, bool have_hist, cudaStream_t st) {
    if (!have_hist) rs_hist_kernel<BITS><<<(unsigned)ntiles, kRsThreads, 0, st>>>(kin, n, shift, sc.counts, ntiles);
    scan_exclusive(sc.counts, ntiles << BITS, sc.bsum, st);
    if (scatter_threads() == 512)
        launch_scatter<BITS, 512, false>(kin, vin, n, shift, sc.counts, ntiles, kout, vout, st);
    else if (scatter_late_v())
        launch_scatter<BITS, 256, true>(kin, vin, n, shift, sc.counts, ntiles, kout, vout, st);
    else
        launch_scatter<BITS, 256, false>(kin, vin, n, shift, sc.counts, ntiles, kout, vout, st);
}

// Level sort for the Wang-tile sampler: key = the record's lower level l0 (255 = invalid), the tile
// histogram fused as in bin_keys_kernel, then one stable 8-bit radix pass -> permutation.  Lanes of a
// warp then sample footprints of the same size, whose row loops have similar trip counts.
__global__ void __launch_bounds__(kRsThreads) level_keys_kernel(const QParams p, const pndf_query* __restrict__ q,
                                                                int64_t n, uint32_t* keys, uint32_t* counts,
                                                                int64_t ntiles) {
    __shared__ uint32_t h[256];
    for (int d = threadIdx.x; d < 256; d += kRsThreads) h[d] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * kRsTile;
    for (int i = 0; i < kRsItems; ++i) {
        const int64_t k = t0 + (int64_t)i * kRsThreads + threadIdx.x;
        if (k >= n) continue;
        const pndf_query rec = ldg_query(q + k);
        int x1, x2, y1, y2;
        uint32_t key = 255u;
        if (record_valid(p, rec, x1, x2, y1, y2)) {
            int l0;
            float t;
            level_select(p, rec.size, l0, t);
            key = (uint32_t)l0;
        }
        keys[k] = key;
        atomicAdd(&h[key], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += kRsThreads) counts[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

cudaError_t launch_level_sort(const QParams& p, const pndf_query* q, int64_t n, BinScratch& sc, cudaStream_t st,
                              int* launches, const uint32_t** perm) {
    const int64_t ntiles = radix_tiles(n);
    level_keys_kernel<<<(unsigned)ntiles, kRsThreads, 0, st>>>(p, q, n, sc.keys[0], sc.counts, ntiles);
    radix_pass<8>(sc.keys[0], nullptr, n, 0, sc, ntiles, nullptr, sc.vals[1], true, st);
    *launches += 5;
    *perm = sc.vals[1];
    return cudaGetLastError();
}

int64_t bin_key_space(int64_t P, int* half) {
    // half-cell keys (4 per cell) when they fit in 32 bits, else cell keys
    *half = (4 * P + 1 < (int64_t)0xffffffffLL) ? 1 : 0;
    return (*half ? 4 * P : P) + 1;
}

cudaError_t launch_binning(const QParams& p, const pndf_query* q, int64_t n, int64_t P, BinScratch& sc,
                           int num_sms, cudaStream_t st, int* launches, const uint32_t** perm,
                           const uint32_t** sorted_keys) {
    int half;
    const int64_t nkeys = bin_key_space(P, &half);
    int kbits = 1;
    while (kbits < 32 && ((int64_t)1 << kbits) < nkeys) ++kbits;
    // <= 24 bits: 8-bit digits; <= 27: 9-bit digits (3 passes); else 8-bit digits (4 passes)
    const int bits = (kbits > 24 && kbits <= 27) ? 9 : 8;
    const int passes = (kbits + bits - 1) / bits;
    const int64_t ntiles = radix_tiles(n);
    if (bits == 9)
        bin_keys_kernel<9><<<(unsigned)ntiles, kRsThreads, 0, st>>>(p, q, n, sc.keys[0], (uint32_t)(nkeys - 1), half,
                                                                   sc.counts, ntiles);
    else
        bin_keys_kernel<8><<<(unsigned)ntiles, kRsThreads, 0, st>>>(p, q, n, sc.keys[0], (uint32_t)(nkeys - 1), half,
                                                                   sc.counts, ntiles);
    *launches += 1;
    int cur = 0;
    const uint32_t* vals = nullptr;  // pass 0: identity permutation
    for (int ps = 0; ps < passes; ++ps) {
        // the last pass writes sorted keys only when the caller asks for them
        uint32_t* kout = (ps + 1 < passes || sorted_keys) ? sc.keys[cur ^ 1] : nullptr;
        if (bits == 9)
            radix_pass<9>(sc.keys[cur], vals, n, 9 * ps, sc, ntiles, kout, sc.vals[cur ^ 1], ps == 0, st);
        else
            radix_pass<8>(sc.keys[cur], vals, n, 8 * ps, sc, ntiles, kout, sc.vals[cur ^ 1], ps == 0, st);
        vals = sc.vals[cur ^ 1];
        cur ^= 1;
        *launches += ps == 0 ? 4 : 5;
    }
    *perm = vals;
    if (sorted_keys) *sorted_keys = sc.keys[cur];
    return cudaGetLastError();
}

}  // namespace pndf
