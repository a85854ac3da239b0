// query.cu -- sm_100a kernels of the batched NDF range query (the hot path).
//
// Rows of SURVEY.md §8(a) implemented here:
//   a1  query binning        bin_keys_kernel, scan_*_kernel, bin_scatter_kernel
//   a2  decode + level select  decode()
//   a3  spatial neighbours     decode()
//   a4  positional gather + interpolation  query_kernel: 8 rows of Zc, float4 per lane
//   a5  angular prefix differencing        query_kernel: 4 prefix rows (hi,lo)
//   a6  rank product + reduce + write      query_kernel: Eq. 6, xor-shuffle
//                                          reduction over the G lanes of a query
// This is a gather-and-reduce (~11 flop per rank per query), bound by the memory
// system, so there are no tensor cores here.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"
#include "launch.h"

namespace pndf {

// ------------------------------------------------------------ helpers --
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

__device__ __forceinline__ pndf_query ldg_query(const pndf_query* q) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(q));
    pndf_query r;
    r.u = __uint_as_float(v.x);
    r.v = __uint_as_float(v.y);
    r.size = __uint_as_float(v.z);
    r.rect = v.w;
    return r;
}

// off_l = sum_{m<l} (n0 >> m)^2 = 4 (n0^2 - n_l^2) / 3 for power-of-two n0 (exact)
__device__ __forceinline__ int64_t level_offset(int64_t n0, int l) {
    const int64_t nl = n0 >> l;
    return 4 * (n0 * n0 - nl * nl) / 3;
}

__device__ __forceinline__ uint32_t part1by1(uint32_t x) {
    x &= 0x0000ffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

__device__ __forceinline__ bool record_valid(const QParams& p, const pndf_query& q, int& x1, int& x2, int& y1,
                                             int& y2) {
    x1 = (int)(q.rect & 255u);
    x2 = (int)((q.rect >> 8) & 255u);
    y1 = (int)((q.rect >> 16) & 255u);
    y2 = (int)(q.rect >> 24);
    return isfinite(q.u) && isfinite(q.v) && isfinite(q.size) && fabsf(q.u) <= 4194304.f &&
           fabsf(q.v) <= 4194304.f && q.size > 0.f && x1 <= x2 && x2 < p.A && y1 <= y2 && y2 < p.A;
}

// a2: level select.  l* = clamp(log2(S/s0), 0, L-1), l0 = min(floor(l*), L-2),
// t = l* - l0.  floor(log2(S/s0)) is taken exactly from the fp32 exponent of
// S/s0 (s0 is a power of two, so the division is exact); t = log2 of the
// mantissa.  Above the top level: (L-2, t=1) = "directly clamp".
__device__ __forceinline__ void level_select(const QParams& p, float size, int& l0, float& t) {
    int e;
    const float m = frexpf(size * p.inv_s0, &e);  // S/s0 = m 2^e, m in [0.5, 1)
    const int el = e - 1;                         // floor(log2(S/s0))
    if (el < 0) {
        l0 = 0;
        t = 0.f;
    } else if (el >= p.L - 1) {
        l0 = p.L - 2;
        t = 1.f;
    } else {
        l0 = el;
        t = log2f(2.f * m);
    }
}

// a3: neighbour cell along one axis at level l: f = u/s_l - 1/2 (exact in fp32
// for |u| <= 2^22), i0 = floor(f), a = f - i0; wrap (power-of-two grid) or clamp.
__device__ __forceinline__ void axis_cells(const QParams& p, float u, int l, int& i0, int& i1, float& a) {
    const int n = p.n0 >> l;
    const float f = fmaf(u, ldexpf(p.inv_s0, -l), -0.5f);
    const float fl = floorf(f);
    a = f - fl;
    i0 = (int)fl;
    i1 = i0 + 1;
    if (p.wrap) {
        i0 &= n - 1;
        i1 &= n - 1;
    } else {
        i0 = min(max(i0, 0), n - 1);
        i1 = min(max(i1, 0), n - 1);
    }
}

// a2 + a3: the 8 (row, weight) pairs of a valid record.
__device__ __forceinline__ void neighbours(const QParams& p, const pndf_query& q, int64_t (&row)[8], float (&w)[8]) {
    int l0;
    float t;
    level_select(p, q.size, l0, t);
#pragma unroll
    for (int dl = 0; dl < 2; ++dl) {
        const int l = l0 + dl;
        const float wl = dl ? t : 1.f - t;
        int i0, i1, j0, j1;
        float a, b;
        axis_cells(p, q.u, l, i0, i1, a);
        axis_cells(p, q.v, l, j0, j1, b);
        const int64_t n = p.n0 >> l;
        const int64_t off = level_offset(p.n0, l);
        row[4 * dl + 0] = off + (int64_t)j0 * n + i0;
        row[4 * dl + 1] = off + (int64_t)j0 * n + i1;
        row[4 * dl + 2] = off + (int64_t)j1 * n + i0;
        row[4 * dl + 3] = off + (int64_t)j1 * n + i1;
        const float wa = wl * (1.f - a), wb = wl * a;
        w[4 * dl + 0] = wa * (1.f - b);
        w[4 * dl + 1] = wb * (1.f - b);
        w[4 * dl + 2] = wa * b;
        w[4 * dl + 3] = wb * b;
    }
}

// ------------------------------------------------------- query kernel --
// G lanes share one query; each lane owns NV float4 rank chunks at float
// offsets (gl + v*G)*4, so the G lanes of a query read each 4*G-float slice of
// a row contiguously (coalesced 16-byte loads).  Per lane and chunk: 8 Zc
// loads (a4) + 8 prefix loads (a5, hi/lo of 4 rows), all issued before use.
// Per-query results do not depend on the query's position in the batch, so
// binned and unbinned batches are bitwise identical.
template <int G, int NV, bool BINNED>
__global__ void __launch_bounds__(kThreads) query_kernel(const QParams p, const pndf_query* __restrict__ q,
                                                         const uint32_t* __restrict__ idx, int64_t n,
                                                         float* __restrict__ out) {
    constexpr int QPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane % G;
    const int grp = lane / G;
    const int64_t gw = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
    const size_t Rp = (size_t)p.Rp;
    const float* __restrict__ PX = p.PXY;
    const float* __restrict__ PY = p.PXY + (size_t)(p.A + 1) * 2 * Rp;
    const float* __restrict__ Zc = p.Zc;

    for (int64_t base = gw * QPW; base < n; base += nw * QPW) {
        const int64_t qi = base + grp;
        float part = 0.f;
        int status = 0;  // 0: no query, 1: valid, 2: invalid record
        float area = 1.f;
        int64_t oi = qi;
        if (qi < n) {
            const pndf_query rec = ldg_query(q + qi);
            if (BINNED) oi = (int64_t)__ldg(idx + qi);
            int x1, x2, y1, y2;
            if (record_valid(p, rec, x1, x2, y1, y2)) {
                status = 1;
                area = (float)((x2 - x1 + 1) * (y2 - y1 + 1));
                int64_t row[8];
                float w[8];
                neighbours(p, rec, row, w);
                const float* px0 = PX + (size_t)(2 * x1) * Rp;
                const float* px1 = PX + (size_t)(2 * (x2 + 1)) * Rp;
                const float* py0 = PY + (size_t)(2 * y1) * Rp;
                const float* py1 = PY + (size_t)(2 * (y2 + 1)) * Rp;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int c = (gl + v * G) * 4;
                    float4 zr[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        zr[k] = (w[k] != 0.f) ? ldg4(Zc + (size_t)row[k] * Rp + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float4 xh1 = ldg4(px1 + c), xh0 = ldg4(px0 + c);
                    const float4 xl1 = ldg4(px1 + Rp + c), xl0 = ldg4(px0 + Rp + c);
                    const float4 yh1 = ldg4(py1 + c), yh0 = ldg4(py0 + c);
                    const float4 yl1 = ldg4(py1 + Rp + c), yl0 = ldg4(py0 + Rp + c);
                    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        z.x = fmaf(w[k], zr[k].x, z.x);
                        z.y = fmaf(w[k], zr[k].y, z.y);
                        z.z = fmaf(w[k], zr[k].z, z.z);
                        z.w = fmaf(w[k], zr[k].w, z.w);
                    }
                    // Xbar, Ybar numerators: (hi1 - hi0) + (lo1 - lo0); hi1 - hi0 is exact
                    // under cancellation (Sterbenz), lo carries the fp64 residual.
                    const float dx0 = (xh1.x - xh0.x) + (xl1.x - xl0.x), dy0 = (yh1.x - yh0.x) + (yl1.x - yl0.x);
                    const float dx1 = (xh1.y - xh0.y) + (xl1.y - xl0.y), dy1 = (yh1.y - yh0.y) + (yl1.y - yl0.y);
                    const float dx2 = (xh1.z - xh0.z) + (xl1.z - xl0.z), dy2 = (yh1.z - yh0.z) + (yl1.z - yl0.z);
                    const float dx3 = (xh1.w - xh0.w) + (xl1.w - xl0.w), dy3 = (yh1.w - yh0.w) + (yl1.w - yl0.w);
                    part = fmaf(dx0 * dy0, z.x, part);
                    part = fmaf(dx1 * dy1, z.y, part);
                    part = fmaf(dx2 * dy2, z.z, part);
                    part = fmaf(dx3 * dy3, z.w, part);
                }
            } else {
                status = 2;
            }
        }
        // a6: fixed xor-butterfly over the G lanes of the query (IEEE + is commutative,
        // so every lane of the group ends with the same bits).
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (gl == 0 && status != 0) {
            out[oi] = (status == 1) ? (p.mean ? part / area : part) : __int_as_float(0x7fc00000);
            if (status == 2) atomicOr(p.err, 1u);
        }
    }
}

// ------------------------------------------------------------ binning --
// a1: key = off_{l0} + Morton(i0, j0) -- the record's lower-left neighbour cell
// on its lower level l0, in Z-order within the level, so queries that share Zc
// rows become neighbours in the binned order.  Invalid records -> last bin.
__global__ void bin_keys_kernel(const QParams p, const pndf_query* __restrict__ q, int64_t n, uint32_t* keys,
                                uint32_t* hist, uint32_t invalid_key) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const pndf_query rec = ldg_query(q + i);
        int x1, x2, y1, y2;
        uint32_t key = invalid_key;
        if (record_valid(p, rec, x1, x2, y1, y2)) {
            int l0;
            float t;
            level_select(p, rec.size, l0, t);
            int i0, i1, j0, j1;
            float a, b;
            axis_cells(p, rec.u, l0, i0, i1, a);
            axis_cells(p, rec.v, l0, j0, j1, b);
            key = (uint32_t)level_offset(p.n0, l0) + (part1by1((uint32_t)i0) | (part1by1((uint32_t)j0) << 1));
        }
        keys[i] = key;
        atomicAdd(hist + key, 1u);
    }
}

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

__global__ void bin_scatter_kernel(const pndf_query* __restrict__ q, const uint32_t* __restrict__ keys, int64_t n,
                                   uint32_t* cursor, pndf_query* binned, uint32_t* idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t pos = atomicAdd(cursor + keys[i], 1u);
        reinterpret_cast<uint4*>(binned)[pos] = __ldg(reinterpret_cast<const uint4*>(q + i));
        idx[pos] = (uint32_t)i;
    }
}

// ----------------------------------------------------------- launchers --
template <int G, int NV, bool B>
static cudaError_t launch_q(const QParams& p, const pndf_query* q, const uint32_t* idx, int64_t n, float* out,
                            int num_sms, cudaStream_t st) {
    static int occ = -1;
    if (occ < 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, query_kernel<G, NV, B>, kThreads, 0) != cudaSuccess ||
            occ < 1)
            occ = 1;
    }
    const int64_t qpb = (int64_t)(kThreads / 32) * (32 / G);
    int64_t grid = (n + qpb - 1) / qpb;
    const int64_t cap = (int64_t)num_sms * occ;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    query_kernel<G, NV, B><<<(unsigned)grid, kThreads, 0, st>>>(p, q, idx, n, out);
    return cudaGetLastError();
}

template <int G, bool B>
static cudaError_t dispatch_nv(int NV, const QParams& p, const pndf_query* q, const uint32_t* idx, int64_t n,
                               float* out, int num_sms, cudaStream_t st) {
    switch (NV) {
        case 1: return launch_q<G, 1, B>(p, q, idx, n, out, num_sms, st);
        case 2: return launch_q<G, 2, B>(p, q, idx, n, out, num_sms, st);
        case 3: return launch_q<G, 3, B>(p, q, idx, n, out, num_sms, st);
        case 4: return launch_q<G, 4, B>(p, q, idx, n, out, num_sms, st);
        case 8: return launch_q<G, 8, B>(p, q, idx, n, out, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

template <bool B>
static cudaError_t dispatch_g(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx, int64_t n,
                              float* out, int num_sms, cudaStream_t st) {
    switch (G) {
        case 1: return dispatch_nv<1, B>(NV, p, q, idx, n, out, num_sms, st);
        case 2: return dispatch_nv<2, B>(NV, p, q, idx, n, out, num_sms, st);
        case 4: return dispatch_nv<4, B>(NV, p, q, idx, n, out, num_sms, st);
        case 8: return dispatch_nv<8, B>(NV, p, q, idx, n, out, num_sms, st);
        case 16: return dispatch_nv<16, B>(NV, p, q, idx, n, out, num_sms, st);
        case 32: return dispatch_nv<32, B>(NV, p, q, idx, n, out, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

bool lanes_supported(int G, int NV) {
    const bool g = (G == 1 || G == 2 || G == 4 || G == 8 || G == 16 || G == 32);
    const bool v = (NV == 1 || NV == 2 || NV == 3 || NV == 4 || NV == 8);
    return g && v;
}

cudaError_t launch_query(const QParams& p, int G, int NV, const pndf_query* q, const uint32_t* idx, int64_t n,
                         float* out, int num_sms, cudaStream_t st) {
    if (idx) return dispatch_g<true>(G, NV, p, q, idx, n, out, num_sms, st);
    return dispatch_g<false>(G, NV, p, q, idx, n, out, num_sms, st);
}

int64_t scan_blocks(int64_t nbins) { return (nbins + kScanTile - 1) / kScanTile; }

cudaError_t launch_binning(const QParams& p, const pndf_query* q, int64_t n, uint32_t* keys, uint32_t* hist,
                           int64_t nbins, uint32_t* bsum, pndf_query* binned, uint32_t* idx, int num_sms,
                           cudaStream_t st, int* launches) {
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)nbins, st);
    if (e != cudaSuccess) return e;
    const int eg = num_sms * 8;
    int64_t g = (n + 255) / 256;
    if (g > eg) g = eg;
    if (g < 1) g = 1;
    bin_keys_kernel<<<(unsigned)g, 256, 0, st>>>(p, q, n, keys, hist, (uint32_t)(nbins - 1));
    const int64_t nblk = scan_blocks(nbins);
    scan_reduce_kernel<<<(unsigned)nblk, kScanThreads, 0, st>>>(hist, nbins, bsum);
    scan_bsum_kernel<<<1, kScanThreads, 0, st>>>(bsum, nblk);
    scan_apply_kernel<<<(unsigned)nblk, kScanThreads, 0, st>>>(hist, nbins, bsum);
    bin_scatter_kernel<<<(unsigned)g, 256, 0, st>>>(q, keys, n, hist, binned, idx);
    *launches += 5;
    return cudaGetLastError();
}

}  // namespace pndf
