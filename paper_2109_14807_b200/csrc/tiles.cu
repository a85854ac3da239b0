// tiles.cu -- range queries on an implicitly Wang-tiled normal map (Sec. 5.5,
// P:438-454).  Each of the 8 trilinear neighbours (world
// cell centres) gathers the Zc row of every tile whose extended grid holds it
// (the tiles' partial NDFs add up to the footprint's NDF); the tile of a
// world cell comes from the edge colours hashed at its corner vertices (P:444,
// P:450-451).  X, Y are shared by the tiles, so Z-hat = sum_k w_k sum_tiles Zc
// is accumulated first and the SAT product runs once, as in query_kernel.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.h"
#include "sample_kernel.cuh"

namespace pndf {

__device__ __forceinline__ uint64_t tile_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t tile_vertex(uint64_t seed_mixed, int64_t vx, int64_t vy) {
    return tile_mix(seed_mixed ^ ((uint64_t)(uint32_t)vx | ((uint64_t)(uint32_t)vy << 32)));
}
// tile id = N | E<<1 | S<<2 | W<<3 from the corner vertices' edge colours
__device__ __forceinline__ int tile_of(uint64_t seed_mixed, int64_t cx, int64_t cy) {
    const uint64_t a = tile_vertex(seed_mixed, cx, cy);
    const int n = (int)(a & 1u), w = (int)((a >> 1) & 1u);
    const int sth = (int)(tile_vertex(seed_mixed, cx, cy + 1) & 1u);
    const int e = (int)((tile_vertex(seed_mixed, cx + 1, cy) >> 1) & 1u);
    return n | (e << 1) | (sth << 2) | (w << 3);
}

template <int G, int NV, bool U32>
__global__ void __launch_bounds__(256) tiled_query_kernel(const QParams p, const TileParams tp,
                                                          const pndf_query* __restrict__ q,
                                                          const uint32_t* __restrict__ idx, int64_t n,
                                                          float* __restrict__ out) {
    constexpr int QPW = 32 / G;
    constexpr int RP = 4 * G * NV;
    constexpr int PSTRIDE = U32 ? RP : 2 * RP;
    const int lane = threadIdx.x & 31, gl = lane % G, grp = lane / G;
    const float* __restrict__ PX = p.PXY;
    const float* __restrict__ PY = p.PXY + (size_t)(p.A + 1) * PSTRIDE;
    const uint64_t seed_mixed = tile_mix(tp.seed);
    // per group: tile ids of the level's candidate-tile box, hashed once by the group's lanes
    constexpr int TBOX = G >= 8 ? 64 : 16;  // 6 x 6 candidate tiles at the top levels (8 KB of smem at G = 8)
    __shared__ int s_tile[8][32 / G][TBOX];
    int* my_tiles = s_tile[threadIdx.x >> 5][grp];
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
    const int M = tp.margin;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = gw * QPW; base < n; base += nw * QPW) {
        const int64_t qo = base + grp;
        const bool active = qo < n;
        const int64_t qi = active ? (idx ? (int64_t)__ldg(idx + qo) : qo) : 0;  // record (level-sorted order)
        const pndf_query rec = ldg_query(q + qi);
        int x1, x2, y1, y2;
        const bool valid = active && record_valid(p, rec, x1, x2, y1, y2);
        float4 zh[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) zh[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
            int l0;
            float t;
            level_select(p, rec.size, l0, t);
            for (int dl = 0; dl < 2; ++dl) {
                const int l = l0 + dl;
                const float wl = dl ? t : 1.f - t;
                const int sh = __ffs(p.n0 >> l) - 1;  // log2 n_l
                // 32-bit index math: world cells |i| <= 2^22, tile rows < 2^31 (the 64-bit products
                // were a third of the kernel's instructions)
                const int nl = 1 << sh, ne = nl + 2 * M;
                int off = 0;
                for (int m = 0; m < l; ++m) {
                    const int e2 = (p.n0 >> m) + 2 * M;
                    off += e2 * e2;
                }
                const float inv_s = __int_as_float(__float_as_int(p.inv_s0) - (l << 23));
                const float fu = fmaf(rec.u, inv_s, -0.5f), fv = fmaf(rec.v, inv_s, -0.5f);
                const float flu = floorf(fu), flv = floorf(fv);
                const float a = fu - flu, b = fv - flv;
                const int iu = (int)flu, iv = (int)flv;
                const float wa = wl * (1.f - a), wb = wl * a;
                const float wk4[4] = {wa * (1.f - b), wb * (1.f - b), wa * b, wb * b};
                // candidate tiles of all 4 neighbours lie in one small box: hash each cell once
                const int MA = tp.reach;  // rows beyond it are zero (measured at load)
                const int bx0 = (iu - (nl + MA) + 1) >> sh, bx1 = (iu + 1 + MA) >> sh;
                const int by0 = (iv - (nl + MA) + 1) >> sh, by1 = (iv + 1 + MA) >> sh;
                const int bw = bx1 - bx0 + 1;
                const int nc = bw * (by1 - by0 + 1);
                const bool boxed = nc <= TBOX;  // group-uniform
                __syncwarp(gmask);              // the previous level's readers are done
                if (boxed)
                    for (int c = gl; c < nc; c += G) my_tiles[c] = tile_of(seed_mixed, bx0 + c % bw, by0 + c / bw);
                __syncwarp(gmask);
                const int base_rows = off + M * ne + M;  // (jl + M) ne + (il + M) = jl ne + il + base
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int iw = iu + (k & 1), jw = iv + (k >> 1);
                    const float wk = wk4[k];
                    // tiles whose extended grid holds this centre with a possibly nonzero row: local cell
                    // il in [-reach, nl + reach - 1]; rows further out are all zero (checked at load) and
                    // skipped, which is exact (they would add +0)
                    const int tx0 = (iw - (nl + MA) + 1) >> sh, tx1 = (iw + MA) >> sh;
                    const int ty0 = (jw - (nl + MA) + 1) >> sh, ty1 = (jw + MA) >> sh;
                    for (int ty = ty0; ty <= ty1; ++ty)
                        for (int tx = tx0; tx <= tx1; ++tx) {
                            const int il = iw - (tx << sh), jl = jw - (ty << sh);
                            if (il < -MA || il >= nl + MA || jl < -MA || jl >= nl + MA) continue;
                            const int tile = boxed ? my_tiles[(ty - by0) * bw + (tx - bx0)]
                                                   : tile_of(seed_mixed, tx, ty);
                            const int row = tile * (int)tp.p_ext + base_rows + jl * ne + il;
                            const float* zr0 = p.Zc + (size_t)row * RP + gl * 4;
#pragma unroll
                            for (int v = 0; v < NV; ++v) {
                                const float4 zr = ldg4(zr0 + v * G * 4);
                                zh[v].x = fmaf(wk, zr.x, zh[v].x);
                                zh[v].y = fmaf(wk, zr.y, zh[v].y);
                                zh[v].z = fmaf(wk, zr.z, zh[v].z);
                                zh[v].w = fmaf(wk, zr.w, zh[v].w);
                            }
                        }
                }
            }
        }
        float part = 0.f;
        if (valid) {
            const float* px0 = PX + (size_t)x1 * PSTRIDE;
            const float* px1 = PX + (size_t)(x2 + 1) * PSTRIDE;
            const float* py0 = PY + (size_t)y1 * PSTRIDE;
            const float* py1 = PY + (size_t)(y2 + 1) * PSTRIDE;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int c = (gl + v * G) * 4;
                float4 dx, dy;
                if (U32) {
                    const uint4 qx1 = __ldg(reinterpret_cast<const uint4*>(px1 + c));
                    const uint4 qx0 = __ldg(reinterpret_cast<const uint4*>(px0 + c));
                    const uint4 qy1 = __ldg(reinterpret_cast<const uint4*>(py1 + c));
                    const uint4 qy0 = __ldg(reinterpret_cast<const uint4*>(py0 + c));
                    dx = make_float4(__uint2float_rn(qx1.x - qx0.x), __uint2float_rn(qx1.y - qx0.y),
                                     __uint2float_rn(qx1.z - qx0.z), __uint2float_rn(qx1.w - qx0.w));
                    dy = make_float4(__uint2float_rn(qy1.x - qy0.x), __uint2float_rn(qy1.y - qy0.y),
                                     __uint2float_rn(qy1.z - qy0.z), __uint2float_rn(qy1.w - qy0.w));
                } else {
                    const float4 xh1 = ldg4(px1 + c), xh0 = ldg4(px0 + c);
                    const float4 xl1 = ldg4(px1 + RP + c), xl0 = ldg4(px0 + RP + c);
                    const float4 yh1 = ldg4(py1 + c), yh0 = ldg4(py0 + c);
                    const float4 yl1 = ldg4(py1 + RP + c), yl0 = ldg4(py0 + RP + c);
                    dx = make_float4((xh1.x - xh0.x) + (xl1.x - xl0.x), (xh1.y - xh0.y) + (xl1.y - xl0.y),
                                     (xh1.z - xh0.z) + (xl1.z - xl0.z), (xh1.w - xh0.w) + (xl1.w - xl0.w));
                    dy = make_float4((yh1.x - yh0.x) + (yl1.x - yl0.x), (yh1.y - yh0.y) + (yl1.y - yl0.y),
                                     (yh1.z - yh0.z) + (yl1.z - yl0.z), (yh1.w - yh0.w) + (yl1.w - yl0.w));
                }
                part = fmaf(dx.x * dy.x, zh[v].x, part);
                part = fmaf(dx.y * dy.y, zh[v].y, part);
                part = fmaf(dx.z * dy.z, zh[v].z, part);
                part = fmaf(dx.w * dy.w, zh[v].w, part);
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (active && gl == 0) {
            if (!valid) {
                out[qi] = __int_as_float(0x7fc00000);
                atomicOr(p.err, 1u);
            } else {
                out[qi] = p.mean ? part / (float)((x2 - x1 + 1) * (y2 - y1 + 1)) : part;
            }
        }
    }
}

// Importance sampling over the implicit Wang tiles (Sec. 5.5; DESIGN.md
// reading 25): "choose one Wang tile from all the Wang tiles covered by the
// pixel footprint with equal probability", descend on that tile's partial NDF
// as in sample_kernel (Sec. 5.2), and set the pdf to the full (all-tile) NDF
// value of the sampled pixel.  A tile instance is covered when its partial
// NDF has positive mass over the whole angular domain (it holds texels of the
// footprint).  Pass 1 walks the query's rows once: it accumulates Z-hat of all
// tiles (pdf) and, per row, the row's full-domain mass sum_r PX[A] PY[A] Zc,
// setting the instance's bit in a 64-bit mask over the (ty, tx) box of
// candidate instances (row-major, so bit order = the (ty, tx) order).  The
// c-th set bit, c = floor(xi[10] * popc(mask)) in fp32, is the chosen tile;
// pass 2 re-reads only its rows (L1/L2-hot) into Z-hat of the tile.
template <int G>
__device__ __forceinline__ float group_sum_m(float v, unsigned gmask) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
    return v;
}

template <int G, int NV, bool U32>
__global__ void __launch_bounds__(256) tiled_sample_kernel(const QParams p, const TileParams tp,
                                                           const pndf_query* __restrict__ q,
                                                           const float* __restrict__ xi,
                                                           const uint32_t* __restrict__ idx, int64_t n,
                                                           pndf_sample* __restrict__ out,
                                                           int32_t* __restrict__ tile_out) {
    constexpr int QPW = 32 / G;
    constexpr int RP = 4 * G * NV;
    constexpr int PSTRIDE = U32 ? RP : 2 * RP;
    const int REACH = tp.reach;  // rows beyond it are zero (measured at load; <= 4 for sampling)
    const int lane = threadIdx.x & 31, gl = lane % G, grp = lane / G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
    const float* __restrict__ PX = p.PXY;
    const float* __restrict__ PY = p.PXY + (size_t)(p.A + 1) * PSTRIDE;
    const uint64_t seed_mixed = tile_mix(tp.seed);
    const int M = tp.margin;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = gw * QPW; base < n; base += nw * QPW) {  // warp-uniform trip count
        const int64_t qi = base + grp;
        const bool active = qi < n;
        const int64_t si = active ? (idx ? (int64_t)__ldg(idx + qi) : qi) : 0;  // record (level-sorted order)
        const pndf_query rec = ldg_query(q + si);
        int x1, x2, y1, y2;
        bool valid = active && record_valid(p, rec, x1, x2, y1, y2);
        if (!valid) x1 = x2 = y1 = y2 = 0;
        const float* sxi = xi + (size_t)si * 11;
        int l0;
        float t;
        level_select(p, valid ? rec.size : 1.f, l0, t);
        // per-level geometry; candidate instances: the union box of both levels' reach
        int iu[2], iv[2], sh[2], offl[2];
        float fa[2], fb[2], wlv[2];
        bool use[2];
        int bx0 = 0x7fffffff, bx1 = -0x7fffffff, by0 = 0x7fffffff, by1 = -0x7fffffff;
#pragma unroll
        for (int dl = 0; dl < 2; ++dl) {
            const int l = l0 + dl;
            wlv[dl] = dl ? t : 1.f - t;
            sh[dl] = __ffs(p.n0 >> l) - 1;
            const float inv_s = __int_as_float(__float_as_int(p.inv_s0) - (l << 23));
            const float fu = fmaf(valid ? rec.u : 0.f, inv_s, -0.5f), fv = fmaf(valid ? rec.v : 0.f, inv_s, -0.5f);
            const float flu = floorf(fu), flv = floorf(fv);
            fa[dl] = fu - flu;
            fb[dl] = fv - flv;
            iu[dl] = (int)flu;
            iv[dl] = (int)flv;
            use[dl] = valid && wlv[dl] > 0.f;
            int off = 0;
            for (int m = 0; m < l; ++m) {
                const int e2 = (p.n0 >> m) + 2 * M;
                off += e2 * e2;
            }
            offl[dl] = off;
            if (use[dl]) {
                bx0 = min(bx0, (iu[dl] - REACH) >> sh[dl]);
                bx1 = max(bx1, (iu[dl] + REACH + 1) >> sh[dl]);
                by0 = min(by0, (iv[dl] - REACH) >> sh[dl]);
                by1 = max(by1, (iv[dl] + REACH + 1) >> sh[dl]);
            }
        }
        const int bw = bx1 - bx0 + 1;
        // the union box is at most 2 reach + 2 tiles per side: <= 100 candidates for reach <= 4
        // (pndf_sample_tiles rejects larger reaches), held in a 128-bit mask
        if (valid && bw * (by1 - by0 + 1) > 128) valid = false;
        // full-domain angular factor sum_x X_r sum_y Y_r (C folded into Zc)
        float4 full[NV];
        {
            SatV<U32> a0, a1, b0, b1;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int c = (gl + v * G) * 4;
                a0.load(PX, c, RP);
                a1.load(PX + (size_t)p.A * PSTRIDE, c, RP);
                b0.load(PY, c, RP);
                b1.load(PY + (size_t)p.A * PSTRIDE, c, RP);
                const float4 dx = SatV<U32>::diff(a0, a1), dy = SatV<U32>::diff(b0, b1);
                full[v] = make_float4(dx.x * dy.x, dx.y * dy.y, dx.z * dy.z, dx.w * dy.w);
            }
        }
        // pass 1: Z-hat of all tiles + covered-instance mask
        float4 zt[NV], za[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) zt[v] = za[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        uint64_t mask = 0, mask_hi = 0;  // bits 0-63, 64-127 of the candidate box
#pragma unroll
        for (int dl = 0; dl < 2; ++dl) {
            if (!use[dl]) continue;
            const int s_ = sh[dl], nl = 1 << s_, ne = nl + 2 * M;
            const int base_rows = offl[dl] + M * ne + M;
            const float wa = wlv[dl] * (1.f - fa[dl]), wb = wlv[dl] * fa[dl];
            const float wk4[4] = {wa * (1.f - fb[dl]), wb * (1.f - fb[dl]), wa * fb[dl], wb * fb[dl]};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float wk = wk4[k];
                if (!(wk > 0.f)) continue;
                const int iw = iu[dl] + (k & 1), jw = iv[dl] + (k >> 1);
                const int tx0 = (iw - REACH) >> s_, tx1 = (iw + REACH) >> s_;
                const int ty0 = (jw - REACH) >> s_, ty1 = (jw + REACH) >> s_;
                for (int ty = ty0; ty <= ty1; ++ty)
                    for (int tx = tx0; tx <= tx1; ++tx) {
                        const int il = iw - (tx << s_), jl = jw - (ty << s_);
                        const int tile = tile_of(seed_mixed, tx, ty);
                        const int row = tile * (int)tp.p_ext + base_rows + jl * ne + il;
                        const float* zr0 = p.Zc + (size_t)row * RP + gl * 4;
                        float m = 0.f;
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            const float4 zr = ldg4(zr0 + v * G * 4);
                            za[v].x = fmaf(wk, zr.x, za[v].x);
                            za[v].y = fmaf(wk, zr.y, za[v].y);
                            za[v].z = fmaf(wk, zr.z, za[v].z);
                            za[v].w = fmaf(wk, zr.w, za[v].w);
                            m = fmaf(full[v].x, zr.x, m);
                            m = fmaf(full[v].y, zr.y, m);
                            m = fmaf(full[v].z, zr.z, m);
                            m = fmaf(full[v].w, zr.w, m);
                        }
                        m = group_sum_m<G>(m, gmask);
                        const int bit = (ty - by0) * bw + (tx - bx0);
                        if (m > 0.f) {
                            if (bit < 64)
                                mask |= 1ull << bit;
                            else
                                mask_hi |= 1ull << (bit - 64);
                        }
                    }
            }
        }
        const int count_lo = __popcll(mask);
        const int count = count_lo + __popcll(mask_hi);
        int ptx = 0, pty = 0;
        if (count > 0) {
            int c = (int)floorf(__fmul_rn(__ldg(sxi + 10), (float)count));
            if (c > count - 1) c = count - 1;
            const bool in_lo = c < count_lo;
            uint64_t mm = in_lo ? mask : mask_hi;
            for (int j = in_lo ? c : c - count_lo; j > 0; --j) mm &= mm - 1;  // drop the lower set bits
            const int bit = __ffsll((long long)mm) - 1 + (in_lo ? 0 : 64);
            ptx = bx0 + bit % bw;
            pty = by0 + bit / bw;
            // pass 2: Z-hat of the chosen tile (its rows only)
#pragma unroll
            for (int dl = 0; dl < 2; ++dl) {
                if (!use[dl]) continue;
                const int s_ = sh[dl], nl = 1 << s_, ne = nl + 2 * M;
                const int base_rows = offl[dl] + M * ne + M;
                const int tile = tile_of(seed_mixed, ptx, pty);
                const float wa = wlv[dl] * (1.f - fa[dl]), wb = wlv[dl] * fa[dl];
                const float wk4[4] = {wa * (1.f - fb[dl]), wb * (1.f - fb[dl]), wa * fb[dl], wb * fb[dl]};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float wk = wk4[k];
                    const int il = iu[dl] + (k & 1) - (ptx << s_), jl = iv[dl] + (k >> 1) - (pty << s_);
                    if (!(wk > 0.f) || il < -REACH || il >= nl + REACH || jl < -REACH || jl >= nl + REACH) continue;
                    const float* zr0 = p.Zc + (size_t)(tile * (int)tp.p_ext + base_rows + jl * ne + il) * RP + gl * 4;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const float4 zr = ldg4(zr0 + v * G * 4);
                        zt[v].x = fmaf(wk, zr.x, zt[v].x);
                        zt[v].y = fmaf(wk, zr.y, zt[v].y);
                        zt[v].z = fmaf(wk, zr.z, zt[v].z);
                        zt[v].w = fmaf(wk, zr.w, zt[v].w);
                    }
                }
            }
        }
        // SAT values at the current range's corners [xa, xb) x [ya, yb)
        int xa = x1, xb = x2 + 1, ya = y1, yb = y2 + 1;
        SatV<U32> sxa[NV], sxb[NV], sya[NV], syb[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int c = (gl + v * G) * 4;
            sxa[v].load(PX + (size_t)xa * PSTRIDE, c, RP);
            sxb[v].load(PX + (size_t)xb * PSTRIDE, c, RP);
            sya[v].load(PY + (size_t)ya * PSTRIDE, c, RP);
            syb[v].load(PY + (size_t)yb * PSTRIDE, c, RP);
        }
        float root = 0.f, root_all = 0.f;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 dx = SatV<U32>::diff(sxa[v], sxb[v]), dy = SatV<U32>::diff(sya[v], syb[v]);
            const float4 e = make_float4(dx.x * dy.x, dx.y * dy.y, dx.z * dy.z, dx.w * dy.w);
            root = fmaf(e.x, zt[v].x, root);
            root = fmaf(e.y, zt[v].y, root);
            root = fmaf(e.z, zt[v].z, root);
            root = fmaf(e.w, zt[v].w, root);
            root_all = fmaf(e.x, za[v].x, root_all);
            root_all = fmaf(e.y, za[v].y, root_all);
            root_all = fmaf(e.z, za[v].z, root_all);
            root_all = fmaf(e.w, za[v].w, root_all);
        }
        root = group_sum<G>(root);
        root_all = group_sum<G>(root_all);
        const bool live = valid && count > 0 && root > 0.f;
        int lvl = 0;
        while (__any_sync(0xffffffffu, live && (xb - xa > 1 || yb - ya > 1))) {
            const bool go = live && (xb - xa > 1 || yb - ya > 1);
            const int xm = go && xb - xa > 1 ? xa + (xb - xa + 1) / 2 : xb;
            const int ym = go && yb - ya > 1 ? ya + (yb - ya + 1) / 2 : yb;
            SatV<U32> sxm[NV], sym[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int c = (gl + v * G) * 4;
                sxm[v].load(PX + (size_t)xm * PSTRIDE, c, RP);
                sym[v].load(PY + (size_t)ym * PSTRIDE, c, RP);
            }
            float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float4 dxl = SatV<U32>::diff(sxa[v], sxm[v]), dxr = SatV<U32>::diff(sxm[v], sxb[v]);
                const float4 dyb = SatV<U32>::diff(sya[v], sym[v]), dyt = SatV<U32>::diff(sym[v], syb[v]);
                const float4 u = make_float4(dyb.x * zt[v].x, dyb.y * zt[v].y, dyb.z * zt[v].z, dyb.w * zt[v].w);
                const float4 w = make_float4(dyt.x * zt[v].x, dyt.y * zt[v].y, dyt.z * zt[v].z, dyt.w * zt[v].w);
                q0 = fmaf(dxl.x, u.x, fmaf(dxl.y, u.y, fmaf(dxl.z, u.z, fmaf(dxl.w, u.w, q0))));
                q1 = fmaf(dxr.x, u.x, fmaf(dxr.y, u.y, fmaf(dxr.z, u.z, fmaf(dxr.w, u.w, q1))));
                q2 = fmaf(dxl.x, w.x, fmaf(dxl.y, w.y, fmaf(dxl.z, w.z, fmaf(dxl.w, w.w, q2))));
                q3 = fmaf(dxr.x, w.x, fmaf(dxr.y, w.y, fmaf(dxr.z, w.z, fmaf(dxr.w, w.w, q3))));
            }
            quad_reduce<G>(q0, q1, q2, q3, gl, lane);
            if (go) {
                const float qs[4] = {q0, q1, q2, q3};
                const float tot = ((q0 + q1) + q2) + q3;
                const float tt = __ldg(sxi + lvl) * tot;
                float c = 0.f;
                int k = -1;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    c += qs[j];
                    if (k < 0 && tt < c) k = j;
                }
                if (k < 0) k = qs[3] > 0.f ? 3 : (qs[2] > 0.f ? 2 : (qs[1] > 0.f ? 1 : 0));
                if (k & 1) {
                    xa = xm;
#pragma unroll
                    for (int v = 0; v < NV; ++v) sxa[v] = sxm[v];
                } else {
                    xb = xm;
#pragma unroll
                    for (int v = 0; v < NV; ++v) sxb[v] = sxm[v];
                }
                if (k & 2) {
                    ya = ym;
#pragma unroll
                    for (int v = 0; v < NV; ++v) sya[v] = sym[v];
                } else {
                    yb = ym;
#pragma unroll
                    for (int v = 0; v < NV; ++v) syb[v] = sym[v];
                }
                ++lvl;
            }
        }
        // pdf: the full NDF's mass in the sampled pixel over its mass in the domain
        float pix = 0.f;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 dx = SatV<U32>::diff(sxa[v], sxb[v]), dy = SatV<U32>::diff(sya[v], syb[v]);
            pix = fmaf(dx.x * dy.x, za[v].x, pix);
            pix = fmaf(dx.y * dy.y, za[v].y, pix);
            pix = fmaf(dx.z * dy.z, za[v].z, pix);
            pix = fmaf(dx.w * dy.w, za[v].w, pix);
        }
        pix = group_sum<G>(pix);
        if (active && gl == 0) {
            pndf_sample o;
            if (!valid) {
                atomicOr(p.err, 1u);
                o.hx = o.hy = o.pdf = __int_as_float(0x7fc00000);
                o.pixel = 0xffffffffu;
            } else if (!live) {
                o.hx = o.hy = __int_as_float(0x7fc00000);
                o.pdf = 0.f;
                o.pixel = 0xffffffffu;
            } else {
                const float inv = 2.f / (float)p.A;
                o.hx = ((float)xa + __ldg(sxi + 8)) * inv - 1.f;
                o.hy = ((float)ya + __ldg(sxi + 9)) * inv - 1.f;
                o.pdf = (pix / root_all) / (inv * inv);
                o.pixel = (uint32_t)xa | ((uint32_t)ya << 16);
            }
            out[si] = o;
            if (tile_out) {
                tile_out[2 * si] = valid ? ptx : 0;
                tile_out[2 * si + 1] = valid ? pty : 0;
            }
        }
    }
}

// One thread per row of the 16 tiles' extended grids: a row with any nonzero entry raises *reach to
// its distance beyond the tile's own cells (Chebyshev, in cells of its level).
__global__ void tile_reach_kernel(const float* __restrict__ Zc, int Rp, TileParams tp, int n0, int L,
                                  uint32_t* reach) {
    const int64_t rows = 16 * tp.p_ext;
    const int M = tp.margin;
    for (int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; z < rows; z += (int64_t)gridDim.x * blockDim.x) {
        const float4* r4 = reinterpret_cast<const float4*>(Zc + (size_t)z * Rp);
        bool nz = false;
        for (int c = 0; c < Rp / 4 && !nz; ++c) {
            const float4 v = __ldg(r4 + c);
            nz = v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f;
        }
        if (!nz) continue;
        int64_t k = z % tp.p_ext;
        int l = 0;
        int64_t ne = (int64_t)n0 + 2 * M;
        while (l + 1 < L && k >= ne * ne) {
            k -= ne * ne;
            ++l;
            ne = (int64_t)(n0 >> l) + 2 * M;
        }
        const int nl = n0 >> l;
        const int il = (int)(k % ne) - M, jl = (int)(k / ne) - M;
        const int d = max(max(max(-il, il - (nl - 1)), max(-jl, jl - (nl - 1))), 0);
        if (d > 0) atomicMax(reach, (uint32_t)d);
    }
}

cudaError_t launch_tile_reach(const float* Zc, int Rp, const TileParams& tp, int n0, int L, uint32_t* reach,
                              cudaStream_t st) {
    const int64_t rows = 16 * tp.p_ext;
    int64_t grid = (rows + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    if (grid < 1) grid = 1;
    tile_reach_kernel<<<(unsigned)grid, 256, 0, st>>>(Zc, Rp, tp, n0, L, reach);
    return cudaGetLastError();
}

template <int G, int NV, bool U>
static cudaError_t launch_ts(const QParams& p, const TileParams& tp, const pndf_query* q, const float* xi,
                             const uint32_t* idx, int64_t n, pndf_sample* out, int32_t* tile_out, int num_sms,
                             cudaStream_t st) {
    const int64_t spb = 8 * (32 / G);
    int64_t grid = (n + spb - 1) / spb;
    if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
    if (grid < 1) grid = 1;
    tiled_sample_kernel<G, NV, U><<<(unsigned)grid, 256, 0, st>>>(p, tp, q, xi, idx, n, out, tile_out);
    return cudaGetLastError();
}

template <int G, bool U>
static cudaError_t ts_nv(int NV, const QParams& p, const TileParams& tp, const pndf_query* q, const float* xi,
                         const uint32_t* ix, int64_t n, pndf_sample* out, int32_t* to, int sms, cudaStream_t st) {
    switch (NV) {
        case 1: return launch_ts<G, 1, U>(p, tp, q, xi, ix, n, out, to, sms, st);
        case 2: return launch_ts<G, 2, U>(p, tp, q, xi, ix, n, out, to, sms, st);
        case 3: return launch_ts<G, 3, U>(p, tp, q, xi, ix, n, out, to, sms, st);
        case 4: return launch_ts<G, 4, U>(p, tp, q, xi, ix, n, out, to, sms, st);
        case 8: return launch_ts<G, 8, U>(p, tp, q, xi, ix, n, out, to, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

template <bool U>
static cudaError_t ts_g(int G, int NV, const QParams& p, const TileParams& tp, const pndf_query* q, const float* xi,
                        const uint32_t* ix, int64_t n, pndf_sample* out, int32_t* to, int sms, cudaStream_t st) {
    switch (G) {
        case 1: return ts_nv<1, U>(NV, p, tp, q, xi, ix, n, out, to, sms, st);
        case 2: return ts_nv<2, U>(NV, p, tp, q, xi, ix, n, out, to, sms, st);
        case 4: return ts_nv<4, U>(NV, p, tp, q, xi, ix, n, out, to, sms, st);
        case 8: return ts_nv<8, U>(NV, p, tp, q, xi, ix, n, out, to, sms, st);
        case 16: return ts_nv<16, U>(NV, p, tp, q, xi, ix, n, out, to, sms, st);
        case 32: return ts_nv<32, U>(NV, p, tp, q, xi, ix, n, out, to, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tiled_sample(const QParams& p, const TileParams& tp, int G, int NV, const pndf_query* q,
                                const float* xi, const uint32_t* idx, int64_t n, pndf_sample* out,
                                int32_t* tile_out, int num_sms, cudaStream_t st) {
    if (4 * G * NV != p.Rp) return cudaErrorInvalidValue;
    if (p.prefix_u32) return ts_g<true>(G, NV, p, tp, q, xi, idx, n, out, tile_out, num_sms, st);
    return ts_g<false>(G, NV, p, tp, q, xi, idx, n, out, tile_out, num_sms, st);
}

template <int G, int NV, bool U>
static cudaError_t launch_t(const QParams& p, const TileParams& tp, const pndf_query* q, const uint32_t* idx,
                            int64_t n, float* out, int num_sms, cudaStream_t st) {
    const int64_t qpb = 8 * (32 / G);
    int64_t grid = (n + qpb - 1) / qpb;
    if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
    if (grid < 1) grid = 1;
    tiled_query_kernel<G, NV, U><<<(unsigned)grid, 256, 0, st>>>(p, tp, q, idx, n, out);
    return cudaGetLastError();
}

template <int G, bool U>
static cudaError_t t_nv(int NV, const QParams& p, const TileParams& tp, const pndf_query* q, const uint32_t* ix,
                        int64_t n, float* out, int sms, cudaStream_t st) {
    switch (NV) {
        case 1: return launch_t<G, 1, U>(p, tp, q, ix, n, out, sms, st);
        case 2: return launch_t<G, 2, U>(p, tp, q, ix, n, out, sms, st);
        case 3: return launch_t<G, 3, U>(p, tp, q, ix, n, out, sms, st);
        case 4: return launch_t<G, 4, U>(p, tp, q, ix, n, out, sms, st);
        case 8: return launch_t<G, 8, U>(p, tp, q, ix, n, out, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

template <bool U>
static cudaError_t t_g(int G, int NV, const QParams& p, const TileParams& tp, const pndf_query* q,
                       const uint32_t* ix, int64_t n, float* out, int sms, cudaStream_t st) {
    switch (G) {
        case 1: return t_nv<1, U>(NV, p, tp, q, ix, n, out, sms, st);
        case 2: return t_nv<2, U>(NV, p, tp, q, ix, n, out, sms, st);
        case 4: return t_nv<4, U>(NV, p, tp, q, ix, n, out, sms, st);
        case 8: return t_nv<8, U>(NV, p, tp, q, ix, n, out, sms, st);
        case 16: return t_nv<16, U>(NV, p, tp, q, ix, n, out, sms, st);
        case 32: return t_nv<32, U>(NV, p, tp, q, ix, n, out, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_tiled_query(const QParams& p, const TileParams& tp, int G, int NV, const pndf_query* q,
                               const uint32_t* idx, int64_t n, float* out, int num_sms, cudaStream_t st) {
    if (4 * G * NV != p.Rp) return cudaErrorInvalidValue;
    if (p.prefix_u32) return t_g<true>(G, NV, p, tp, q, idx, n, out, num_sms, st);
    return t_g<false>(G, NV, p, tp, q, idx, n, out, num_sms, st);
}

}  // namespace pndf
