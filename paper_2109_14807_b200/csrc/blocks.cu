// blocks.cu -- the paper-faithful blocked / clustered store (Sec. 4.2,
// P:294-311): build kernels and the query kernel.
//
// Query: for each of the 8 trilinear neighbours (row z, weight w) and each t x t
// angular block b the rectangle overlaps ("we subdivide it into smaller ones
// according to the boundary of the image blocks"): slab = slab_ptr[z][b]
// (-1: blank block, pruned -- contributes 0), set = group_set[region(z), b], and
// Eq. 6 on the block-local sub-rectangle with that set's SATs and the slab's
// Zc row.  Unlike the one-group store the SAT rows depend on the neighbour (its
// group), so they are fetched per neighbour and block, as the paper's P:327.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.h"

namespace pndf {

// one thread per (set, table, rank): fp64 running sum -> (hi, lo) fp32, layout
// pool[set][table][t+1][2][Rp]; flags bit 0 on a negative / non-finite factor
__global__ void block_prefix_kernel(const float* __restrict__ X, const float* __restrict__ Y, int sets, int t, int R,
                                    int Rp, float* pool, uint32_t* flags) {
    const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (int64_t)sets * 2 * Rp) return;
    const int r = (int)(id % Rp);
    const int table = (int)((id / Rp) % 2);
    const int64_t set = id / (2 * Rp);
    const float* F = (table ? Y : X) + set * t * R;
    float* o = pool + ((set * 2 + table) * (t + 1)) * 2 * (int64_t)Rp;
    double S = 0.0;
    bool bad = false;
    for (int k = 0; k <= t; ++k) {
        const float hi = (float)S;
        o[(2 * k) * (int64_t)Rp + r] = hi;
        o[(2 * k + 1) * (int64_t)Rp + r] = (float)(S - (double)hi);
        if (k < t && r < R) {
            const float v = F[(int64_t)k * R + r];
            bad |= !(v >= 0.f) || isinf(v);
            S += (double)v;
        }
    }
    if (bad) atomicOr(flags, 1u);
}

// Zc[slab][r] = fl32(C[set(slab)][r] * Z[slab][r]), padded ranks 0
__global__ void block_fold_kernel(const float* Z, int64_t slabs, int R, const float* __restrict__ C,
                                  const int32_t* __restrict__ slab_set, float* Zc, int Rp, uint32_t* flags) {
    bool bad = false;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < slabs * Rp;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sl = e / Rp;
        const int r = (int)(e - sl * Rp);
        float v = 0.f;
        if (r < R) {
            const float z = Z[sl * R + r], c = C[(int64_t)slab_set[sl] * R + r];
            bad |= !(z >= 0.f) || isinf(z) || !(c >= 0.f) || isinf(c);
            v = c * z;
        }
        Zc[e] = v;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

template <int G, int NV, bool WRAP>
__global__ void __launch_bounds__(256) blocked_query_kernel(const QParams p, const BlockParams bp,
                                                            const pndf_query* __restrict__ q, int64_t n,
                                                            float* __restrict__ out) {
    constexpr int QPW = 32 / G;
    constexpr int RP = 4 * G * NV;
    const int lane = threadIdx.x & 31, gl = lane % G, grp = lane / G;
    const int t = bp.t, nb = bp.nb, nb2 = bp.nb * bp.nb;
    const int64_t tstride = (int64_t)(t + 1) * 2 * RP;  // one SAT table of a set
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = gw * QPW; base < n; base += nw * QPW) {
        const int64_t qi = base + grp;
        const bool active = qi < n;
        const pndf_query rec = ldg_query(q + (active ? qi : 0));
        int x1, x2, y1, y2;
        const bool valid = active && record_valid(p, rec, x1, x2, y1, y2);
        float part = 0.f;
        if (valid) {
            int l0;
            float tl;
            level_select(p, rec.size, l0, tl);
            const int bx0 = x1 / t, bx1 = x2 / t, by0 = y1 / t, by1 = y2 / t;  // the rectangle's blocks
            for (int dl = 0; dl < 2; ++dl) {
                const int l = l0 + dl;
                const float wl = dl ? tl : 1.f - tl;
                int i0, i1, j0, j1;
                float a, b;
                axis_cells<WRAP>(p, rec.u, l, i0, i1, a);
                axis_cells<WRAP>(p, rec.v, l, j0, j1, b);
                const int nl = p.n0 >> l;
                const int lsh = __ffs(p.N / p.n0) - 1 + l;  // log2(s0 * 2^l)
                const int off = (int)level_offset(p.n0, l);  // 32-bit row math: P < 2^31
                const float wa = wl * (1.f - a), wb = wl * a;
                const float wk4[4] = {wa * (1.f - b), wb * (1.f - b), wa * b, wb * b};
                for (int k = 0; k < 4; ++k) {
                    const float wk = wk4[k];
                    if (wk == 0.f) continue;  // group-uniform
                    const int i = (k & 1) ? i1 : i0, j = (k >> 1) ? j1 : j0;
                    const int z = off + j * nl + i;
                    // region of the centre ((i+1/2)s, (j+1/2)s) = floor((2i+1) s / (2 region)); s and region
                    // are powers of two, so a shift (a 64-bit division here costs ~70 instructions)
                    const int rsh = lsh - 1 - bp.r_shift;
                    const int reg = (rsh >= 0 ? ((2 * j + 1) << rsh) : ((2 * j + 1) >> -rsh)) * bp.nr +
                                    (rsh >= 0 ? ((2 * i + 1) << rsh) : ((2 * i + 1) >> -rsh));
                    const int32_t* __restrict__ slab_row = bp.slab_ptr + (int64_t)z * nb2;
                    const int32_t* __restrict__ set_row = bp.group_set + (int64_t)reg * nb2;
                    for (int byb = by0; byb <= by1; ++byb)
                        for (int bxb = bx0; bxb <= bx1; ++bxb) {
                            const int blk = byb * nb + bxb;
                            const int32_t slab = __ldg(slab_row + blk);
                            if (slab < 0) continue;  // blank block
                            const int32_t set = __ldg(set_row + blk);
                            if (set < 0) continue;
                            const int lx1 = max(x1, bxb * t) - bxb * t, lx2 = min(x2, bxb * t + t - 1) - bxb * t;
                            const int ly1 = max(y1, byb * t) - byb * t, ly2 = min(y2, byb * t + t - 1) - byb * t;
                            const float* SX = p.PXY + (int64_t)set * 2 * tstride;
                            const float* SY = SX + tstride;
                            const float* px0 = SX + (int64_t)(2 * lx1) * RP;
                            const float* px1 = SX + (int64_t)(2 * (lx2 + 1)) * RP;
                            const float* py0 = SY + (int64_t)(2 * ly1) * RP;
                            const float* py1 = SY + (int64_t)(2 * (ly2 + 1)) * RP;
#pragma unroll
                            for (int v = 0; v < NV; ++v) {
                                const int c = (gl + v * G) * 4;
                                const float4 xh1 = ldg4(px1 + c), xh0 = ldg4(px0 + c);
                                const float4 xl1 = ldg4(px1 + RP + c), xl0 = ldg4(px0 + RP + c);
                                const float4 yh1 = ldg4(py1 + c), yh0 = ldg4(py0 + c);
                                const float4 yl1 = ldg4(py1 + RP + c), yl0 = ldg4(py0 + RP + c);
                                const float4 zr = ldg4(p.Zc + (int64_t)slab * RP + c);
                                const float dx0 = (xh1.x - xh0.x) + (xl1.x - xl0.x), dy0 = (yh1.x - yh0.x) + (yl1.x - yl0.x);
                                const float dx1 = (xh1.y - xh0.y) + (xl1.y - xl0.y), dy1 = (yh1.y - yh0.y) + (yl1.y - yl0.y);
                                const float dx2 = (xh1.z - xh0.z) + (xl1.z - xl0.z), dy2 = (yh1.z - yh0.z) + (yl1.z - yl0.z);
                                const float dx3 = (xh1.w - xh0.w) + (xl1.w - xl0.w), dy3 = (yh1.w - yh0.w) + (yl1.w - yl0.w);
                                float acc = dx0 * dy0 * zr.x;
                                acc = fmaf(dx1 * dy1, zr.y, acc);
                                acc = fmaf(dx2 * dy2, zr.z, acc);
                                acc = fmaf(dx3 * dy3, zr.w, acc);
                                part = fmaf(wk, acc, part);
                            }
                        }
                }
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

// ---------------------------------------------------------------- importance sampling --
// The footprint's 8 neighbours on the blocked store: Zc row, region and weight.
struct BFoot {
    int32_t z[8], reg[8];
    float w[8];
};

template <bool WRAP>
__device__ __forceinline__ void blocked_foot(const QParams& p, const BlockParams& bp, const pndf_query& rec,
                                             BFoot& f) {
    int l0;
    float tl;
    level_select(p, rec.size, l0, tl);
    for (int dl = 0; dl < 2; ++dl) {
        const int l = l0 + dl;
        const float wl = dl ? tl : 1.f - tl;
        int i0, i1, j0, j1;
        float a, b;
        axis_cells<WRAP>(p, rec.u, l, i0, i1, a);
        axis_cells<WRAP>(p, rec.v, l, j0, j1, b);
        const int nl = p.n0 >> l;
        const int lsh = __ffs(p.N / p.n0) - 1 + l;
        const int off = (int)level_offset(p.n0, l);
        const float wa = wl * (1.f - a), wb = wl * a;
        const float wk4[4] = {wa * (1.f - b), wb * (1.f - b), wa * b, wb * b};
        for (int k = 0; k < 4; ++k) {
            const int i = (k & 1) ? i1 : i0, j = (k >> 1) ? j1 : j0;
            const int rsh = lsh - 1 - bp.r_shift;
            f.z[4 * dl + k] = off + j * nl + i;
            f.reg[4 * dl + k] = (rsh >= 0 ? ((2 * j + 1) << rsh) : ((2 * j + 1) >> -rsh)) * bp.nr +
                                (rsh >= 0 ? ((2 * i + 1) << rsh) : ((2 * i + 1) >> -rsh));
            f.w[4 * dl + k] = wk4[k];
        }
    }
}

// This lane's part of the Eq. 6 SUM over bins [xa, xb) x [ya, yb) inside angular block (bx, by), blended over
// the 8 neighbours (each with its group's SATs); 0 outside the block or on blank blocks.
template <int G, int NV>
__device__ __forceinline__ float block_rect_part(const QParams& p, const BlockParams& bp, const BFoot& f, int bx,
                                                 int by, int xa, int xb, int ya, int yb, int gl) {
    constexpr int RP = 4 * G * NV;
    const int t = bp.t, nb2 = bp.nb * bp.nb;
    const int lx1 = max(xa, bx * t) - bx * t, lx2 = min(xb, bx * t + t) - bx * t;
    const int ly1 = max(ya, by * t) - by * t, ly2 = min(yb, by * t + t) - by * t;
    if (lx2 <= lx1 || ly2 <= ly1) return 0.f;
    const int blk = by * bp.nb + bx;
    const int64_t tstride = (int64_t)(t + 1) * 2 * RP;
    float part = 0.f;
    for (int k = 0; k < 8; ++k) {
        const float wk = f.w[k];
        if (wk == 0.f) continue;
        const int32_t slab = __ldg(bp.slab_ptr + (int64_t)f.z[k] * nb2 + blk);
        if (slab < 0) continue;  // blank block
        const int32_t set = __ldg(bp.group_set + (int64_t)f.reg[k] * nb2 + blk);
        if (set < 0) continue;
        const float* SX = p.PXY + (int64_t)set * 2 * tstride;
        const float* SY = SX + tstride;
        const float* px0 = SX + (int64_t)(2 * lx1) * RP;
        const float* px1 = SX + (int64_t)(2 * lx2) * RP;
        const float* py0 = SY + (int64_t)(2 * ly1) * RP;
        const float* py1 = SY + (int64_t)(2 * ly2) * RP;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int c = (gl + v * G) * 4;
            const float4 xh1 = ldg4(px1 + c), xh0 = ldg4(px0 + c);
            const float4 xl1 = ldg4(px1 + RP + c), xl0 = ldg4(px0 + RP + c);
            const float4 yh1 = ldg4(py1 + c), yh0 = ldg4(py0 + c);
            const float4 yl1 = ldg4(py1 + RP + c), yl0 = ldg4(py0 + RP + c);
            const float4 zr = ldg4(p.Zc + (int64_t)slab * RP + c);
            float acc = ((xh1.x - xh0.x) + (xl1.x - xl0.x)) * ((yh1.x - yh0.x) + (yl1.x - yl0.x)) * zr.x;
            acc = fmaf(((xh1.y - xh0.y) + (xl1.y - xl0.y)) * ((yh1.y - yh0.y) + (yl1.y - yl0.y)), zr.y, acc);
            acc = fmaf(((xh1.z - xh0.z) + (xl1.z - xl0.z)) * ((yh1.z - yh0.z) + (yl1.z - yl0.z)), zr.z, acc);
            acc = fmaf(((xh1.w - xh0.w) + (xl1.w - xl0.w)) * ((yh1.w - yh0.w) + (yl1.w - yl0.w)), zr.w, acc);
            part = fmaf(wk, acc, part);
        }
    }
    return part;
}

template <int G>
__device__ __forceinline__ float bgroup_sum(float v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One sample per group of G lanes: (1) the record rectangle's angular blocks weighted by their blended sums,
// one chosen with xi[10]; (2) the quad descent inside it with xi[0..7]; jitter xi[8..9].
// The choice rules are the oracle's (oracle_blocked_sample_batch), taken in fp32.  Every loop runs until all
// groups of the warp are done, so the shuffles stay warp-uniform.
constexpr int kMaxBlocks = 256;
template <int G, int NV, bool WRAP>
__global__ void __launch_bounds__(256) blocked_sample_kernel(const QParams p, const BlockParams bp,
                                                             const pndf_query* __restrict__ q,
                                                             const float* __restrict__ xi, int64_t n,
                                                             pndf_sample* __restrict__ out, int32_t* block_out) {
    constexpr int QPW = 32 / G;
    extern __shared__ float sS[];  // [8 * QPW][nb^2] block weights of each group's sample
    const int lane = threadIdx.x & 31, gl = lane % G, grp = lane / G;
    const int t = bp.t, nb = bp.nb, nb2 = bp.nb * bp.nb;
    float* S = sS + ((threadIdx.x >> 5) * QPW + grp) * nb2;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = gw * QPW; base < n; base += nw * QPW) {
        const int64_t si = base + grp;
        const bool active = si < n;
        const pndf_query rec = ldg_query(q + (active ? si : 0));
        int x1, x2, y1, y2;
        const bool valid = active && record_valid(p, rec, x1, x2, y1, y2);
        if (!valid) x1 = x2 = y1 = y2 = 0;
        BFoot f;
        blocked_foot<WRAP>(p, bp, valid ? rec : pndf_query{0.f, 0.f, 1.f, 0u}, f);
        if (!valid)
            for (int k = 0; k < 8; ++k) f.w[k] = 0.f;
        const float* sxi = xi + (size_t)(active ? si : 0) * 11;
        // 1. block weights over the rectangle, in block order (by, bx)
        float total = 0.f;
        for (int j = 0; j < nb2; ++j) {
            const float sb = bgroup_sum<G>(block_rect_part<G, NV>(p, bp, f, j % nb, j / nb, x1, x2 + 1, y1, y2 + 1, gl));
            if (gl == 0) S[j] = sb;
            total += sb;
        }
        __syncwarp();
        const bool live = valid && total > 0.f;
        int kb = -1;
        if (live) {
            const float tb = __ldg(sxi + 10) * total;
            float cum = 0.f;
            int lastnz = -1;
            for (int j = 0; j < nb2; ++j) {
                const float sb = S[j];
                cum += sb;
                if (sb > 0.f) lastnz = j;
                if (kb < 0 && tb < cum) kb = j;
            }
            if (kb < 0) kb = lastnz;
        }
        __syncwarp();
        const int bx = kb >= 0 ? kb % nb : 0, by = kb >= 0 ? kb / nb : 0;
        // 2. quad descent inside the chosen block (as sample_kernel)
        int xa = max(x1, bx * t), xb = min(x2 + 1, bx * t + t), ya = max(y1, by * t), yb = min(y2 + 1, by * t + t);
        float last = live ? S[kb] : 0.f;
        int lvl = 0;
        while (__any_sync(0xffffffffu, live && (xb - xa > 1 || yb - ya > 1))) {
            const bool go = live && (xb - xa > 1 || yb - ya > 1);
            const int xm = go ? xa + (xb - xa + 1) / 2 : xb, ym = go ? ya + (yb - ya + 1) / 2 : yb;
            float qs[4];
            qs[0] = bgroup_sum<G>(go ? block_rect_part<G, NV>(p, bp, f, bx, by, xa, xm, ya, ym, gl) : 0.f);
            qs[1] = bgroup_sum<G>(go ? block_rect_part<G, NV>(p, bp, f, bx, by, xm, xb, ya, ym, gl) : 0.f);
            qs[2] = bgroup_sum<G>(go ? block_rect_part<G, NV>(p, bp, f, bx, by, xa, xm, ym, yb, gl) : 0.f);
            qs[3] = bgroup_sum<G>(go ? block_rect_part<G, NV>(p, bp, f, bx, by, xm, xb, ym, yb, gl) : 0.f);
            if (go) {
                const float tot = ((qs[0] + qs[1]) + qs[2]) + qs[3];
                const float tt = __ldg(sxi + lvl) * tot;
                float c = 0.f;
                int k = -1;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    c += qs[j];
                    if (k < 0 && tt < c) k = j;
                }
                if (k < 0) k = qs[3] > 0.f ? 3 : (qs[2] > 0.f ? 2 : (qs[1] > 0.f ? 1 : 0));
                if (k & 1) xa = xm; else xb = xm;
                if (k & 2) ya = ym; else yb = ym;
                last = qs[k];
                ++lvl;
            }
        }
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
                o.pdf = (last / total) / (inv * inv);
                o.pixel = (uint32_t)xa | ((uint32_t)ya << 16);
            }
            out[si] = o;
            if (block_out) block_out[si] = live ? kb : -1;
        }
    }
}

template <int G, int NV, bool W>
static cudaError_t launch_bs(const QParams& p, const BlockParams& bp, const pndf_query* q, const float* xi, int64_t n,
                             pndf_sample* out, int32_t* blk, int num_sms, cudaStream_t st) {
    const int64_t spb = 8 * (32 / G);
    int64_t grid = (n + spb - 1) / spb;
    if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
    if (grid < 1) grid = 1;
    const size_t smem = sizeof(float) * 8 * (32 / G) * bp.nb * bp.nb;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(blocked_sample_kernel<G, NV, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    blocked_sample_kernel<G, NV, W><<<(unsigned)grid, 256, smem, st>>>(p, bp, q, xi, n, out, blk);
    return cudaGetLastError();
}

template <bool W>
static cudaError_t bs_g(int G, int NV, const QParams& p, const BlockParams& bp, const pndf_query* q, const float* xi,
                        int64_t n, pndf_sample* out, int32_t* blk, int sms, cudaStream_t st) {
    // the lane splits of the configs' blocked stores (R <= 128); others: EINVAL from the caller
    if (G == 8 && NV == 1) return launch_bs<8, 1, W>(p, bp, q, xi, n, out, blk, sms, st);
    if (G == 16 && NV == 1) return launch_bs<16, 1, W>(p, bp, q, xi, n, out, blk, sms, st);
    if (G == 32 && NV == 1) return launch_bs<32, 1, W>(p, bp, q, xi, n, out, blk, sms, st);
    if (G == 4 && NV == 1) return launch_bs<4, 1, W>(p, bp, q, xi, n, out, blk, sms, st);
    if (G == 2 && NV == 1) return launch_bs<2, 1, W>(p, bp, q, xi, n, out, blk, sms, st);
    if (G == 1 && NV == 1) return launch_bs<1, 1, W>(p, bp, q, xi, n, out, blk, sms, st);
    return cudaErrorInvalidValue;
}

cudaError_t launch_blocked_sample(const QParams& p, const BlockParams& bp, int G, int NV, const pndf_query* q,
                                  const float* xi, int64_t n, pndf_sample* out, int32_t* blk, int num_sms,
                                  cudaStream_t st) {
    if (4 * G * NV != p.Rp || bp.nb * bp.nb > kMaxBlocks) return cudaErrorInvalidValue;
    if (p.wrap) return bs_g<true>(G, NV, p, bp, q, xi, n, out, blk, num_sms, st);
    return bs_g<false>(G, NV, p, bp, q, xi, n, out, blk, num_sms, st);
}

template <int G, int NV, bool W>
static cudaError_t launch_b(const QParams& p, const BlockParams& bp, const pndf_query* q, int64_t n, float* out,
                            int num_sms, cudaStream_t st) {
    const int64_t qpb = 8 * (32 / G);
    int64_t grid = (n + qpb - 1) / qpb;
    if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
    if (grid < 1) grid = 1;
    blocked_query_kernel<G, NV, W><<<(unsigned)grid, 256, 0, st>>>(p, bp, q, n, out);
    return cudaGetLastError();
}

template <int G, bool W>
static cudaError_t b_nv(int NV, const QParams& p, const BlockParams& bp, const pndf_query* q, int64_t n, float* out,
                        int sms, cudaStream_t st) {
    switch (NV) {
        case 1: return launch_b<G, 1, W>(p, bp, q, n, out, sms, st);
        case 2: return launch_b<G, 2, W>(p, bp, q, n, out, sms, st);
        case 3: return launch_b<G, 3, W>(p, bp, q, n, out, sms, st);
        case 4: return launch_b<G, 4, W>(p, bp, q, n, out, sms, st);
        case 8: return launch_b<G, 8, W>(p, bp, q, n, out, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

template <bool W>
static cudaError_t b_g(int G, int NV, const QParams& p, const BlockParams& bp, const pndf_query* q, int64_t n,
                       float* out, int sms, cudaStream_t st) {
    switch (G) {
        case 1: return b_nv<1, W>(NV, p, bp, q, n, out, sms, st);
        case 2: return b_nv<2, W>(NV, p, bp, q, n, out, sms, st);
        case 4: return b_nv<4, W>(NV, p, bp, q, n, out, sms, st);
        case 8: return b_nv<8, W>(NV, p, bp, q, n, out, sms, st);
        case 16: return b_nv<16, W>(NV, p, bp, q, n, out, sms, st);
        case 32: return b_nv<32, W>(NV, p, bp, q, n, out, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_blocked_query(const QParams& p, const BlockParams& bp, int G, int NV, const pndf_query* q,
                                 int64_t n, float* out, int num_sms, cudaStream_t st) {
    if (4 * G * NV != p.Rp) return cudaErrorInvalidValue;
    if (p.wrap) return b_g<true>(G, NV, p, bp, q, n, out, num_sms, st);
    return b_g<false>(G, NV, p, bp, q, n, out, num_sms, st);
}

cudaError_t launch_block_build(const float* X, const float* Y, int sets, int t, int R, int Rp, float* pool,
                               const float* Z, int64_t slabs, const float* C, const int32_t* slab_set, float* Zc,
                               uint32_t* flags, int num_sms, cudaStream_t st) {
    const int64_t th = (int64_t)sets * 2 * Rp;
    block_prefix_kernel<<<(unsigned)((th + 127) / 128), 128, 0, st>>>(X, Y, sets, t, R, Rp, pool, flags);
    int64_t g = (slabs * Rp + 255) / 256;
    if (g > (int64_t)num_sms * 16) g = (int64_t)num_sms * 16;
    if (g < 1) g = 1;
    if (slabs > 0) block_fold_kernel<<<(unsigned)g, 256, 0, st>>>(Z, slabs, R, C, slab_set, Zc, Rp, flags);
    return cudaGetLastError();
}

}  // namespace pndf
