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
