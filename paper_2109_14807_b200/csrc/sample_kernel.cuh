// sample_kernel.cuh -- the importance-sampling kernel template and its launch
// dispatch; instantiated per SAT format in sample_u32.cu / sample_hilo.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.h"

namespace pndf {

// a SAT value of the lane's 4 ranks: uint32 fixed point, or fp32 (hi, lo)
template <bool U32>
struct SatV;
template <>
struct SatV<true> {
    uint4 q;
    __device__ __forceinline__ void load(const float* row, int c, int /*RP*/) {
        q = __ldg(reinterpret_cast<const uint4*>(row + c));
    }
    __device__ __forceinline__ static float4 diff(const SatV& a, const SatV& b) {  // b - a
        return make_float4(__uint2float_rn(b.q.x - a.q.x), __uint2float_rn(b.q.y - a.q.y),
                           __uint2float_rn(b.q.z - a.q.z), __uint2float_rn(b.q.w - a.q.w));
    }
};
template <>
struct SatV<false> {
    float4 hi, lo;
    __device__ __forceinline__ void load(const float* row, int c, int RP) {
        hi = ldg4(row + c);
        lo = ldg4(row + RP + c);
    }
    __device__ __forceinline__ static float4 diff(const SatV& a, const SatV& b) {
        return make_float4((b.hi.x - a.hi.x) + (b.lo.x - a.lo.x), (b.hi.y - a.hi.y) + (b.lo.y - a.lo.y),
                           (b.hi.z - a.hi.z) + (b.lo.z - a.lo.z), (b.hi.w - a.hi.w) + (b.lo.w - a.lo.w));
    }
};

template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum q0..q3 over the G lanes of each group with recursive halving (log2 G + 1 shuffles instead of
// 4 log2 G), then gather the four totals into every lane of the group (3 more shuffles).
template <int G>
__device__ __forceinline__ void quad_reduce(float& q0, float& q1, float& q2, float& q3, int gl, int lane) {
    if (G >= 4) {
        constexpr int H = G / 2, Q = G / 4;
        const bool up = (gl & H) != 0;  // upper half keeps (q2, q3)
        float k0 = up ? q2 : q0, k1 = up ? q3 : q1;
        const float s0 = up ? q0 : q2, s1 = up ? q1 : q3;
        k0 += __shfl_xor_sync(0xffffffffu, s0, H);
        k1 += __shfl_xor_sync(0xffffffffu, s1, H);
        const bool up2 = (gl & Q) != 0;  // then keeps k1
        float k = up2 ? k1 : k0;
        k += __shfl_xor_sync(0xffffffffu, up2 ? k0 : k1, Q);
#pragma unroll
        for (int o = Q / 2; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
        // lane gl now holds quad 2*[gl & H] + [gl & Q]
        const int g0 = lane - gl;
        q0 = __shfl_sync(0xffffffffu, k, g0);
        q1 = __shfl_sync(0xffffffffu, k, g0 + Q);
        q2 = __shfl_sync(0xffffffffu, k, g0 + H);
        q3 = __shfl_sync(0xffffffffu, k, g0 + H + Q);
    } else {
        q0 = group_sum<G>(q0);
        q1 = group_sum<G>(q1);
        q2 = group_sum<G>(q2);
        q3 = group_sum<G>(q3);
    }
}

#ifndef PNDF_SRELOAD
#define PNDF_SRELOAD 1  // 1: re-read the range corners each level (fewer registers, no corner moves)
#endif

#ifndef PNDF_SMINB
#define PNDF_SMINB 2  // resident CTAs per SM the register budget targets
#endif

template <int G, int NV, bool WRAP, bool BINNED, bool U32>
__global__ void __launch_bounds__(256, PNDF_SMINB) sample_kernel(const QParams p, const pndf_query* __restrict__ q,
                                                     const float* __restrict__ xi, const uint32_t* __restrict__ idx,
                                                     int64_t n, pndf_sample* __restrict__ out) {
    constexpr int QPW = 32 / G;
    constexpr int RP = 4 * G * NV;
    constexpr int PSTRIDE = U32 ? RP : 2 * RP;
    const int lane = threadIdx.x & 31, gl = lane % G, grp = lane / G;
    const float* __restrict__ PX = p.PXY;
    const float* __restrict__ PY = p.PXY + (size_t)(p.A + 1) * PSTRIDE;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = gw * QPW; base < n; base += nw * QPW) {  // warp-uniform trip count
        const int64_t si = base + grp;
        const bool active = si < n;
        const int64_t src = active ? (BINNED ? (int64_t)__ldg(idx + si) : si) : 0;
        const pndf_query rec = ldg_query(q + src);
        int x1, x2, y1, y2;
        const bool valid = active && record_valid(p, rec, x1, x2, y1, y2);
        if (!valid) {
            x1 = x2 = y1 = y2 = 0;
        }
        // a2/a3: neighbours; a4: Z-hat once per sample
        int l0;
        float t;
        level_select(p, valid ? rec.size : 1.f, l0, t);
        float4 zh[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) zh[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int dl = 0; dl < 2; ++dl) {
            const int l = l0 + dl;
            const float wl = dl ? t : 1.f - t;
            int i0, i1, j0, j1;
            float a, b;
            axis_cells<WRAP>(p, valid ? rec.u : 0.f, l, i0, i1, a);
            axis_cells<WRAP>(p, valid ? rec.v : 0.f, l, j0, j1, b);
            const int32_t nl = p.n0 >> l;
            const int32_t off = (int32_t)level_offset(p.n0, l);
            const int row[4] = {off + j0 * nl + i0, off + j0 * nl + i1, off + j1 * nl + i0, off + j1 * nl + i1};
            const float wa = wl * (1.f - a), wb = wl * a;
            const float w[4] = {wa * (1.f - b), wb * (1.f - b), wa * b, wb * b};
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int c = (gl + v * G) * 4;
                float4 zr[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) zr[k] = ldg4(p.Zc + (size_t)row[k] * RP + c);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    zh[v].x = fmaf(w[k], zr[k].x, zh[v].x);
                    zh[v].y = fmaf(w[k], zr[k].y, zh[v].y);
                    zh[v].z = fmaf(w[k], zr[k].z, zh[v].z);
                    zh[v].w = fmaf(w[k], zr[k].w, zh[v].w);
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
        float root = 0.f;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 dx = SatV<U32>::diff(sxa[v], sxb[v]), dy = SatV<U32>::diff(sya[v], syb[v]);
            root = fmaf(dx.x * dy.x, zh[v].x, root);
            root = fmaf(dx.y * dy.y, zh[v].y, root);
            root = fmaf(dx.z * dy.z, zh[v].z, root);
            root = fmaf(dx.w * dy.w, zh[v].w, root);
        }
        root = group_sum<G>(root);
        const bool live = valid && root > 0.f;
        float last = root;
        const float* sxi = xi + (size_t)src * 10;
        // descent: the loop bound depends only on the record, uniform within the group;
        // groups of a warp may differ, so every lane keeps shuffling until all are done
        int lvl = 0;
        while (__any_sync(0xffffffffu, live && (xb - xa > 1 || yb - ya > 1))) {
            const bool go = live && (xb - xa > 1 || yb - ya > 1);
            const int xm = go && xb - xa > 1 ? xa + (xb - xa + 1) / 2 : xb;
            const int ym = go && yb - ya > 1 ? ya + (yb - ya + 1) / 2 : yb;
            SatV<U32> sxm[NV], sym[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int c = (gl + v * G) * 4;
#if PNDF_SRELOAD
                // the current range's corners are re-read with the midpoints (L1-resident rows, issued
                // together, so no extra round trip) instead of being carried across levels in registers
                sxa[v].load(PX + (size_t)xa * PSTRIDE, c, RP);
                sxb[v].load(PX + (size_t)xb * PSTRIDE, c, RP);
                sya[v].load(PY + (size_t)ya * PSTRIDE, c, RP);
                syb[v].load(PY + (size_t)yb * PSTRIDE, c, RP);
#endif
                sxm[v].load(PX + (size_t)xm * PSTRIDE, c, RP);
                sym[v].load(PY + (size_t)ym * PSTRIDE, c, RP);
            }
            // quad sums: (x-lo|x-hi) x (y-lo|y-hi), two ranks per packed FFMA2; the y factor and Z-hat
            // are multiplied first (u = ey z, w = fy z) so each quad costs one FMA per rank
            float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float4 dxl = SatV<U32>::diff(sxa[v], sxm[v]), dxr = SatV<U32>::diff(sxm[v], sxb[v]);
                const float4 dyb = SatV<U32>::diff(sya[v], sym[v]), dyt = SatV<U32>::diff(sym[v], syb[v]);
                const float2 z01 = make_float2(zh[v].x, zh[v].y), z23 = make_float2(zh[v].z, zh[v].w);
                const float2 u01 = __fmul2_rn(make_float2(dyb.x, dyb.y), z01);
                const float2 u23 = __fmul2_rn(make_float2(dyb.z, dyb.w), z23);
                const float2 w01 = __fmul2_rn(make_float2(dyt.x, dyt.y), z01);
                const float2 w23 = __fmul2_rn(make_float2(dyt.z, dyt.w), z23);
                const float2 e01 = make_float2(dxl.x, dxl.y), e23 = make_float2(dxl.z, dxl.w);
                const float2 f01 = make_float2(dxr.x, dxr.y), f23 = make_float2(dxr.z, dxr.w);
                a0 = __ffma2_rn(e01, u01, a0);
                a0 = __ffma2_rn(e23, u23, a0);
                a1 = __ffma2_rn(f01, u01, a1);
                a1 = __ffma2_rn(f23, u23, a1);
                a2 = __ffma2_rn(e01, w01, a2);
                a2 = __ffma2_rn(e23, w23, a2);
                a3 = __ffma2_rn(f01, w01, a3);
                a3 = __ffma2_rn(f23, w23, a3);
            }
            float q0 = a0.x + a0.y, q1 = a1.x + a1.y, q2 = a2.x + a2.y, q3 = a3.x + a3.y;
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
#if !PNDF_SRELOAD
#pragma unroll
                    for (int v = 0; v < NV; ++v) sxa[v] = sxm[v];
#endif
                } else {
                    xb = xm;
#if !PNDF_SRELOAD
#pragma unroll
                    for (int v = 0; v < NV; ++v) sxb[v] = sxm[v];
#endif
                }
                if (k & 2) {
                    ya = ym;
#if !PNDF_SRELOAD
#pragma unroll
                    for (int v = 0; v < NV; ++v) sya[v] = sym[v];
#endif
                } else {
                    yb = ym;
#if !PNDF_SRELOAD
#pragma unroll
                    for (int v = 0; v < NV; ++v) syb[v] = sym[v];
#endif
                }
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
            } else if (!live) {  // blank domain: no sample
                o.hx = o.hy = __int_as_float(0x7fc00000);
                o.pdf = 0.f;
                o.pixel = 0xffffffffu;
            } else {
                const float inv = 2.f / (float)p.A;
                o.hx = ((float)xa + __ldg(sxi + 8)) * inv - 1.f;
                o.hy = ((float)ya + __ldg(sxi + 9)) * inv - 1.f;
                o.pdf = (last / root) / (inv * inv);  // pmf / pixel area in projected-h space
                o.pixel = (uint32_t)xa | ((uint32_t)ya << 16);
            }
            out[src] = o;
        }
    }
}

template <int G, int NV, bool W, bool B, bool U>
static cudaError_t launch_s(const QParams& p, const pndf_query* q, const float* xi, const uint32_t* idx, int64_t n,
                            pndf_sample* out, int num_sms, cudaStream_t st) {
    const int64_t spb = 8 * (32 / G);
    int64_t grid = (n + spb - 1) / spb;
    if (grid > (int64_t)num_sms * 8) grid = (int64_t)num_sms * 8;
    if (grid < 1) grid = 1;
    sample_kernel<G, NV, W, B, U><<<(unsigned)grid, 256, 0, st>>>(p, q, xi, idx, n, out);
    return cudaGetLastError();
}

template <int G, bool W, bool B, bool U>
static cudaError_t s_nv(int NV, const QParams& p, const pndf_query* q, const float* xi, const uint32_t* idx,
                        int64_t n, pndf_sample* out, int sms, cudaStream_t st) {
    switch (NV) {
        case 1: return launch_s<G, 1, W, B, U>(p, q, xi, idx, n, out, sms, st);
        case 2: return launch_s<G, 2, W, B, U>(p, q, xi, idx, n, out, sms, st);
        case 3: return launch_s<G, 3, W, B, U>(p, q, xi, idx, n, out, sms, st);
        case 4: return launch_s<G, 4, W, B, U>(p, q, xi, idx, n, out, sms, st);
        case 8: return launch_s<G, 8, W, B, U>(p, q, xi, idx, n, out, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

template <bool W, bool B, bool U>
static cudaError_t s_g(int G, int NV, const QParams& p, const pndf_query* q, const float* xi, const uint32_t* idx,
                       int64_t n, pndf_sample* out, int sms, cudaStream_t st) {
    switch (G) {
        case 1: return s_nv<1, W, B, U>(NV, p, q, xi, idx, n, out, sms, st);
        case 2: return s_nv<2, W, B, U>(NV, p, q, xi, idx, n, out, sms, st);
        case 4: return s_nv<4, W, B, U>(NV, p, q, xi, idx, n, out, sms, st);
        case 8: return s_nv<8, W, B, U>(NV, p, q, xi, idx, n, out, sms, st);
        case 16: return s_nv<16, W, B, U>(NV, p, q, xi, idx, n, out, sms, st);
        case 32: return s_nv<32, W, B, U>(NV, p, q, xi, idx, n, out, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pndf
