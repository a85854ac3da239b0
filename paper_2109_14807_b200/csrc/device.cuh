// device.cuh -- device helpers shared by the query and sampling kernels:
// record decode (a2 level select, a3 neighbour cells),
// the binning key, and TMA / mbarrier wrappers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace pndf {

// ------------------------------------------------------------ helpers --
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// L1 cache policies for the gather (experiments; both off by default): stream the
// positional rows past L1 (ZNA) / keep SAT rows with evict_last priority (SATEL).
// Measured on B200, config 5: ZNA 20% slower, SATEL 21% slower than plain LDG.
#ifndef PNDF_ZNA
#define PNDF_ZNA 0
#endif
#ifndef PNDF_SATEL
#define PNDF_SATEL 0
#endif
__device__ __forceinline__ float4 ldg4_stream(const float* p) {
#if PNDF_ZNA
    float4 r;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
#else
    return ldg4(p);
#endif
}
__device__ __forceinline__ uint4 ldg_sat(const void* p) {
#if PNDF_SATEL
    uint4 r;
    asm("ld.global.nc.L1::evict_last.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
#else
    return __ldg(reinterpret_cast<const uint4*>(p));
#endif
}

__device__ __forceinline__ pndf_query ldg_query(const pndf_query* q) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(q));
    pndf_query r;
    r.u = __uint_as_float(v.x);
    r.v = __uint_as_float(v.y);
    r.size = __uint_as_float(v.z);
    r.rect = v.w;
    return r;
}

// --------------------------------------------- TMA bulk copy + mbarrier --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// one contiguous global -> shared copy on the TMA engine, completion counted on bar
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// off_l = sum_{m<l} (n0 >> m)^2 = 4 n_l^2 (4^l - 1)/3 for power-of-two n0, and
// (4^l - 1)/3 = 0x5555... (l bit pairs): exact, no division.
__device__ __forceinline__ int64_t level_offset(int64_t n0, int l) {
    const int64_t nl = n0 >> l;
    const uint64_t m = l ? (0x5555555555555555ULL >> (64 - 2 * l)) : 0ULL;
    return (int64_t)((uint64_t)(nl * nl) * 4ULL * m);
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
template <bool WRAP>
__device__ __forceinline__ void axis_cells(const QParams& p, float u, int l, int& i0, int& i1, float& a) {
    const int n = p.n0 >> l;
    const float f = fmaf(u, __int_as_float(__float_as_int(p.inv_s0) - (l << 23)), -0.5f);  // u / (s0 2^l) - 1/2
    const float fl = floorf(f);
    a = f - fl;
    i0 = (int)fl;
    i1 = i0 + 1;
    if (WRAP) {
        i0 &= n - 1;
        i1 &= n - 1;
    } else {
        i0 = min(max(i0, 0), n - 1);
        i1 = min(max(i1, 0), n - 1);
    }
}

// a1 key: the record's half cell on its lower level l0, Z-ordered within the level:
//   key = 4 off_{l0} + Morton(floor(2 f_u) mod 2n, floor(2 f_v) mod 2n).
// With wrapped neighbours, equal keys <=> the same 8 Zc rows (level l0's cell is
// floor(f) and level l0+1's cell floor((floor(2f) - 1)/4) -- both functions of
// floor(2f)).  half = 0 falls back to cell keys off_{l0} + Morton(i0, j0).
__device__ __forceinline__ uint64_t part1by1_64(uint64_t x) {
    x &= 0x00000000ffffffffULL;
    x = (x | (x << 16)) & 0x0000ffff0000ffffULL;
    x = (x | (x << 8)) & 0x00ff00ff00ff00ffULL;
    x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0fULL;
    x = (x | (x << 2)) & 0x3333333333333333ULL;
    x = (x | (x << 1)) & 0x5555555555555555ULL;
    return x;
}

__device__ __forceinline__ uint32_t cell_key(const QParams& p, const pndf_query& rec, int l0, int half) {
    const int64_t n_l = p.n0 >> l0;
    const float inv_s = __int_as_float(__float_as_int(p.inv_s0) - (l0 << 23));
    const int64_t m = (n_l << half) - 1;
    const float fu = fmaf(rec.u, inv_s, -0.5f), fv = fmaf(rec.v, inv_s, -0.5f);
    const int64_t hu = (int64_t)floorf(half ? 2.f * fu : fu) & m;
    const int64_t hv = (int64_t)floorf(half ? 2.f * fv : fv) & m;
    return (uint32_t)((level_offset(p.n0, l0) << (2 * half)) +
                      (int64_t)(part1by1_64((uint64_t)hu) | (part1by1_64((uint64_t)hv) << 1)));
}


}  // namespace pndf
