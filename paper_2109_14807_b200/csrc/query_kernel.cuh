// query_kernel.cuh -- the query kernel template (rows a2-a6) and its launch
// dispatch; instantiated per SAT format in query_u32.cu / query_hilo.cu so the
// two halves compile in parallel.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "device.cuh"
#include "launch.h"

namespace pndf {

// ------------------------------------------------- decoded query (smem) --
// One warp decodes 32 records at once (one per lane) into these descriptors,
// then the whole warp gathers for them G lanes per query.
struct __align__(16) QDesc {
    int32_t row[8];  // Zc rows of the 8 neighbours (level l0: (i0,j0),(i1,j0),(i0,j1),(i1,j1); then l0+1)
    float w[8];      // trilinear weights (1-t)(1-a)(1-b), ...
    int32_t sat[4];  // SAT rows (entries of PXY) x1, x2+1, A+1+y1, A+1+y2+1 (the 4 look-ups)
    float div;       // rectangle area (MEAN), 1 (SUM), NaN (invalid record)
    int32_t out;     // output index within the (sub-)batch, -1 = no query
    int32_t mode;    // bit 0: x range from the range table DT (sat[0] = its row), bit 1: y likewise (sat[2])
    int32_t pad;
};
static_assert(sizeof(QDesc) == 96, "QDesc layout");

// returns false for an invalid record (its descriptor then yields NaN)
template <bool WRAP, bool USE_DT>  // USE_DT: narrow ranges read the range table (not with TMA staging)
__device__ __forceinline__ bool decode(const QParams& p, const pndf_query& rec, int32_t out_index, QDesc& d) {
    int x1, x2, y1, y2;
    if (!record_valid(p, rec, x1, x2, y1, y2)) {
        atomicOr(p.err, 1u);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            d.row[k] = 0;
            d.w[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) d.sat[k] = 0;
        d.mode = 0;
        d.div = __int_as_float(0x7fc00000);
        d.out = out_index;
        return false;
    }
    int l0;
    float t;
    level_select(p, rec.size, l0, t);
#pragma unroll
    for (int dl = 0; dl < 2; ++dl) {
        const int l = l0 + dl;
        const float wl = dl ? t : 1.f - t;
        int i0, i1, j0, j1;
        float a, b;
        axis_cells<WRAP>(p, rec.u, l, i0, i1, a);
        axis_cells<WRAP>(p, rec.v, l, j0, j1, b);
        const int32_t n = p.n0 >> l;
        const int32_t off = (int32_t)level_offset(p.n0, l);
        d.row[4 * dl + 0] = off + j0 * n + i0;
        d.row[4 * dl + 1] = off + j0 * n + i1;
        d.row[4 * dl + 2] = off + j1 * n + i0;
        d.row[4 * dl + 3] = off + j1 * n + i1;
        const float wa = wl * (1.f - a), wb = wl * a;
        d.w[4 * dl + 0] = wa * (1.f - b);
        d.w[4 * dl + 1] = wb * (1.f - b);
        d.w[4 * dl + 2] = wa * b;
        d.w[4 * dl + 3] = wb * b;
    }
    d.sat[0] = x1;  // PY follows PX: its entries are rows A+1 ...
    d.sat[1] = x2 + 1;
    d.sat[2] = p.A + 1 + y1;
    d.sat[3] = p.A + 2 + y2;
    d.mode = 0;
    if (USE_DT && x2 - x1 < p.dt_w) {  // narrow range: one table row DT[0][x1][w-1] instead of two SAT rows
        d.sat[0] = x1 * p.dt_w + (x2 - x1);
        d.mode |= 1;
    }
    if (USE_DT && y2 - y1 < p.dt_w) {
        d.sat[2] = (p.A + y1) * p.dt_w + (y2 - y1);
        d.mode |= 2;
    }
    d.div = p.mean ? (float)((x2 - x1 + 1) * (y2 - y1 + 1)) : 1.f;
    d.out = out_index;
    return true;
}

// Which of a warp's 32 decoded queries repeat the previous query's Zc rows, per level:
// bit j of *same_lo = query j has query j-1's 4 level-l0 rows, *same_hi likewise for level l0+1.
// A level's 4 rows are fixed by its first and last row: (i0, j0) and (i1, j1) give (i1, j0) and
// (i0, j1).  With wrapped borders the first alone fixes them (i1 = i0 + 1 mod n), but clamped borders
// map f in [-1/2, 0) to cells (0, 0) and f in [0, 1) to (0, 1): same first row, different others,
// so CLAMP compares both.  Equal rows imply the same level (levels own disjoint row ranges).
template <bool WRAP>
__device__ __forceinline__ void reuse_masks(const QDesc& d, bool valid, bool first_ok, int32_t prev_lo,
                                            int32_t prev_lo3, int32_t prev_hi, int32_t prev_hi3,
                                            uint32_t* same_lo, uint32_t* same_hi, int32_t (&mine)[4]) {
    mine[0] = valid ? d.row[0] : -1;
    mine[1] = valid ? d.row[3] : -1;
    mine[2] = valid ? d.row[4] : -1;
    mine[3] = valid ? d.row[7] : -1;
    int32_t plo = __shfl_up_sync(0xffffffffu, mine[0], 1), phi = __shfl_up_sync(0xffffffffu, mine[2], 1);
    int32_t plo3 = 0, phi3 = 0;
    if (!WRAP) {
        plo3 = __shfl_up_sync(0xffffffffu, mine[1], 1);
        phi3 = __shfl_up_sync(0xffffffffu, mine[3], 1);
    }
    const int lane = threadIdx.x & 31;
    if (lane == 0) {  // the query before lane 0 (previous 32-query batch of a segment; -1 = none)
        plo = prev_lo;
        plo3 = prev_lo3;
        phi = prev_hi;
        phi3 = prev_hi3;
    }
    const bool ok = first_ok && valid;
    *same_lo = __ballot_sync(0xffffffffu, ok && mine[0] == plo && (WRAP || mine[1] == plo3));
    *same_hi = __ballot_sync(0xffffffffu, ok && mine[2] == phi && (WRAP || mine[3] == phi3));
}

// Reduce NB per-lane partials v[0..NB) over the G lanes of each group by
// recursive halving: at level o the lanes with bit o set keep the upper half.
// Every value is summed along the same pairing tree (xor G/2, G/4, ..., 1) as a
// plain butterfly, so the result does not depend on the value's slot.
// Afterwards lane gl holds the totals of slots (slot_base(gl) + i) for i < NB/G'.
template <int G, int NB>
__device__ __forceinline__ void group_reduce(float (&v)[NB], int gl) {
    int nv = NB;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        if (nv > 1) {
            const bool upper = (gl & o) != 0;
            const int half = nv / 2;
#pragma unroll
            for (int i = 0; i < NB / 2; ++i) {
                if (i < half) {
                    const float send = upper ? v[i] : v[i + half];
                    const float keep = upper ? v[i + half] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            nv = half;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        }
    }
}

// ------------------------------------------------------- query kernel --
// Work split: CTA b owns the contiguous query range [b*chunk, (b+1)*chunk), so
// binned (sorted) queries that share Zc rows run on the same SM and hit in L1.
// Each warp takes 32 consecutive queries of the CTA's range at a time:
//   1. decode: lane i decodes query i into a QDesc in shared memory, and notes
//      whether it has the same 8 Zc rows as query i-1 (equal half-cell key);
//   2. gather: G lanes per query (QPW = 32/G queries per step); each lane owns
//      NV float4 rank chunks at float offsets (gl + v*G)*4, so a query's G lanes
//      read each row slice contiguously (RP = 4*G*NV is a compile-time stride).
//      With G == 32 the previous query's Zc rows stay in registers and are not
//      re-read when the rows repeat (binned neighbours);
//   3. reduce: per-lane partials of 8 steps are reduced together over the G lanes
//      (group_reduce: 1 shuffle per query instead of log2 G, and no shuffle chain
//      between consecutive queries), then routed to lane (query index) and the
//      warp writes 32 results at once.
// A query's result never depends on where it sits in the batch, so binned and
// unbinned batches are bitwise identical.
constexpr int kWarpsPerBlock = kThreads / 32;
#ifndef PNDF_MINB
#define PNDF_MINB 2  // min resident blocks per SM (tuned on B200: 2 beats 1 and 3, see profiles/)
#endif
#ifndef PNDF_KSTEPS
#define PNDF_KSTEPS 8
#endif
constexpr int kSteps = PNDF_KSTEPS;  // gather steps whose partials are reduced together

#ifndef PNDF_F2
#define PNDF_F2 1  // 1: packed fp32 FFMA2/FMUL2 for the interpolation and rank product (sm_100)
#endif
#ifndef PNDF_WSEG
#define PNDF_WSEG 0  // 1: contiguous per-warp segments with row reuse across 32-query batches (experiment)
#endif
#ifndef PNDF_PREUSE
#define PNDF_PREUSE 1  // 1: per-level Zc row reuse (rows 0-3 / 4-7 separately); 0: all 8 rows or none
#endif
#ifndef PNDF_NOREUSE
#define PNDF_NOREUSE 0  // 1: no cross-step register reuse of Zc rows (fewer live registers; experiment)
#endif
#ifndef PNDF_PF
#define PNDF_PF 0  // 1: prefetch the next step's SAT rows into L1; 2: and its Zc rows (experiment)
#endif
#ifndef PNDF_TMA
#define PNDF_TMA 0  // 1: stage SAT rows of the next query in smem with TMA bulk copies (measured slower on B200)
#endif
constexpr int kSlots = 2;  // per-warp SAT staging slots (prefetch distance 1)

// SAT rows are staged by TMA when a warp runs one query per step (G == 32) and a
// slot (4 rows) is at most 4 KB, so 8 warps x 2 slots fit beside the descriptors.
template <int G, int NV, bool U32>
struct QLayout {
    static constexpr int RP = 4 * G * NV;
    static constexpr int PSTRIDE = U32 ? RP : 2 * RP;  // floats (or uint32) per SAT entry row
    static constexpr bool TMA = PNDF_TMA && G == 32 && PSTRIDE <= 256;
    static constexpr int ROW_BYTES = PSTRIDE * 4;
    static constexpr size_t DESC = sizeof(QDesc) * kWarpsPerBlock * 32;
    static constexpr size_t REUSE = 128;
    static constexpr size_t BARS = TMA ? 128 : 0;
    static constexpr size_t SLOTS = TMA ? (size_t)kWarpsPerBlock * kSlots * 4 * ROW_BYTES : 0;
    static constexpr size_t BYTES = DESC + REUSE + BARS + SLOTS;
};

template <int G, int NV, bool WRAP, bool BINNED, bool U32>
__global__ void __launch_bounds__(kThreads, PNDF_MINB) query_kernel(const QParams p, const pndf_query* __restrict__ q,
                                                         const uint32_t* __restrict__ idx, int64_t n,
                                                         int64_t chunk, float* __restrict__ out) {
    using LY = QLayout<G, NV, U32>;
    constexpr int QPW = 32 / G;
    constexpr int RP = LY::RP;
    constexpr int NSTEP = 32 / QPW;                       // steps per 32-query warp batch
    constexpr int SB = NSTEP < kSteps ? NSTEP : kSteps;   // steps per reduction batch
    constexpr int VPL = SB / G > 0 ? SB / G : 1;          // reduced values left per lane
    constexpr bool TMA = LY::TMA;
    extern __shared__ __align__(128) unsigned char qsmem[];
    QDesc(*sdesc)[32] = reinterpret_cast<QDesc(*)[32]>(qsmem);
    uint32_t* sreuse = reinterpret_cast<uint32_t*>(qsmem + LY::DESC);  // bit j: query j repeats j-1's rows
    uint64_t* sbar = reinterpret_cast<uint64_t*>(qsmem + LY::DESC + LY::REUSE);
    uint32_t* sslot = reinterpret_cast<uint32_t*>(qsmem + LY::DESC + LY::REUSE + LY::BARS);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gl = lane % G, grp = lane / G;
    QDesc* wd = sdesc[warp];
    const float* __restrict__ Zc = p.Zc;
    // SAT rows: HILO = [hi row | lo row] per entry (stride 2*RP floats), U32 = one uint32 row
    constexpr int PSTRIDE = LY::PSTRIDE;
    const float* __restrict__ PXl = p.PXY + gl * 4;  // this lane's first rank chunk of SAT row 0
    const float* __restrict__ DTl = p.DT + gl * 4;   // ... and of range-table row 0
    uint64_t* wbar = sbar + warp * kSlots;
    uint32_t* wslot = sslot + (size_t)warp * kSlots * 4 * PSTRIDE;
    uint32_t phase = 0;  // bit k: parity of slot k's next completion
    if (TMA) {
        if (lane == 0)
            for (int k = 0; k < kSlots; ++k) mbar_init(wbar + k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
    }
    // lane 0: TMA the 4 SAT rows (x1, x2+1, y1, y2+1) of warp-batch query s into slot s % kSlots
    auto issue_sat = [&](int s) {
        if (lane == 0) {
            const QDesc& d = wd[s];
            const int k = s % kSlots;
            uint32_t* dst = wslot + (size_t)k * 4 * PSTRIDE;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // slot was last read by the generic proxy
            mbar_arrive_expect_tx(wbar + k, 4 * LY::ROW_BYTES);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                tma_load_1d(dst + e * PSTRIDE, p.PXY + (size_t)d.sat[e] * PSTRIDE, LY::ROW_BYTES, wbar + k);
        }
    };

    const int64_t c0 = (int64_t)blockIdx.x * chunk;
    float4 zc[NV][8];
#if PNDF_WSEG
    // each warp walks its own contiguous segment of the CTA's range, so the rows of one batch's last
    // query can be reused by the next batch's first
    const int64_t wlen = (((chunk + kWarpsPerBlock - 1) / kWarpsPerBlock) + 31) / 32 * 32;
    const int64_t ws = c0 + (int64_t)warp * wlen;
    const int64_t c1 = min(min(n, c0 + chunk), ws + wlen);
    int32_t prev_r[4] = {-1, -1, -1, -1};
    for (int64_t base = ws; base < c1; base += 32) {
#else
    const int64_t c1 = min(n, c0 + chunk);
    for (int64_t base = c0 + (int64_t)warp * 32; base < c1; base += (int64_t)kWarpsPerBlock * 32) {
#endif
        // 1. decode 32 records, one per lane
        {
            const int64_t qi = base + lane;
            bool valid = false;
            if (qi < c1) {
                // binned: idx is the radix-sorted permutation; gather the record through it
                const int64_t src = BINNED ? (int64_t)__ldg(idx + qi) : qi;
                const pndf_query rec = ldg_query(q + src);
                valid = decode<WRAP, !TMA>(p, rec, (int32_t)src, wd[lane]);
            } else {
                wd[lane].out = -1;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    wd[lane].row[k] = 0;
                    wd[lane].w[k] = 0.f;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) wd[lane].sat[k] = 0;
                wd[lane].mode = 0;
                wd[lane].div = 1.f;
            }
            uint32_t same_lo, same_hi;
            int32_t mine[4];
#if PNDF_WSEG
            // the previous batch's last query (its rows are still in zc)
            reuse_masks<WRAP>(wd[lane], valid, true, prev_r[0], prev_r[1], prev_r[2], prev_r[3], &same_lo,
                              &same_hi, mine);
#pragma unroll
            for (int e = 0; e < 4; ++e) prev_r[e] = __shfl_sync(0xffffffffu, mine[e], 31);
#else
            reuse_masks<WRAP>(wd[lane], valid, lane > 0, -1, -1, -1, -1, &same_lo, &same_hi, mine);
#endif
#if !PNDF_PREUSE
            same_lo = same_hi = same_lo & same_hi;  // all 8 rows or none
#endif
            if (lane == 0) {
                sreuse[2 * warp] = same_lo;
                sreuse[2 * warp + 1] = same_hi;
            }
        }
        __syncwarp();
        const uint32_t reuse_mask = (G == 32) ? (sreuse[2 * warp] & sreuse[2 * warp + 1]) : 0u;
        const uint32_t reuse_lo = (G == 32) ? sreuse[2 * warp] : 0u;
        const uint32_t reuse_hi = (G == 32) ? sreuse[2 * warp + 1] : 0u;
        if (TMA) issue_sat(0);
        // 2-3. gather + batched reduce
        float res = 0.f;
#pragma unroll 1
        for (int s0 = 0; s0 < NSTEP; s0 += SB) {
            float part[SB];
#pragma unroll
            for (int j = 0; j < SB; ++j) {
                const int s = s0 + j;  // step: queries s*QPW + grp
                const QDesc& d = wd[s * QPW + grp];
                if (TMA) {
                    if (s + 1 < NSTEP) issue_sat(s + 1);  // prefetch the next query's SAT rows
                    const int k = s % kSlots;
                    while (!mbar_try_wait(wbar + k, (phase >> k) & 1u)) {
                    }
                    phase ^= 1u << k;
                }
                const float4 w03 = *reinterpret_cast<const float4*>(&d.w[0]);
                const float4 w47 = *reinterpret_cast<const float4*>(&d.w[4]);
                const int4 so = *reinterpret_cast<const int4*>(&d.sat[0]);
                const int dmode = d.mode;  // warp-uniform for G == 32
                const float w[8] = {w03.x, w03.y, w03.z, w03.w, w47.x, w47.y, w47.z, w47.w};
                const bool tx = dmode & 1, ty = (dmode >> 1) & 1;
                const float* px0 = tx ? DTl + (int64_t)so.x * RP : PXl + (int64_t)so.x * PSTRIDE;
                const float* px1 = PXl + (int64_t)so.y * PSTRIDE;
                const float* py0 = ty ? DTl + (int64_t)so.z * RP : PXl + (int64_t)so.z * PSTRIDE;
                const float* py1 = PXl + (int64_t)so.w * PSTRIDE;
#if PNDF_PF
                // software prefetch (into L1) of the next step's SAT rows (and Zc rows with PNDF_PF=2), so
                // their L2 latency overlaps this step's arithmetic; costs no registers or shared memory
                if (!TMA && s + 1 < NSTEP) {
                    const QDesc& dn = wd[(s + 1) * QPW + grp];
                    const int4 sn = *reinterpret_cast<const int4*>(&dn.sat[0]);
                    const int sr[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float* pp = PXl + (int64_t)sr[e] * PSTRIDE;
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            prefetch_l1(pp + v * G * 4);
                            if (!U32) prefetch_l1(pp + RP + v * G * 4);
                        }
                    }
                    if (PNDF_PF >= 2 && !((G == 32) && ((reuse_mask >> (s + 1)) & 1u))) {
#pragma unroll
                        for (int k = 0; k < 8; ++k)
#pragma unroll
                            for (int v = 0; v < NV; ++v) prefetch_l1(Zc + (size_t)dn.row[k] * RP + (gl + v * G) * 4);
                    }
                }
#endif
                // warp-uniform for G == 32 (every lane reads the same descriptor)
                // warp-uniform for G == 32: level l0's rows (0-3) and level l0+1's rows (4-7) are
                // re-read only when they differ from the previous query's
                const bool reuse0 = (G == 32) && (PNDF_WSEG || s > 0) && ((reuse_lo >> s) & 1u);
                const bool reuse1 = (G == 32) && (PNDF_WSEG || s > 0) && ((reuse_hi >> s) & 1u);
                // outer warp-uniform branch: a fully reused step (the common binned case) skips the
                // whole load block instead of issuing it predicated off
                if (__builtin_expect(!PNDF_NOREUSE && !(reuse0 && reuse1), 0)) {
                if (!reuse0) {
                    const uint4 r03 = *reinterpret_cast<const uint4*>(&d.row[0]);
                    const int row[4] = {(int)r03.x, (int)r03.y, (int)r03.z, (int)r03.w};
#pragma unroll
                    for (int v = 0; v < NV; ++v)
#pragma unroll
                        for (int k = 0; k < 4; ++k) zc[v][k] = ldg4_stream(Zc + (size_t)row[k] * RP + (gl + v * G) * 4);
                }
                if (!reuse1) {
                    const uint4 r47 = *reinterpret_cast<const uint4*>(&d.row[4]);
                    const int row[4] = {(int)r47.x, (int)r47.y, (int)r47.z, (int)r47.w};
#pragma unroll
                    for (int v = 0; v < NV; ++v)
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            zc[v][4 + k] = ldg4_stream(Zc + (size_t)row[k] * RP + (gl + v * G) * 4);
                }
                }
                float acc = 0.f;
                float2 acc2 = make_float2(0.f, 0.f);
                float4 dxv[NV], dyv[NV];
                if (!TMA && dmode == 3) {
                    // both ranges narrow (every BJ config): one range-table row per axis; a real
                    // (warp-uniform) branch, so the SAT path below costs no issue slots here
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        dxv[v] = ldg4(px0 + v * G * 4);
                        dyv[v] = ldg4(py0 + v * G * 4);
                    }
                } else {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int c = (gl + v * G) * 4;
                    float4 dx, dy;
                    const uint32_t* sl = wslot + (size_t)(s % kSlots) * 4 * PSTRIDE;
                    if (TMA && U32) {
                        const uint4 qx0 = *reinterpret_cast<const uint4*>(sl + 0 * PSTRIDE + c);
                        const uint4 qx1 = *reinterpret_cast<const uint4*>(sl + 1 * PSTRIDE + c);
                        const uint4 qy0 = *reinterpret_cast<const uint4*>(sl + 2 * PSTRIDE + c);
                        const uint4 qy1 = *reinterpret_cast<const uint4*>(sl + 3 * PSTRIDE + c);
                        dx = make_float4(__uint2float_rn(qx1.x - qx0.x), __uint2float_rn(qx1.y - qx0.y),
                                         __uint2float_rn(qx1.z - qx0.z), __uint2float_rn(qx1.w - qx0.w));
                        dy = make_float4(__uint2float_rn(qy1.x - qy0.x), __uint2float_rn(qy1.y - qy0.y),
                                         __uint2float_rn(qy1.z - qy0.z), __uint2float_rn(qy1.w - qy0.w));
                    } else if (TMA) {
                        const float* sf = reinterpret_cast<const float*>(sl);
                        const float4 xh0 = *reinterpret_cast<const float4*>(sf + 0 * PSTRIDE + c);
                        const float4 xl0 = *reinterpret_cast<const float4*>(sf + 0 * PSTRIDE + RP + c);
                        const float4 xh1 = *reinterpret_cast<const float4*>(sf + 1 * PSTRIDE + c);
                        const float4 xl1 = *reinterpret_cast<const float4*>(sf + 1 * PSTRIDE + RP + c);
                        const float4 yh0 = *reinterpret_cast<const float4*>(sf + 2 * PSTRIDE + c);
                        const float4 yl0 = *reinterpret_cast<const float4*>(sf + 2 * PSTRIDE + RP + c);
                        const float4 yh1 = *reinterpret_cast<const float4*>(sf + 3 * PSTRIDE + c);
                        const float4 yl1 = *reinterpret_cast<const float4*>(sf + 3 * PSTRIDE + RP + c);
                        dx = make_float4((xh1.x - xh0.x) + (xl1.x - xl0.x), (xh1.y - xh0.y) + (xl1.y - xl0.y),
                                         (xh1.z - xh0.z) + (xl1.z - xl0.z), (xh1.w - xh0.w) + (xl1.w - xl0.w));
                        dy = make_float4((yh1.x - yh0.x) + (yl1.x - yl0.x), (yh1.y - yh0.y) + (yl1.y - yl0.y),
                                         (yh1.z - yh0.z) + (yl1.z - yl0.z), (yh1.w - yh0.w) + (yl1.w - yl0.w));
                    } else if (U32) {
                        // exact integer differences of the fixed-point SATs (scale folded into Zc)
                        if (tx) {
                            dx = ldg4(px0 + v * G * 4);
                        } else {
                            const uint4 qx1 = ldg_sat(px1 + v * G * 4);
                            const uint4 qx0 = ldg_sat(px0 + v * G * 4);
                            dx = make_float4(__uint2float_rn(qx1.x - qx0.x), __uint2float_rn(qx1.y - qx0.y),
                                             __uint2float_rn(qx1.z - qx0.z), __uint2float_rn(qx1.w - qx0.w));
                        }
                        if (ty) {
                            dy = ldg4(py0 + v * G * 4);
                        } else {
                            const uint4 qy1 = ldg_sat(py1 + v * G * 4);
                            const uint4 qy0 = ldg_sat(py0 + v * G * 4);
                            dy = make_float4(__uint2float_rn(qy1.x - qy0.x), __uint2float_rn(qy1.y - qy0.y),
                                             __uint2float_rn(qy1.z - qy0.z), __uint2float_rn(qy1.w - qy0.w));
                        }
                    } else {
                        // Xbar, Ybar numerators: (hi1 - hi0) + (lo1 - lo0); hi1 - hi0 is exact
                        // under cancellation (Sterbenz), lo carries the fp64 residual.
                        const int cv = v * G * 4;
                        if (tx) {
                            dx = ldg4(px0 + cv);
                        } else {
                            const float4 xh1 = ldg4(px1 + cv), xh0 = ldg4(px0 + cv);
                            const float4 xl1 = ldg4(px1 + RP + cv), xl0 = ldg4(px0 + RP + cv);
                            dx = make_float4((xh1.x - xh0.x) + (xl1.x - xl0.x), (xh1.y - xh0.y) + (xl1.y - xl0.y),
                                             (xh1.z - xh0.z) + (xl1.z - xl0.z), (xh1.w - xh0.w) + (xl1.w - xl0.w));
                        }
                        if (ty) {
                            dy = ldg4(py0 + cv);
                        } else {
                            const float4 yh1 = ldg4(py1 + cv), yh0 = ldg4(py0 + cv);
                            const float4 yl1 = ldg4(py1 + RP + cv), yl0 = ldg4(py0 + RP + cv);
                            dy = make_float4((yh1.x - yh0.x) + (yl1.x - yl0.x), (yh1.y - yh0.y) + (yl1.y - yl0.y),
                                             (yh1.z - yh0.z) + (yl1.z - yl0.z), (yh1.w - yh0.w) + (yl1.w - yl0.w));
                        }
                    }
                    dxv[v] = dx;
                    dyv[v] = dy;
                }
                }
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float4 dx = dxv[v], dy = dyv[v];
#if PNDF_NOREUSE
                    {  // experiment: Zc rows loaded per rank chunk, no cross-step register copy
                        const uint4 r03 = *reinterpret_cast<const uint4*>(&d.row[0]);
                        const uint4 r47 = *reinterpret_cast<const uint4*>(&d.row[4]);
                        const int row[8] = {(int)r03.x, (int)r03.y, (int)r03.z, (int)r03.w,
                                            (int)r47.x, (int)r47.y, (int)r47.z, (int)r47.w};
#pragma unroll
                        for (int k = 0; k < 8; ++k) zc[v][k] = ldg4_stream(Zc + (size_t)row[k] * RP + (gl + v * G) * 4);
                    }
#endif
#if PNDF_F2
                    // packed fp32 (FFMA2/FMUL2, sm_100): two ranks per instruction, same per-element
                    // rounding as the scalar chain; the rank sum runs in two interleaved halves
                    float2 zxy = make_float2(0.f, 0.f), zzw = make_float2(0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const float2 wk = make_float2(w[k], w[k]);
                        zxy = __ffma2_rn(wk, make_float2(zc[v][k].x, zc[v][k].y), zxy);
                        zzw = __ffma2_rn(wk, make_float2(zc[v][k].z, zc[v][k].w), zzw);
                    }
                    acc2 = __ffma2_rn(__fmul2_rn(make_float2(dx.x, dx.y), make_float2(dy.x, dy.y)), zxy, acc2);
                    acc2 = __ffma2_rn(__fmul2_rn(make_float2(dx.z, dx.w), make_float2(dy.z, dy.w)), zzw, acc2);
#else
                    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        z.x = fmaf(w[k], zc[v][k].x, z.x);
                        z.y = fmaf(w[k], zc[v][k].y, z.y);
                        z.z = fmaf(w[k], zc[v][k].z, z.z);
                        z.w = fmaf(w[k], zc[v][k].w, z.w);
                    }
                    acc = fmaf(dx.x * dy.x, z.x, acc);
                    acc = fmaf(dx.y * dy.y, z.y, acc);
                    acc = fmaf(dx.z * dy.z, z.z, acc);
                    acc = fmaf(dx.w * dy.w, z.w, acc);
#endif
                }
                part[j] = PNDF_F2 ? acc2.x + acc2.y : acc;
                if (TMA) __syncwarp();  // every lane is done with this slot before it is refilled
            }
            group_reduce<G, SB>(part, gl);
            // lane gl holds slots [slot0, slot0 + VPL) of its group: slot bits from the halving levels
            int slot0 = 0;
            {
                int nv = SB, o = G / 2;
                while (nv > 1 && o > 0) {
                    nv >>= 1;
                    if (gl & o) slot0 += nv;
                    o >>= 1;
                }
            }
            // route: query (s0 + j) * QPW + g of this batch goes to lane (s0 + j) * QPW + g
#pragma unroll
            for (int i = 0; i < VPL; ++i) {
                const int dst_rel = lane - s0 * QPW;  // this lane's query, relative to the batch
                const int j = dst_rel / QPW, g = dst_rel % QPW;
                // source lane: group g, a lane whose slot range starts at j - (j % VPL) when i == j % VPL
                int src_gl = 0;
                {
                    int nv = SB, o = G / 2, rem = j;
                    while (nv > 1 && o > 0) {
                        nv >>= 1;
                        if (rem >= nv) {
                            src_gl |= o;
                            rem -= nv;
                        }
                        o >>= 1;
                    }
                }
                const float got = __shfl_sync(0xffffffffu, part[i], (g * G + src_gl) & 31);
                const bool mine = dst_rel >= 0 && dst_rel < SB * QPW && (j % VPL) == i;
                if (mine) res = got;
            }
            (void)slot0;
        }
        const QDesc& mine = wd[lane];
        const int32_t oi = mine.out;
        const float div = mine.div;
        __syncwarp();
        if (oi >= 0) out[oi] = res / div;  // a6: Eq. 6 mean (div = area) or sum (div = 1)
    }
}

// --------------------------------------- gather4-staged query kernel (G == 32) --
// query_kernel with a5's range-table rows staged by the bulk-copy engine: each warp owns PNDF_G4D slots
// of shared memory, each holding the dx and dy rows of two consecutive queries; lane 0 fills a slot with
// ONE cp.async.bulk.tensor ... tile::gather4 (4 arbitrary rows of the DT tensor map), completion on the
// slot's mbarrier, 2 PNDF_G4D queries ahead.  The consumer's loads no longer sit on its scoreboards, so
// the FFMA2 / FMUL2 chain of step s waits only for step s's own Zc rows.  Same arithmetic and order as
// query_kernel: results are bitwise identical.
#ifndef PNDF_G4D
#define PNDF_G4D 2  // pair slots per warp (0: off)
#endif

template <int NV>
struct G4Layout {
    static constexpr int RP = 128 * NV;
    static constexpr int D2 = PNDF_G4D > 0 ? PNDF_G4D : 1;
    static constexpr int SLOT_F = 4 * RP;  // [q0 dx | q0 dy | q1 dx | q1 dy]
    static constexpr size_t DESC = sizeof(QDesc) * kWarpsPerBlock * 32;
    static constexpr size_t REUSE = 128;
    static constexpr size_t ROWS = (size_t)kWarpsPerBlock * 32 * 2 * 4;  // per query: its dx, dy table rows
    static constexpr size_t BARS = 128 * ((kWarpsPerBlock * D2 * 8 + 127) / 128);
    static constexpr size_t RING = (size_t)kWarpsPerBlock * D2 * SLOT_F * 4;
    static constexpr size_t BYTES = DESC + REUSE + ROWS + BARS + RING;
};

template <int NV, bool WRAP, bool BINNED, bool U32>
__global__ void __launch_bounds__(kThreads, PNDF_MINB)
    query_g4_kernel(const __grid_constant__ CUtensorMap tm, const QParams p, const pndf_query* __restrict__ q,
                    const uint32_t* __restrict__ idx, int64_t n, int64_t chunk, float* __restrict__ out) {
    using LY = G4Layout<NV>;
    constexpr int G = 32;
    constexpr int RP = LY::RP;
    constexpr int D2 = LY::D2;
    constexpr int SB = kSteps;
    static_assert(SB % 2 == 0 && (SB / 2) % D2 == 0, "pair slots must tile a reduction batch");
    constexpr int PSTRIDE = U32 ? RP : 2 * RP;
    extern __shared__ __align__(128) unsigned char qsmem[];
    QDesc(*sdesc)[32] = reinterpret_cast<QDesc(*)[32]>(qsmem);
    uint32_t* sreuse = reinterpret_cast<uint32_t*>(qsmem + LY::DESC);
    int2* srows = reinterpret_cast<int2*>(qsmem + LY::DESC + LY::REUSE);
    uint64_t* sbar = reinterpret_cast<uint64_t*>(qsmem + LY::DESC + LY::REUSE + LY::ROWS);
    float* sring = reinterpret_cast<float*>(qsmem + LY::DESC + LY::REUSE + LY::ROWS + LY::BARS);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    QDesc* wd = sdesc[warp];
    int2* wrows = srows + warp * 32;  // gather4 row coordinates of the batch (decoded once per query)
    uint64_t* wbar = sbar + warp * D2;
    float* wring = sring + (size_t)warp * D2 * LY::SLOT_F;
    const float* __restrict__ Zc = p.Zc;
    const float* __restrict__ PXl = p.PXY + lane * 4;
    if (lane == 0)
        for (int k = 0; k < D2; ++k) mbar_init(wbar + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t phase = 0;
    // lane 0: one gather4 of the dx / dy rows of queries 2 pr, 2 pr + 1 into slot pr % D2 (row 0 stands in
    // for an axis whose range is wider than the table: its SAT rows are read at its step)
    auto issue_pair = [&](int pr) {
        if (lane == 0) {
            const int4 rr = *reinterpret_cast<const int4*>(wrows + 2 * pr);
            const int r0 = rr.x, r1 = rr.y, r2 = rr.z, r3 = rr.w;
            const int k = pr % D2;
            // (the slot's previous contents were consumed by every lane's FFMA2s before the __syncwarp that
            // precedes this issue, so the bulk copy cannot overwrite a pending read)
            mbar_arrive_expect_tx(wbar + k, 4 * RP * 4);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(wring + k * LY::SLOT_F)),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
                "r"(smem_u32(wbar + k))
                : "memory");
        }
    };

    const int64_t c0 = (int64_t)blockIdx.x * chunk;
    const int64_t c1 = min(n, c0 + chunk);
    float4 zc[NV][8];
    for (int64_t base = c0 + (int64_t)warp * 32; base < c1; base += (int64_t)kWarpsPerBlock * 32) {
        {
            const int64_t qi = base + lane;
            bool valid = false;
            QDesc& d = wd[lane];
            if (qi < c1) {
                const int64_t src = BINNED ? (int64_t)__ldg(idx + qi) : qi;
                const pndf_query rec = ldg_query(q + src);
                valid = decode<WRAP, true>(p, rec, (int32_t)src, d);
            } else {
                d.out = -1;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    d.row[k] = 0;
                    d.w[k] = 0.f;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) d.sat[k] = 0;
                d.mode = 0;
                d.div = 1.f;
            }
            uint32_t same_lo, same_hi;
            int32_t mine[4];
            reuse_masks<WRAP>(d, valid, lane > 0, -1, -1, -1, -1, &same_lo, &same_hi, mine);
            if (lane == 0) {
                sreuse[2 * warp] = same_lo;
                sreuse[2 * warp + 1] = same_hi;
            }
            wrows[lane] = make_int2((d.mode & 1) ? d.sat[0] : 0, (d.mode & 2) ? d.sat[2] : 0);
        }
        __syncwarp();
        const uint32_t reuse_lo = sreuse[2 * warp];
        const uint32_t reuse_hi = sreuse[2 * warp + 1];
#pragma unroll
        for (int pr = 0; pr < D2; ++pr) issue_pair(pr);
        float res = 0.f;
#pragma unroll 1
        for (int s0 = 0; s0 < 32; s0 += SB) {
            float part[SB];
#pragma unroll
            for (int j = 0; j < SB; ++j) {
                const int s = s0 + j;
                const int k = (j / 2) % D2;  // == (s / 2) % D2: SB / 2 is a multiple of D2
                if ((j & 1) == 0) {
                    while (!mbar_try_wait(wbar + k, (phase >> k) & 1u)) {
                    }
                    phase ^= 1u << k;
                }
                const QDesc& d = wd[s];
                const float4 w03 = *reinterpret_cast<const float4*>(&d.w[0]);
                const float4 w47 = *reinterpret_cast<const float4*>(&d.w[4]);
                const int dmode = d.mode;
                const float w[8] = {w03.x, w03.y, w03.z, w03.w, w47.x, w47.y, w47.z, w47.w};
                const bool reuse0 = s > 0 && ((reuse_lo >> s) & 1u);
                const bool reuse1 = s > 0 && ((reuse_hi >> s) & 1u);
                if (__builtin_expect(!(reuse0 && reuse1), 0)) {
                    if (!reuse0) {
                        const uint4 r03 = *reinterpret_cast<const uint4*>(&d.row[0]);
                        const int row[4] = {(int)r03.x, (int)r03.y, (int)r03.z, (int)r03.w};
#pragma unroll
                        for (int v = 0; v < NV; ++v)
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                zc[v][kk] = ldg4_stream(Zc + (size_t)row[kk] * RP + (lane + v * G) * 4);
                    }
                    if (!reuse1) {
                        const uint4 r47 = *reinterpret_cast<const uint4*>(&d.row[4]);
                        const int row[4] = {(int)r47.x, (int)r47.y, (int)r47.z, (int)r47.w};
#pragma unroll
                        for (int v = 0; v < NV; ++v)
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                zc[v][4 + kk] = ldg4_stream(Zc + (size_t)row[kk] * RP + (lane + v * G) * 4);
                    }
                }
                const float* sl = wring + k * LY::SLOT_F + (j & 1) * 2 * RP + lane * 4;
                float4 dxv[NV], dyv[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    dxv[v] = *reinterpret_cast<const float4*>(sl + v * G * 4);
                    dyv[v] = *reinterpret_cast<const float4*>(sl + RP + v * G * 4);
                }
                if (__builtin_expect(dmode != 3, 0)) {  // a wide range: its two SAT rows, read directly
                    const int4 so = *reinterpret_cast<const int4*>(&d.sat[0]);
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const int cv = v * G * 4;
                        if (!(dmode & 1)) {
                            const float* px0 = PXl + (int64_t)so.x * PSTRIDE;
                            const float* px1 = PXl + (int64_t)so.y * PSTRIDE;
                            if (U32) {
                                const uint4 qx1 = ldg_sat(px1 + cv), qx0 = ldg_sat(px0 + cv);
                                dxv[v] = make_float4(__uint2float_rn(qx1.x - qx0.x), __uint2float_rn(qx1.y - qx0.y),
                                                     __uint2float_rn(qx1.z - qx0.z), __uint2float_rn(qx1.w - qx0.w));
                            } else {
                                const float4 xh1 = ldg4(px1 + cv), xh0 = ldg4(px0 + cv);
                                const float4 xl1 = ldg4(px1 + RP + cv), xl0 = ldg4(px0 + RP + cv);
                                dxv[v] = make_float4((xh1.x - xh0.x) + (xl1.x - xl0.x), (xh1.y - xh0.y) + (xl1.y - xl0.y),
                                                     (xh1.z - xh0.z) + (xl1.z - xl0.z), (xh1.w - xh0.w) + (xl1.w - xl0.w));
                            }
                        }
                        if (!(dmode & 2)) {
                            const float* py0 = PXl + (int64_t)so.z * PSTRIDE;
                            const float* py1 = PXl + (int64_t)so.w * PSTRIDE;
                            if (U32) {
                                const uint4 qy1 = ldg_sat(py1 + cv), qy0 = ldg_sat(py0 + cv);
                                dyv[v] = make_float4(__uint2float_rn(qy1.x - qy0.x), __uint2float_rn(qy1.y - qy0.y),
                                                     __uint2float_rn(qy1.z - qy0.z), __uint2float_rn(qy1.w - qy0.w));
                            } else {
                                const float4 yh1 = ldg4(py1 + cv), yh0 = ldg4(py0 + cv);
                                const float4 yl1 = ldg4(py1 + RP + cv), yl0 = ldg4(py0 + RP + cv);
                                dyv[v] = make_float4((yh1.x - yh0.x) + (yl1.x - yl0.x), (yh1.y - yh0.y) + (yl1.y - yl0.y),
                                                     (yh1.z - yh0.z) + (yl1.z - yl0.z), (yh1.w - yh0.w) + (yl1.w - yl0.w));
                            }
                        }
                    }
                }
                float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float4 dx = dxv[v], dy = dyv[v];
                    float2 zxy = make_float2(0.f, 0.f), zzw = make_float2(0.f, 0.f);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const float2 wk = make_float2(w[kk], w[kk]);
                        zxy = __ffma2_rn(wk, make_float2(zc[v][kk].x, zc[v][kk].y), zxy);
                        zzw = __ffma2_rn(wk, make_float2(zc[v][kk].z, zc[v][kk].w), zzw);
                    }
                    acc2 = __ffma2_rn(__fmul2_rn(make_float2(dx.x, dx.y), make_float2(dy.x, dy.y)), zxy, acc2);
                    acc2 = __ffma2_rn(__fmul2_rn(make_float2(dx.z, dx.w), make_float2(dy.z, dy.w)), zzw, acc2);
                }
                part[j] = acc2.x + acc2.y;
                if (j & 1) {  // both queries of the pair are done with the slot: refill it D2 pairs ahead
                    __syncwarp();
                    if (s / 2 + D2 < 16) issue_pair(s / 2 + D2);
                }
            }
            group_reduce<G, SB>(part, lane);
            const int jj = lane - s0;
            int src_gl = 0;
            {
                int nv = SB, o = G / 2, rem = jj;
                while (nv > 1 && o > 0) {
                    nv >>= 1;
                    if (rem >= nv) {
                        src_gl |= o;
                        rem -= nv;
                    }
                    o >>= 1;
                }
            }
            const float got = __shfl_sync(0xffffffffu, part[0], src_gl & 31);
            if (jj >= 0 && jj < SB) res = got;
        }
        const QDesc& mine = wd[lane];
        const int32_t oi = mine.out;
        const float div = mine.div;
        __syncwarp();
        if (oi >= 0) out[oi] = res / div;
    }
}

template <int NV, bool W, bool B, bool U>
static cudaError_t launch_g4(const QParams& p, const pndf_query* q, const uint32_t* idx, int64_t n, float* out,
                             int num_sms, cudaStream_t st) {
    constexpr size_t smem = G4Layout<NV>::BYTES;
    auto* kfn = query_g4_kernel<NV, W, B, U>;
    static int occ = -1;
    if (occ < 0) {
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kThreads, smem) != cudaSuccess || occ < 1)
            occ = 1;
    }
    int64_t grid = (int64_t)num_sms * occ;
    const int64_t need = (n + kThreads - 1) / kThreads;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = (chunk + 31) / 32 * 32;
    grid = (n + chunk - 1) / chunk;
    kfn<<<(unsigned)grid, kThreads, smem, st>>>(*p.dt_tmap, p, q, idx, n, chunk, out);
    return cudaGetLastError();
}

// ------------------------------------------- lean gather4 query kernel (G == 32) --
// query_g4_kernel's data path (range-table rows staged by tile::gather4, Zc rows reused in registers)
// with a leaner step, the per-step control and reduction work cut down:
//   * one warp-uniform reload branch per step (either level changed); the two levels' row loads inside it
//     are predicated, not branched;
//   * batches whose 32 records all take both ranges from the range table (every BJ config) run a step
//     with no wide-range path at all (ballot at decode);
//   * no shuffle reduction: each pair of steps stores its 32 per-lane partials over its own (consumed)
//     descriptor slots, and at the end of the batch lane q sums query q's 32 partials in a fixed order.  A query's result still does not depend on where it sits in the batch
//     (binned == unbinned bitwise), but it is not bitwise query_g4_kernel's (different summation order).
#ifndef PNDF_G5D
#define PNDF_G5D 2  // pair slots per warp
#endif
#ifndef PNDF_G5SB
#define PNDF_G5SB 4  // steps per unrolled block (8: 197.8 ms, 4: 194.9 ms on config 5 -- half the code, fewer instruction-cache misses)
#endif
#ifndef PNDF_G5EARLY
#define PNDF_G5EARLY 1  // 1: a step's Zc reload is issued at the end of the previous step (0: at its own start)
#endif
#ifndef PNDF_G5ELECT
#define PNDF_G5ELECT 1  // 1: the pair copies are issued by an elect.sync lane with predicated instructions (no branch)
#endif

// a query's descriptor, then (after its step) its 32 per-lane partials.  144 B = 9 16-byte bank groups: the
// decode's per-lane 16-byte stores to 32 consecutive slots and the end-of-batch per-lane reads of them are
// bank-conflict free (a 128 B stride puts every lane on the same banks)
struct __align__(16) QSlot {
    QDesc d;
    int32_t pad[8];
    int4 fin;  // dx row, dy row of the range table, out index, div: past the 128 B the partials overwrite
};
static_assert(sizeof(QSlot) == 144, "QSlot layout");

template <int NV>
struct G5Layout {
    static constexpr int RP = 128 * NV;
    static constexpr int D2 = PNDF_G5D;
    static constexpr int SLOT_F = 4 * RP;  // [q0 dx | q0 dy | q1 dx | q1 dy]
    static constexpr size_t SLOTS = sizeof(QSlot) * kWarpsPerBlock * 32;
    static constexpr size_t BARS = 128 * ((kWarpsPerBlock * D2 * 8 + 127) / 128);
    static constexpr size_t RING = (size_t)kWarpsPerBlock * D2 * SLOT_F * 4;
    static constexpr size_t RECS = (size_t)kWarpsPerBlock * 32 * 20;  // next batch: records (16 B), idx (4 B)
    static constexpr size_t BYTES = SLOTS + BARS + RING + RECS;
};

__device__ __forceinline__ void cp_async_4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int NV, bool WRAP, bool BINNED, bool U32>
__global__ void __launch_bounds__(kThreads, PNDF_MINB)
    query_g5_kernel(const __grid_constant__ CUtensorMap tm, const QParams p, const pndf_query* __restrict__ q,
                    const uint32_t* __restrict__ idx, int64_t n, int64_t chunk, int rot, float* __restrict__ out) {
    using LY = G5Layout<NV>;
    constexpr int G = 32;
    constexpr int RP = LY::RP;
    constexpr int D2 = LY::D2;
    constexpr int SB = PNDF_G5SB;  // steps per unrolled block
    static_assert((SB / 2) % D2 == 0, "pair slots must tile an unrolled block");
    constexpr int PSTRIDE = U32 ? RP : 2 * RP;
    extern __shared__ __align__(128) unsigned char qsmem[];
    QSlot* wslot = reinterpret_cast<QSlot*>(qsmem) + (threadIdx.x >> 5) * 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t* wbar = reinterpret_cast<uint64_t*>(qsmem + LY::SLOTS) + warp * D2;
    float* wring = reinterpret_cast<float*>(qsmem + LY::SLOTS + LY::BARS) + (size_t)warp * D2 * LY::SLOT_F;
    // the next batch's records (and, binned, their idx entries) arrive by cp.async while this batch runs
    uint4* srec = reinterpret_cast<uint4*>(qsmem + LY::SLOTS + LY::BARS + LY::RING) + warp * 32;
    uint32_t* sidx = reinterpret_cast<uint32_t*>(qsmem + LY::SLOTS + LY::BARS + LY::RING +
                                                 (size_t)kWarpsPerBlock * 32 * 16) + warp * 32;
    const float* __restrict__ Zc = p.Zc + lane * 4;
    if (lane == 0)
        for (int k = 0; k < D2; ++k) mbar_init(wbar + k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t phase = 0;
    auto issue_pair = [&](int pr) {
#if PNDF_G5ELECT
        // every lane reads the (warp-uniform) coordinates; one elected lane arrives and issues the copy
        const int4 ra = wslot[2 * pr].fin, rb = wslot[2 * pr + 1].fin;
        const int k = pr % D2;
        asm volatile(
            "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
            " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%7], %8;\n"
            " @p cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n}" ::"r"(smem_u32(wring + k * LY::SLOT_F)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(ra.x), "r"(ra.y), "r"(rb.x), "r"(rb.y),
            "r"(smem_u32(wbar + k)), "r"(4 * RP * 4)
            : "memory");
#else
        if (lane == 0) {
            const int4 ra = wslot[2 * pr].fin, rb = wslot[2 * pr + 1].fin;
            const int4 rr = make_int4(ra.x, ra.y, rb.x, rb.y);
            const int k = pr % D2;
            mbar_arrive_expect_tx(wbar + k, 4 * RP * 4);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(wring + k * LY::SLOT_F)),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(rr.x), "r"(rr.y), "r"(rr.z), "r"(rr.w),
                "r"(smem_u32(wbar + k))
                : "memory");
        }
#endif
    };

    // one step of query s = s0 + j; NARROW: every query of the batch reads both ranges from the table
    float4 zc[NV][8];
    float pe = 0.f;  // the even step's partial, stored with the odd step's
    // (re)load the Zc rows of the levels that differ from the previous query's (rl: level l0, rh: l0 + 1)
    auto reload = [&](const QDesc& d, bool rl, bool rh) {
        const int4 r03 = *reinterpret_cast<const int4*>(&d.row[0]);
        const int4 r47 = *reinterpret_cast<const int4*>(&d.row[4]);
        const int row[8] = {r03.x, r03.y, r03.z, r03.w, r47.x, r47.y, r47.z, r47.w};
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (rl) zc[v][kk] = ldg4_stream(Zc + (size_t)row[kk] * RP + v * G * 4);
                if (rh) zc[v][4 + kk] = ldg4_stream(Zc + (size_t)row[4 + kk] * RP + v * G * 4);
            }
    };
    auto step = [&](auto narrow_tag, int s0, int j, uint32_t nb, uint32_t lob, uint32_t hib) {
        constexpr bool NARROW = decltype(narrow_tag)::value;
        const int s = s0 + j;
        const int k = (j / 2) % D2;
        if ((j & 1) == 0) {
            while (!mbar_try_wait(wbar + k, (phase >> k) & 1u)) {
            }
            phase ^= 1u << k;
        }
        const QDesc& d = wslot[s].d;
        const float4 w03 = *reinterpret_cast<const float4*>(&d.w[0]);
        const float4 w47 = *reinterpret_cast<const float4*>(&d.w[4]);
        const float w[8] = {w03.x, w03.y, w03.z, w03.w, w47.x, w47.y, w47.z, w47.w};
#if !PNDF_G5EARLY
        if ((nb >> j) & 1u) reload(d, !((lob >> j) & 1u), !((hib >> j) & 1u));
#endif
        const float* sl = wring + k * LY::SLOT_F + (j & 1) * 2 * RP + lane * 4;
        float4 dxv[NV], dyv[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            dxv[v] = *reinterpret_cast<const float4*>(sl + v * G * 4);
            dyv[v] = *reinterpret_cast<const float4*>(sl + RP + v * G * 4);
        }
        if constexpr (!NARROW) {
            const int dmode = d.mode;
            if (dmode != 3) {  // a wide range: its two SAT rows, read directly
                const int4 so = *reinterpret_cast<const int4*>(&d.sat[0]);
                const float* __restrict__ PXl = p.PXY + lane * 4;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int cv = v * G * 4;
                    if (!(dmode & 1)) {
                        const float* px0 = PXl + (int64_t)so.x * PSTRIDE;
                        const float* px1 = PXl + (int64_t)so.y * PSTRIDE;
                        if (U32) {
                            const uint4 qx1 = ldg_sat(px1 + cv), qx0 = ldg_sat(px0 + cv);
                            dxv[v] = make_float4(__uint2float_rn(qx1.x - qx0.x), __uint2float_rn(qx1.y - qx0.y),
                                                 __uint2float_rn(qx1.z - qx0.z), __uint2float_rn(qx1.w - qx0.w));
                        } else {
                            const float4 xh1 = ldg4(px1 + cv), xh0 = ldg4(px0 + cv);
                            const float4 xl1 = ldg4(px1 + RP + cv), xl0 = ldg4(px0 + RP + cv);
                            dxv[v] = make_float4((xh1.x - xh0.x) + (xl1.x - xl0.x), (xh1.y - xh0.y) + (xl1.y - xl0.y),
                                                 (xh1.z - xh0.z) + (xl1.z - xl0.z), (xh1.w - xh0.w) + (xl1.w - xl0.w));
                        }
                    }
                    if (!(dmode & 2)) {
                        const float* py0 = PXl + (int64_t)so.z * PSTRIDE;
                        const float* py1 = PXl + (int64_t)so.w * PSTRIDE;
                        if (U32) {
                            const uint4 qy1 = ldg_sat(py1 + cv), qy0 = ldg_sat(py0 + cv);
                            dyv[v] = make_float4(__uint2float_rn(qy1.x - qy0.x), __uint2float_rn(qy1.y - qy0.y),
                                                 __uint2float_rn(qy1.z - qy0.z), __uint2float_rn(qy1.w - qy0.w));
                        } else {
                            const float4 yh1 = ldg4(py1 + cv), yh0 = ldg4(py0 + cv);
                            const float4 yl1 = ldg4(py1 + RP + cv), yl0 = ldg4(py0 + RP + cv);
                            dyv[v] = make_float4((yh1.x - yh0.x) + (yl1.x - yl0.x), (yh1.y - yh0.y) + (yl1.y - yl0.y),
                                                 (yh1.z - yh0.z) + (yl1.z - yl0.z), (yh1.w - yh0.w) + (yl1.w - yl0.w));
                        }
                    }
                }
            }
        }
        // a6: (Xbar Ybar) . (sum_k w_k Zc_k) over this lane's 4 NV ranks; two accumulators (xy / zw lanes of
        // the packed pairs) keep the product chain two deep
        float2 exy[NV], ezw[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            exy[v] = __fmul2_rn(make_float2(dxv[v].x, dxv[v].y), make_float2(dyv[v].x, dyv[v].y));
            ezw[v] = __fmul2_rn(make_float2(dxv[v].z, dxv[v].w), make_float2(dyv[v].z, dyv[v].w));
        }
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            float2 zxy = __fmul2_rn(make_float2(w[0], w[0]), make_float2(zc[v][0].x, zc[v][0].y));
            float2 zzw = __fmul2_rn(make_float2(w[0], w[0]), make_float2(zc[v][0].z, zc[v][0].w));
#pragma unroll
            for (int kk = 1; kk < 8; ++kk) {
                const float2 wk = make_float2(w[kk], w[kk]);
                zxy = __ffma2_rn(wk, make_float2(zc[v][kk].x, zc[v][kk].y), zxy);
                zzw = __ffma2_rn(wk, make_float2(zc[v][kk].z, zc[v][kk].w), zzw);
            }
            a0 = __ffma2_rn(exy[v], zxy, a0);
            a1 = __ffma2_rn(ezw[v], zzw, a1);
        }
#if PNDF_G5EARLY
        // the Zc registers are free again: the next query's reload (warp-uniform) is issued here, so its
        // latency overlaps this step's tail, the pair copy and the next step's shared-memory loads
        if ((nb >> (j + 1)) & 1u)
            reload(wslot[s + 1].d, !((lob >> (j + 1)) & 1u), !((hib >> (j + 1)) & 1u));
#endif
        const float2 a = __fadd2_rn(a0, a1);
        const float part = a.x + a.y;
        if ((j & 1) == 0) {
            pe = part;
        } else {
            // both queries of the pair are done with their descriptors and the ring slot: the descriptor
            // slots take the pair's partials, and the ring slot is refilled D2 pairs ahead
            __syncwarp();
            reinterpret_cast<float*>(wslot + s - 1)[lane] = pe;
            reinterpret_cast<float*>(wslot + s)[lane] = part;
            if (s / 2 + D2 < 16) issue_pair(s / 2 + D2);
        }
    };

    // CTA b takes the chunks b, b + gridDim.x, ... of the batch: a binned batch is ordered by level, and a
    // level-0 query (nearly every one reloads its rows) costs several coarse-level ones, so contiguous
    // per-CTA ranges leave most SMs idle while the level-0 CTAs finish; interleaved chunks give every CTA
    // the same level mix (and all CTAs work on one region of the map at a time: better L2 locality)
    // rot: each CTA starts its round at a different point of the batch, so at any time the CTAs are spread
    // over all levels and the reload-heavy level-0 phase does not hit DRAM from every SM at once
    const int64_t nch = (n + chunk - 1) / chunk;
    const int64_t cnt = (nch - blockIdx.x + gridDim.x - 1) / gridDim.x;  // chunks of this CTA
    const int64_t r0 = rot ? ((int64_t)blockIdx.x * cnt) / gridDim.x : 0;
    int64_t c0 = 0;
    int nloc = 0;  // the current chunk's queries (chunk < 2^31)
    // each lane fetches its own record of the next batch (no cross-lane hand-off, so no warp sync)
    auto fetch_idx = [&](int blq) {
        if (BINNED && blq + lane < nloc) cp_async_4(sidx + lane, idx + c0 + blq + lane);
    };
    auto fetch_rec = [&](int blq) {
        if (blq + lane < nloc)
            cp_async_16(srec + lane, q + (BINNED ? (int64_t)sidx[lane] : c0 + blq + lane));
        cp_async_commit();
    };
    for (int64_t kq = 0; kq < cnt; ++kq) {
    const int64_t kk = kq + r0 < cnt ? kq + r0 : kq + r0 - cnt;
    c0 = ((int64_t)blockIdx.x + kk * gridDim.x) * chunk;
    nloc = (int)(min(n, c0 + chunk) - c0);
    fetch_idx(warp * 32);
    cp_async_commit_wait_all();
    fetch_rec(warp * 32);
    for (int bl = warp * 32; bl < nloc; bl += kWarpsPerBlock * 32) {
        cp_async_commit_wait_all();
        uint32_t same_lo, same_hi;
        bool narrow_ok;
        {
            const int ql = bl + lane;
            bool valid = false;
            QDesc& d = wslot[lane].d;
            d.out = -1;
            d.div = 1.f;
            if (ql < nloc) {
                const int64_t src = BINNED ? (int64_t)sidx[lane] : c0 + ql;
                const uint4 rv = srec[lane];
                pndf_query rec;
                rec.u = __uint_as_float(rv.x);
                rec.v = __uint_as_float(rv.y);
                rec.size = __uint_as_float(rv.z);
                rec.rect = rv.w;
                valid = decode<WRAP, true>(p, rec, (int32_t)src, d);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    d.row[k] = 0;
                    d.w[k] = 0.f;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) d.sat[k] = 0;
                d.mode = 0;
            }
            int32_t mine[4];
            reuse_masks<WRAP>(d, valid, lane > 0, -1, -1, -1, -1, &same_lo, &same_hi, mine);
            // invalid / absent records (mode 0, zero weights, NaN or no output) may take the narrow step:
            // it reads range-table row 0, finite, and their result is discarded or NaN anyway
            narrow_ok = __all_sync(0xffffffffu, d.mode == 3 || !valid);
            wslot[lane].fin = make_int4((d.mode & 1) ? d.sat[0] : 0, (d.mode & 2) ? d.sat[2] : 0, d.out,
                                    __float_as_int(d.div));
        }
        __syncwarp();
#pragma unroll
        for (int pr = 0; pr < D2; ++pr) issue_pair(pr);
        const int bn = bl + kWarpsPerBlock * 32;  // this warp's next batch
        fetch_idx(bn);
        cp_async_commit();
        uint32_t nb = ~(same_lo & same_hi);  // bit j: step j reloads (shifted down a block at a time)
#if PNDF_G5EARLY
        reload(wslot[0].d, true, true);  // query 0 never repeats a previous query's rows
#endif
        if (narrow_ok) {
#pragma unroll 1
            for (int s0 = 0; s0 < 32; s0 += SB) {
#pragma unroll
                for (int j = 0; j < SB; ++j) step(std::true_type{}, s0, j, nb, same_lo, same_hi);
                nb >>= SB;
                same_lo >>= SB;
                same_hi >>= SB;
                if (s0 == 0) {  // the next batch's idx entries have landed: fetch its records
                    cp_async_commit_wait_all();
                    fetch_rec(bn);
                }
            }
        } else {
#pragma unroll 1
            for (int s0 = 0; s0 < 32; s0 += SB) {
#pragma unroll
                for (int j = 0; j < SB; ++j) step(std::false_type{}, s0, j, nb, same_lo, same_hi);
                nb >>= SB;
                same_lo >>= SB;
                same_hi >>= SB;
                if (s0 == 0) {
                    cp_async_commit_wait_all();
                    fetch_rec(bn);
                }
            }
        }
        __syncwarp();
        // lane q: query q's 32 partials (chunk c = lanes 4c..4c+3)
        const float4* pr4 = reinterpret_cast<const float4*>(wslot + lane);
        float4 t[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) t[c] = pr4[c];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            t[c].x += t[c + 4].x;
            t[c].y += t[c + 4].y;
            t[c].z += t[c + 4].z;
            t[c].w += t[c + 4].w;
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            t[c].x += t[c + 2].x;
            t[c].y += t[c + 2].y;
            t[c].z += t[c + 2].z;
            t[c].w += t[c + 2].w;
        }
        const float res = ((t[0].x + t[1].x) + (t[0].y + t[1].y)) + ((t[0].z + t[1].z) + (t[0].w + t[1].w));
        const int4 mo = wslot[lane].fin;
        __syncwarp();  // the slots are rewritten by the next batch's decode
        if (mo.z >= 0) out[mo.z] = res / __int_as_float(mo.w);  // a6: Eq. 6 mean (div = area) or sum (div = 1)
    }
    cp_async_commit_wait_all();  // nothing of this chunk's last (empty) prefetch is left in flight
    }
}

template <int NV, bool W, bool B, bool U>
static cudaError_t launch_g5(const QParams& p, const pndf_query* q, const uint32_t* idx, int64_t n, float* out,
                             int num_sms, cudaStream_t st) {
    constexpr size_t smem = G5Layout<NV>::BYTES;
    auto* kfn = query_g5_kernel<NV, W, B, U>;
    static int occ = -1;
    if (occ < 0) {
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kThreads, smem) != cudaSuccess || occ < 1)
            occ = 1;
    }
    int64_t grid = (int64_t)num_sms * occ;
    const int64_t need = (n + kThreads - 1) / kThreads;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = (chunk + 31) / 32 * 32;
    if (chunk > g5_chunk()) chunk = g5_chunk();  // large batches: interleaved chunks (see the kernel)
    const int64_t nchunks = (n + chunk - 1) / chunk;
    if (grid > nchunks) grid = nchunks;
    kfn<<<(unsigned)grid, kThreads, smem, st>>>(*p.dt_tmap, p, q, idx, n, chunk, g5_rot() ? 1 : 0, out);
    return cudaGetLastError();
}

// ----------------------------------------------------------- launchers --
template <int G, int NV, bool W, bool B, bool U>
static cudaError_t launch_q(const QParams& p, const pndf_query* q, const uint32_t* idx, int64_t n, float* out,
                            int num_sms, cudaStream_t st) {
    if constexpr (G == 32 && NV <= 2) {
        if (p.dt_tmap && p.dt_w > 0 && !g5_disabled()) return launch_g5<NV, W, B, U>(p, q, idx, n, out, num_sms, st);
    }
    if constexpr (G == 32 && PNDF_G4D > 0 && NV <= 2) {
        if (p.dt_tmap && p.dt_w > 0 && !g4_disabled()) return launch_g4<NV, W, B, U>(p, q, idx, n, out, num_sms, st);
    }
    constexpr size_t smem = QLayout<G, NV, U>::BYTES;
    cudaFuncSetAttribute(query_kernel<G, NV, W, B, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    static int occ = -1;
    if (occ < 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, query_kernel<G, NV, W, B, U>, kThreads, smem) !=
                cudaSuccess ||
            occ < 1)
            occ = 1;
    }
    int64_t grid = (int64_t)num_sms * occ;
    const int64_t need = (n + kThreads - 1) / kThreads;  // at least one query per lane per block
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    int64_t chunk = (n + grid - 1) / grid;
    chunk = (chunk + 31) / 32 * 32;
    grid = (n + chunk - 1) / chunk;
    query_kernel<G, NV, W, B, U><<<(unsigned)grid, kThreads, smem, st>>>(p, q, idx, n, chunk, out);
    return cudaGetLastError();
}

template <int G, bool W, bool B, bool U>
static cudaError_t dispatch_nv(int NV, const QParams& p, const pndf_query* q, const uint32_t* idx, int64_t n,
                               float* out, int num_sms, cudaStream_t st) {
    switch (NV) {
        case 1: return launch_q<G, 1, W, B, U>(p, q, idx, n, out, num_sms, st);
        case 2: return launch_q<G, 2, W, B, U>(p, q, idx, n, out, num_sms, st);
        case 3: return launch_q<G, 3, W, B, U>(p, q, idx, n, out, num_sms, st);
        case 4: return launch_q<G, 4, W, B, U>(p, q, idx, n, out, num_sms, st);
        case 8: return launch_q<G, 8, W, B, U>(p, q, idx, n, out, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

template <bool W, bool B, bool U>
static cudaError_t dispatch_g(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx, int64_t n,
                              float* out, int num_sms, cudaStream_t st) {
    switch (G) {
        case 1: return dispatch_nv<1, W, B, U>(NV, p, q, idx, n, out, num_sms, st);
        case 2: return dispatch_nv<2, W, B, U>(NV, p, q, idx, n, out, num_sms, st);
        case 4: return dispatch_nv<4, W, B, U>(NV, p, q, idx, n, out, num_sms, st);
        case 8: return dispatch_nv<8, W, B, U>(NV, p, q, idx, n, out, num_sms, st);
        case 16: return dispatch_nv<16, W, B, U>(NV, p, q, idx, n, out, num_sms, st);
        case 32: return dispatch_nv<32, W, B, U>(NV, p, q, idx, n, out, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace pndf
