// query_tc.cuh -- tensor-core run kernel (rows a4-a6 for binned runs; Rp == 256).
//
// After binning, an aligned block of 128 consecutive queries with one key shares all 8 Zc rows
// (DESIGN.md section 5), so Eq. 6 for the block is a dense contraction
//   D[q][k] = sum_r (dx_q[r] dy_q[r]) Z_k[r],   result_q = (sum_k w_qk D[q][k]) / area_q
// i.e. [128 x 256] . [256 x 8].  It runs as tcgen05.mma kind::tf32 (M = 128, N = 16, K = 8 per instruction,
// fp32 accumulator in TMEM) with both operands split into a tf32 part and its fp32 remainder:
//   B = [hi(Z_0..7) ; lo(Z_0..7)]  (16 columns),  A = hi(P) then lo(P),  P = dx . dy
// so every product that matters (hi hi, hi lo, lo hi) is accumulated and the dropped lo lo term is 2^-22
// relative.  The warps write the operands straight into the 128-byte-swizzled K-major layout the UMMA
// descriptors of als.cu use; one thread issues the MMAs; the 8 trilinear weights are applied to the
// accumulator row in the epilogue (thread q = query q = TMEM lane q).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.h"
#include "query_kernel.cuh"

namespace pndf {
namespace tc {

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// K-major operand tile in the 128-byte swizzle layout (8-row atoms of 1024 B): start >> 4, LBO = 1
// (unused for swizzled K-major), SBO = 1024 B, version 1, layout SWIZZLE_128B
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// x = hi + lo with hi holding the 11 leading significand bits (exactly a tf32 value)
__device__ __forceinline__ void split4(const float4 x, float4& hi, float4& lo) {
    hi.x = __uint_as_float(__float_as_uint(x.x) & 0xffffe000u);
    hi.y = __uint_as_float(__float_as_uint(x.y) & 0xffffe000u);
    hi.z = __uint_as_float(__float_as_uint(x.z) & 0xffffe000u);
    hi.w = __uint_as_float(__float_as_uint(x.w) & 0xffffe000u);
    lo = make_float4(x.x - hi.x, x.y - hi.y, x.z - hi.z, x.w - hi.w);
}
// byte offset of (row r, 16-byte chunk c) inside a [rows][32 fp32] SW128 tile
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

struct Layout {
    static constexpr int M = 128;                         // queries per block
    static constexpr int RP = 256;                        // ranks (K)
    static constexpr int KC = 32;                         // ranks per A chunk (one K-block)
    static constexpr int NCH = RP / KC;                   // chunks per block
    static constexpr int A_TILE = M * 128;                // one [128 x 32 fp32] tile
    static constexpr int A_BUF = 2 * A_TILE;              // hi tile then lo tile
    static constexpr int A_BYTES = 2 * A_BUF;             // two buffers
    static constexpr int B_TILE = 16 * 128;               // one [16 x 32 fp32] tile
    static constexpr int B_BYTES = (RP / 32) * B_TILE;
    static constexpr int DESC = M * (int)sizeof(QDesc);
    static constexpr int BYTES = 1024 + A_BYTES + B_BYTES + DESC + 128;
    static constexpr int TMEM_COLS = 32;
    static constexpr int PRODUCERS = 256;                 // warps 0-7 build the operands, warp 8 issues the MMAs
    static constexpr int THREADS = PRODUCERS + 32;
};

}  // namespace tc

__device__ __forceinline__ void sts4(uint32_t addr, const float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// dx or dy of one query over 4 ranks from its two SAT rows (wide range: rows a0, a1 of PXY)
template <bool U32>
__device__ __forceinline__ float4 sat_diff4(const float* __restrict__ PXY, int a0, int a1, int rank) {
    constexpr int RP = tc::Layout::RP;
    constexpr int PSTRIDE = U32 ? RP : 2 * RP;
    const float* p0 = PXY + (int64_t)a0 * PSTRIDE + rank;
    const float* p1 = PXY + (int64_t)a1 * PSTRIDE + rank;
    if (U32) {
        const uint4 q1 = ldg_sat(p1), q0 = ldg_sat(p0);
        return make_float4(__uint2float_rn(q1.x - q0.x), __uint2float_rn(q1.y - q0.y), __uint2float_rn(q1.z - q0.z),
                           __uint2float_rn(q1.w - q0.w));
    }
    const float4 h1 = ldg4(p1), h0 = ldg4(p0), l1 = ldg4(p1 + RP), l0 = ldg4(p0 + RP);
    return make_float4((h1.x - h0.x) + (l1.x - l0.x), (h1.y - h0.y) + (l1.y - l0.y), (h1.z - h0.z) + (l1.z - l0.z),
                       (h1.w - h0.w) + (l1.w - l0.w));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void producer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// list[0 .. *count): ids of the eligible 128-query blocks of the binned order (query.cu: tc_classify_kernel);
// perm: the binning permutation; each CTA takes a contiguous share of the list.
// Warps 0-7 decode the block's queries, build the operands and run the epilogue; warp 8 issues the MMAs.
// The A operand is built 32 ranks (one K-block) at a time into two buffers: full[buf] (8 producer-warp
// arrivals) hands a chunk to the issuer, the issuer's tcgen05.commit on empty[buf] hands the buffer back, and
// its commit on dfull after a block's last chunk releases the accumulator to the epilogue.
template <bool WRAP, bool U32>
__global__ void __launch_bounds__(tc::Layout::THREADS, 2)
    query_tc_kernel(const QParams p, const pndf_query* __restrict__ q, const uint32_t* __restrict__ perm,
                    const uint32_t* __restrict__ list, const uint32_t* __restrict__ count, float* __restrict__ out) {
    using LY = tc::Layout;
    extern __shared__ __align__(16) unsigned char tc_raw[];
    // 1024-byte alignment of the operand tiles, computed on the shared-space address
    unsigned char* sm = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);
    unsigned char* sB = sm + LY::A_BYTES;
    QDesc* sd = reinterpret_cast<QDesc*>(sB + LY::B_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sd) + LY::DESC);
    uint64_t* empty = full + 2;
    uint64_t* dfull = empty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dfull + 1);
    int* s_wide = reinterpret_cast<int*>(tmem_slot + 1);  // [2]: a query of the block has a wide range
    const uint32_t sA_u = smem_u32(sm), sB_u = smem_u32(sB);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int k = 0; k < 2; ++k) {
            mbar_init(full + k, 8);
            mbar_init(empty + k, 1);
        }
        mbar_init(dfull, 1);
        s_wide[0] = 0;
        s_wide[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(LY::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    // kind::tf32, D fp32, A/B K-major, N = 16, M = 128
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) |
                               ((uint32_t)(LY::M >> 4) << 24);

    const uint32_t nb = *count;
    const uint32_t per = (nb + gridDim.x - 1) / gridDim.x;
    const uint32_t b0 = blockIdx.x * per;
    const uint32_t b1 = b0 + per < nb ? b0 + per : nb;

    if (warp == 8) {
        // ---- MMA issuer: one thread; chunk u of the CTA's stream uses buffer u & 1
        if (lane == 0) {
            uint32_t u = 0;
            for (uint32_t b = b0; b < b1; ++b) {
#pragma unroll 1
                for (int kc = 0; kc < LY::NCH; ++kc, ++u) {
                    const uint32_t buf = u & 1u;
                    tc::mbar_wait(full + buf, (u >> 1) & 1u);
                    tc::fence_after();
                    const uint64_t dah = tc::sw128_desc(sA_u + buf * LY::A_BUF);
                    const uint64_t dal = tc::sw128_desc(sA_u + buf * LY::A_BUF + LY::A_TILE);
                    const uint64_t db = tc::sw128_desc(sB_u + kc * LY::B_TILE);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {  // UMMA K = 8 tf32 = 32 bytes = +2 in the address field
                        tc::mma_tf32(tmem, dah + 2 * k, db + 2 * k, idesc, (kc | k) != 0);
                        tc::mma_tf32(tmem, dal + 2 * k, db + 2 * k, idesc, 1u);
                    }
                    tc::mma_commit(empty + buf);  // the buffer is free when these MMAs have read it
                }
                tc::mma_commit(dfull);  // the block's accumulator is complete
            }
        }
    } else {
        // ---- producers: a quarter warp per query, 4 ranks per lane; this thread's 4 queries of a block and
        // where their 16-byte chunks go in the hi tile never change
        const int l8 = lane & 7;
        uint32_t aoff[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) aoff[i] = tc::sw128_off(warp * 16 + 4 * i + (lane >> 3), l8);
        // thread t < 128 decodes query t of a block; its perm entry and record are fetched one block ahead
        uint32_t src_n = 0;
        pndf_query rec_n;
        if (tid < LY::M && b0 < b1) {
            src_n = __ldg(perm + (int64_t)__ldg(list + b0) * LY::M + tid);
            rec_n = ldg_query(q + src_n);
        }
        uint32_t u = 0;
        int prev0 = -1, prev3 = -1, prev4 = -1, prev7 = -1;
        for (uint32_t b = b0; b < b1; ++b) {
            const int wb = (int)((b - b0) & 1u);
            if (tid < LY::M) {  // a2/a3
                decode<WRAP, true>(p, rec_n, (int32_t)src_n, sd[tid]);
                if (sd[tid].mode != 3) s_wide[wb] = 1;
                if (b + 1 < b1) src_n = __ldg(perm + (int64_t)__ldg(list + b + 1) * LY::M + tid);
            }
            producer_sync();
            const bool all_narrow = s_wide[wb] == 0;
            if (tid == 0) s_wide[wb ^ 1] = 0;
            // B operand: the block's 8 Zc rows (one key => the same rows for every query), rebuilt when they
            // change; the previous block's MMAs (which read B) are complete: every producer waited on dfull
            const int4 r03 = *reinterpret_cast<const int4*>(&sd[0].row[0]);
            const int4 r47 = *reinterpret_cast<const int4*>(&sd[0].row[4]);
            if (r03.x != prev0 || r03.w != prev3 || r47.x != prev4 || r47.w != prev7) {
                const float* zr = p.Zc + (size_t)sd[0].row[warp] * LY::RP;  // warp k splits row k
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rank = h * 128 + 4 * lane;
                    float4 hi, lo;
                    tc::split4(ldg4(zr + rank), hi, lo);
                    const uint32_t tile = sB_u + (uint32_t)((rank >> 5) * LY::B_TILE);
                    const int c = (rank & 31) >> 2;
                    sts4(tile + tc::sw128_off(warp, c), hi);
                    sts4(tile + tc::sw128_off(8 + warp, c), lo);
                }
                prev0 = r03.x;
                prev3 = r03.w;
                prev4 = r47.x;
                prev7 = r47.w;
            }
            int rx[4], ry[4];  // range-table rows of this thread's 4 queries (narrow ranges)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const QDesc& d = sd[warp * 16 + 4 * i + (lane >> 3)];
                rx[i] = d.sat[0];
                ry[i] = d.sat[2];
            }
            float4 dx[4], dy[4];
            // dx, dy of this thread's 4 (query, 4-rank) items of chunk kc
            auto load_chunk = [&](int kc) {
                const int rank = kc * LY::KC + 4 * l8;
                if (all_narrow) {
                    const float* dt = p.DT + rank;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        dx[i] = ldg4(dt + (size_t)rx[i] * LY::RP);
                        dy[i] = ldg4(dt + (size_t)ry[i] * LY::RP);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const QDesc& d = sd[warp * 16 + 4 * i + (lane >> 3)];
                        const int4 so = *reinterpret_cast<const int4*>(&d.sat[0]);
                        dx[i] = (d.mode & 1) ? ldg4(p.DT + (size_t)so.x * LY::RP + rank)
                                             : sat_diff4<U32>(p.PXY, so.x, so.y, rank);
                        dy[i] = (d.mode & 2) ? ldg4(p.DT + (size_t)so.z * LY::RP + rank)
                                             : sat_diff4<U32>(p.PXY, so.z, so.w, rank);
                    }
                }
            };
            load_chunk(0);
#pragma unroll 1
            for (int kc = 0; kc < LY::NCH; ++kc, ++u) {
                const uint32_t buf = u & 1u;
                float4 hi[4], lo[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 pxy = __fmul2_rn(make_float2(dx[i].x, dx[i].y), make_float2(dy[i].x, dy[i].y));
                    const float2 pzw = __fmul2_rn(make_float2(dx[i].z, dx[i].w), make_float2(dy[i].z, dy[i].w));
                    hi[i].x = __uint_as_float(__float_as_uint(pxy.x) & 0xffffe000u);
                    hi[i].y = __uint_as_float(__float_as_uint(pxy.y) & 0xffffe000u);
                    hi[i].z = __uint_as_float(__float_as_uint(pzw.x) & 0xffffe000u);
                    hi[i].w = __uint_as_float(__float_as_uint(pzw.y) & 0xffffe000u);
                    const float2 lxy = __fadd2_rn(pxy, make_float2(-hi[i].x, -hi[i].y));
                    const float2 lzw = __fadd2_rn(pzw, make_float2(-hi[i].z, -hi[i].w));
                    lo[i] = make_float4(lxy.x, lxy.y, lzw.x, lzw.y);
                }
                // the next chunk's rows (or, after the last chunk, the next block's record) are in flight
                // while this chunk is stored and multiplied
                if (kc + 1 < LY::NCH)
                    load_chunk(kc + 1);
                else if (tid < LY::M && b + 1 < b1)
                    rec_n = ldg_query(q + src_n);
                tc::mbar_wait(empty + buf, ((u >> 1) & 1u) ^ 1u);  // the MMAs of chunk u - 2 have read the buffer
                const uint32_t ab = sA_u + buf * LY::A_BUF;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    sts4(ab + aoff[i], hi[i]);
                    sts4(ab + LY::A_TILE + aoff[i], lo[i]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> tcgen05.mma reads
                __syncwarp();
                if (lane == 0) mbar_arrive(full + buf);
            }
            tc::mbar_wait(dfull, (b - b0) & 1u);  // every MMA of the block is complete (D final, B and sd free)
            tc::fence_after();
            if (warp < 4) {  // a6: thread t owns accumulator row t (TMEM lane t): weights, area, write
                float v[16];
                tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
                const QDesc& d = sd[tid];
                const float4 w03 = *reinterpret_cast<const float4*>(&d.w[0]);
                const float4 w47 = *reinterpret_cast<const float4*>(&d.w[4]);
                const float w[8] = {w03.x, w03.y, w03.z, w03.w, w47.x, w47.y, w47.z, w47.w};
                float res = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) res = fmaf(w[k], v[k] + v[8 + k], res);
                if (d.out >= 0) out[d.out] = res / d.div;
                tc::fence_before();
            }
            producer_sync();  // the descriptors are rewritten by the next block's decode
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 8) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(LY::TMEM_COLS)
                     : "memory");
    }
}

template <bool W, bool U>
static cudaError_t launch_tc(const QParams& p, const pndf_query* q, const uint32_t* perm, const uint32_t* list,
                             const uint32_t* count, float* out, int num_sms, cudaStream_t st) {
    constexpr int smem = tc::Layout::BYTES;
    auto* kfn = query_tc_kernel<W, U>;
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    kfn<<<2 * num_sms, tc::Layout::THREADS, smem, st>>>(p, q, perm, list, count, out);
    return cudaGetLastError();
}

}  // namespace pndf
