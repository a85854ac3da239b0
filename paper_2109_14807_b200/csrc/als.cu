// als.cu -- the GPU factor builder: the footprint NDF tensor the paper compresses
// (Eq. 2) and its nonnegative CP decomposition by alternating least squares (Eq. 5),
// one global group (readings 14, 23).  Declarations and contracts: include/pndf.h.
//
// Per ALS sweep (modes Z, X, Y; DESIGN.md §5 "Factor builder"):
//   MTTKRP_Z = D_(z) (X kr Y)        tcgen05 GEMM  [P x A^2] . [A^2 x Rp]         -> fp32 rows
//   MTTKRP_X = sum_z Z_z (D_z Y)     tcgen05 GEMM  [(P A) x A] . [A x Rp], epilogue scales the
//                                    accumulator row (z, x) by Z[z] and reduces over z in registers
//   MTTKRP_Y = same on Dt = D with x, y swapped
//   HALS column updates in fp64 (warp per row), Gram matrices in fp64, fit error, norm balance.
// D is tf32-exact by construction (pndf_hist_tensor rounds it); the factor operand B is split into
// tf32 hi + lo parts and both products accumulate in the same TMEM tile, so the contraction is
// accurate to ~2^-22 relative plus fp32 accumulation.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "device.cuh"
#include "pndf.h"

namespace pndf {
void set_last_error(const char* msg);  // store.cu: the text pndf_last_cuda_error returns
}

namespace pndf {
namespace als {

constexpr int BM = 128;  // UMMA M: accumulator rows = TMEM lanes
constexpr int BK = 32;   // K elements per pipeline stage: one 128-byte swizzle row of fp32
constexpr double kEps = 1e-30;  // HALS floor (oracle/als.py HALS_EPS)

// ------------------------------------------------------------------------------ histogram --
struct HistLevel {
    int64_t off;   // first row of the level
    int32_t s, n;  // stride, grid side
    int32_t qmin, wf;
    int32_t woff;  // offset of the level's weights in the table
    double tot;    // (sum w)^2
};

// round to nearest-even at 11 significant bits (tf32), from fp64; exact as fp32 (oracle.als.tf32_round)
__device__ __forceinline__ float tf32_rne(double v) {
    if (v == 0.0) return 0.f;
    int e;
    const double m = frexp(v, &e);
    return (float)ldexp(rint(ldexp(m, 11)), e - 11);
}

// One CTA per footprint row: exact uint64 counts of the footprint-weighted texel bins in shared memory
// (padded [y][A+1] so the transposed write below is conflict-free), then D[z][x][y] and Dt[z][y][x].
__global__ void __launch_bounds__(256) hist_kernel(const uint16_t* __restrict__ bins, int N, int A,
                                                   const HistLevel* __restrict__ lv, int L,
                                                   const uint32_t* __restrict__ wtab, int64_t P,
                                                   float* __restrict__ D, float* __restrict__ Dt) {
    extern __shared__ unsigned long long cnt[];  // [A][A+1]
    const int AP = A + 1;
    for (int64_t z = blockIdx.x; z < P; z += gridDim.x) {
        int l = 0;
        while (l + 1 < L && z >= lv[l + 1].off) ++l;
        const HistLevel h = lv[l];
        const int64_t c = z - h.off;
        const int64_t i = c % h.n, j = c / h.n;
        for (int b = threadIdx.x; b < A * AP; b += blockDim.x) cnt[b] = 0ull;
        __syncthreads();
        const int bu = (int)((((int64_t)i * h.s + h.qmin) % N + N) % N);
        const int bv = (int)((((int64_t)j * h.s + h.qmin) % N + N) % N);
        const uint32_t* w = wtab + h.woff;
        const int nwin = h.wf * h.wf;  // <= N^2 < 2^31; 32-bit division (the 64-bit one costs ~70 instructions)
        for (int t = threadIdx.x; t < nwin; t += blockDim.x) {
            const int q = t / h.wf, p = t - q * h.wf;
            int v = bv + q, u = bu + p;
            if (v >= N) v -= N;
            if (u >= N) u = 0 + (u - N);
            const int b = bins[(int64_t)v * N + u];  // x + A*y
            const int x = b % A, y = b / A;
            atomicAdd(&cnt[y * AP + x], (unsigned long long)w[q] * (unsigned long long)w[p]);
        }
        __syncthreads();
        // counts -> tf32 values in place (once per bin; most bins of a footprint are empty), then both
        // layouts are written with coalesced stores
        for (int b = threadIdx.x; b < A * AP; b += blockDim.x) {
            const unsigned long long k = cnt[b];
            cnt[b] = k ? (unsigned long long)__float_as_uint(tf32_rne((double)k / h.tot)) : 0ull;
        }
        __syncthreads();
        const int64_t base = z * (int64_t)A * A;
        for (int o = threadIdx.x; o < A * A; o += blockDim.x) {
            const int x = o / A, y = o % A;  // D[z][x][y]
            D[base + o] = __uint_as_float((uint32_t)cnt[y * AP + x]);
        }
        if (Dt)
            for (int o = threadIdx.x; o < A * A; o += blockDim.x) {
                const int y = o / A, x = o % A;  // Dt[z][y][x]
                Dt[base + o] = __uint_as_float((uint32_t)cnt[y * AP + x]);
            }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------ operand staging --
// B operands are [Rp][K] fp32, K-contiguous (UMMA K-major), split v = hi + lo with hi tf32-exact.
__device__ __forceinline__ void split_store(double v, float* hi, float* lo, int64_t i) {
    const float h = tf32_rne(v);
    hi[i] = h;
    lo[i] = (float)(v - (double)h);
}

// Khatri-Rao operand of mode Z: B[r][x*A + y] = X[x][r] Y[y][r] (the column order of D_(z))
__global__ void kr_operand_kernel(const double* __restrict__ X, const double* __restrict__ Y, int A, int R, int RP,
                                  float* __restrict__ hi, float* __restrict__ lo) {
    const int64_t K = (int64_t)A * A, n = (int64_t)RP * K;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / K);
        const int k = (int)(e % K);
        const double v = r < R ? X[(int64_t)(k / A) * R + r] * Y[(int64_t)(k % A) * R + r] : 0.0;
        split_store(v, hi, lo, e);
    }
}

// operand of modes X / Y: B[r][k] = F[k][r]
__global__ void t_operand_kernel(const double* __restrict__ F, int A, int R, int RP, float* __restrict__ hi,
                                 float* __restrict__ lo) {
    const int64_t n = (int64_t)RP * A;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / A), k = (int)(e % A);
        split_store(r < R ? F[(int64_t)k * R + r] : 0.0, hi, lo, e);
    }
}

// ------------------------------------------------------------------ tcgen05 MTTKRP GEMM --
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// K-major operand tile in the 128-byte swizzle layout TMA writes (8-row atoms of 1024 B):
// start >> 4, LBO = 1 (unused for swizzled K-major), SBO = 1024 B, version 1, layout SWIZZLE_128B
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
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
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

struct GemmArgs {
    int64_t rows;      // A-operand rows (P for mode Z, P*A for modes X/Y)
    int64_t ntiles;    // ceil(rows / BM)
    int32_t kblocks;   // K / BK
    int32_t stages;
    int32_t a_shift;   // log2(A): z = row >> a_shift (epilogue 1)
    int32_t bres;      // 1: the whole B operand (kblocks x hi/lo) is loaded once and stays in shared memory
    int32_t kbs;       // K-blocks per pipeline stage (> 1 only with bres: one 3-D TMA box per tile row block)
    float* out;        // epilogue 0: [rows][RP]
    const float* Zf;   // epilogue 1: [P][RP] fp32 Z
    float* part;       // epilogue 1: [grid][BM][RP] per-thread partial sums
};

template <int RP>
struct GemmLayout {
    static constexpr int A_BYTES = BM * BK * 4;
    static constexpr int B_BYTES = RP * BK * 4;
    static constexpr int STAGE = A_BYTES + 2 * B_BYTES;  // A, B hi, B lo (all 1024-byte multiples)
    static constexpr int TMEM_COLS = (2 * RP <= 32) ? 32 : (2 * RP <= 64) ? 64 : (2 * RP <= 128) ? 128 : 256;
    static int stages() { return std::min(8, (200 * 1024) / STAGE); }
    static size_t smem(int st) { return 1024 + (size_t)st * STAGE + 256; }
    // B-resident variant (short K: modes X / Y): B region [kblocks][hi | lo] then A-only stages
    __host__ __device__ static int bres_bytes(int kblocks) { return kblocks * 2 * B_BYTES; }
    static bool bres_fits(int kblocks) { return bres_bytes(kblocks) <= 64 * 1024; }
    static int bres_stages(int kblocks, int kbs) {
        return std::min(8, (200 * 1024 - bres_bytes(kblocks)) / (kbs * A_BYTES));
    }
    static size_t bres_smem(int kblocks, int kbs, int st) {
        return 1024 + (size_t)bres_bytes(kblocks) + (size_t)st * kbs * A_BYTES + 256;
    }
};

// Warp-specialised persistent GEMM, one CTA per SM: warps 0-3 epilogue (TMEM lanes 32w..32w+31),
// warp 4 TMA producer, warp 5 TMEM owner + MMA issuer.  Accumulators double-buffered in TMEM so the
// epilogue of tile i overlaps the MMAs of tile i+1.
template <int RP, int EPI>
__global__ void __launch_bounds__(192, 1) mttkrp_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                             const __grid_constant__ CUtensorMap tmBh,
                                                             const __grid_constant__ CUtensorMap tmBl,
                                                             const GemmArgs g) {
    using LY = GemmLayout<RP>;
    extern __shared__ unsigned char gsm_raw[];
    unsigned char* gsm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gsm_raw) + 1023) & ~uintptr_t(1023));
    const int S = g.stages;
    const bool bres = g.bres != 0;
    const int stage_bytes = bres ? g.kbs * LY::A_BYTES : LY::STAGE;
    unsigned char* bsm = gsm;                                                   // resident B (bres)
    unsigned char* asm_ = gsm + (bres ? LY::bres_bytes(g.kblocks) : 0);          // stages
    uint64_t* full = reinterpret_cast<uint64_t*>(asm_ + (size_t)S * stage_bytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint64_t* bfull = tempty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull + b, 1);
            mbar_init(tempty + b, 4 * 32);
        }
        mbar_init(bfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(LY::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        if (lane == 0) {
            if (bres) {
                mbar_arrive_expect_tx(bfull, LY::bres_bytes(g.kblocks));
                for (int kb = 0; kb < g.kblocks; ++kb) {
                    tma_2d(bsm + (size_t)(2 * kb) * LY::B_BYTES, &tmBh, kb * BK, 0, bfull);
                    tma_2d(bsm + (size_t)(2 * kb + 1) * LY::B_BYTES, &tmBl, kb * BK, 0, bfull);
                }
            }
            int s = 0;
            uint32_t ph = 0;
            for (int64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
                for (int kb = 0; kb < g.kblocks; kb += g.kbs) {
                    mbar_wait(empty + s, ph ^ 1u);
                    unsigned char* st = asm_ + (size_t)s * stage_bytes;
                    mbar_arrive_expect_tx(full + s, stage_bytes);
                    if (g.kbs > 1)  // [kb][128 rows][32] in one box: whole 128-row x K slab, read contiguously
                        tma_3d(st, &tmA, 0, (int)(tile * BM), kb, full + s);
                    else
                        tma_2d(st, &tmA, kb * BK, (int)(tile * BM), full + s);
                    if (!bres) {
                        tma_2d(st + LY::A_BYTES, &tmBh, kb * BK, 0, full + s);
                        tma_2d(st + LY::A_BYTES + LY::B_BYTES, &tmBl, kb * BK, 0, full + s);
                    }
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 5) {
        // kind::tf32, D fp32, A/B K-major, N = RP, M = 128
        constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(RP >> 3) << 17) |
                                   ((uint32_t)(BM >> 4) << 24);
        int s = 0;
        uint32_t ph = 0;
        int i = 0;
        if (bres) mbar_wait(bfull, 0);
        for (int64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++i) {
            const int b = i & 1;
            mbar_wait(tempty + b, ((uint32_t)(i >> 1) & 1u) ^ 1u);
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(b * RP);
            for (int kb0 = 0; kb0 < g.kblocks; kb0 += g.kbs) {
                mbar_wait(full + s, ph);
                tc_fence_after();
                if (lane == 0) {
                    for (int j = 0; j < g.kbs; ++j) {
                        const int kb = kb0 + j;
                        const uint32_t sa = smem_u32(asm_ + (size_t)s * stage_bytes) + (uint32_t)(j * LY::A_BYTES);
                        const uint32_t sb = bres ? smem_u32(bsm + (size_t)(2 * kb) * LY::B_BYTES) : sa + LY::A_BYTES;
                        const uint64_t da = sw128_desc(sa);
                        const uint64_t dh = sw128_desc(sb);
                        const uint64_t dl = sw128_desc(sb + LY::B_BYTES);
#pragma unroll
                        for (int k = 0; k < BK / 8; ++k) {  // UMMA K = 8 tf32 = 32 bytes = +2 in the address field
                            mma_tf32(d, da + 2 * k, dh + 2 * k, idesc, (kb | k) != 0);
                            mma_tf32(d, da + 2 * k, dl + 2 * k, idesc, 1u);
                        }
                    }
                    mma_commit(empty + s);  // frees the stage when these MMAs complete
                }
                __syncwarp();
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
            if (lane == 0) mma_commit(tfull + b);
            __syncwarp();
        }
    } else {
        // epilogue: thread t owns accumulator row t of the tile (TMEM lane t)
        const int t = threadIdx.x;
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        float acc[EPI == 1 ? RP : 1];
        if (EPI == 1)
#pragma unroll
            for (int r = 0; r < RP; ++r) acc[r] = 0.f;
        int i = 0;
        for (int64_t tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x, ++i) {
            const int b = i & 1;
            const int64_t row = tile * BM + t;
            const bool ok = row < g.rows;
            mbar_wait(tfull + b, (uint32_t)(i >> 1) & 1u);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < RP / 16; ++c) {
                float v[16];
                tmem_ld16(tmem + lane_base + (uint32_t)(b * RP + c * 16), v);
                if (EPI == 0) {
                    if (ok) {
                        float4* o = reinterpret_cast<float4*>(g.out + row * RP + c * 16);
#pragma unroll
                        for (int q = 0; q < 4; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    }
                } else if (ok) {
                    const float4* zr = reinterpret_cast<const float4*>(g.Zf + (row >> g.a_shift) * RP + c * 16);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float4 zz = __ldg(zr + q);
                        acc[c * 16 + 4 * q + 0] = fmaf(zz.x, v[4 * q + 0], acc[c * 16 + 4 * q + 0]);
                        acc[c * 16 + 4 * q + 1] = fmaf(zz.y, v[4 * q + 1], acc[c * 16 + 4 * q + 1]);
                        acc[c * 16 + 4 * q + 2] = fmaf(zz.z, v[4 * q + 2], acc[c * 16 + 4 * q + 2]);
                        acc[c * 16 + 4 * q + 3] = fmaf(zz.w, v[4 * q + 3], acc[c * 16 + 4 * q + 3]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty + b);
        }
        if (EPI == 1) {
            float* p = g.part + ((int64_t)blockIdx.x * BM + t) * RP;
#pragma unroll
            for (int r = 0; r < RP; ++r) p[r] = acc[r];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(LY::TMEM_COLS)
                     : "memory");
    }
}

// M[x][r] = sum over CTAs and accumulator rows t = x (mod A) of the partials (fp64, fixed order):
// one block per output, strided partial sums then a shared-memory tree
__global__ void __launch_bounds__(128) part_reduce_kernel(const float* __restrict__ part, int grid, int A, int R,
                                                          int RP, double* __restrict__ M) {
    __shared__ double red[128];
    const int e = blockIdx.x;
    const int x = e / R, r = e % R;
    const int per_cta = BM / A;  // accumulator rows of one CTA holding x
    const int n = grid * per_cta;
    double s = 0.0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const int c = k / per_cta, t = x + (k % per_cta) * A;
        s += (double)part[((int64_t)c * BM + t) * RP + r];
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 64; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) M[e] = red[0];
}

// ------------------------------------------------------------------------- small kernels --
// per-block partial Gram matrices F^T F over a row range (fp64)
__global__ void gram_part_kernel(const double* __restrict__ F, int64_t rows, int R, double* __restrict__ part) {
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
        const int a = e / R, b = e % R;
        double s = 0.0;
        for (int64_t i = r0; i < r1; ++i) s += F[i * R + a] * F[i * R + b];
        part[(int64_t)blockIdx.x * R * R + e] = s;
    }
}
// out[e] = sum_p part[p][e]: one block per entry (fixed order: strided sums, then a tree)
__global__ void __launch_bounds__(128) sum_parts_kernel(const double* __restrict__ part, int nparts, int n,
                                                        double* __restrict__ out) {
    __shared__ double red[128];
    const int e = blockIdx.x;
    double s = 0.0;
    for (int p = threadIdx.x; p < nparts; p += blockDim.x) s += part[(int64_t)p * n + e];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 64; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[e] = red[0];
}

// HALS column pass with one THREAD per row (R <= 64: the row lives in registers, G is broadcast from
// shared memory, no shuffles), fused with the block's partial Gram matrix F^T F of the updated rows
// (rows staged in shared memory, each thread owns RT*RT/TPB Gram entries).  Same update as hals_kernel.
template <int RT, int TPB>
__global__ void __launch_bounds__(TPB) hals_rows_kernel(double* __restrict__ F, int64_t rows, int R, int RP,
                                                        const float* __restrict__ Mf, const double* __restrict__ Md,
                                                        const double* __restrict__ G1, const double* __restrict__ G2,
                                                        float* __restrict__ Ff, double* __restrict__ gpart) {
    constexpr int NE = (RT * RT + TPB - 1) / TPB;  // Gram entries per thread
    constexpr int RS = RT + 1;                     // padded row stride in shared memory
    __shared__ double G[RT * RT];
    __shared__ double inv[RT];
    extern __shared__ double rowbuf[];  // [TPB][RS]
    for (int e = threadIdx.x; e < RT * RT; e += TPB) {
        const int a = e / RT, b = e % RT;
        G[e] = (a < R && b < R) ? G1[a * R + b] * G2[a * R + b] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < RT; r += TPB) inv[r] = (r < R && G[r * RT + r] > 0.0) ? 1.0 / G[r * RT + r] : 0.0;
    __syncthreads();
    double gacc[NE];
#pragma unroll
    for (int k = 0; k < NE; ++k) gacc[k] = 0.0;
    for (int64_t base = (int64_t)blockIdx.x * TPB; base < rows; base += (int64_t)gridDim.x * TPB) {
        const int64_t z = base + threadIdx.x;
        const bool valid = z < rows;
        double f[RT];
#pragma unroll
        for (int s = 0; s < RT; ++s) f[s] = (valid && s < R) ? F[z * R + s] : 0.0;
        if (valid) {
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                if (r < R && inv[r] > 0.0) {
                    double dot = 0.0;
#pragma unroll
                    for (int s = 0; s < RT; ++s) dot = fma(f[s], G[s * RT + r], dot);
                    const double m = Mf ? (double)Mf[z * RP + r] : Md[z * R + r];
                    f[r] = fmax(kEps, f[r] + (m - dot) * inv[r]);
                }
            }
#pragma unroll
            for (int s = 0; s < RT; ++s)
                if (s < R) F[z * R + s] = f[s];
            if (Ff) {
#pragma unroll
                for (int s = 0; s < RT; ++s) Ff[z * RP + s] = s < R ? (float)f[s] : 0.f;
                for (int s = RT; s < RP; ++s) Ff[z * RP + s] = 0.f;
            }
        }
        if (gpart) {
#pragma unroll
            for (int s = 0; s < RT; ++s) rowbuf[threadIdx.x * RS + s] = f[s];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NE; ++k) {
                const int e = threadIdx.x + k * TPB;
                if (e < RT * RT) {
                    const int a = e / RT, b = e % RT;
                    double acc = gacc[k];
                    for (int t = 0; t < TPB; ++t) acc = fma(rowbuf[t * RS + a], rowbuf[t * RS + b], acc);
                    gacc[k] = acc;
                }
            }
            __syncthreads();
        }
    }
    if (gpart)
#pragma unroll
        for (int k = 0; k < NE; ++k) {
            const int e = threadIdx.x + k * TPB;
            if (e < RT * RT) {
                const int a = e / RT, b = e % RT;
                if (a < R && b < R) gpart[(int64_t)blockIdx.x * R * R + a * R + b] = gacc[k];
            }
        }
}

// G[r][s] *= a_r a_s (the Gram matrix of a column-scaled factor)
__global__ void scale_gram_kernel(double* __restrict__ G, int R, const double* __restrict__ a) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < R * R) G[e] *= a[e / R] * a[e % R];
}

// HALS column pass (oracle/als.py hals_update), one warp per row, G = G1 * G2 (Hadamard) in shared memory:
// for r in order: F[r] <- max(eps, F[r] + (M[r] - sum_s F[s] G[s][r]) / G[r][r])
template <int KR>  // ranks per lane = ceil(R / 32)
__global__ void __launch_bounds__(256) hals_kernel(double* __restrict__ F, int64_t rows, int R, int RP,
                                                   const float* __restrict__ Mf, const double* __restrict__ Md,
                                                   const double* __restrict__ G1, const double* __restrict__ G2,
                                                   float* __restrict__ Ff) {
    extern __shared__ double G[];
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) G[e] = G1[e] * G2[e];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t z = w0; z < rows; z += nw) {
        double f[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int s = lane + 32 * k;
            f[k] = s < R ? F[z * R + s] : 0.0;
        }
        for (int r = 0; r < R; ++r) {
            double dot = 0.0;
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int s = lane + 32 * k;
                if (s < R) dot = fma(f[k], G[s * R + r], dot);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            const double grr = G[r * R + r];
            if (grr > 0.0 && lane == (r & 31)) {
                const double m = Mf ? (double)Mf[z * RP + r] : Md[z * R + r];
#pragma unroll
                for (int k = 0; k < KR; ++k)
                    if (k == (r >> 5)) f[k] = fmax(kEps, f[k] + (m - dot) / grr);
            }
        }
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int s = lane + 32 * k;
            if (s < R) F[z * R + s] = f[k];
        }
        if (Ff)
            for (int s = lane; s < RP; s += 32) Ff[z * RP + s] = s < R ? (float)F[z * R + s] : 0.f;
    }
}

// fp32 input factors -> fp64 master (+ fp32 padded copy); flags negative / non-finite entries
__global__ void load_factor_kernel(const float* __restrict__ in, int64_t rows, int R, int RP, double* __restrict__ F,
                                   float* __restrict__ Ff, uint32_t* __restrict__ bad) {
    const int64_t n = rows * RP;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = e / RP;
        const int r = (int)(e % RP);
        float v = 0.f;
        if (r < R) {
            v = in[z * R + r];
            if (!(v >= 0.f) || isinf(v)) atomicOr(bad, 1u);
            F[z * R + r] = (double)v;
        }
        if (Ff) Ff[e] = v;
    }
}

__global__ void sumsq_part_kernel(const float* __restrict__ D, int64_t n, double* __restrict__ part) {
    double s = 0.0;
    const float4* D4 = reinterpret_cast<const float4*>(D);  // n % 4 == 0 (A >= 32)
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n / 4; e += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(D4 + e);
        s = fma((double)v.x, (double)v.x, s);
        s = fma((double)v.y, (double)v.y, s);
        s = fma((double)v.z, (double)v.z, s);
        s = fma((double)v.w, (double)v.w, s);
    }
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// out[0] = <D, D_hat> = sum My * Y, out[1] = ||D_hat||^2 = sum GZ * GX * GY (oracle/als.py fit_error)
__global__ void err_terms_kernel(const double* __restrict__ My, const double* __restrict__ Y, int A, int R,
                                 const double* __restrict__ GZ, const double* __restrict__ GX,
                                 const double* __restrict__ GY, double* __restrict__ out) {
    __shared__ double red[2][256];
    double a = 0.0, b = 0.0;
    for (int e = threadIdx.x; e < A * R; e += blockDim.x) a += My[e] * Y[e];
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) b += GZ[e] * GX[e] * GY[e];
    red[0][threadIdx.x] = a;
    red[1][threadIdx.x] = b;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = red[0][0];
        out[1] = red[1][0];
    }
}

// per-rank multipliers of the norm balance (oracle/als.py balance): geometric mean of the three norms
__global__ void balance_scale_kernel(const double* __restrict__ GZ, const double* __restrict__ GX,
                                     const double* __restrict__ GY, int R, double* __restrict__ sc /*[3][R]*/) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const double nz = sqrt(GZ[r * R + r]), nx = sqrt(GX[r * R + r]), ny = sqrt(GY[r * R + r]);
    const bool ok = nz > 0.0 && nx > 0.0 && ny > 0.0;
    const double g = ok ? cbrt(nz * nx * ny) : 1.0;
    sc[r] = ok ? g / nz : 1.0;
    sc[R + r] = ok ? g / nx : 1.0;
    sc[2 * R + r] = ok ? g / ny : 1.0;
}
__global__ void scale_cols_kernel(double* __restrict__ F, int64_t rows, int R, const double* __restrict__ sc,
                                  int mode /*0: multiply, 1: divide*/, float* __restrict__ Ff, int RP) {
    const int64_t n = rows * R;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % R);
        const double v = mode ? F[e] / sc[r] : F[e] * sc[r];
        F[e] = v;
        if (Ff) Ff[(e / R) * RP + r] = (float)v;
    }
}

// normalise (oracle/als.py normalise): column sums / maxima and row masses
__global__ void col_reduce_kernel(const double* __restrict__ F, int64_t rows, int R, int op /*0 sum, 1 max*/,
                                  double* __restrict__ part) {
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
        double s = 0.0;
        for (int64_t i = r0; i < r1; ++i) s = op ? fmax(s, F[i * R + r]) : s + F[i * R + r];
        part[(int64_t)blockIdx.x * R + r] = s;
    }
}
__global__ void col_finish_kernel(const double* __restrict__ part, int nparts, int R, int op,
                                  double* __restrict__ out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s = op ? fmax(s, part[(int64_t)p * R + r]) : s + part[(int64_t)p * R + r];
    out[r] = s > 0.0 ? s : 1.0;  // zero sums / maxima keep the rank unscaled
}
__global__ void mul2_kernel(const double* __restrict__ a, const double* __restrict__ b, int R, double* __restrict__ o) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < R) o[r] = a[r] * b[r];
}
__global__ void row_renorm_kernel(double* __restrict__ Z, int64_t rows, int R, const double* __restrict__ C) {
    const int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= rows) return;
    double m = 0.0;
    for (int r = 0; r < R; ++r) m += Z[z * R + r] * C[r];
    if (m > 0.0)
        for (int r = 0; r < R; ++r) Z[z * R + r] /= m;
}
__global__ void to_f32_kernel(const double* __restrict__ F, int64_t n, float* __restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = (float)F[e];
}
__global__ void fill_kernel(float* __restrict__ out, int n, float v) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) out[e] = v;
}
__global__ void rows_to_f64_kernel(const float* __restrict__ in, int64_t rows, int R, int RP, double* __restrict__ out) {
    const int64_t n = rows * R;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = (double)in[(e / R) * RP + e % R];
}


// ---------------------------------------------------------------- map-domain MTTKRP (no D) --
// The footprint tensor is a blur of the texels' one-hot angular histograms (Eq. 2: D[z][x][y] =
// sum over z's window of w_p w_q [bin(t) = (x, y)] / tot), so every MTTKRP contracts over TEXELS instead of
// over the P x A x A tensor, and D is never formed (DESIGN.md §5 "Factor builder"):
//   mode Z  M_Z[z] = (1/tot) sum_q w_q sum_p w_p  X[bx(t)] o Y[by(t)],   t = texel (p, q) of z's window
//   mode X  M_X[x] = sum_{t: bx(t) = x} Y[by(t)] o U[t],   U[t] = sum_z (1/tot) w_p w_q Z[z]  (the adjoint)
//   mode Y  M_Y[y] = sum_{t: by(t) = y} X[bx(t)] o U[t]
// Both blurs are separable: a pass along u at the level's stride, then one along v.  Work per sweep is
// ~3 x 3.5 N^2 L R FMAs instead of 3 P A^2 R, all in fp64 (the GEMM path's tf32(D) rounding is gone).
// Warps own one output row; lane k handles rank c0 + k of the 32-rank chunk blockIdx.y.
struct MapLevel {
    int64_t off;      // first Zc row of the level
    int64_t hoff;     // first row of the level's [N][n] block in the pass buffer
    int32_t s, n, qmin, wf, woff;
    double inv_tot;   // 1 / (sum w)^2
};

// level of row g among levels [l0, l1) (pass-buffer rows when by_hoff, else Zc rows)
__device__ __forceinline__ int map_level(const MapLevel* lv, int l0, int l1, int64_t g, bool by_hoff) {
    int l = l0;
    while (l + 1 < l1 && g >= (by_hoff ? lv[l + 1].hoff : lv[l + 1].off)) ++l;
    return l;
}

// H[hoff + v n + i][r] = sum_p w_p X[bx][r] Y[by][r] over texels (v, (i s + qmin + p) mod N), levels [l0, l1)
__global__ void __launch_bounds__(256) mz_h_kernel(const uint16_t* __restrict__ bins, int N, int A, int ash,
                                                   const MapLevel* __restrict__ lv, int l0, int l1,
                                                   const uint32_t* __restrict__ wtab, const double* __restrict__ X,
                                                   const double* __restrict__ Y, int R, double* __restrict__ H) {
    extern __shared__ double xs[];  // [2][A][32]: X, Y columns of this rank chunk
    double* ys = xs + A * 32;
    const int c0 = blockIdx.y * 32, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < A * 32; e += blockDim.x) {
        const int r = c0 + (e & 31);
        xs[e] = r < R ? X[(e >> 5) * R + r] : 0.0;
        ys[e] = r < R ? Y[(e >> 5) * R + r] : 0.0;
    }
    __syncthreads();
    const int64_t g0 = lv[l0].hoff, g1 = lv[l1 - 1].hoff + (int64_t)N * lv[l1 - 1].n;
    const int r = c0 + lane;
    for (int64_t g = g0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); g < g1;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const MapLevel h = lv[map_level(lv, l0, l1, g, true)];
        const int64_t c = g - h.hoff;
        const int v = (int)(c / h.n), i = (int)(c % h.n);
        int u = (int)((((int64_t)i * h.s + h.qmin) % N + N) % N);
        const uint16_t* brow = bins + (int64_t)v * N;
        const uint32_t* w = wtab + h.woff;
        double acc = 0.0;
#pragma unroll 4
        for (int p = 0; p < h.wf; ++p) {
            const int b = __ldg(brow + u);
            acc = fma((double)__ldg(w + p), xs[(b & (A - 1)) * 32 + lane] * ys[(b >> ash) * 32 + lane], acc);
            if (++u == N) u = 0;
        }
        if (r < R) H[g * R + r] = acc;
    }
}

// M[z][r] = inv_tot sum_q w_q H[hoff + ((j s + qmin + q) mod N) n + i][r], rows z of levels [l0, l1)
__global__ void __launch_bounds__(256) mz_v_kernel(int N, const MapLevel* __restrict__ lv, int l0, int l1,
                                                   const uint32_t* __restrict__ wtab, const double* __restrict__ H,
                                                   int R, double* __restrict__ M) {
    const int r = blockIdx.y * 32 + (threadIdx.x & 31);
    const int64_t z0 = lv[l0].off, z1 = lv[l1 - 1].off + (int64_t)lv[l1 - 1].n * lv[l1 - 1].n;
    for (int64_t z = z0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); z < z1;
         z += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const MapLevel h = lv[map_level(lv, l0, l1, z, false)];
        const int64_t c = z - h.off;
        const int j = (int)(c / h.n), i = (int)(c % h.n);
        int v = (int)((((int64_t)j * h.s + h.qmin) % N + N) % N);
        const uint32_t* w = wtab + h.woff;
        double acc = 0.0;
        if (r < R)
#pragma unroll 4
            for (int q = 0; q < h.wf; ++q) {
                acc = fma((double)__ldg(w + q), H[(h.hoff + (int64_t)v * h.n + i) * R + r], acc);
                if (++v == N) v = 0;
            }
        if (r < R) M[z * R + r] = acc * h.inv_tot;
    }
}

// adjoint along v: G[hoff + v n + i][r] = inv_tot sum_j sum_q [(j s + qmin + q) = v mod N] w_q Z[off + j n + i][r]
// (for d = (v - qmin) mod N the terms are q = d mod s + k s, j = d div s - k mod n, k = 0, 1, ... while q < wf)
__global__ void __launch_bounds__(256) u_g_kernel(int N, const MapLevel* __restrict__ lv, int l0, int l1,
                                                  const uint32_t* __restrict__ wtab, const double* __restrict__ Z,
                                                  int R, double* __restrict__ G) {
    const int r = blockIdx.y * 32 + (threadIdx.x & 31);
    const int64_t g0 = lv[l0].hoff, g1 = lv[l1 - 1].hoff + (int64_t)N * lv[l1 - 1].n;
    for (int64_t g = g0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); g < g1;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const MapLevel h = lv[map_level(lv, l0, l1, g, true)];
        const int64_t c = g - h.hoff;
        const int v = (int)(c / h.n), i = (int)(c % h.n);
        const int d = (int)((((int64_t)v - h.qmin) % N + N) % N);
        int j = d / h.s;
        const uint32_t* w = wtab + h.woff;
        double acc = 0.0;
        if (r < R)
#pragma unroll 4
            for (int q = d % h.s; q < h.wf; q += h.s) {
                acc = fma((double)__ldg(w + q), Z[(h.off + (int64_t)j * h.n + i) * R + r], acc);
                if (--j < 0) j = h.n - 1;
            }
        if (r < R) G[g * R + r] = acc * h.inv_tot;
    }
}

// adjoint along u, summed over levels [l0, l1): U[v N + u][r] (+)= sum_l sum_k w_{p0 + k s} G_l[v][i0 - k mod n][r]
__global__ void __launch_bounds__(256) u_h_kernel(int N, const MapLevel* __restrict__ lv, int l0, int l1,
                                                  const uint32_t* __restrict__ wtab, const double* __restrict__ G,
                                                  int R, int accumulate, double* __restrict__ U) {
    const int r = blockIdx.y * 32 + (threadIdx.x & 31);
    const int64_t nt = (int64_t)N * N;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nt;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        if (r >= R) continue;
        const int v = (int)(t / N), u = (int)(t % N);
        double acc = accumulate ? U[t * R + r] : 0.0;
        for (int l = l0; l < l1; ++l) {
            const MapLevel h = lv[l];
            const int d = (int)((((int64_t)u - h.qmin) % N + N) % N);
            int i = d / h.s;
            const uint32_t* w = wtab + h.woff;
            const double* Gv = G + (h.hoff + (int64_t)v * h.n) * R + r;
#pragma unroll 4
            for (int p = d % h.s; p < h.wf; p += h.s) {
                acc = fma((double)__ldg(w + p), Gv[(int64_t)i * R], acc);
                if (--i < 0) i = h.n - 1;
            }
        }
        U[t * R + r] = acc;
    }
}

// mode X (key = bx, other = Y[by]) or Y (key = by, other = X[bx]): per-CTA partial sums over its texels,
// part[blockIdx.x][key][r] (smem fp64 atomics; the partials are then summed in a fixed order)
__global__ void __launch_bounds__(256) mxy_kernel(const uint16_t* __restrict__ bins, int N, int A, int ash, int mode,
                                                  const double* __restrict__ O, const double* __restrict__ U, int R,
                                                  double* __restrict__ part) {
    extern __shared__ double sacc[];  // [A][32] accumulators, then [A][32] other factor
    double* so = sacc + A * 32;
    const int c0 = blockIdx.y * 32, lane = threadIdx.x & 31, r = c0 + lane;
    for (int e = threadIdx.x; e < A * 32; e += blockDim.x) {
        sacc[e] = 0.0;
        const int rr = c0 + (e & 31);
        so[e] = rr < R ? O[(e >> 5) * R + rr] : 0.0;
    }
    __syncthreads();
    const int64_t nt = (int64_t)N * N;
    if (r < R)
        for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nt;
             t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
            const int b = __ldg(bins + t);
            const int x = b & (A - 1), y = b >> ash;
            const int key = mode == 1 ? x : y, oth = mode == 1 ? y : x;
            atomicAdd(&sacc[key * 32 + lane], so[oth * 32 + lane] * U[t * R + r]);
        }
    __syncthreads();
    for (int e = threadIdx.x; e < A * 32; e += blockDim.x) {
        const int rr = c0 + (e & 31);
        if (rr < R) part[((int64_t)blockIdx.x * A + (e >> 5)) * R + rr] = sacc[e];
    }
}

// ||D||^2 = sum_z sum_b (cnt_b / tot)^2 without forming D: exact uint64 bin counts of each footprint in
// shared memory, read back (and cleared) by a second walk of the same window -- so a row costs O(window),
// not O(A^2); bins with y in [y0, y0 + AS) per slab when A^2 counts exceed shared memory.
__global__ void __launch_bounds__(256) sumsq_rows_kernel(const uint16_t* __restrict__ bins, int N, int A, int ash,
                                                         int AS, const MapLevel* __restrict__ lv, int L,
                                                         const uint32_t* __restrict__ wtab, int64_t z0, int64_t P,
                                                         double* __restrict__ part) {
    extern __shared__ unsigned long long cnt[];  // [AS][A]
    for (int e = threadIdx.x; e < AS * A; e += blockDim.x) cnt[e] = 0ull;
    __syncthreads();
    double acc = 0.0;
    for (int64_t z = z0 + blockIdx.x; z < P; z += gridDim.x) {
        const MapLevel h = lv[map_level(lv, 0, L, z, false)];
        const int64_t c = z - h.off;
        const int i = (int)(c % h.n), j = (int)(c / h.n);
        const int bu = (int)((((int64_t)i * h.s + h.qmin) % N + N) % N);
        const int bv = (int)((((int64_t)j * h.s + h.qmin) % N + N) % N);
        const uint32_t* w = wtab + h.woff;
        const int nwin = h.wf * h.wf;
        double rs = 0.0;
        for (int y0 = 0; y0 < A; y0 += AS) {
            for (int pass = 0; pass < 2; ++pass) {
                for (int t = threadIdx.x; t < nwin; t += blockDim.x) {
                    const int q = t / h.wf, p = t - q * h.wf;
                    int v = bv + q, u = bu + p;
                    if (v >= N) v -= N;
                    if (u >= N) u -= N;
                    const int b = bins[(int64_t)v * N + u];
                    const int y = (b >> ash) - y0;
                    if (y < 0 || y >= AS) continue;
                    unsigned long long* cp = &cnt[y * A + (b & (A - 1))];
                    if (pass == 0) {
                        atomicAdd(cp, (unsigned long long)__ldg(w + q) * (unsigned long long)__ldg(w + p));
                    } else {
                        const unsigned long long k = atomicExch(cp, 0ull);
                        if (k) rs = fma((double)k, (double)k, rs);
                    }
                }
                __syncthreads();
            }
        }
        acc = fma(rs, h.inv_tot * h.inv_tot, acc);
    }
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// ||D||^2 over the rows [0, z1) of the small-window levels (wf^2 <= 64): one warp per row, the window's
// (bin, weight) pairs merged in a 128-slot open-addressing table in the warp's shared memory (exact uint64
// counts), whose squares are summed and cleared -- no CTA barrier per row.
__global__ void __launch_bounds__(256) sumsq_small_kernel(const uint16_t* __restrict__ bins, int N,
                                                          const MapLevel* __restrict__ lv, int L,
                                                          const uint32_t* __restrict__ wtab, int64_t z1,
                                                          double* __restrict__ part) {
    constexpr int TS = 128;
    __shared__ int skey[8][TS];
    __shared__ unsigned long long scnt[8][TS];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* key = skey[wib];
    unsigned long long* cnt = scnt[wib];
    for (int e = lane; e < TS; e += 32) {
        key[e] = -1;
        cnt[e] = 0ull;
    }
    __syncwarp();
    double acc = 0.0;
    for (int64_t z = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; z < z1;
         z += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const MapLevel h = lv[map_level(lv, 0, L, z, false)];
        const int64_t c = z - h.off;
        const int i = (int)(c % h.n), j = (int)(c / h.n);
        const int bu = (int)((((int64_t)i * h.s + h.qmin) % N + N) % N);
        const int bv = (int)((((int64_t)j * h.s + h.qmin) % N + N) % N);
        const uint32_t* w = wtab + h.woff;
        for (int t = lane; t < h.wf * h.wf; t += 32) {
            const int q = t / h.wf, p = t - q * h.wf;
            int v = bv + q, u = bu + p;
            if (v >= N) v -= N;
            if (u >= N) u -= N;
            const int b = bins[(int64_t)v * N + u];
            const unsigned long long wt = (unsigned long long)__ldg(w + q) * (unsigned long long)__ldg(w + p);
            int k = (int)(((uint32_t)b * 2654435761u) >> 25);
            while (true) {
                const int old = atomicCAS(&key[k], -1, b);
                if (old == -1 || old == b) {
                    atomicAdd(&cnt[k], wt);
                    break;
                }
                k = (k + 1) & (TS - 1);
            }
        }
        __syncwarp();
        double rs = 0.0;
        for (int e = lane; e < TS; e += 32) {
            if (key[e] != -1) {
                const double k = (double)cnt[e];
                rs = fma(k, k, rs);
                key[e] = -1;
                cnt[e] = 0ull;
            }
        }
        __syncwarp();
        acc = fma(rs, h.inv_tot * h.inv_tot, acc);
    }
    __shared__ double red[256];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// HALS column pass for R > 128 (G = G1 * G2 too large for shared memory: read from global / L2)
template <int KR>
__global__ void __launch_bounds__(256) hals_global_kernel(double* __restrict__ F, int64_t rows, int R,
                                                          const double* __restrict__ Md,
                                                          const double* __restrict__ G1,
                                                          const double* __restrict__ G2) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t z = w0; z < rows; z += nw) {
        double f[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int s = lane + 32 * k;
            f[k] = s < R ? F[z * R + s] : 0.0;
        }
        for (int r = 0; r < R; ++r) {
            double dot = 0.0;
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int s = lane + 32 * k;
                if (s < R) dot = fma(f[k], __ldg(G1 + s * R + r) * __ldg(G2 + s * R + r), dot);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            const double grr = G1[r * R + r] * G2[r * R + r];
            if (grr > 0.0 && lane == (r & 31)) {
                const double m = Md[z * R + r];
#pragma unroll
                for (int k = 0; k < KR; ++k)
                    if (k == (r >> 5)) f[k] = fmax(kEps, f[k] + (m - dot) / grr);
            }
        }
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int s = lane + 32 * k;
            if (s < R) F[z * R + s] = f[k];
        }
    }
}

}  // namespace als
}  // namespace pndf

// ======================================================================================= host ==
using namespace pndf::als;

namespace {

struct Fail {
    pndf_status st;
};

#define ACK(call)                                                                      \
    do {                                                                               \
        cudaError_t _e = (call);                                                       \
        if (_e != cudaSuccess) {                                                       \
            char _m[256];                                                              \
            snprintf(_m, sizeof(_m), "%s: %s", #call, cudaGetErrorString(_e));         \
            pndf::set_last_error(_m);                                                  \
            throw Fail{_e == cudaErrorMemoryAllocation ? PNDF_ENOMEM : PNDF_ECUDA};    \
        }                                                                              \
    } while (0)

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D fp32 tensor map [rows][cols], box BK x box_rows, 128-byte swizzle (the UMMA K-major SW128 layout)
CUtensorMap make_map(const float* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    CUtensorMap m;
    auto fn = encode_fn();
    if (!fn) {
        pndf::set_last_error("cuTensorMapEncodeTiled unavailable");
        throw Fail{PNDF_ECUDA};
    }
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char m[64];
        snprintf(m, sizeof(m), "cuTensorMapEncodeTiled failed (%d)", (int)r);
        pndf::set_last_error(m);
        throw Fail{PNDF_ECUDA};
    }
    return m;
}

// 3-D view [kblock][rows][32] of a row-major [rows][K] fp32 operand (K = 32 * kblocks): box {32, box_rows,
// kblocks} lands as kblocks stacked 128-byte-swizzled [box_rows][32] tiles, i.e. the UMMA K-major layout
CUtensorMap make_map3(const float* base, uint64_t rows, uint64_t K, uint32_t box_rows) {
    CUtensorMap m;
    auto fn = encode_fn();
    if (!fn) {
        pndf::set_last_error("cuTensorMapEncodeTiled unavailable");
        throw Fail{PNDF_ECUDA};
    }
    const uint32_t kb = (uint32_t)(K / BK);
    cuuint64_t dims[3] = {(cuuint64_t)BK, rows, kb};
    cuuint64_t strides[2] = {K * sizeof(float), BK * sizeof(float)};
    cuuint32_t box[3] = {(cuuint32_t)BK, box_rows, kb};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        char msg[64];
        snprintf(msg, sizeof(msg), "cuTensorMapEncodeTiled (3-D) failed (%d)", (int)r);
        pndf::set_last_error(msg);
        throw Fail{PNDF_ECUDA};
    }
    return m;
}

int ilog2i(int64_t x) {
    int l = 0;
    while ((int64_t(1) << (l + 1)) <= x) ++l;
    return l;
}

struct Geometry {
    int N, s0, L, A, R, RP, a_shift;
    int64_t P;
    std::vector<int64_t> off;
};

pndf_status check_desc(const pndf_desc* d, Geometry& g) {
    if (!d || d->abi_version != PNDF_ABI_VERSION) return PNDF_EINVAL;
    const int N = d->map_size, s0 = d->base_stride, L = d->num_levels, A = d->ang_res, R = d->rank;
    auto pow2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
    if (!pow2(N) || !pow2(s0) || s0 > N || L < 2 || L > 24 || (N / s0) < (1 << (L - 1))) return PNDF_EINVAL;
    if (!pow2(A) || A < 32 || A > 128 || R < 1 || R > 128 || N > 32768) return PNDF_EINVAL;
    g.N = N;
    g.s0 = s0;
    g.L = L;
    g.A = A;
    g.R = R;
    g.RP = R <= 16 ? 16 : R <= 32 ? 32 : R <= 64 ? 64 : 128;
    g.a_shift = ilog2i(A);
    g.P = 0;
    g.off.clear();
    for (int l = 0; l < L; ++l) {
        g.off.push_back(g.P);
        const int64_t n = N / ((int64_t)s0 << l);
        g.P += n * n;
    }
    if (g.P * A >= (int64_t(1) << 31)) return PNDF_EINVAL;
    return PNDF_OK;
}

int num_sms() {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

// device scratch of one builder call (freed on every exit path)
// stream-ordered allocations from the device's default memory pool: reused across builder calls, so a
// call's setup costs no cudaMalloc round trips; freed in stream order when the call's work is done
struct Buffers {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Buffers(cudaStream_t s) : st(s) { keep_pool(); }
    // keep freed blocks cached in the device's default pool (the default release threshold of 0 hands
    // them back to the driver at every synchronisation, so each call would re-map ~10^8 bytes)
    static void keep_pool() {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
    }
    template <class T>
    T* alloc(size_t n) {
        void* p = nullptr;
        ACK(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), st));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~Buffers() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

template <int RP, int EPI>
void launch_gemm_rp(const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, GemmArgs g, int grid,
                    cudaStream_t st) {
    using LY = GemmLayout<RP>;
    // short K (modes X / Y, a3d map): B resident, all K-blocks of a tile in one stage (one 3-D TMA box)
    g.bres = g.kbs > 1 ? 1 : 0;
    g.stages = g.bres ? LY::bres_stages(g.kblocks, g.kbs) : LY::stages();
    const size_t sm = g.bres ? LY::bres_smem(g.kblocks, g.kbs, g.stages) : LY::smem(g.stages);
    ACK(cudaFuncSetAttribute(mttkrp_gemm_kernel<RP, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    mttkrp_gemm_kernel<RP, EPI><<<grid, 192, sm, st>>>(a, bh, bl, g);
    ACK(cudaGetLastError());
}

template <int EPI>
void launch_gemm(int RP, const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, const GemmArgs& g,
                 int grid, cudaStream_t st) {
    switch (RP) {
        case 16: return launch_gemm_rp<16, EPI>(a, bh, bl, g, grid, st);
        case 32: return launch_gemm_rp<32, EPI>(a, bh, bl, g, grid, st);
        case 64: return launch_gemm_rp<64, EPI>(a, bh, bl, g, grid, st);
        default: return launch_gemm_rp<128, EPI>(a, bh, bl, g, grid, st);
    }
}

// The builder's device state: fp64 master factors, fp32 Z for the GEMM epilogue, operands, maps.
struct Builder {
    Geometry g;
    cudaStream_t st;
    int sms;
    Buffers buf{nullptr};  // stream set in the constructor
    double *Z, *X, *Y;          // masters [rows][R]
    float* Zf;                  // [P][RP]
    float *kr_hi, *kr_lo;       // [RP][A^2]
    float *t_hi, *t_lo;         // [RP][A]
    float* Mz;                  // [P][RP]
    double *Mx, *My;            // [A][R]
    float* part;                // [grid][BM][RP]
    double *GZ, *GX, *GY;       // [R][R]
    double* gpart;              // Gram partials
    double* sc;                 // [3][R]
    double* terms;              // [2]
    uint32_t* bad;
    int ggrid;                  // Gram partial blocks
    CUtensorMap mD_z, mD_x, mDt_y, mKr_h, mKr_l, mT_h, mT_l;
    int kbs_xy = 1;  // K-blocks per stage of the mode X / Y GEMMs

    Builder(const Geometry& geo, cudaStream_t s, const float* D, const float* Dt) : g(geo), st(s) {
        buf.st = s;
        sms = num_sms();
        const int A = g.A, R = g.R, RP = g.RP;
        const int64_t P = g.P;
        Z = buf.alloc<double>(P * R);
        X = buf.alloc<double>((size_t)A * R);
        Y = buf.alloc<double>((size_t)A * R);
        Mx = buf.alloc<double>((size_t)A * R);
        My = buf.alloc<double>((size_t)A * R);
        GZ = buf.alloc<double>((size_t)R * R);
        GX = buf.alloc<double>((size_t)R * R);
        GY = buf.alloc<double>((size_t)R * R);
        ggrid = (int)std::min<int64_t>(4 * sms, std::max<int64_t>(1, P / 64));
        gpart = buf.alloc<double>((size_t)(4 * sms + 1) * R * R + 1024);  // Gram / HALS / sum-of-squares partials
        sc = buf.alloc<double>((size_t)3 * R);
        terms = buf.alloc<double>(2);
        bad = buf.alloc<uint32_t>(1);
        if (!D) {  // map-domain builder (pndf_cp_als_map): no tensor, no GEMM operands
            Zf = nullptr;
            Mz = nullptr;
            return;
        }
        Zf = buf.alloc<float>(P * RP);
        kr_hi = buf.alloc<float>((size_t)RP * A * A);
        kr_lo = buf.alloc<float>((size_t)RP * A * A);
        t_hi = buf.alloc<float>((size_t)RP * A);
        t_lo = buf.alloc<float>((size_t)RP * A);
        Mz = buf.alloc<float>(P * RP);
        part = buf.alloc<float>((size_t)sms * BM * RP);
        mD_z = make_map(D, (uint64_t)P, (uint64_t)A * A, BM);
        const int64_t bres_b = (int64_t)(A / BK) * 2 * RP * BK * sizeof(float);  // resident B (hi + lo)
        kbs_xy = (A / BK > 1 && bres_b <= 64 * 1024) ? A / BK : 1;
        mD_x = kbs_xy > 1 ? make_map3(D, (uint64_t)P * A, (uint64_t)A, BM) : make_map(D, (uint64_t)P * A, (uint64_t)A, BM);
        if (Dt)
            mDt_y = kbs_xy > 1 ? make_map3(Dt, (uint64_t)P * A, (uint64_t)A, BM)
                               : make_map(Dt, (uint64_t)P * A, (uint64_t)A, BM);
        mKr_h = make_map(kr_hi, RP, (uint64_t)A * A, RP);
        mKr_l = make_map(kr_lo, RP, (uint64_t)A * A, RP);
        mT_h = make_map(t_hi, RP, A, RP);
        mT_l = make_map(t_lo, RP, A, RP);
    }

    int blocks(int64_t n, int per = 256) const {
        return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 8 * sms));
    }

    void load(const float* in, int64_t rows, double* F, float* Ff) {
        load_factor_kernel<<<blocks(rows * g.RP), 256, 0, st>>>(in, rows, g.R, g.RP, F, Ff, bad);
        ACK(cudaGetLastError());
    }

    void gram(const double* F, int64_t rows, double* G) {
        const int R = g.R;
        const int nb = rows >= 4096 ? ggrid : 1;
        gram_part_kernel<<<nb, 256, 0, st>>>(F, rows, R, gpart);
        sum_parts_kernel<<<R * R, 128, 0, st>>>(gpart, nb, R * R, G);
        ACK(cudaGetLastError());
    }

    void mttkrp_z() {
        const int A = g.A;
        kr_operand_kernel<<<blocks((int64_t)g.RP * A * A), 256, 0, st>>>(X, Y, A, g.R, g.RP, kr_hi, kr_lo);
        ACK(cudaGetLastError());
        GemmArgs a{};
        a.rows = g.P;
        a.ntiles = (g.P + BM - 1) / BM;
        a.kblocks = A * A / BK;
        a.kbs = 1;
        a.out = Mz;
        launch_gemm<0>(g.RP, mD_z, mKr_h, mKr_l, a, (int)std::min<int64_t>(a.ntiles, sms), st);
    }

    // mode 1: M_X from D with Y; mode 2: M_Y from Dt with X
    void mttkrp_xy(int mode, double* M) {
        const int A = g.A;
        t_operand_kernel<<<blocks((int64_t)g.RP * A), 256, 0, st>>>(mode == 1 ? Y : X, A, g.R, g.RP, t_hi, t_lo);
        ACK(cudaGetLastError());
        GemmArgs a{};
        a.rows = g.P * A;
        a.ntiles = (a.rows + BM - 1) / BM;
        a.kblocks = A / BK;
        a.kbs = kbs_xy;
        a.a_shift = g.a_shift;
        a.Zf = Zf;
        a.part = part;
        const int grid = (int)std::min<int64_t>(a.ntiles, sms);
        launch_gemm<1>(g.RP, mode == 1 ? mD_x : mDt_y, mT_h, mT_l, a, grid, st);
        part_reduce_kernel<<<A * g.R, 128, 0, st>>>(part, grid, A, g.R, g.RP, M);
        ACK(cudaGetLastError());
    }

    template <int RT, int TPB>
    void hals_rows(double* F, int64_t rows, const float* Mf, const double* Md, const double* G1, const double* G2,
                   float* Ff, double* Gout) {
        const size_t sm = (size_t)TPB * (RT + 1) * sizeof(double);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + TPB - 1) / TPB, 4 * sms));
        ACK(cudaFuncSetAttribute(hals_rows_kernel<RT, TPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        hals_rows_kernel<RT, TPB><<<grid, TPB, sm, st>>>(F, rows, g.R, g.RP, Mf, Md, G1, G2, Ff, gpart);
        ACK(cudaGetLastError());
        sum_parts_kernel<<<g.R * g.R, 128, 0, st>>>(gpart, grid, g.R * g.R, Gout);
        ACK(cudaGetLastError());
    }

    // HALS pass over F's columns with G = G1 * G2, then Gout = F^T F of the updated factor
    void hals(double* F, int64_t rows, const float* Mf, const double* Md, const double* G1, const double* G2,
              float* Ff, double* Gout) {
        const int R = g.R;
        if (R <= 8) return hals_rows<8, 256>(F, rows, Mf, Md, G1, G2, Ff, Gout);
        if (R <= 16) return hals_rows<16, 256>(F, rows, Mf, Md, G1, G2, Ff, Gout);
        if (R <= 32) return hals_rows<32, 256>(F, rows, Mf, Md, G1, G2, Ff, Gout);
        if (R <= 64) return hals_rows<64, 128>(F, rows, Mf, Md, G1, G2, Ff, Gout);
        const int KR = (R + 31) / 32;
        const size_t sm = (size_t)R * R * sizeof(double);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, 16 * sms));
        if (KR <= 4) {
            ACK(cudaFuncSetAttribute(hals_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            hals_kernel<4><<<grid, 256, sm, st>>>(F, rows, R, g.RP, Mf, Md, G1, G2, Ff);
        } else {  // R <= 256 (map-domain builder only: Md in fp64, no fp32 copy)
            hals_global_kernel<8><<<grid, 256, 0, st>>>(F, rows, R, Md, G1, G2);
        }
        ACK(cudaGetLastError());
        gram(F, rows, Gout);
    }
};


// Geometry of the map-domain builder: as check_desc, plus A <= 256, R <= 256 and no P * A limit (no GEMM)
pndf_status check_desc_map(const pndf_desc* d, Geometry& g) {
    if (!d || d->abi_version != PNDF_ABI_VERSION) return PNDF_EINVAL;
    const int N = d->map_size, s0 = d->base_stride, L = d->num_levels, A = d->ang_res, R = d->rank;
    auto pow2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
    if (!pow2(N) || !pow2(s0) || s0 > N || L < 2 || L > 24 || (N / s0) < (1 << (L - 1))) return PNDF_EINVAL;
    if (!pow2(A) || A < 2 || A > 256 || R < 1 || R > 256 || N > 32768 || !(d->flags & PNDF_WRAP)) return PNDF_EINVAL;
    g.N = N;
    g.s0 = s0;
    g.L = L;
    g.A = A;
    g.R = R;
    g.RP = (R + 31) / 32 * 32;
    g.a_shift = ilog2i(A);
    g.P = 0;
    g.off.clear();
    for (int l = 0; l < L; ++l) {
        g.off.push_back(g.P);
        const int64_t n = N / ((int64_t)s0 << l);
        g.P += n * n;
    }
    return PNDF_OK;
}

// integer footprint weights of every level (reading 11; oracle/als.py footprint_weights): w is
// the concatenated table, lv[l] = {qmin, wf, woff, tot = (sum w)^2} of level l
void level_weights(const Geometry& g, std::vector<uint32_t>& w, std::vector<int64_t>& qmin, std::vector<int>& wf,
                   std::vector<int>& woff, std::vector<double>& tot) {
    for (int l = 0; l < g.L; ++l) {
        const int sl = g.s0 << l;
        const double sigma = 1.5 * sl / sqrt(12.0), c = 0.5 * (1.0 - sl);
        const int64_t q0 = (int64_t)ceil(-4.0 * sigma - c), q1 = (int64_t)floor(4.0 * sigma - c);
        const int f = (int)std::min<int64_t>(q1 - q0 + 1, g.N);
        const size_t w0 = w.size();
        w.resize(w0 + f, 0u);
        for (int64_t q = q0; q <= q1; ++q) {
            const double d = (double)q + c;
            w[w0 + (size_t)((q - q0) % f)] += (uint32_t)llround(65536.0 * exp(-d * d / (2.0 * sigma * sigma)));
        }
        uint64_t sw = 0;
        for (int p = 0; p < f; ++p) sw += w[w0 + p];
        qmin.push_back(q0);
        wf.push_back(f);
        woff.push_back((int)w0);
        tot.push_back((double)sw * (double)sw);
    }
}

// Map-domain MTTKRPs (pndf_cp_als_map / pndf_mttkrp_map): level tables on the device, the pass buffer
// (level 0's [N][n0] rows, or levels >= 1 stacked), U [N^2][R] and the mode-X/Y partials.
struct MapOps {
    const Geometry& g;
    cudaStream_t st;
    int sms;
    const uint16_t* bins;
    MapLevel* d_lv = nullptr;
    uint32_t* d_w = nullptr;
    double *HG = nullptr, *U = nullptr, *part = nullptr;
    int pgrid = 0;
    std::vector<MapLevel> lv;

    MapOps(const Geometry& geo, cudaStream_t s, int nsm, Buffers& buf, const uint16_t* b)
        : g(geo), st(s), sms(nsm), bins(b) {
        std::vector<uint32_t> w;
        std::vector<int64_t> qmin;
        std::vector<int> wf, woff;
        std::vector<double> tot;
        level_weights(g, w, qmin, wf, woff, tot);
        lv.resize(g.L);
        int64_t hb = 0;  // group A = level 0 at pass row 0; group B = levels >= 1 stacked from row 0
        for (int l = 0; l < g.L; ++l) {
            const int sl = g.s0 << l;
            if (l == 1) hb = 0;
            lv[l] = MapLevel{g.off[l], hb, sl, g.N / sl, (int)qmin[l], wf[l], woff[l], 1.0 / tot[l]};
            hb += (int64_t)g.N * (g.N / sl);
        }
        const int64_t n0 = g.N / g.s0;
        const int64_t rows = std::max<int64_t>((int64_t)g.N * n0, hb);
        d_lv = buf.alloc<MapLevel>(lv.size());
        d_w = buf.alloc<uint32_t>(w.size());
        ACK(cudaMemcpyAsync(d_lv, lv.data(), lv.size() * sizeof(MapLevel), cudaMemcpyHostToDevice, st));
        ACK(cudaMemcpyAsync(d_w, w.data(), w.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        HG = buf.alloc<double>((size_t)rows * g.R);
        U = buf.alloc<double>((size_t)g.N * g.N * g.R);
        pgrid = 2 * sms;
        part = buf.alloc<double>((size_t)pgrid * g.A * g.R);
    }
    dim3 grid(int64_t warps) const {
        return dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 16 * sms)), (g.R + 31) / 32);
    }
    // M [P][R] = D_(z) (X kr Y), fp64
    void mz(const double* X, const double* Y, double* M) {
        const size_t sm = (size_t)2 * g.A * 32 * sizeof(double);
        ACK(cudaFuncSetAttribute(mz_h_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        for (int grp = 0; grp < 2; ++grp) {
            const int l0 = grp ? 1 : 0, l1 = grp ? g.L : 1;
            int64_t hrows = 0, zrows = 0;
            for (int l = l0; l < l1; ++l) {
                hrows += (int64_t)g.N * lv[l].n;
                zrows += (int64_t)lv[l].n * lv[l].n;
            }
            mz_h_kernel<<<grid(hrows), 256, sm, st>>>(bins, g.N, g.A, g.a_shift, d_lv, l0, l1, d_w, X, Y, g.R, HG);
            mz_v_kernel<<<grid(zrows), 256, 0, st>>>(g.N, d_lv, l0, l1, d_w, HG, g.R, M);
            ACK(cudaGetLastError());
        }
    }
    // U [N^2][R] = the adjoint blur of Z
    void u(const double* Z) {
        for (int grp = 0; grp < 2; ++grp) {
            const int l0 = grp ? 1 : 0, l1 = grp ? g.L : 1;
            int64_t hrows = 0;
            for (int l = l0; l < l1; ++l) hrows += (int64_t)g.N * lv[l].n;
            u_g_kernel<<<grid(hrows), 256, 0, st>>>(g.N, d_lv, l0, l1, d_w, Z, g.R, HG);
            u_h_kernel<<<grid((int64_t)g.N * g.N), 256, 0, st>>>(g.N, d_lv, l0, l1, d_w, HG, g.R, grp, U);
            ACK(cudaGetLastError());
        }
    }
    // mode 1: M [A][R] = D_(x) (Z kr Y) with O = Y; mode 2: D_(y) (Z kr X) with O = X (needs u() first)
    void mxy(int mode, const double* O, double* M, double* sumbuf_unused = nullptr) {
        (void)sumbuf_unused;
        const size_t sm = (size_t)2 * g.A * 32 * sizeof(double);
        ACK(cudaFuncSetAttribute(mxy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        mxy_kernel<<<dim3(pgrid, (g.R + 31) / 32), 256, sm, st>>>(bins, g.N, g.A, g.a_shift, mode, O, U, g.R, part);
        sum_parts_kernel<<<g.A * g.R, 128, 0, st>>>(part, pgrid, g.A * g.R, M);
        ACK(cudaGetLastError());
    }
    // ||D||^2 (fp64), synchronous
    double sumsq(double* scratch /* >= 6 sms + 1 doubles */) {
        const int AS = std::min(g.A, (int)((128 * 1024) / (8 * g.A)));
        const size_t sm = (size_t)AS * g.A * sizeof(unsigned long long);
        ACK(cudaFuncSetAttribute(sumsq_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int64_t zs = 0;  // rows of the levels whose windows have <= 64 texels (a prefix: wf grows with l)
        for (int l = 0; l < g.L && (int64_t)lv[l].wf * lv[l].wf <= 64; ++l) zs = lv[l].off + (int64_t)lv[l].n * lv[l].n;
        const int g1 = (int)std::max<int64_t>(1, std::min<int64_t>((zs + 7) / 8, 4 * sms));
        const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(g.P - zs, 2 * sms));
        sumsq_small_kernel<<<g1, 256, 0, st>>>(bins, g.N, d_lv, g.L, d_w, zs, scratch);
        sumsq_rows_kernel<<<g2, 256, sm, st>>>(bins, g.N, g.A, g.a_shift, AS, d_lv, g.L, d_w, zs, g.P, scratch + g1);
        sum_parts_kernel<<<1, 128, 0, st>>>(scratch, g1 + g2, 1, scratch + g1 + g2);
        ACK(cudaGetLastError());
        double v = 0.0;
        ACK(cudaMemcpyAsync(&v, scratch + g1 + g2, sizeof(double), cudaMemcpyDeviceToHost, st));
        ACK(cudaStreamSynchronize(st));
        return v;
    }
};

}  // namespace

extern "C" pndf_status pndf_hist_tensor(const pndf_desc* desc, const uint16_t* d_bins, float* d_D, float* d_Dt,
                                        void* cuda_stream) {
    Geometry g;
    pndf_status s = check_desc(desc, g);
    if (s != PNDF_OK) return s;
    if (!(desc->flags & PNDF_WRAP) || !d_bins || !d_D) return PNDF_EINVAL;
    try {
        cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
        // integer footprint weights per level (reading 11; oracle/als.py footprint_weights)
        std::vector<HistLevel> lv(g.L);
        std::vector<uint32_t> w;
        for (int l = 0; l < g.L; ++l) {
            const int sl = g.s0 << l;
            const double sigma = 1.5 * sl / sqrt(12.0), c = 0.5 * (1.0 - sl);
            const int64_t qmin = (int64_t)ceil(-4.0 * sigma - c), qmax = (int64_t)floor(4.0 * sigma - c);
            const int64_t W = qmax - qmin + 1;
            const int wf = (int)std::min<int64_t>(W, g.N);
            const size_t w0 = w.size();
            w.resize(w0 + wf, 0u);
            for (int64_t q = qmin; q <= qmax; ++q) {
                const double d = (double)q + c;
                w[w0 + (size_t)((q - qmin) % wf)] += (uint32_t)llround(65536.0 * exp(-d * d / (2.0 * sigma * sigma)));
            }
            uint64_t sw = 0;
            for (int p = 0; p < wf; ++p) sw += w[w0 + p];
            lv[l] = HistLevel{g.off[l], sl, g.N / sl, (int)qmin, wf, (int)w0, (double)sw * (double)sw};
        }
        Buffers buf(st);
        HistLevel* d_lv = buf.alloc<HistLevel>(lv.size());
        uint32_t* d_w = buf.alloc<uint32_t>(w.size());
        ACK(cudaMemcpyAsync(d_lv, lv.data(), lv.size() * sizeof(HistLevel), cudaMemcpyHostToDevice, st));
        ACK(cudaMemcpyAsync(d_w, w.data(), w.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        const size_t sm = (size_t)g.A * (g.A + 1) * sizeof(unsigned long long);
        ACK(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        const int grid = (int)std::min<int64_t>(g.P, 8 * num_sms());
        hist_kernel<<<grid, 256, sm, st>>>(d_bins, g.N, g.A, d_lv, g.L, d_w, g.P, d_D, d_Dt);
        ACK(cudaGetLastError());
        ACK(cudaStreamSynchronize(st));  // the weight tables are freed on return
    } catch (const Fail& f) {
        return f.st;
    }
    return PNDF_OK;
}

extern "C" pndf_status pndf_mttkrp(const pndf_desc* desc, const float* d_D, const float* d_Dt, const float* d_Z,
                                   const float* d_X, const float* d_Y, int32_t mode, double* d_M,
                                   void* cuda_stream) {
    Geometry g;
    pndf_status s = check_desc(desc, g);
    if (s != PNDF_OK) return s;
    if (!d_D || !d_Z || !d_X || !d_Y || !d_M || mode < 0 || mode > 2 || (mode == 2 && !d_Dt)) return PNDF_EINVAL;
    try {
        cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
        Builder b(g, st, d_D, d_Dt);
        ACK(cudaMemsetAsync(b.bad, 0, sizeof(uint32_t), st));
        b.load(d_Z, g.P, b.Z, b.Zf);
        b.load(d_X, g.A, b.X, nullptr);
        b.load(d_Y, g.A, b.Y, nullptr);
        if (mode == 0) {
            b.mttkrp_z();
            rows_to_f64_kernel<<<b.blocks(g.P * g.R), 256, 0, st>>>(b.Mz, g.P, g.R, g.RP, d_M);
            ACK(cudaGetLastError());
        } else {
            b.mttkrp_xy(mode, d_M);
        }
        uint32_t bad = 0;
        ACK(cudaMemcpyAsync(&bad, b.bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
        ACK(cudaStreamSynchronize(st));
        if (bad) return PNDF_EINVAL;
    } catch (const Fail& f) {
        return f.st;
    }
    return PNDF_OK;
}

// The sweep loop shared by the tensor (GEMM) and map-domain builders: modes Z, X, Y with HALS updates, fit
// error, norm balance (oracle/als.py hals_sweep), stopping rule (reading 15), then normalise (reading 16).
// mz() fills the Z-mode MTTKRP (fp32 Mf or fp64 Md), prep_xy() runs after the Z update, mxy(mode, M) the
// X / Y modes.
template <class MZ, class PREP, class MXY>
void als_loop(Builder& b, double nD2, const pndf_als_opts* o, double* h_err, int32_t* sweeps_out, float* d_C,
              float* d_X, float* d_Y, float* d_Z, const float* Mf, const double* Md, MZ mz, PREP prep_xy, MXY mxy) {
    const Geometry& g = b.g;
    cudaStream_t st = b.st;
    const int R = g.R, A = g.A;
    const int64_t P = g.P;
    double prev = -1.0, terms[2];
    int sweeps = 0;
    b.gram(b.X, A, b.GX);
    b.gram(b.Y, A, b.GY);
    for (int it = 0; it < o->max_sweeps; ++it) {
        // Z: M_Z with (X, Y), G = (X'X) * (Y'Y); the pass also yields Z'Z
        mz();
        b.hals(b.Z, P, Mf, Md, b.GX, b.GY, b.Zf, b.GZ);
        prep_xy();
        // X: M_X with (Z, Y), G = (Z'Z) * (Y'Y)
        mxy(1, b.Mx);
        b.hals(b.X, A, nullptr, b.Mx, b.GZ, b.GY, nullptr, b.GX);
        // Y: M_Y with (Z, X), G = (Z'Z) * (X'X)
        mxy(2, b.My);
        b.hals(b.Y, A, nullptr, b.My, b.GZ, b.GX, nullptr, b.GY);
        err_terms_kernel<<<1, 256, 0, st>>>(b.My, b.Y, A, R, b.GZ, b.GX, b.GY, b.terms);
        // norm balance; the next sweep's X'X and Y'Y follow by scaling
        balance_scale_kernel<<<(R + 127) / 128, 128, 0, st>>>(b.GZ, b.GX, b.GY, R, b.sc);
        scale_cols_kernel<<<b.blocks(P * R), 256, 0, st>>>(b.Z, P, R, b.sc, 0, b.Zf, g.RP);
        scale_cols_kernel<<<1, 256, 0, st>>>(b.X, A, R, b.sc + R, 0, nullptr, g.RP);
        scale_cols_kernel<<<1, 256, 0, st>>>(b.Y, A, R, b.sc + 2 * R, 0, nullptr, g.RP);
        scale_gram_kernel<<<(R * R + 255) / 256, 256, 0, st>>>(b.GX, R, b.sc + R);
        scale_gram_kernel<<<(R * R + 255) / 256, 256, 0, st>>>(b.GY, R, b.sc + 2 * R);
        ACK(cudaGetLastError());
        ACK(cudaMemcpyAsync(terms, b.terms, sizeof(terms), cudaMemcpyDeviceToHost, st));
        ACK(cudaStreamSynchronize(st));
        const double err = sqrt(std::max(0.0, nD2 - 2.0 * terms[0] + terms[1]) / nD2);
        if (h_err) h_err[it] = err;
        sweeps = it + 1;
        if (prev >= 0.0 && fabs(prev - err) < o->tol * std::max(prev, 1e-300)) break;
        prev = err;
    }
    if (sweeps_out) *sweeps_out = sweeps;

    if (o->flags & PNDF_ALS_NORMALISE) {
        const int nb = (int)std::min<int64_t>(b.ggrid, std::max<int64_t>(1, P / 64));
        double* sx = b.sc;           // [R]
        double* sy = b.sc + R;       // [R]
        double* sxy = b.sc + 2 * R;  // [R]
        const int rb = (R + 127) / 128;
        col_reduce_kernel<<<1, 128, 0, st>>>(b.X, A, R, 0, b.gpart);
        col_finish_kernel<<<rb, 128, 0, st>>>(b.gpart, 1, R, 0, sx);
        col_reduce_kernel<<<1, 128, 0, st>>>(b.Y, A, R, 0, b.gpart);
        col_finish_kernel<<<rb, 128, 0, st>>>(b.gpart, 1, R, 0, sy);
        mul2_kernel<<<rb, 128, 0, st>>>(sx, sy, R, sxy);
        scale_cols_kernel<<<1, 256, 0, st>>>(b.X, A, R, sx, 1, nullptr, g.RP);
        scale_cols_kernel<<<1, 256, 0, st>>>(b.Y, A, R, sy, 1, nullptr, g.RP);
        scale_cols_kernel<<<b.blocks(P * R), 256, 0, st>>>(b.Z, P, R, sxy, 0, nullptr, g.RP);
        // C_r = max_z Z_r, Z /= C (GX's storage holds C: R doubles)
        double* C = b.GX;
        col_reduce_kernel<<<nb, 128, 0, st>>>(b.Z, P, R, 1, b.gpart);
        col_finish_kernel<<<rb, 128, 0, st>>>(b.gpart, nb, R, 1, C);
        scale_cols_kernel<<<b.blocks(P * R), 256, 0, st>>>(b.Z, P, R, C, 1, nullptr, g.RP);
        row_renorm_kernel<<<(int)((P + 255) / 256), 256, 0, st>>>(b.Z, P, R, C);
        if (d_C) to_f32_kernel<<<1, 128, 0, st>>>(C, R, d_C);
        ACK(cudaGetLastError());
    } else if (d_C) {
        fill_kernel<<<(R + 127) / 128, 128, 0, st>>>(d_C, R, 1.f);
    }
    to_f32_kernel<<<b.blocks(P * R), 256, 0, st>>>(b.Z, P * R, d_Z);
    to_f32_kernel<<<1, 256, 0, st>>>(b.X, (int64_t)A * R, d_X);
    to_f32_kernel<<<1, 256, 0, st>>>(b.Y, (int64_t)A * R, d_Y);
    ACK(cudaGetLastError());
    ACK(cudaStreamSynchronize(st));
}

extern "C" pndf_status pndf_cp_als(const pndf_desc* desc, const float* d_D, const float* d_Dt, float* d_C,
                                   float* d_X, float* d_Y, float* d_Z, const pndf_als_opts* o, double* h_err,
                                   int32_t* sweeps_out, void* cuda_stream) {
    Geometry g;
    pndf_status s = check_desc(desc, g);
    if (s != PNDF_OK) return s;
    if (!d_D || !d_Dt || !d_X || !d_Y || !d_Z || !o || o->abi_version != PNDF_ABI_VERSION || o->max_sweeps < 1 ||
        !(o->tol >= 0.0))
        return PNDF_EINVAL;
    try {
        cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
        Builder b(g, st, d_D, d_Dt);
        const int A = g.A;
        const int64_t P = g.P;
        ACK(cudaMemsetAsync(b.bad, 0, sizeof(uint32_t), st));
        b.load(d_Z, P, b.Z, b.Zf);
        b.load(d_X, A, b.X, nullptr);
        b.load(d_Y, A, b.Y, nullptr);
        // ||D||^2 (fp64)
        const int64_t nD = P * (int64_t)A * A;
        const int sg = std::min(1024, 4 * b.sms);
        sumsq_part_kernel<<<sg, 256, 0, st>>>(d_D, nD, b.gpart);
        sum_parts_kernel<<<1, 128, 0, st>>>(b.gpart, sg, 1, b.terms);
        ACK(cudaGetLastError());
        double nD2 = 0.0;
        uint32_t bad = 0;
        ACK(cudaMemcpyAsync(&nD2, b.terms, sizeof(double), cudaMemcpyDeviceToHost, st));
        ACK(cudaMemcpyAsync(&bad, b.bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
        ACK(cudaStreamSynchronize(st));
        if (bad || !(nD2 > 0.0)) return PNDF_EINVAL;
        als_loop(b, nD2, o, h_err, sweeps_out, d_C, d_X, d_Y, d_Z, b.Mz, nullptr, [&] { b.mttkrp_z(); }, [] {},
                 [&](int mode, double* M) { b.mttkrp_xy(mode, M); });
    } catch (const Fail& f) {
        return f.st;
    }
    return PNDF_OK;
}

extern "C" pndf_status pndf_cp_als_map(const pndf_desc* desc, const uint16_t* d_bins, float* d_C, float* d_X,
                                       float* d_Y, float* d_Z, const pndf_als_opts* o, double* h_err,
                                       int32_t* sweeps_out, void* cuda_stream) {
    Geometry g;
    pndf_status s = check_desc_map(desc, g);
    if (s != PNDF_OK) return s;
    if (!d_bins || !d_X || !d_Y || !d_Z || !o || o->abi_version != PNDF_ABI_VERSION || o->max_sweeps < 1 ||
        !(o->tol >= 0.0))
        return PNDF_EINVAL;
    try {
        cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
        Builder b(g, st, nullptr, nullptr);
        MapOps m(g, st, b.sms, b.buf, d_bins);
        double* Mz = b.buf.alloc<double>((size_t)g.P * g.R);
        ACK(cudaMemsetAsync(b.bad, 0, sizeof(uint32_t), st));
        b.load(d_Z, g.P, b.Z, nullptr);
        b.load(d_X, g.A, b.X, nullptr);
        b.load(d_Y, g.A, b.Y, nullptr);
        uint32_t bad = 0;
        ACK(cudaMemcpyAsync(&bad, b.bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
        const double nD2 = m.sumsq(b.gpart);  // synchronises
        if (bad || !(nD2 > 0.0)) return PNDF_EINVAL;
        als_loop(b, nD2, o, h_err, sweeps_out, d_C, d_X, d_Y, d_Z, nullptr, Mz, [&] { m.mz(b.X, b.Y, Mz); },
                 [&] { m.u(b.Z); }, [&](int mode, double* M) { m.mxy(mode, mode == 1 ? b.Y : b.X, M); });
    } catch (const Fail& f) {
        return f.st;
    }
    return PNDF_OK;
}

extern "C" pndf_status pndf_mttkrp_map(const pndf_desc* desc, const uint16_t* d_bins, const float* d_Z,
                                       const float* d_X, const float* d_Y, int32_t mode, double* d_M,
                                       double* h_sumsq, void* cuda_stream) {
    Geometry g;
    pndf_status s = check_desc_map(desc, g);
    if (s != PNDF_OK) return s;
    if (!d_bins || !d_Z || !d_X || !d_Y || !d_M || mode < 0 || mode > 2) return PNDF_EINVAL;
    try {
        cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
        Builder b(g, st, nullptr, nullptr);
        MapOps m(g, st, b.sms, b.buf, d_bins);
        ACK(cudaMemsetAsync(b.bad, 0, sizeof(uint32_t), st));
        b.load(d_Z, g.P, b.Z, nullptr);
        b.load(d_X, g.A, b.X, nullptr);
        b.load(d_Y, g.A, b.Y, nullptr);
        if (mode == 0) {
            m.mz(b.X, b.Y, d_M);
        } else {
            m.u(b.Z);
            m.mxy(mode, mode == 1 ? b.Y : b.X, d_M);
        }
        uint32_t bad = 0;
        ACK(cudaMemcpyAsync(&bad, b.bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
        ACK(cudaStreamSynchronize(st));
        if (bad) return PNDF_EINVAL;
        if (h_sumsq) *h_sumsq = m.sumsq(b.gpart);
    } catch (const Fail& f) {
        return f.st;
    }
    return PNDF_OK;
}
