// build.cu -- store build kernels (once per store, untimed).
//
// The 1-D SATs of the angular factors ("a 1D SAT for each 1D vector ...
// gives exact results"): S_k = sum_{i<k} X_r(i) accumulated in fp64 in index
// order, stored in one of two formats (chosen per store):
//   HILO  hi = fl32(S_k), lo = fl32(S_k - hi)     -- 8 B/entry, ~1 ulp for any store
//   U32   q_k = round(S_k 2^e_r), uint32 fixed point with a per-rank power-of-two
//         scale e_r (the largest with q_A < 2^32) -- 4 B/entry; differences are
//         exact integers, so Xbar has error <= 2^-e_r; used only when that is
//         <= 2^-15 of the smallest nonzero factor entry of every rank.
// Zc[z][r] = fl32(M_r * Z_r(z)) with M_r = C_r (HILO) or C_r 2^-(ex_r+ey_r) (U32,
// a power-of-two rescale that is exact unless it underflows -- flagged).
#include <cuda_runtime.h>

#include <algorithm>
#include <float.h>
#include <stdint.h>

#include "launch.h"

namespace pndf {

__device__ __forceinline__ bool bad_factor(float v) { return !(v >= 0.0f) || isinf(v); }

// flags: bit 0 = negative / non-finite factor, bit 1 = a nonzero product underflowed
__global__ void fold_rows_kernel(const float* Zsrc, int64_t rows, int R, const float* __restrict__ M, float* Zc,
                                 int Rp, uint32_t* flags) {
    const int64_t total = rows * (int64_t)Rp;
    bool any_bad = false, any_uflow = false;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = t / Rp;
        const int r = (int)(t - z * Rp);
        float v = 0.0f;
        if (r < R) {
            const float zr = Zsrc[z * R + r];
            any_bad |= bad_factor(zr);
            v = M ? M[r] * zr : zr;
            any_uflow |= (zr != 0.0f && M && M[r] != 0.0f && fabsf(v) < FLT_MIN);
        }
        Zc[t] = v;
    }
    if (__any_sync(0xffffffffu, any_bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
    if (__any_sync(0xffffffffu, any_uflow) && (threadIdx.x & 31) == 0) atomicOr(flags, 2u);
}

// One thread per (table, rank): fp64 total and smallest nonzero entry.
__global__ void prefix_stats_kernel(const float* __restrict__ X, const float* __restrict__ Y, int A, int R, int Rp,
                                    double* total, float* minnz, uint32_t* flags) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * Rp) return;
    const int table = t / Rp, r = t % Rp;
    const float* F = table ? Y : X;
    double S = 0.0;
    float mn = FLT_MAX;
    bool any_bad = false;
    if (r < R)
        for (int k = 0; k < A; ++k) {
            const float v = F[(size_t)k * R + r];
            any_bad |= bad_factor(v);
            S += (double)v;
            if (v > 0.0f && v < mn) mn = v;
        }
    total[t] = S;
    minnz[t] = mn;
    if (any_bad) atomicOr(flags, 1u);
}

// HILO: PXY[table][k][0|1][Rp]
__global__ void prefix_hilo_kernel(const float* __restrict__ X, const float* __restrict__ Y, int A, int R, int Rp,
                                   float* PXY) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * Rp) return;
    const int table = t / Rp, r = t % Rp;
    const float* F = table ? Y : X;
    float* out = PXY + (size_t)table * (A + 1) * 2 * Rp;
    double S = 0.0;
    for (int k = 0; k <= A; ++k) {
        const float hi = (float)S;
        const float lo = (float)(S - (double)hi);
        out[(size_t)(2 * k) * Rp + r] = hi;
        out[(size_t)(2 * k + 1) * Rp + r] = lo;
        if (k < A && r < R) S += (double)F[(size_t)k * R + r];
    }
}

// U32: PQ[table][k][Rp], q_k = round(S_k 2^e)
__global__ void prefix_u32_kernel(const float* __restrict__ X, const float* __restrict__ Y, int A, int R, int Rp,
                                  const int* __restrict__ exps, uint32_t* PQ) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * Rp) return;
    const int table = t / Rp, r = t % Rp;
    const float* F = table ? Y : X;
    uint32_t* out = PQ + (size_t)table * (A + 1) * Rp;
    const int e = exps[t];
    double S = 0.0;
    for (int k = 0; k <= A; ++k) {
        out[(size_t)k * Rp + r] = __double2uint_rn(ldexp(S, e));
        if (k < A && r < R) S += (double)F[(size_t)k * R + r];
    }
}

// DT[axis][x1][w-1][r] = the prefix difference of [x1, x1+w) computed exactly as query_kernel does
// (U32: float of the integer difference; HILO: (hi1 - hi0) + (lo1 - lo0) in fp32), so a table look-up
// returns the same bits as the two SAT look-ups it replaces.  Entries with x1 + w > A are 0.
__global__ void range_table_kernel(const float* __restrict__ PXY, int A, int Rp, int u32, int W,
                                   float* __restrict__ DT) {
    const int64_t n = (int64_t)2 * A * W * Rp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % Rp);
        const int64_t row = e / Rp;
        const int w = (int)(row % W) + 1;
        const int x1 = (int)((row / W) % A);
        const int axis = (int)(row / ((int64_t)W * A));
        float v = 0.f;
        if (x1 + w <= A) {
            if (u32) {
                const uint32_t* Q = reinterpret_cast<const uint32_t*>(PXY) + (size_t)axis * (A + 1) * Rp;
                v = __uint2float_rn(Q[(size_t)(x1 + w) * Rp + r] - Q[(size_t)x1 * Rp + r]);
            } else {
                const float* T = PXY + (size_t)axis * (A + 1) * 2 * Rp;
                const float h1 = T[(size_t)(2 * (x1 + w)) * Rp + r], h0 = T[(size_t)(2 * x1) * Rp + r];
                const float l1 = T[(size_t)(2 * (x1 + w) + 1) * Rp + r], l0 = T[(size_t)(2 * x1 + 1) * Rp + r];
                v = __fadd_rn(__fsub_rn(h1, h0), __fsub_rn(l1, l0));
            }
        }
        DT[e] = v;
    }
}

cudaError_t launch_range_table(const float* PXY, int A, int Rp, int u32, int W, float* DT, cudaStream_t st) {
    const int64_t n = (int64_t)2 * A * W * Rp;
    range_table_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(PXY, A, Rp, u32, W, DT);
    return cudaGetLastError();
}

static int grid_for(int64_t total, int threads, int cap_blocks) {
    int64_t g = (total + threads - 1) / threads;
    if (g > cap_blocks) g = cap_blocks;
    return g < 1 ? 1 : (int)g;
}

cudaError_t launch_fold_rows(const float* Zsrc, int64_t rows, int R, const float* Mdev, float* Zc_dst, int Rp,
                             uint32_t* flags, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    fold_rows_kernel<<<grid_for(rows * (int64_t)Rp, 256, sms * 16), 256, 0, st>>>(Zsrc, rows, R, Mdev, Zc_dst, Rp,
                                                                                  flags);
    return cudaGetLastError();
}

cudaError_t launch_prefix_stats(const float* Xdev, const float* Ydev, int A, int R, int Rp, double* total,
                                float* minnz, uint32_t* flags, cudaStream_t st) {
    prefix_stats_kernel<<<grid_for(2 * Rp, 128, 1 << 20), 128, 0, st>>>(Xdev, Ydev, A, R, Rp, total, minnz, flags);
    return cudaGetLastError();
}

cudaError_t launch_prefix(const float* Xdev, const float* Ydev, int A, int R, int Rp, int u32, const int* exps,
                          void* table, cudaStream_t st) {
    if (u32)
        prefix_u32_kernel<<<grid_for(2 * Rp, 128, 1 << 20), 128, 0, st>>>(Xdev, Ydev, A, R, Rp, exps,
                                                                          (uint32_t*)table);
    else
        prefix_hilo_kernel<<<grid_for(2 * Rp, 128, 1 << 20), 128, 0, st>>>(Xdev, Ydev, A, R, Rp, (float*)table);
    return cudaGetLastError();
}

}  // namespace pndf
