// build.cu -- store build kernels (once per store, untimed).
//
//   fold_rows_kernel  Zc[z][r] = fl32(C_r * Z_r(z)) for r < R, 0 for R <= r < Rp;
//                     flags any negative or non-finite factor (nonnegative store).
//   prefix_kernel     1-D SATs of the angular factors ("a 1D SAT for each
//                     1D vector"): S_k = sum_{i<k} X_r(i) accumulated in fp64 in
//                     index order, stored as hi = fl32(S_k), lo = fl32(S_k - hi).
#include <cuda_runtime.h>
#include <stdint.h>

#include "launch.h"

namespace pndf {

__device__ __forceinline__ bool bad_factor(float v) { return !(v >= 0.0f) || isinf(v); }

__global__ void fold_rows_kernel(const float* Zsrc, int64_t rows, int R, const float* __restrict__ C,
                                 float* Zc, int Rp, uint32_t* bad) {
    const int64_t total = rows * (int64_t)Rp;
    bool any_bad = false;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = t / Rp;
        const int r = (int)(t - z * Rp);
        float v = 0.0f;
        if (r < R) {
            const float zr = Zsrc[z * R + r];
            any_bad |= bad_factor(zr);
            v = C ? C[r] * zr : zr;
        }
        Zc[t] = v;
    }
    if (__any_sync(0xffffffffu, any_bad) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// One thread per (table, rank); A <= 256 so the sequential fp64 scan is short.
__global__ void prefix_kernel(const float* __restrict__ X, const float* __restrict__ Y, int A, int R, int Rp,
                              float* PXY, uint32_t* bad) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * Rp) return;
    const int table = t / Rp, r = t % Rp;
    const float* F = table ? Y : X;
    float* out = PXY + (size_t)table * (A + 1) * 2 * Rp;
    double S = 0.0;
    bool any_bad = false;
    for (int k = 0; k <= A; ++k) {
        const float hi = (float)S;
        const float lo = (float)(S - (double)hi);
        out[(size_t)(2 * k) * Rp + r] = hi;
        out[(size_t)(2 * k + 1) * Rp + r] = lo;
        if (k < A && r < R) {
            const float v = F[(size_t)k * R + r];
            any_bad |= bad_factor(v);
            S += (double)v;
        }
    }
    if (any_bad) atomicOr(bad, 1u);
}

cudaError_t launch_fold_rows(const float* Zsrc, int64_t rows, int R, const float* Cdev, float* Zc_dst, int Rp,
                             uint32_t* bad, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t total = rows * (int64_t)Rp;
    int64_t g = (total + 255) / 256;
    if (g > (int64_t)sms * 16) g = (int64_t)sms * 16;
    if (g < 1) g = 1;
    fold_rows_kernel<<<(unsigned)g, 256, 0, st>>>(Zsrc, rows, R, Cdev, Zc_dst, Rp, bad);
    return cudaGetLastError();
}

cudaError_t launch_prefix(const float* Xdev, const float* Ydev, int A, int R, int Rp, float* PXY, uint32_t* bad,
                          cudaStream_t st) {
    const int threads = 128;
    const int g = (2 * Rp + threads - 1) / threads;
    prefix_kernel<<<g, threads, 0, st>>>(Xdev, Ydev, A, R, Rp, PXY, bad);
    return cudaGetLastError();
}

}  // namespace pndf
