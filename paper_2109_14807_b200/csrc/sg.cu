// sg.cu -- environment-light prefiltering rectangles (Sec. 5.4, P:408-428;
// SURVEY §8(f) row 4): one spherical-Gaussian light sample -> the angular
// rectangle over which the NDF is averaged by the range query.
//   theta = arccos((ln eps - ln A) / lambda + 1)   compact-eps support
//   Q     = A_res theta / pi                       square side (P:426-428, 256 -> A_res)
// Readings (same as oracle.c): arccos argument clamped (theta = pi below -1,
// 0 above 1), side = clamp(floor(Q + 1/2), 1, A_res), centred on the bin of the
// projected half vector and shifted inside the grid.  Invalid inputs produce an
// invalid rectangle (x1 > x2), which the query batch then reports.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "launch.h"

namespace pndf {

__device__ __forceinline__ int bin_of(float h, int A) {
    const int b = (int)floorf((h + 1.f) * 0.5f * (float)A);
    return min(max(b, 0), A - 1);
}

__global__ void sg_rect_kernel(const pndf_sg_light* __restrict__ in, int64_t n, float log_eps, int A,
                               pndf_query* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(in + i));
        const float4 b = __ldg(reinterpret_cast<const float4*>(in + i) + 1);
        const float hx = a.w, hy = b.x, lam = b.y, amp = b.z;
        pndf_query q;
        q.u = a.x;
        q.v = a.y;
        q.size = a.z;
        if (!(lam > 0.f) || !(amp > 0.f) || !isfinite(lam) || !isfinite(amp) || !isfinite(hx) || !isfinite(hy)) {
            q.rect = 0x000000ffu;  // x1 = 255 > x2 = 0: invalid
        } else {
            const float arg = (log_eps - logf(amp)) / lam + 1.f;
            const float th = arg <= -1.f ? 3.14159265358979f : (arg >= 1.f ? 0.f : acosf(arg));
            const float Q = (float)A * th / 3.14159265358979f;
            const int side = min(max((int)floorf(Q + 0.5f), 1), A);
            const int x1 = min(max(bin_of(hx, A) - (side - 1) / 2, 0), A - side);
            const int y1 = min(max(bin_of(hy, A) - (side - 1) / 2, 0), A - side);
            q.rect = (uint32_t)x1 | ((uint32_t)(x1 + side - 1) << 8) | ((uint32_t)y1 << 16) |
                     ((uint32_t)(y1 + side - 1) << 24);
        }
        out[i] = q;
    }
}

cudaError_t launch_sg_rects(const pndf_sg_light* in, int64_t n, float eps, int A, pndf_query* out, int num_sms,
                            cudaStream_t st) {
    int64_t g = (n + 255) / 256;
    if (g > (int64_t)num_sms * 16) g = (int64_t)num_sms * 16;
    if (g < 1) g = 1;
    sg_rect_kernel<<<(unsigned)g, 256, 0, st>>>(in, n, logf(eps), A, out);
    return cudaGetLastError();
}

}  // namespace pndf
