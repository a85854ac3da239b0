// sample_u32_clamp.cu -- sampling kernel instantiations: uint32 fixed-point SATs,
// clamped neighbours.
#include "sample_kernel.cuh"

namespace pndf {

cudaError_t launch_sample_u32_clamp(int G, int NV, const QParams& p, const pndf_query* q, const float* xi,
                                  const uint32_t* idx, int64_t n, pndf_sample* out, int num_sms, cudaStream_t st) {
    if (idx) return s_g<false, true, true>(G, NV, p, q, xi, idx, n, out, num_sms, st);
    return s_g<false, false, true>(G, NV, p, q, xi, idx, n, out, num_sms, st);
}

}  // namespace pndf
