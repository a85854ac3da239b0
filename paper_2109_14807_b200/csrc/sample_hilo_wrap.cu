// sample_hilo_wrap.cu -- sampling kernel instantiations: fp32 (hi, lo) SATs,
// wrapped neighbours.
#include "sample_kernel.cuh"

namespace pndf {

cudaError_t launch_sample_hilo_wrap(int G, int NV, const QParams& p, const pndf_query* q, const float* xi,
                                  const uint32_t* idx, int64_t n, pndf_sample* out, int num_sms, cudaStream_t st) {
    if (idx) return s_g<true, true, false>(G, NV, p, q, xi, idx, n, out, num_sms, st);
    return s_g<true, false, false>(G, NV, p, q, xi, idx, n, out, num_sms, st);
}

}  // namespace pndf
