// query_hilo_wrap.cu -- query kernel instantiations: fp32 (hi, lo) SATs,
// wrapped neighbours (one translation unit per variant so they compile in parallel).
#include "query_kernel.cuh"

namespace pndf {

cudaError_t launch_query_hilo_wrap(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx,
                                 int64_t n, float* out, int num_sms, cudaStream_t st) {
    if (idx) return dispatch_g<true, true, false>(G, NV, p, q, idx, n, out, num_sms, st);
    return dispatch_g<true, false, false>(G, NV, p, q, idx, n, out, num_sms, st);
}

}  // namespace pndf
