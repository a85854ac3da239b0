// query_u32_wrap.cu -- query kernel instantiations: uint32 fixed-point SATs,
// wrapped neighbours (one translation unit per variant so they compile in parallel).
#include "query_kernel.cuh"

namespace pndf {

cudaError_t launch_query_u32_wrap(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx,
                                 int64_t n, float* out, int num_sms, cudaStream_t st) {
    if (idx) return dispatch_g<true, true, true>(G, NV, p, q, idx, n, out, num_sms, st);
    return dispatch_g<true, false, true>(G, NV, p, q, idx, n, out, num_sms, st);
}

}  // namespace pndf
