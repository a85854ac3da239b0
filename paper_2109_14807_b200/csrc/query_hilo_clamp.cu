// query_hilo_clamp.cu -- query kernel instantiations: fp32 (hi, lo) SATs,
// clamped neighbours (one translation unit per variant so they compile in parallel).
#include "query_kernel.cuh"
#include "query_tc.cuh"

namespace pndf {

cudaError_t launch_query_hilo_clamp(int G, int NV, const QParams& p, const pndf_query* q, const uint32_t* idx,
                                 int64_t n, float* out, int num_sms, cudaStream_t st) {
    if (idx) return dispatch_g<false, true, false>(G, NV, p, q, idx, n, out, num_sms, st);
    return dispatch_g<false, false, false>(G, NV, p, q, idx, n, out, num_sms, st);
}

cudaError_t launch_tc_hilo_clamp(const QParams& p, const pndf_query* q, const uint32_t* perm, const uint32_t* list,
                               const uint32_t* count, float* out, int num_sms, cudaStream_t st) {
    return launch_tc<false, false>(p, q, perm, list, count, out, num_sms, st);
}

}  // namespace pndf
