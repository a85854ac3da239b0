// sample.cu -- batched hierarchical importance sampling of the footprint NDF
// (Sec. 5.2), built on the range query.
//
// "We start from the entire NDF image, and subdivide it evenly into four quads
// ... acquire the average values in these four quads ... use the four average
// values as relative probabilities, and randomly choose one quad to proceed ...
// until reaching the bottom level, i.e. a pixel"; "when we reach a pixel,
// we uniformly perturb the sample location inside it"; the pdf is the
// evaluated NDF value.  Readings (same as oracle.c):
// the descent starts from the record's rectangle; a width-w range splits into
// ceil(w/2) | floor(w/2); quads are chosen by their sums (order x-lo/y-lo,
// x-hi/y-lo, x-lo/y-hi, x-hi/y-hi) with one variate per level, xi[8..9] jitter.
//
// Per sample, G lanes share the work as in the query kernel: the 8 Zc rows are
// interpolated ONCE (Z-hat stays in registers), the 4 SAT values of the current
// range stay in registers, and each level loads only the two midpoint SAT rows
// (x_mid, y_mid): 8 + 4 + 2 per level row loads instead of 8 + 4 per range query.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.cuh"
#include "launch.h"

namespace pndf {

cudaError_t launch_sample(const QParams& p, int G, int NV, const pndf_query* q, const float* xi, const uint32_t* idx,
                          int64_t n, pndf_sample* out, int num_sms, cudaStream_t st) {
    if (4 * G * NV != p.Rp) return cudaErrorInvalidValue;
    if (p.prefix_u32)
        return p.wrap ? launch_sample_u32_wrap(G, NV, p, q, xi, idx, n, out, num_sms, st)
                      : launch_sample_u32_clamp(G, NV, p, q, xi, idx, n, out, num_sms, st);
    return p.wrap ? launch_sample_hilo_wrap(G, NV, p, q, xi, idx, n, out, num_sms, st)
                  : launch_sample_hilo_clamp(G, NV, p, q, xi, idx, n, out, num_sms, st);
}

}  // namespace pndf
