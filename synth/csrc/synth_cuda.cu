// synth_cuda.cu -- CUDA twin of synth_build_z_exact (synth.c): the exact-rank
// positional factors Z[z][k] of the synthetic INPUT (not the query path).
//
// Bit-identical to the C version: the footprint weights are the same integer
// tables (built on the host by synth_footprint_table and uploaded), every
// footprint sum is accumulated in uint64 (order-independent), and the final
// value is (float)((double)acc / (double)total) on both sides.  It exists so
// that an 8-rank run can build its 22.9 GB replica of config 5 on each GPU
// instead of in host RAM.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr int kWarps = 8;

// grid: one warp per row (grid-stride over the level's rows);
// acc: kWarps * R uint64 in shared memory.
__global__ void z_exact_level_kernel(int N, const uint16_t* __restrict__ atom_map, int R, int s, int n, int qmin,
                                     int Wf, const uint32_t* __restrict__ w, double tot, int64_t row0,
                                     float* __restrict__ Z) {
    extern __shared__ unsigned long long acc_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* acc = acc_all + (size_t)warp * R;
    const int64_t rows = (int64_t)n * n;
    const int64_t W2 = (int64_t)Wf * Wf;
    for (int64_t c = (int64_t)blockIdx.x * kWarps + warp; c < rows; c += (int64_t)gridDim.x * kWarps) {
        for (int k = lane; k < R; k += 32) acc[k] = 0ull;
        __syncwarp();
        const int64_t i = c % n, j = c / n;
        const int64_t bu = (((i * s + qmin) % N) + N) % N, bv = (((j * s + qmin) % N) + N) % N;
        for (int64_t t = lane; t < W2; t += 32) {
            const int q = (int)(t / Wf), p = (int)(t - (int64_t)q * Wf);
            int64_t v = bv + q, u = bu + p;
            if (v >= N) v -= N;
            if (u >= N) u -= N;
            const uint16_t a = atom_map[v * N + u];
            atomicAdd(&acc[a], (unsigned long long)w[q] * (unsigned long long)w[p]);
        }
        __syncwarp();
        float* out = Z + (row0 + c) * (int64_t)R;
        for (int k = lane; k < R; k += 32) out[k] = (float)((double)acc[k] / tot);
        __syncwarp();
    }
}

}  // namespace

extern "C" {

// tables: concatenated per-level weights; tab_off[l], tab_len[l], tab_qmin[l] and
// tab_tot[l] = (double)(sum w) * (double)(sum w) are host arrays (as in synth.c).
// atom_map, tables_dev, Z: device pointers.  Returns a cudaError_t value.
__attribute__((visibility("default"))) int synth_cuda_build_z_exact(int N, const uint16_t* atom_map, int R, int s0,
                                                                    int L, const uint32_t* tables_dev,
                                                                    const int64_t* tab_off, const int32_t* tab_len,
                                                                    const int32_t* tab_qmin, const double* tab_tot,
                                                                    float* Z, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const size_t smem = (size_t)kWarps * R * sizeof(unsigned long long);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(z_exact_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return (int)e;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t row0 = 0;
    for (int l = 0; l < L; ++l) {
        const int s = s0 << l, n = N / s;
        const int32_t Wf = tab_len[l];
        const int64_t rows = (int64_t)n * n;
        int64_t grid = (rows + kWarps - 1) / kWarps;
        if (grid > (int64_t)sms * 64) grid = (int64_t)sms * 64;
        z_exact_level_kernel<<<(unsigned)grid, kWarps * 32, smem, st>>>(
            N, atom_map, R, s, n, tab_qmin[l], Wf, tables_dev + tab_off[l], tab_tot[l], row0, Z);
        row0 += rows;
    }
    return (int)cudaGetLastError();
}

}
