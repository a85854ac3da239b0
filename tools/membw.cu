// membw.cu -- bandwidth probes for the roofline denominators that
// MEASURED_PEAKS.json does not carry: L2-resident read bandwidth and
// L1-resident read bandwidth of the B200 load path (float4 LDG), plus an HBM
// read probe for comparison.  Usage: membw [reps]
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membw tools/membw.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

__global__ void read_kernel(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            float4 v = __ldg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 123.456f) *sink = acc;
}

// Per-SM private window: block b reads its own window (L1-resident when small).
__global__ void l1_kernel(const float4* __restrict__ p, size_t win4, int reps, float* sink) {
    float acc = 0.f;
    const float4* base = p + (size_t)blockIdx.x * win4;
    for (int r = 0; r < reps; ++r)
        for (size_t i = threadIdx.x; i < win4; i += blockDim.x) {
            float4 v = __ldg(base + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 123.456f) *sink = acc;
}

static double time_ms(void (*fn)(void*), void* arg) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    fn(arg);  // warm-up
    cudaEventRecord(a);
    fn(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

struct Arg { const float4* p; size_t n4; int reps; float* sink; int grid; int block; };
static void run_read(void* v) {
    Arg* a = (Arg*)v;
    read_kernel<<<a->grid, a->block>>>(a->p, a->n4, a->reps, a->sink);
}
static void run_l1(void* v) {
    Arg* a = (Arg*)v;
    l1_kernel<<<a->grid, a->block>>>(a->p, a->n4, a->reps, a->sink);
}

// Library entry for bench.py: best-of-3 L2-resident float4 read bandwidth (GB/s)
// over a working set of ws_mb MB on the current device; < 0 on error.
extern "C" __attribute__((visibility("default"))) double membw_l2_read_gbs(int ws_mb) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t ws = (size_t)ws_mb << 20;
    float4* buf = nullptr;
    float* sink = nullptr;
    if (cudaMalloc(&buf, ws) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess) return -1.0;
    cudaMemset(buf, 0, ws);
    double best = 0.0;
    for (int r = 0; r < 3; ++r) {
        Arg a{buf, ws / 16, 40, sink, sms * 8, 512};
        const double ms = time_ms(run_read, &a);
        const double gbs = (double)ws * 40 / ms / 1e6;
        if (gbs > best) best = gbs;
    }
    cudaFree(buf);
    cudaFree(sink);
    return best;
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    float* sink;
    cudaMalloc(&sink, 4);
    const size_t big = (size_t)8 << 30;  // 8 GB for HBM
    float4* buf;
    if (cudaMalloc(&buf, big) != cudaSuccess) return 1;
    cudaMemset(buf, 0, big);
    printf("{\"sms\": %d, \"l2_bytes\": %d", sms, l2);
    // HBM read
    {
        Arg a{buf, big / 16, 1, sink, sms * 8, 512};
        double ms = time_ms(run_read, &a);
        printf(", \"hbm_read_gbs\": %.1f", big / ms / 1e6);
    }
    // L2-resident: 48 MB working set read many times
    for (size_t ws : {(size_t)24 << 20, (size_t)48 << 20}) {
        Arg a{buf, ws / 16, 40, sink, sms * 8, 512};
        double ms = time_ms(run_read, &a);
        printf(", \"l2_read_gbs_%zuMB\": %.1f", ws >> 20, (double)ws * 40 / ms / 1e6);
    }
    // L1-resident: 64 KB window per block, one block per SM
    {
        size_t win = 64 << 10;
        Arg a{buf, win / 16, 400, sink, sms, 1024};
        double ms = time_ms(run_l1, &a);
        printf(", \"l1_read_gbs\": %.1f", (double)win * sms * 400 / ms / 1e6);
    }
    printf("}\n");
    return 0;
}
