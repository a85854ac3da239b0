// store.cu -- the C ABI of libpndf: store build, batch
// enqueue (a1-a6 via query.cu), sync/errors (a7) and the end-to-end host
// pipeline.  Declarations and argument contracts: include/pndf.h.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <vector>
#include <mutex>
#include <cstdlib>
#include <new>

#include "internal.cuh"

#ifndef PNDF_DTW
#define PNDF_DTW 48  // widest range (bins) served by the range table (SG rectangles reach ~40)
#endif
#ifndef PNDF_DTAB
#define PNDF_DTAB 1  // build the small-range difference table (query_kernel: one load per axis and rank chunk)
#endif
#include "launch.h"

using namespace pndf;

namespace {

thread_local char g_cuda_err[256] = "";

pndf_status cuda_fail(cudaError_t e, const char* what) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? PNDF_ENOMEM : PNDF_ECUDA;
}

#define CK(call)                                                   \
    do {                                                           \
        cudaError_t _e = (call);                                   \
        if (_e != cudaSuccess) return cuda_fail(_e, #call);        \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
int ilog2(int64_t x) {
    int l = 0;
    while ((int64_t(1) << (l + 1)) <= x) ++l;
    return l;
}

// Binning scratch for one in-flight batch.
struct Scratch : BinScratch {
    void release() {
        for (int i = 0; i < 2; ++i) {
            cudaFree(keys[i]);
            cudaFree(vals[i]);
        }
        cudaFree(counts);
        cudaFree(bsum);
        *this = Scratch();
    }
};

// One stage of the host pipeline.
struct Slot {
    Scratch scratch;
    pndf_query* d_rec = nullptr;
    float* d_out = nullptr;
    int64_t cap = 0;
    cudaStream_t st = nullptr;
    void release() {
        scratch.release();
        cudaFree(d_rec);
        cudaFree(d_out);
        if (st) cudaStreamDestroy(st);
        *this = Slot();
    }
};

constexpr int kSlots = 3;

}  // namespace

struct pndf_store_s {
    pndf_desc d;
    int device = 0;
    int num_sms = 148;
    int64_t l2_bytes = 0;
    int64_t P = 0;
    int Rp = 0, G0 = 0, NV0 = 0, G = 0, NV = 0;
    int64_t nbins = 0;  // P + 1 (last = invalid records); 0 if binning infeasible
    bool tiled = false;  // Wang-tile store (pndf_load_tiles)
    TileParams tp{};
    bool blocked = false;  // blocked / clustered store (pndf_load_blocked)
    BlockParams bp{};
    int32_t* d_slab_ptr = nullptr;
    int32_t* d_group_set = nullptr;
    QParams qp{};
    float* Zc = nullptr;
    float* PXY = nullptr;
    float* DT = nullptr;
    CUtensorMap dt_tmap;  // DT as a 2-D tensor [rows][Rp] for query_g4_kernel's gather4 copies
    uint32_t* err = nullptr;
    Scratch main;
    Slot slots[kSlots];
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    bool timing_pending = false;
    bool pending_binned = false;
    pndf_store_stats stats{};
    std::mutex mu;
};

namespace {

pndf_status validate_desc(const pndf_desc* d) {
    if (!d) return PNDF_EINVAL;
    if (d->abi_version != PNDF_ABI_VERSION) return PNDF_EFORMAT;
    if (!is_pow2(d->map_size) || d->map_size > (1 << 20)) return PNDF_EINVAL;
    if (!is_pow2(d->base_stride) || d->base_stride > d->map_size) return PNDF_EINVAL;
    const int maxL = ilog2(d->map_size / d->base_stride) + 1;
    if (d->num_levels < 2 || d->num_levels > maxL || d->num_levels > kMaxLevels) return PNDF_EINVAL;
    if (d->ang_res < 1 || d->ang_res > 256) return PNDF_EINVAL;
    if (d->rank < 1 || d->rank > 1024) return PNDF_EINVAL;
    {  // positional rows are addressed with int32 indices
        const int64_t n0 = d->map_size / d->base_stride;
        int64_t P = 0;
        for (int l = 0; l < d->num_levels; ++l) P += (n0 >> l) * (n0 >> l);
        if (P >= (int64_t(1) << 31)) return PNDF_EINVAL;
    }
    if (d->flags & ~(PNDF_WRAP | PNDF_PREFIX_MASK)) return PNDF_EINVAL;
    if ((d->flags & PNDF_PREFIX_MASK) == PNDF_PREFIX_MASK) return PNDF_EINVAL;
    return PNDF_OK;
}

// Default lane split: G = lanes sharing a query, NV float4 chunks per lane.
void choose_lanes(int R, int* G, int* NV) {
    const int q4 = (R + 3) / 4;
    int g = 1;
    while (g < q4 && g < 32) g <<= 1;
    int nv = (q4 + g - 1) / g;
    if (nv > 4) nv = 8;
    *G = g;
    *NV = nv;
}

// DT [rows][Rp] fp32 as a 2-D tensor map with a one-row box of the whole row (gather4 fetches 4 such rows);
// false when the driver entry point is unavailable or the shape is outside TMA's limits (Rp > 256)
bool encode_dt_map(const float* DT, int64_t rows, int Rp, CUtensorMap* out) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    if (!fn || Rp > 256 || rows < 1) return false;
    cuuint64_t dims[2] = {(cuuint64_t)Rp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)Rp * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)Rp, 1};
    cuuint32_t es[2] = {1, 1};
    return fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(DT), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return st && cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

pndf_status ensure_scratch(Scratch& s, int64_t n, cudaStream_t st) {
    if (s.cap >= n && s.counts) return PNDF_OK;
    if (capturing(st)) return PNDF_EINVAL;  // no allocation while a CUDA graph is being captured
    s.release();
    const int64_t nb = radix_tiles(n) * 512;
    for (int i = 0; i < 2; ++i) {
        CK(cudaMalloc(&s.keys[i], sizeof(uint32_t) * n));
        CK(cudaMalloc(&s.vals[i], sizeof(uint32_t) * n));
    }
    CK(cudaMalloc(&s.counts, sizeof(uint32_t) * nb));
    CK(cudaMalloc(&s.bsum, sizeof(uint32_t) * scan_blocks(nb)));
    s.cap = n;
    return PNDF_OK;
}

bool want_bins(const pndf_store_s* s, int64_t n, uint32_t opts) {
    if (s->nbins == 0 || (opts & PNDF_BIN_OFF)) return false;
    if (opts & PNDF_BIN_ON) return true;
    // AUTO: the factor set does not stay in L2, and the batch reuses rows enough
    // (>= 4 queries per positional row) for the sort to pay for itself (measured on
    // B200: config 5 at 5.6 queries/row gains 27%, config 4 at 18/row 11%; config 3
    // at 1.8/row loses 40%).
    return (int64_t)s->stats.zc_bytes > s->l2_bytes / 2 && n >= 4 * s->P;
}

// Enqueue one batch (device records) on st using scratch sc.
pndf_status enqueue(pndf_store_s* s, Scratch& sc, const pndf_query* q, int64_t n, float* out, uint32_t opts,
                    cudaStream_t st, bool timing) {
    QParams p = s->qp;
    p.mean = (opts & PNDF_SUM) ? 0u : 1u;
    if (s->blocked) {  // blocked / clustered store: one kernel, never binned
        if (opts & PNDF_BIN_ON) return PNDF_EINVAL;
        if (timing) CK(cudaEventRecord(s->ev[0], st));
        if (timing) CK(cudaEventRecord(s->ev[1], st));
        CK(launch_blocked_query(p, s->bp, s->G, s->NV, q, n, out, s->num_sms, st));
        if (timing) CK(cudaEventRecord(s->ev[2], st));
        s->stats.kernel_launches += 1;
        s->stats.last_binned = 0;
        return PNDF_OK;
    }
    if (s->tiled) {  // Wang-tiled world queries: not binned by cell; batches >= 64K sorted by level
        if (opts & PNDF_BIN_ON) return PNDF_EINVAL;
        // level sort (as in pndf_sample_tiles): the lanes of a warp then serve footprints of one size,
        // whose tile-row loops have similar trip counts; PNDF_BIN_OFF keeps the caller's order
        // (results are bitwise identical either way, so a batch captured into a CUDA graph before the
        // sort scratch exists -- no allocation during capture -- simply runs unsorted)
        const bool sorted = !(opts & PNDF_BIN_OFF) && n >= (int64_t(1) << 16) && n <= (int64_t(1) << 30) &&
                            (sc.cap >= n || !capturing(st));
        int launches = 1;
        const uint32_t* perm = nullptr;
        if (sorted) {
            pndf_status r = ensure_scratch(sc, n, st);
            if (r != PNDF_OK) return r;
        }
        if (timing) CK(cudaEventRecord(s->ev[0], st));
        if (sorted) CK(launch_level_sort(p, q, n, sc, st, &launches, &perm));
        if (timing) CK(cudaEventRecord(s->ev[1], st));
        CK(launch_tiled_query(p, s->tp, s->G, s->NV, q, perm, n, out, s->num_sms, st));
        if (timing) CK(cudaEventRecord(s->ev[2], st));
        s->stats.kernel_launches += (uint64_t)launches;
        s->stats.last_binned = sorted ? 1 : 0;
        return PNDF_OK;
    }
    const bool binned = want_bins(s, n, opts);
    if ((opts & PNDF_BIN_ON) && s->nbins == 0) return PNDF_EINVAL;
    int launches = 0;
    if (timing) CK(cudaEventRecord(s->ev[0], st));
    // sub-batches keep per-query indices in int32 (kernel descriptors, binning permutation)
    const int64_t step = int64_t(1) << 30;
    if (binned) {
        pndf_status r = ensure_scratch(sc, std::min(n, step), st);
        if (r != PNDF_OK) return r;
    }
    bool first = true;
    for (int64_t a = 0; a < n; a += step) {
        const int64_t m = std::min(step, n - a);
        if (binned) {
            const uint32_t* perm = nullptr;
            CK(launch_binning(p, q + a, m, s->P, sc, s->num_sms, st, &launches, &perm));
            if (timing && first) CK(cudaEventRecord(s->ev[1], st));
            CK(launch_query(p, s->G, s->NV, q + a, perm, m, out + a, s->num_sms, st));
        } else {
            if (timing && first) CK(cudaEventRecord(s->ev[1], st));
            CK(launch_query(p, s->G, s->NV, q + a, nullptr, m, out + a, s->num_sms, st));
        }
        launches += 1;
        first = false;
    }
    if (timing) CK(cudaEventRecord(s->ev[2], st));
    s->stats.kernel_launches += (uint64_t)launches;
    s->stats.last_binned = binned ? 1 : 0;
    return PNDF_OK;
}

pndf_status read_sticky(pndf_store_s* s) {
    uint32_t e = 0;
    CK(cudaMemcpy(&e, s->err, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    if (e) {
        CK(cudaMemset(s->err, 0, sizeof(uint32_t)));
        return PNDF_EQUERY;
    }
    return PNDF_OK;
}

void destroy(pndf_store_s* s) {
    if (!s) return;
    DeviceGuard g(s->device);
    cudaDeviceSynchronize();
    cudaFree(s->Zc);
    cudaFree(s->PXY);
    cudaFree(s->DT);
    cudaFree(s->err);
    cudaFree(s->d_slab_ptr);
    cudaFree(s->d_group_set);
    s->main.release();
    for (auto& sl : s->slots) sl.release();
    for (auto& e : s->ev)
        if (e) cudaEventDestroy(e);
    delete s;
}

}  // namespace

// ----------------------------------------------------------------- API --
namespace pndf {
void set_last_error(const char* msg) { snprintf(g_cuda_err, sizeof(g_cuda_err), "%s", msg); }
}  // namespace pndf

extern "C" {

uint32_t pndf_abi_version(void) { return PNDF_ABI_VERSION; }

const char* pndf_error_string(pndf_status st) {
    switch (st) {
        case PNDF_OK: return "ok";
        case PNDF_EINVAL: return "invalid argument";
        case PNDF_ENOMEM: return "out of memory";
        case PNDF_ECUDA: return "CUDA error";
        case PNDF_EFORMAT: return "ABI version mismatch";
        case PNDF_EQUERY: return "invalid query record(s) in batch (results NaN)";
        default: return "unknown pndf status";
    }
}

const char* pndf_last_cuda_error(void) { return g_cuda_err; }

static pndf_status load_impl(const pndf_desc* desc, int64_t P_override, const float* C, const float* X,
                             const float* Y, const float* Z, int device, void* cuda_stream, pndf_store* out);

pndf_status pndf_load_factors(const pndf_desc* desc, const float* C, const float* X, const float* Y, const float* Z,
                              int device, void* cuda_stream, pndf_store* out) {
    if (!out) return PNDF_EINVAL;
    *out = nullptr;
    pndf_status r = validate_desc(desc);
    if (r != PNDF_OK) return r;
    return load_impl(desc, 0, C, X, Y, Z, device, cuda_stream, out);
}

pndf_status pndf_load_tiles(const pndf_tile_desc* td, const float* C, const float* X, const float* Y, const float* Z,
                            int device, void* cuda_stream, pndf_store* out) {
    if (!out || !td) return PNDF_EINVAL;
    *out = nullptr;
    if (td->abi_version != PNDF_ABI_VERSION) return PNDF_EFORMAT;
    if (!is_pow2(td->tile_size) || td->tile_size > (1 << 16) || td->margin < 2 || td->margin > 64) return PNDF_EINVAL;
    pndf_desc d;
    d.abi_version = PNDF_ABI_VERSION;
    d.map_size = td->tile_size;
    d.base_stride = td->base_stride;
    d.num_levels = td->num_levels;
    d.ang_res = td->ang_res;
    d.rank = td->rank;
    d.flags = td->flags & PNDF_PREFIX_MASK;
    pndf_status r = validate_desc(&d);
    if (r != PNDF_OK) return r;
    int64_t pext = 0;
    const int64_t n0 = td->tile_size / td->base_stride;
    for (int l = 0; l < td->num_levels; ++l) {
        const int64_t ne = (n0 >> l) + 2 * td->margin;
        pext += ne * ne;
    }
    if (16 * pext >= (int64_t(1) << 31)) return PNDF_EINVAL;
    r = load_impl(&d, 16 * pext, C, X, Y, Z, device, cuda_stream, out);
    if (r != PNDF_OK) return r;
    pndf_store_s* s = *out;
    s->tiled = true;
    s->nbins = 0;  // tiled queries are not binned
    s->tp.T = td->tile_size;
    s->tp.margin = td->margin;
    s->tp.p_ext = pext;
    s->tp.seed = td->seed;
    s->tp.reach = td->margin;
    s->qp.wrap = 0;
    {  // measured reach: rows beyond it are all zero, so the kernels skip them exactly
        cudaStream_t st = (cudaStream_t)cuda_stream;
        DeviceGuard guard(device);
        cudaError_t e = cudaMemsetAsync(s->err + 1, 0, sizeof(uint32_t), st);
        if (e == cudaSuccess) e = launch_tile_reach(s->Zc, s->Rp, s->tp, (int)(td->tile_size / td->base_stride),
                                                    td->num_levels, s->err + 1, st);
        uint32_t reach = 0;
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaMemcpy(&reach, s->err + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) e = cudaMemsetAsync(s->err + 1, 0, sizeof(uint32_t), st);
        if (e != cudaSuccess) {
            destroy(s);
            *out = nullptr;
            return cuda_fail(e, "tile reach");
        }
        s->tp.reach = (int32_t)reach;
        s->stats.tile_reach = (int32_t)reach;
        s->stats.kernel_launches += 1;
    }
    return PNDF_OK;
}

pndf_status pndf_load_blocked(const pndf_block_desc* bd, const float* C, const float* X, const float* Y,
                              const int32_t* group_set, const int64_t* slab_ptr, const float* Z, int device,
                              void* cuda_stream, pndf_store* out) {
    if (!out || !bd || !C || !X || !Y || !group_set || !slab_ptr || (bd->num_slabs > 0 && !Z)) return PNDF_EINVAL;
    *out = nullptr;
    if (bd->abi_version != PNDF_ABI_VERSION) return PNDF_EFORMAT;
    pndf_desc d;
    d.abi_version = PNDF_ABI_VERSION;
    d.map_size = bd->map_size;
    d.base_stride = bd->base_stride;
    d.num_levels = bd->num_levels;
    d.ang_res = bd->ang_res;
    d.rank = bd->rank;
    d.flags = bd->flags & PNDF_WRAP;
    pndf_status r = validate_desc(&d);
    if (r != PNDF_OK) return r;
    const int t = bd->block, A = bd->ang_res, R = bd->rank;
    if (t < 1 || t > 64 || A % t != 0) return PNDF_EINVAL;
    if (!is_pow2(bd->region) || bd->region > bd->map_size) return PNDF_EINVAL;
    if (bd->num_sets < 1 || bd->num_slabs < 0 || bd->num_slabs >= (int64_t(1) << 31)) return PNDF_EINVAL;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return PNDF_EINVAL;
    DeviceGuard guard(device);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const int nb = A / t, nb2 = nb * nb;
    const int64_t nr = bd->map_size / bd->region, n0 = bd->map_size / bd->base_stride;
    int64_t P = 0;
    for (int l = 0; l < bd->num_levels; ++l) P += (n0 >> l) * (n0 >> l);
    const int64_t G = nr * nr * nb2, S = bd->num_slabs, sets = bd->num_sets;
    // host copies of the index tables; per-slab factor set for the fold
    std::vector<int32_t> hg(G);
    std::vector<int64_t> hs(P * nb2);
    CK(cudaMemcpy(hg.data(), group_set, sizeof(int32_t) * G, cudaMemcpyDefault));
    CK(cudaMemcpy(hs.data(), slab_ptr, sizeof(int64_t) * P * nb2, cudaMemcpyDefault));
    std::vector<int32_t> hs32(P * nb2), slab_set(S, -1);
    {
        int64_t off = 0;
        for (int l = 0; l < bd->num_levels; ++l) {
            const int64_t nl = n0 >> l, sl = (int64_t)bd->base_stride << l;
            for (int64_t c = 0; c < nl * nl; ++c) {
                const int64_t i = c % nl, j = c / nl;
                const int64_t reg = (((2 * j + 1) * sl) / (2 * bd->region)) * nr + ((2 * i + 1) * sl) / (2 * bd->region);
                for (int b = 0; b < nb2; ++b) {
                    const int64_t slab = hs[(off + c) * nb2 + b];
                    if (slab < -1 || slab >= S) return PNDF_EINVAL;
                    hs32[(off + c) * nb2 + b] = (int32_t)slab;
                    if (slab < 0) continue;
                    const int32_t set = hg[reg * nb2 + b];
                    if (set < 0 || set >= sets) return PNDF_EINVAL;  // a slab without factors
                    slab_set[slab] = set;
                }
            }
            off += nl * nl;
        }
    }
    for (int64_t sl = 0; sl < S; ++sl)
        if (slab_set[sl] < 0) slab_set[sl] = 0;  // unreferenced slab: any valid set
    for (int64_t g = 0; g < G; ++g)
        if (hg[g] < -1 || hg[g] >= sets) return PNDF_EINVAL;

    pndf_store_s* s = new (std::nothrow) pndf_store_s();
    if (!s) return PNDF_ENOMEM;
    s->d = d;
    s->device = device;
    s->P = S;
    choose_lanes(R, &s->G0, &s->NV0);
    s->G = s->G0;
    s->NV = s->NV0;
    s->Rp = 4 * s->G0 * s->NV0;
    const int Rp = s->Rp;
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    s->num_sms = v > 0 ? v : 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device);
    s->l2_bytes = v;
    s->nbins = 0;
    auto fail = [&](pndf_status e) {
        destroy(s);
        return e;
    };
    const size_t zc_bytes = sizeof(float) * (size_t)std::max<int64_t>(S, 1) * Rp;
    const size_t pool_bytes = sizeof(float) * (size_t)sets * 2 * (t + 1) * 2 * Rp;
    float *dC = nullptr, *dX = nullptr, *dY = nullptr, *dZ = nullptr;
    int32_t* dset = nullptr;
    auto free_tmp = [&]() {
        cudaFree(dC);
        cudaFree(dX);
        cudaFree(dY);
        cudaFree(dZ);
        cudaFree(dset);
    };
    cudaError_t e = cudaSuccess;
    auto ok = [&](cudaError_t ce) {
        if (e == cudaSuccess) e = ce;
        return e == cudaSuccess;
    };
    ok(cudaMalloc(&s->Zc, zc_bytes));
    ok(cudaMalloc(&s->PXY, pool_bytes));
    ok(cudaMalloc(&s->err, 2 * sizeof(uint32_t)));
    ok(cudaMalloc(&s->d_slab_ptr, sizeof(int32_t) * P * nb2));
    ok(cudaMalloc(&s->d_group_set, sizeof(int32_t) * G));
    ok(cudaMalloc(&dC, sizeof(float) * sets * R));
    ok(cudaMalloc(&dX, sizeof(float) * sets * t * R));
    ok(cudaMalloc(&dY, sizeof(float) * sets * t * R));
    ok(cudaMalloc(&dZ, sizeof(float) * std::max<int64_t>(S, 1) * R));
    ok(cudaMalloc(&dset, sizeof(int32_t) * std::max<int64_t>(S, 1)));
    for (auto& ev : s->ev) ok(cudaEventCreate(&ev));
    if (e != cudaSuccess) {
        free_tmp();
        return fail(cuda_fail(e, "cudaMalloc(blocked store)"));
    }
    ok(cudaMemsetAsync(s->err, 0, 2 * sizeof(uint32_t), st));
    ok(cudaMemcpy(dC, C, sizeof(float) * sets * R, cudaMemcpyDefault));
    ok(cudaMemcpy(dX, X, sizeof(float) * sets * t * R, cudaMemcpyDefault));
    ok(cudaMemcpy(dY, Y, sizeof(float) * sets * t * R, cudaMemcpyDefault));
    if (S > 0) ok(cudaMemcpy(dZ, Z, sizeof(float) * S * R, cudaMemcpyDefault));
    if (S > 0) ok(cudaMemcpy(dset, slab_set.data(), sizeof(int32_t) * S, cudaMemcpyHostToDevice));
    ok(cudaMemcpy(s->d_slab_ptr, hs32.data(), sizeof(int32_t) * P * nb2, cudaMemcpyHostToDevice));
    ok(cudaMemcpy(s->d_group_set, hg.data(), sizeof(int32_t) * G, cudaMemcpyHostToDevice));
    ok(launch_block_build(dX, dY, (int)sets, t, R, Rp, s->PXY, dZ, S, dC, dset, s->Zc, s->err + 1, s->num_sms, st));
    ok(cudaStreamSynchronize(st));
    uint32_t hflags = 0;
    ok(cudaMemcpy(&hflags, s->err + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    free_tmp();
    if (e != cudaSuccess) return fail(cuda_fail(e, "blocked store build"));
    if (hflags & 1u) return fail(PNDF_EINVAL);
    s->stats.kernel_launches += 2;
    QParams& p = s->qp;
    p.Zc = s->Zc;
    p.PXY = s->PXY;
    p.err = s->err;
    p.N = d.map_size;
    p.n0 = (int32_t)n0;
    p.L = d.num_levels;
    p.A = A;
    p.Rp = Rp;
    p.wrap = (d.flags & PNDF_WRAP) ? 1 : 0;
    p.prefix_u32 = 0;
    p.inv_s0 = 1.0f / (float)d.base_stride;
    p.mean = 1;
    s->blocked = true;
    s->bp.t = t;
    s->bp.nb = nb;
    s->bp.region = bd->region;
    s->bp.nr = (int32_t)nr;
    s->bp.r_shift = ilog2(bd->region);
    s->bp.slab_ptr = s->d_slab_ptr;
    s->bp.group_set = s->d_group_set;
    s->stats.rows = S;
    s->stats.rank_padded = Rp;
    s->stats.lanes_per_query = s->G;
    s->stats.zc_bytes = (int64_t)zc_bytes;
    s->stats.prefix_bytes = (int64_t)pool_bytes;
    s->stats.prefix_format = 0;
    *out = s;
    return PNDF_OK;
}

static pndf_status load_impl(const pndf_desc* desc, int64_t P_override, const float* C, const float* X,
                             const float* Y, const float* Z, int device, void* cuda_stream, pndf_store* out) {
    if (!out || !X || !Y || !Z) return PNDF_EINVAL;
    *out = nullptr;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return PNDF_EINVAL;
    DeviceGuard guard(device);
    cudaStream_t st = (cudaStream_t)cuda_stream;

    pndf_store_s* s = new (std::nothrow) pndf_store_s();
    if (!s) return PNDF_ENOMEM;
    s->d = *desc;
    s->device = device;
    const int N = desc->map_size, s0 = desc->base_stride, L = desc->num_levels, A = desc->ang_res,
              R = desc->rank;
    const int64_t n0 = N / s0;
    for (int l = 0; l < L; ++l) s->P += (n0 >> l) * (n0 >> l);
    if (P_override > 0) s->P = P_override;
    choose_lanes(R, &s->G0, &s->NV0);
    s->G = s->G0;
    s->NV = s->NV0;
    s->Rp = 4 * s->G0 * s->NV0;
    const int Rp = s->Rp;
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    s->num_sms = v > 0 ? v : 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device);
    s->l2_bytes = v;
    // binning keys are uint32 (level offset + Morton code of the cell or half cell)
    s->nbins = (s->P + 1 < (int64_t)0xffffffffLL) ? s->P + 1 : 0;

    auto fail = [&](pndf_status e) {
        destroy(s);
        return e;
    };
    const size_t zc_bytes = sizeof(float) * (size_t)s->P * Rp;
    const size_t pxy_bytes_max = sizeof(float) * (size_t)2 * (A + 1) * 2 * Rp;  // HILO (U32 uses half)
    cudaError_t e;
    if ((e = cudaMalloc(&s->Zc, zc_bytes)) != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(Zc)"));
    if ((e = cudaMalloc(&s->PXY, pxy_bytes_max)) != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(PXY)"));
    if ((e = cudaMalloc(&s->err, 2 * sizeof(uint32_t))) != cudaSuccess) return fail(cuda_fail(e, "cudaMalloc(err)"));
    uint32_t* flags = s->err + 1;  // bit 0: bad factor, bit 1: underflow of the U32 rescale
    cudaMemsetAsync(s->err, 0, 2 * sizeof(uint32_t), st);
    for (auto& ev : s->ev)
        if ((e = cudaEventCreate(&ev)) != cudaSuccess) return fail(cuda_fail(e, "cudaEventCreate"));

    // small factors: C (or ones), X, Y -> device; per-rank stats; multipliers; exponents
    float *dC = nullptr, *dXY = nullptr, *dM = nullptr, *dmin = nullptr;
    double* dtot = nullptr;
    int* dexp = nullptr;
    auto free_small = [&]() {
        cudaFree(dC);
        cudaFree(dXY);
        cudaFree(dM);
        cudaFree(dmin);
        cudaFree(dtot);
        cudaFree(dexp);
    };
    auto fail_small = [&](cudaError_t ce, const char* what) {
        free_small();
        return fail(cuda_fail(ce, what));
    };
    if ((e = cudaMalloc(&dC, sizeof(float) * Rp)) != cudaSuccess) return fail_small(e, "cudaMalloc(C)");
    if ((e = cudaMalloc(&dM, sizeof(float) * Rp)) != cudaSuccess) return fail_small(e, "cudaMalloc(M)");
    if ((e = cudaMalloc(&dXY, sizeof(float) * 2 * (size_t)A * R)) != cudaSuccess) return fail_small(e, "cudaMalloc(XY)");
    if ((e = cudaMalloc(&dtot, sizeof(double) * 2 * Rp)) != cudaSuccess) return fail_small(e, "cudaMalloc(tot)");
    if ((e = cudaMalloc(&dmin, sizeof(float) * 2 * Rp)) != cudaSuccess) return fail_small(e, "cudaMalloc(min)");
    if ((e = cudaMalloc(&dexp, sizeof(int) * 2 * Rp)) != cudaSuccess) return fail_small(e, "cudaMalloc(exp)");
    std::vector<float> hC(Rp, 0.0f);
    for (int i = 0; i < R; ++i) hC[i] = 1.0f;
    if (C && (e = cudaMemcpy(hC.data(), C, sizeof(float) * R, cudaMemcpyDefault)) != cudaSuccess)
        return fail_small(e, "cudaMemcpy(C)");
    if ((e = cudaMemcpy(dC, hC.data(), sizeof(float) * Rp, cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail_small(e, "cudaMemcpy(C)");
    if ((e = cudaMemcpy(dXY, X, sizeof(float) * (size_t)A * R, cudaMemcpyDefault)) != cudaSuccess)
        return fail_small(e, "cudaMemcpy(X)");
    if ((e = cudaMemcpy(dXY + (size_t)A * R, Y, sizeof(float) * (size_t)A * R, cudaMemcpyDefault)) != cudaSuccess)
        return fail_small(e, "cudaMemcpy(Y)");
    // validate C (fold it as a one-row "Z") and X, Y (stats kernel); gather totals / min nonzero
    if ((e = launch_fold_rows(dC, 1, R, nullptr, dC, R, flags, st)) != cudaSuccess) return fail_small(e, "validate C");
    if ((e = launch_prefix_stats(dXY, dXY + (size_t)A * R, A, R, Rp, dtot, dmin, flags, st)) != cudaSuccess)
        return fail_small(e, "prefix stats");
    s->stats.kernel_launches += 2;
    std::vector<double> htot(2 * Rp);
    std::vector<float> hmin(2 * Rp);
    uint32_t hflags = 0;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail_small(e, "store build");
    cudaMemcpy(htot.data(), dtot, sizeof(double) * 2 * Rp, cudaMemcpyDeviceToHost);
    cudaMemcpy(hmin.data(), dmin, sizeof(float) * 2 * Rp, cudaMemcpyDeviceToHost);
    if ((e = cudaMemcpy(&hflags, flags, sizeof(uint32_t), cudaMemcpyDeviceToHost)) != cudaSuccess)
        return fail_small(e, "store build");
    if (hflags & 1u) {  // negative or non-finite C, X or Y
        free_small();
        return fail(PNDF_EINVAL);
    }
    // SAT format: U32 when every rank's fixed-point step 2^-e (~ total 2^-31) is <= 2^-15 of its
    // smallest nonzero entry (so any nonzero range sum is within 2^-15 relative), else HILO.
    const uint32_t pmode = desc->flags & PNDF_PREFIX_MASK;
    std::vector<int> hexp(2 * Rp, 0);
    bool u32_ok = true;
    for (int t = 0; t < 2 * Rp; ++t) {
        const double T = htot[t];
        if (T <= 0.0) continue;
        int ex = (int)std::floor(std::log2(4294967294.0 / T));
        while (std::ldexp(T, ex) > 4294967294.0) --ex;
        hexp[t] = ex;
        if (std::ldexp(1.0, -ex) > std::ldexp((double)hmin[t], -15)) u32_ok = false;
    }
    bool use_u32 = (pmode == PNDF_PREFIX_U32) || (pmode == PNDF_PREFIX_AUTO && u32_ok);

    // positional factors: Zc = fl32(M_r Z_r(z)), padded to Rp; U32 falls back to HILO on underflow
    cudaPointerAttributes pa;
    const bool z_dev = cudaPointerGetAttributes(&pa, Z) == cudaSuccess &&
                       (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    for (int attempt = 0; attempt < 2; ++attempt) {
        std::vector<float> hM(Rp, 0.0f);
        for (int r = 0; r < R; ++r)
            hM[r] = use_u32 ? std::ldexp(hC[r], -(hexp[r] + hexp[Rp + r])) : hC[r];
        if ((e = cudaMemcpy(dM, hM.data(), sizeof(float) * Rp, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail_small(e, "cudaMemcpy(M)");
        if ((e = cudaMemcpy(dexp, hexp.data(), sizeof(int) * 2 * Rp, cudaMemcpyHostToDevice)) != cudaSuccess)
            return fail_small(e, "cudaMemcpy(exp)");
        cudaMemsetAsync(flags, 0, sizeof(uint32_t), st);
        if ((e = launch_prefix(dXY, dXY + (size_t)A * R, A, R, Rp, use_u32 ? 1 : 0, dexp, s->PXY, st)) !=
            cudaSuccess)
            return fail_small(e, "prefix kernel");
        s->stats.kernel_launches += 1;
        if (z_dev) {
            if ((e = launch_fold_rows(Z, s->P, R, dM, s->Zc, Rp, flags, st)) != cudaSuccess)
                return fail_small(e, "fold kernel");
            s->stats.kernel_launches += 1;
        } else {
            // host Z: stream through a device staging buffer (or straight into Zc when Rp == R)
            const int64_t chunk = std::max<int64_t>(1, (int64_t(64) << 20) / R);  // 256 MB of rows
            float* stage = nullptr;
            if (Rp != R && (e = cudaMalloc(&stage, sizeof(float) * (size_t)std::min(chunk, s->P) * R)) !=
                               cudaSuccess)
                return fail_small(e, "cudaMalloc(stage)");
            for (int64_t a = 0; a < s->P && e == cudaSuccess; a += chunk) {
                const int64_t m = std::min(chunk, s->P - a);
                float* dst = stage ? stage : s->Zc + (size_t)a * Rp;
                e = cudaMemcpyAsync(dst, Z + (size_t)a * R, sizeof(float) * (size_t)m * R, cudaMemcpyDefault, st);
                if (e == cudaSuccess) e = launch_fold_rows(dst, m, R, dM, s->Zc + (size_t)a * Rp, Rp, flags, st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                s->stats.kernel_launches += 1;
            }
            cudaFree(stage);
            if (e != cudaSuccess) return fail_small(e, "Z upload");
        }
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail_small(e, "store build");
        if ((e = cudaMemcpy(&hflags, flags, sizeof(uint32_t), cudaMemcpyDeviceToHost)) != cudaSuccess)
            return fail_small(e, "store build");
        if (hflags & 1u) {  // negative or non-finite Z
            free_small();
            return fail(PNDF_EINVAL);
        }
        if ((hflags & 2u) && use_u32 && pmode != PNDF_PREFIX_U32) {
            use_u32 = false;  // the power-of-two rescale underflowed: rebuild with HILO
            continue;
        }
        break;
    }
    free_small();
    cudaMemsetAsync(flags, 0, sizeof(uint32_t), st);
    const size_t pxy_bytes = use_u32 ? pxy_bytes_max / 2 : pxy_bytes_max;

    QParams& p = s->qp;
    p.Zc = s->Zc;
    p.PXY = s->PXY;
    p.err = s->err;
    for (int l = 0; l < kMaxLevels; ++l) p.level_off[l] = 0;
    int64_t off = 0;
    for (int l = 0; l < L; ++l) {
        p.level_off[l] = off;
        off += (n0 >> l) * (n0 >> l);
    }
    p.N = N;
    p.n0 = (int32_t)n0;
    p.L = L;
    p.A = A;
    p.Rp = Rp;
    p.wrap = (desc->flags & PNDF_WRAP) ? 1 : 0;
    p.prefix_u32 = use_u32 ? 1 : 0;
    p.inv_s0 = 1.0f / (float)s0;
    p.mean = 1;
    p.DT = nullptr;
    p.dt_w = 0;
    p.dt_tmap = nullptr;
#if PNDF_DTAB
    {  // range table for rectangles of side <= W (2 A W Rp floats; 8.4 MB for config 5)
        const int W = std::min(PNDF_DTW, A);
        if (cudaMalloc(&s->DT, sizeof(float) * (size_t)2 * A * W * Rp) == cudaSuccess &&
            launch_range_table(s->PXY, A, Rp, use_u32 ? 1 : 0, W, s->DT, st) == cudaSuccess &&
            cudaStreamSynchronize(st) == cudaSuccess) {
            p.DT = s->DT;
            p.dt_w = W;
            p.dt_tmap = encode_dt_map(s->DT, (int64_t)2 * A * W, Rp, &s->dt_tmap) ? &s->dt_tmap : nullptr;
            s->stats.kernel_launches += 1;
            s->stats.range_table_bytes = (int64_t)sizeof(float) * 2 * A * W * Rp;
            s->stats.range_table_width = W;
        } else {
            cudaGetLastError();
            cudaFree(s->DT);
            s->DT = nullptr;
        }
    }
#endif
    s->stats.rows = s->P;
    s->stats.rank_padded = Rp;
    s->stats.lanes_per_query = s->G;
    s->stats.zc_bytes = (int64_t)zc_bytes;
    s->stats.prefix_bytes = (int64_t)pxy_bytes;
    s->stats.prefix_format = use_u32 ? 1 : 0;
    *out = s;
    return PNDF_OK;
}

pndf_status pndf_query_batch(pndf_store s, const pndf_query* d_queries, int64_t n, float* d_out, uint32_t opts,
                             void* cuda_stream) {
    if (!s || n < 0 || (n > 0 && (!d_queries || !d_out))) return PNDF_EINVAL;
    if (opts & ~(PNDF_SUM | PNDF_BIN_ON | PNDF_BIN_OFF | PNDF_TIMING)) return PNDF_EINVAL;
    if ((opts & PNDF_BIN_ON) && (opts & PNDF_BIN_OFF)) return PNDF_EINVAL;
    if (n == 0) return PNDF_OK;
    if ((uintptr_t)d_queries % 16 != 0 || (uintptr_t)d_out % 4 != 0) return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    const bool timing = (opts & PNDF_TIMING) != 0;
    pndf_status r = enqueue(s, s->main, d_queries, n, d_out, opts, (cudaStream_t)cuda_stream, timing);
    if (r == PNDF_OK) {
        s->timing_pending = timing;
        s->pending_binned = s->stats.last_binned != 0;
    }
    return r;
}

pndf_status pndf_sample_batch(pndf_store s, const pndf_query* d_queries, const float* d_xi, int64_t n,
                              pndf_sample* d_out, uint32_t opts, void* cuda_stream) {
    if (!s || n < 0 || (n > 0 && (!d_queries || !d_xi || !d_out))) return PNDF_EINVAL;
    if (opts & ~(PNDF_BIN_ON | PNDF_BIN_OFF | PNDF_TIMING)) return PNDF_EINVAL;
    if ((opts & PNDF_BIN_ON) && (opts & PNDF_BIN_OFF)) return PNDF_EINVAL;
    if (n == 0) return PNDF_OK;
    if ((uintptr_t)d_queries % 16 != 0 || (uintptr_t)d_out % 16 != 0 || (uintptr_t)d_xi % 4 != 0)
        return PNDF_EINVAL;
    if (s->tiled || s->blocked) return PNDF_EINVAL;  // sampling: one-group stores only
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const bool timing = (opts & PNDF_TIMING) != 0;
    const bool binned = want_bins(s, n, opts);
    if ((opts & PNDF_BIN_ON) && s->nbins == 0) return PNDF_EINVAL;
    int launches = 0;
    if (timing) CK(cudaEventRecord(s->ev[0], st));
    const int64_t step = int64_t(1) << 30;
    if (binned) {
        pndf_status r = ensure_scratch(s->main, std::min(n, step), st);
        if (r != PNDF_OK) return r;
    }
    // Lanes per sample: the descent is a chain of dependent L2 loads, so more samples in flight per warp
    // beat wider samples.  With U32 SATs (HILO at 8 float4 per lane spills): Rp >= 128 -> 8 float4 per
    // lane (config 5: G = 8, 4 samples per warp, 3.57e8 vs 3.12e8 samples/s at G = 32, 2.85e8 at G = 16);
    // smaller Rp -> 2 float4 per lane (config 2: G = 4, 2.5e9 vs 2.0e9 at G = 8, 1.9e9 at G = 1).
    // pndf_set_lanes overrides.
    int sg = s->G, snv = s->NV;
    if (s->G == s->G0 && s->qp.prefix_u32) {
        const int nv = s->Rp >= 128 ? 8 : 2;
        if (s->Rp % (4 * nv) == 0 && lanes_supported(s->Rp / (4 * nv), nv)) {
            sg = s->Rp / (4 * nv);
            snv = nv;
        }
    }
    bool first = true;
    for (int64_t a = 0; a < n; a += step) {
        const int64_t m = std::min(step, n - a);
        const uint32_t* perm = nullptr;
        if (binned) CK(launch_binning(s->qp, d_queries + a, m, s->P, s->main, s->num_sms, st, &launches, &perm));
        if (timing && first) CK(cudaEventRecord(s->ev[1], st));
        CK(launch_sample(s->qp, sg, snv, d_queries + a, d_xi + (size_t)a * 10, perm, m, d_out + a, s->num_sms,
                         st));
        launches += 1;
        first = false;
    }
    if (timing) CK(cudaEventRecord(s->ev[2], st));
    s->stats.kernel_launches += (uint64_t)launches;
    s->stats.last_binned = binned ? 1 : 0;
    s->timing_pending = timing;
    return PNDF_OK;
}

pndf_status pndf_sample_blocked(pndf_store s, const pndf_query* d_queries, const float* d_xi, int64_t n,
                                pndf_sample* d_out, int32_t* d_block, uint32_t opts, void* cuda_stream) {
    if (!s || n < 0 || (n > 0 && (!d_queries || !d_xi || !d_out))) return PNDF_EINVAL;
    if (opts & ~PNDF_TIMING) return PNDF_EINVAL;
    if (!s->blocked) return PNDF_EINVAL;
    if (n == 0) return PNDF_OK;
    if ((uintptr_t)d_queries % 16 != 0 || (uintptr_t)d_out % 16 != 0 || (uintptr_t)d_xi % 4 != 0 ||
        (uintptr_t)d_block % 4 != 0)
        return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const bool timing = (opts & PNDF_TIMING) != 0;
    if (timing) CK(cudaEventRecord(s->ev[0], st));
    if (timing) CK(cudaEventRecord(s->ev[1], st));
    QParams p = s->qp;
    CK(launch_blocked_sample(p, s->bp, s->G, s->NV, d_queries, d_xi, n, d_out, d_block, s->num_sms, st));
    if (timing) CK(cudaEventRecord(s->ev[2], st));
    s->stats.kernel_launches += 1;
    s->stats.last_binned = 0;
    s->timing_pending = timing;
    return PNDF_OK;
}

pndf_status pndf_sample_tiles(pndf_store s, const pndf_query* d_queries, const float* d_xi, int64_t n,
                              pndf_sample* d_out, int32_t* d_tile, uint32_t opts, void* cuda_stream) {
    if (!s || n < 0 || (n > 0 && (!d_queries || !d_xi || !d_out))) return PNDF_EINVAL;
    if (opts & ~(PNDF_TIMING | PNDF_BIN_OFF)) return PNDF_EINVAL;
    if (!s->tiled) return PNDF_EINVAL;
    if (n == 0) return PNDF_OK;
    if ((uintptr_t)d_queries % 16 != 0 || (uintptr_t)d_out % 16 != 0 || (uintptr_t)d_xi % 4 != 0 ||
        (uintptr_t)d_tile % 4 != 0)
        return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const bool timing = (opts & PNDF_TIMING) != 0;
    if (s->tp.reach > 4) return PNDF_EINVAL;  // candidate tiles exceed the kernel's 128-bit mask
    // level sort (default for batches >= 64K): lanes of a warp then sample footprints of one size,
    // so their tile-row loops have similar trip counts; PNDF_BIN_OFF samples in the caller's order
    // (bitwise identical results, so a graph capture without sort scratch runs unsorted)
    const bool sorted = !(opts & PNDF_BIN_OFF) && n >= (int64_t(1) << 16) &&
                        (s->main.cap >= std::min(n, int64_t(1) << 30) || !capturing(st));
    const int64_t step = int64_t(1) << 30;
    if (sorted) {
        pndf_status r = ensure_scratch(s->main, std::min(n, step), st);
        if (r != PNDF_OK) return r;
    }
    if (timing) CK(cudaEventRecord(s->ev[0], st));
    // lanes per sample as in pndf_sample_batch: 8 float4 per lane with U32 SATs (the Wang workload, R = 32:
    // one lane per sample, 4.8e8 vs 3.1e8 samples/s at the query kernel's 8 lanes); pndf_set_lanes overrides
    int sg = s->G, snv = s->NV;
    if (s->G == s->G0 && s->qp.prefix_u32 && s->Rp >= 32 && lanes_supported(s->Rp / 32, 8)) {
        sg = s->Rp / 32;
        snv = 8;
    }
    int launches = 0;
    bool first = true;
    for (int64_t a = 0; a < n; a += step) {
        const int64_t m = std::min(step, n - a);
        const uint32_t* perm = nullptr;
        if (sorted) CK(launch_level_sort(s->qp, d_queries + a, m, s->main, st, &launches, &perm));
        if (timing && first) CK(cudaEventRecord(s->ev[1], st));
        CK(launch_tiled_sample(s->qp, s->tp, sg, snv, d_queries + a, d_xi + (size_t)a * 11, perm, m, d_out + a,
                               d_tile ? d_tile + 2 * a : nullptr, s->num_sms, st));
        launches += 1;
        first = false;
    }
    if (timing) CK(cudaEventRecord(s->ev[2], st));
    s->stats.kernel_launches += (uint64_t)launches;
    s->stats.last_binned = sorted ? 1 : 0;
    s->timing_pending = timing;
    return PNDF_OK;
}

pndf_status pndf_sg_queries(const pndf_sg_light* d_in, int64_t n, float eps, int32_t ang_res, pndf_query* d_out,
                            void* cuda_stream) {
    if (n < 0 || (n > 0 && (!d_in || !d_out))) return PNDF_EINVAL;
    if (!(eps > 0.0f) || ang_res < 1 || ang_res > 256) return PNDF_EINVAL;
    if ((uintptr_t)d_in % 16 != 0 || (uintptr_t)d_out % 16 != 0) return PNDF_EINVAL;
    if (n == 0) return PNDF_OK;
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    CK(launch_sg_rects(d_in, n, eps, ang_res, d_out, sms, (cudaStream_t)cuda_stream));
    return PNDF_OK;
}

pndf_status pndf_sync(pndf_store s, void* cuda_stream) {
    if (!s) return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    CK(cudaStreamSynchronize((cudaStream_t)cuda_stream));
    if (s->timing_pending) {
        float t01 = 0.f, t12 = 0.f;
        CK(cudaEventElapsedTime(&t01, s->ev[0], s->ev[1]));
        CK(cudaEventElapsedTime(&t12, s->ev[1], s->ev[2]));
        s->stats.bin_ms += t01;
        s->stats.query_ms += t12;
        s->stats.timed_batches += 1;
        s->timing_pending = false;
    }
    return read_sticky(s);
}

pndf_status pndf_query_batch_host(pndf_store s, const pndf_query* h_queries, int64_t n, float* h_out,
                                  uint32_t opts) {
    if (!s || n < 0 || (n > 0 && (!h_queries || !h_out))) return PNDF_EINVAL;
    if (opts & ~(PNDF_SUM | PNDF_BIN_ON | PNDF_BIN_OFF)) return PNDF_EINVAL;
    if ((opts & PNDF_BIN_ON) && (opts & PNDF_BIN_OFF)) return PNDF_EINVAL;
    if (n == 0) return PNDF_OK;
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    // Chunking: chunks overlap H2D / kernels / D2H on the three slot streams.  When the whole
    // batch qualifies for binning, chunks of n/32 records, but at least 2 queries per positional
    // row so each is still binned on its own (config 5: 44.7M-record chunks, 3.07 G queries/s
    // end to end vs 2.77 with 8 chunks at >= 4 queries/row; measured grid in DESIGN.md);
    // otherwise 1M..64M records each (n/8).
    const bool bin_all = want_bins(s, n, opts);
    static const int64_t kChunks = [] {  // binned chunk count (PNDF_E2E_CHUNKS, for A/B runs)
        const char* e = getenv("PNDF_E2E_CHUNKS");
        const int v = e ? atoi(e) : 32;
        return (int64_t)(v >= 2 && v <= 64 ? v : 32);
    }();
    static const int64_t kMinQ = [] {  // binned chunks hold >= kMinQ queries per row (PNDF_E2E_MINQ)
        const char* e = getenv("PNDF_E2E_MINQ");
        const int v = e ? atoi(e) : 2;
        return (int64_t)(v >= 1 && v <= 64 ? v : 2);
    }();
    int64_t chunk;
    if (bin_all && !(opts & PNDF_BIN_ON))
        chunk = std::max<int64_t>(kMinQ * s->P, (n + kChunks - 1) / kChunks);
    else
        chunk = std::max<int64_t>(int64_t(1) << 20, std::min<int64_t>(int64_t(1) << 26, (n + 7) / 8));
    chunk = std::min(chunk, n);
    const int64_t nchunks = (n + chunk - 1) / chunk;
    const int used = (int)std::min<int64_t>(kSlots, nchunks);  // slot streams this call uses
    bool fits = true;  // buffers of earlier calls already hold this call's chunks: no memory query
    for (int k = 0; k < used; ++k)
        fits = fits && s->slots[k].cap >= chunk && (!bin_all || s->slots[k].scratch.cap >= chunk);
    if (!fits) {  // fit kSlots x (records + results + binning scratch) in free device memory
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            int64_t have = 0;
            for (auto& sl : s->slots) have += sl.cap * 20 + sl.scratch.cap * 16;
            const int64_t budget = (int64_t)(free_b * 0.8) + have;
            const int64_t per_q = 20 + (bin_all ? 18 : 0);
            const int64_t fit = budget / (kSlots * per_q);
            if (chunk > fit) chunk = std::max<int64_t>(int64_t(1) << 20, fit);
        }
    }
    const bool binned = (opts & PNDF_BIN_ON) ? true : (bin_all && chunk >= kMinQ * s->P);
    const uint32_t chunk_opts = (opts & PNDF_SUM) | (binned ? PNDF_BIN_ON : PNDF_BIN_OFF);
    const int nuse = (int)std::min<int64_t>(kSlots, (n + chunk - 1) / chunk);  // chunk may have shrunk
    for (int k = 0; k < nuse; ++k) {
        Slot& sl = s->slots[k];
        if (!sl.st) CK(cudaStreamCreateWithFlags(&sl.st, cudaStreamNonBlocking));
        if (sl.cap < chunk) {
            cudaFree(sl.d_rec);
            cudaFree(sl.d_out);
            sl.d_rec = nullptr;
            sl.d_out = nullptr;
            sl.cap = 0;
            CK(cudaMalloc(&sl.d_rec, sizeof(pndf_query) * chunk));
            CK(cudaMalloc(&sl.d_out, sizeof(float) * chunk));
            sl.cap = chunk;
        }
        if (binned) {
            pndf_status r = ensure_scratch(sl.scratch, chunk, sl.st);
            if (r != PNDF_OK) return r;
        }
    }
    int64_t c = 0;
    for (int64_t a = 0; a < n; a += chunk, ++c) {
        Slot& sl = s->slots[c % kSlots];
        const int64_t m = std::min(chunk, n - a);
        CK(cudaMemcpyAsync(sl.d_rec, h_queries + a, sizeof(pndf_query) * m, cudaMemcpyHostToDevice, sl.st));
        pndf_status r = enqueue(s, sl.scratch, sl.d_rec, m, sl.d_out, chunk_opts, sl.st, false);
        if (r != PNDF_OK) return r;
        CK(cudaMemcpyAsync(h_out + a, sl.d_out, sizeof(float) * m, cudaMemcpyDeviceToHost, sl.st));
    }
    for (int k = 0; k < nuse; ++k) CK(cudaStreamSynchronize(s->slots[k].st));
    return read_sticky(s);
}

pndf_status pndf_free(pndf_store s) {
    destroy(s);
    return PNDF_OK;
}

pndf_status pndf_store_stats_get(pndf_store s, pndf_store_stats* out) {
    if (!s || !out) return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    s->stats.lanes_per_query = s->G;
    *out = s->stats;
    return PNDF_OK;
}

pndf_status pndf_store_stats_reset(pndf_store s) {
    if (!s) return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    s->stats.timed_batches = 0;
    s->stats.query_ms = 0.0;
    s->stats.bin_ms = 0.0;
    return PNDF_OK;
}

pndf_status pndf_store_image(pndf_store s, float* PXY, float* Zc, int64_t z0, int64_t z1) {
    if (!s) return PNDF_EINVAL;
    if (Zc && (z0 < 0 || z1 < z0 || z1 > s->P)) return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    if (PXY) CK(cudaMemcpy(PXY, s->PXY, (size_t)s->stats.prefix_bytes, cudaMemcpyDeviceToHost));
    if (Zc && z1 > z0)
        CK(cudaMemcpy(Zc, s->Zc + (size_t)z0 * s->Rp, sizeof(float) * (size_t)(z1 - z0) * s->Rp,
                      cudaMemcpyDeviceToHost));
    return PNDF_OK;
}

pndf_status pndf_bin_permutation(pndf_store s, const pndf_query* d_queries, int64_t n, uint32_t* d_perm,
                                 uint32_t* d_keys) {
    if (!s || n < 0 || (n > 0 && (!d_queries || !d_perm))) return PNDF_EINVAL;
    if (n == 0) return PNDF_OK;
    if (n > (int64_t(1) << 30) || s->nbins == 0 || s->tiled || s->blocked) return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    pndf_status r = ensure_scratch(s->main, n, nullptr);
    if (r != PNDF_OK) return r;
    int launches = 0;
    const uint32_t *perm = nullptr, *keys = nullptr;
    CK(launch_binning(s->qp, d_queries, n, s->P, s->main, s->num_sms, nullptr, &launches, &perm, &keys));
    CK(cudaMemcpyAsync(d_perm, perm, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, nullptr));
    if (d_keys) CK(cudaMemcpyAsync(d_keys, keys, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, nullptr));
    CK(cudaStreamSynchronize(nullptr));
    s->stats.kernel_launches += (uint64_t)launches;
    return PNDF_OK;
}

pndf_status pndf_rows_touched(pndf_store s, const pndf_query* d_queries, int64_t n, int64_t* d_rows_out) {
    if (!s || n < 0 || !d_rows_out || (n > 0 && !d_queries)) return PNDF_EINVAL;
    if (s->tiled || s->blocked) return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard g(s->device);
    uint32_t* bitmap = nullptr;
    const int64_t words = (s->P + 31) / 32;
    CK(cudaMalloc(&bitmap, sizeof(uint32_t) * words));
    cudaError_t e = cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * words, nullptr);
    if (e == cudaSuccess) e = launch_rows_touched(s->qp, d_queries, n, s->P, bitmap, d_rows_out, s->num_sms, nullptr);
    if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
    cudaFree(bitmap);
    CK(e);
    s->stats.kernel_launches += n > 0 ? 2 : 1;
    return PNDF_OK;
}

pndf_status pndf_set_lanes(pndf_store s, int32_t lanes) {
    if (!s) return PNDF_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    if (lanes == 0) {
        s->G = s->G0;
        s->NV = s->NV0;
        return PNDF_OK;
    }
    if (lanes < 1 || lanes > 32 || (lanes & (lanes - 1)) || s->Rp % (4 * lanes)) return PNDF_EINVAL;
    const int nv = s->Rp / (4 * lanes);
    if (!lanes_supported(lanes, nv)) return PNDF_EINVAL;
    s->G = lanes;
    s->NV = nv;
    return PNDF_OK;
}

}  // extern "C"
