/*
 * synth.c -- seeded synthetic INPUT generators for the NDF range-query path.
 *
 * This module is shared by the oracle (oracle/) and the CUDA product path
 * (paper_2109_14807_b200/).  It holds none of the query arithmetic (Eq. 6,
 * trilinear interpolation, prefix differencing): it only produces the inputs
 * of the query -- normal maps, the footprint NDF tensor or its exact-rank CP
 * factors, and query records.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 *   - normal map n(u)                             P:209-214 (Eq. 2)
 *   - footprint pyramid: stride s*2^l,
 *     sigma_p = 1.5 s/sqrt(12)                    P:279 (Sec. 4.1 "Practical choices")
 *   - footprint NDF = footprint-weighted normal
 *     histogram (Eq. 2 with sigma_r -> 0)
 *   - CP form D = sum_r C_r X_r (x) Y_r (x) Z_r   P:298-303 (Eq. 5)
 *
 * Determinism: every generator is a pure function of (config, seed); the
 * counter-based RNG (splitmix64 of seed, stream, index) makes any shard of
 * the query stream reproducible independently of how it is split.
 * Footprint weights are integers (Gaussian quantised to 16 bits) and all
 * footprint sums are accumulated in uint64, so the tensor / Z factors are
 * bit-identical regardless of summation order or thread count (and equal to
 * the CUDA twin in synth_cuda.cu).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ RNG -- */
static inline uint64_t sm_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* counter-based: value #idx of stream `stream` under `seed` */
static inline uint64_t rng64(uint64_t seed, uint32_t stream, uint64_t idx) {
    uint64_t key = sm_mix(sm_mix(seed) ^ (0xD6E8FEB86659FD93ULL * (uint64_t)(stream + 1)));
    return sm_mix(key + idx * 0x9E3779B97F4A7C15ULL);
}
static inline double rng_unit(uint64_t seed, uint32_t stream, uint64_t idx) {
    return (double)(rng64(seed, stream, idx) >> 11) * 0x1.0p-53; /* [0,1) */
}
static inline double rng_normal(uint64_t seed, uint32_t s0, uint32_t s1, uint64_t idx) {
    double u1 = rng_unit(seed, s0, idx), u2 = rng_unit(seed, s1, idx);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * M_PI * u2);
}

EXPORT uint64_t synth_rng64(uint64_t seed, uint32_t stream, uint64_t idx) { return rng64(seed, stream, idx); }

/* Beckmann-distributed microfacet normal about +z, roughness alpha:
 * tan^2(theta) = -alpha^2 ln(1-xi1), phi = 2 pi xi2.  Returns projected (nx, ny). */
static inline void beckmann_nxy(double alpha, double xi1, double xi2, float* nx, float* ny) {
    double t2 = -alpha * alpha * log(1.0 - xi1);
    double ct = 1.0 / sqrt(1.0 + t2), st = sqrt(t2) * ct;
    double ph = 2.0 * M_PI * xi2;
    *nx = (float)(st * cos(ph));
    *ny = (float)(st * sin(ph));
}

/* --------------------------------------------------------------- maps -- */
/* Output: nxy[(v*N + u)*2 + {0,1}] = projected tangent-space normal (n_x, n_y);
 * n_z = sqrt(1 - n_x^2 - n_y^2) > 0 is implied. All maps are periodic. */

/* Config 1: per-texel i.i.d. Gaussian slopes, n = normalize(-sx, -sy, 1). */
EXPORT void synth_map_gaussian_slopes(int32_t N, uint64_t seed, double sigma, float* nxy) {
    int64_t NN = (int64_t)N * N;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < NN; ++t) {
        double sx = sigma * rng_normal(seed, 0, 1, (uint64_t)t);
        double sy = sigma * rng_normal(seed, 2, 3, (uint64_t)t);
        double inv = 1.0 / sqrt(sx * sx + sy * sy + 1.0);
        nxy[2 * t] = (float)(-sx * inv);
        nxy[2 * t + 1] = (float)(-sy * inv);
    }
}

/* Voronoi metallic flakes on a torus: one jittered seed per cell of a
 * nc x nc grid (cell side N/nc ~= spacing), each flake one Beckmann normal.
 * flake_id (optional) receives the owning seed index per texel. */
EXPORT void synth_map_flakes(int32_t N, uint64_t seed, double spacing, double alpha, float* nxy,
                             int32_t* flake_id) {
    int nc = (int)floor((double)N / spacing + 0.5);
    if (nc < 1) nc = 1;
    double cs = (double)N / nc;
    int64_t NF = (int64_t)nc * nc;
    double* sx = (double*)malloc(sizeof(double) * NF);
    double* sy = (double*)malloc(sizeof(double) * NF);
    float* fnx = (float*)malloc(sizeof(float) * NF);
    float* fny = (float*)malloc(sizeof(float) * NF);
    for (int64_t f = 0; f < NF; ++f) {
        int ci = (int)(f % nc), cj = (int)(f / nc);
        sx[f] = (ci + rng_unit(seed, 10, (uint64_t)f)) * cs;
        sy[f] = (cj + rng_unit(seed, 11, (uint64_t)f)) * cs;
        beckmann_nxy(alpha, rng_unit(seed, 12, (uint64_t)f), rng_unit(seed, 13, (uint64_t)f), &fnx[f], &fny[f]);
    }
    int64_t NN = (int64_t)N * N;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < NN; ++t) {
        double px = (double)(t % N) + 0.5, py = (double)(t / N) + 0.5;
        int ci = (int)floor(px / cs), cj = (int)floor(py / cs);
        double best = 1e300;
        int64_t bf = 0;
        for (int dj = -2; dj <= 2; ++dj)
            for (int di = -2; di <= 2; ++di) {
                int ii = ((ci + di) % nc + nc) % nc, jj = ((cj + dj) % nc + nc) % nc;
                int64_t f = (int64_t)jj * nc + ii;
                double dx = fabs(px - sx[f]), dy = fabs(py - sy[f]);
                if (dx > 0.5 * N) dx = N - dx;
                if (dy > 0.5 * N) dy = N - dy;
                double d2 = dx * dx + dy * dy;
                if (d2 < best || (d2 == best && f < bf)) { best = d2; bf = f; }
            }
        nxy[2 * t] = fnx[bf];
        nxy[2 * t + 1] = fny[bf];
        if (flake_id) flake_id[t] = (int32_t)bf;
    }
    free(sx); free(sy); free(fnx); free(fny);
}

/* Scratched metal: per-texel Beckmann(alpha_base) base, then n_scr straight
 * scratch segments (periodic wrap), width `width` texels, uniform direction,
 * length U[0.1N, 0.5N]; the cross-section normal is tilted by +theta on one
 * side of the centre line and -theta on the other, theta ~ U[0, max_tilt]. */
EXPORT void synth_map_scratches(int32_t N, uint64_t seed, int32_t n_scr, double width, double max_tilt_deg,
                                double alpha_base, float* nxy) {
    int64_t NN = (int64_t)N * N;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < NN; ++t)
        beckmann_nxy(alpha_base, rng_unit(seed, 20, (uint64_t)t), rng_unit(seed, 21, (uint64_t)t), &nxy[2 * t],
                     &nxy[2 * t + 1]);
    double hw = 0.5 * width;
    for (int k = 0; k < n_scr; ++k) { /* sequential: later scratches overwrite earlier ones */
        double x0 = N * rng_unit(seed, 22, (uint64_t)k), y0 = N * rng_unit(seed, 23, (uint64_t)k);
        double phi = M_PI * rng_unit(seed, 24, (uint64_t)k);
        double len = N * (0.1 + 0.4 * rng_unit(seed, 25, (uint64_t)k));
        double th = max_tilt_deg * M_PI / 180.0 * rng_unit(seed, 26, (uint64_t)k);
        double dx = cos(phi), dy = sin(phi), px = -dy, py = dx; /* direction, in-plane perpendicular */
        /* rasterise: walk the segment's bounding strip texel by texel */
        int steps = (int)ceil(len * 2.0);
        for (int st = 0; st <= steps; ++st) {
            double s = len * st / (double)steps;
            for (int w = -2; w <= 2; ++w) {
                double cx = x0 + s * dx + 0.5 * w * hw * px, cy = y0 + s * dy + 0.5 * w * hw * py;
                int64_t ui = (int64_t)floor(cx), vi = (int64_t)floor(cy);
                /* signed perpendicular distance of the texel centre to the centre line */
                double ex = (double)ui + 0.5 - x0, ey = (double)vi + 0.5 - y0;
                double along = ex * dx + ey * dy, d = ex * px + ey * py;
                if (along < 0.0 || along > len || fabs(d) > hw) continue;
                int64_t uu = ((ui % N) + N) % N, vv = ((vi % N) + N) % N;
                double sg = (d >= 0.0) ? 1.0 : -1.0;
                nxy[2 * (vv * N + uu)] = (float)(sg * sin(th) * px);
                nxy[2 * (vv * N + uu) + 1] = (float)(sg * sin(th) * py);
            }
        }
    }
}

/* ------------------------------------------------------- angular bins -- */
/* Projected normal n in [-1,1] -> bin min(floor((n+1) A/2), A-1)
 * (half-open bins, n = 1 goes to the last bin).  id = by*A + bx. */
static inline int bin1(float n, int A) {
    int b = (int)floor(((double)n + 1.0) * 0.5 * A);
    if (b < 0) b = 0;
    if (b > A - 1) b = A - 1;
    return b;
}
EXPORT void synth_bin_map(int32_t N, const float* nxy, int32_t A, uint16_t* bins) {
    int64_t NN = (int64_t)N * N;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < NN; ++t)
        bins[t] = (uint16_t)(bin1(nxy[2 * t + 1], A) * A + bin1(nxy[2 * t], A));
}

/* Atoms = the R most populated bins (ties -> lower bin id; unpopulated bins
 * fill up in increasing id order when fewer than R bins are populated).
 * atom_map[t] = nearest atom to the texel's bin (Euclidean in bin
 * coordinates, ties -> lower atom index). Returns #populated bins. */
EXPORT int32_t synth_select_atoms(int32_t N, const uint16_t* bins, int32_t A, int32_t R, int32_t* atom_bins,
                                  uint16_t* atom_map) {
    int64_t NB = (int64_t)A * A, NN = (int64_t)N * N;
    int64_t* cnt = (int64_t*)calloc(NB, sizeof(int64_t));
    for (int64_t t = 0; t < NN; ++t) cnt[bins[t]]++;
    int32_t npop = 0;
    for (int64_t b = 0; b < NB; ++b) npop += cnt[b] > 0;
    unsigned char* taken = (unsigned char*)calloc(NB, 1);
    for (int r = 0; r < R; ++r) {
        int64_t best = -1;
        for (int64_t b = 0; b < NB; ++b)
            if (!taken[b] && (best < 0 || cnt[b] > cnt[best])) best = b;
        atom_bins[r] = (int32_t)best;
        taken[best] = 1;
    }
    int32_t* lut = (int32_t*)malloc(sizeof(int32_t) * NB);
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < NB; ++b) {
        if (!cnt[b]) { lut[b] = -1; continue; }
        int bx = (int)(b % A), by = (int)(b / A);
        int64_t bd = INT64_MAX;
        int ba = 0;
        for (int r = 0; r < R; ++r) {
            int64_t ax = atom_bins[r] % A, ay = atom_bins[r] / A;
            int64_t d2 = (ax - bx) * (ax - bx) + (ay - by) * (ay - by);
            if (d2 < bd) { bd = d2; ba = r; }
        }
        lut[b] = ba;
    }
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < NN; ++t) atom_map[t] = (uint16_t)lut[bins[t]];
    free(lut); free(taken); free(cnt);
    return npop;
}

/* ------------------------------------------------- footprint weights -- */
/* Level with stride s: centre i at (i+1/2)s, texel u spans [u,u+1)
 * with centre u+1/2.  For texel u = i*s + q the distance to the centre is
 * d(q) = q + (1-s)/2.  Gaussian sigma = 1.5 s / sqrt(12), truncated at
 * |d| <= 4 sigma; weight = round(65536 exp(-d^2 / (2 sigma^2))).
 * Windows longer than the (periodic) map are folded modulo N.
 * Returns the folded length Wf <= N; *qmin = first offset; w[0..Wf). */
EXPORT int32_t synth_footprint_table(int32_t s, int32_t N, int32_t* qmin_out, uint32_t* w /* >= N entries */) {
    double sigma = 1.5 * (double)s / sqrt(12.0);
    double c = 0.5 * (1.0 - (double)s);
    int64_t qmin = (int64_t)ceil(-4.0 * sigma - c), qmax = (int64_t)floor(4.0 * sigma - c);
    int64_t W = qmax - qmin + 1;
    int32_t Wf = (int32_t)(W < N ? W : N);
    for (int32_t p = 0; p < Wf; ++p) w[p] = 0;
    for (int64_t q = qmin; q <= qmax; ++q) {
        double d = (double)q + c;
        uint32_t wi = (uint32_t)llround(65536.0 * exp(-d * d / (2.0 * sigma * sigma)));
        w[(q - qmin) % Wf] += wi;
    }
    *qmin_out = (int32_t)qmin;
    return Wf;
}

static int64_t level_rows(int32_t N, int32_t s0, int32_t l) {
    int64_t n = N / ((int64_t)s0 << l);
    return n * n;
}
EXPORT int64_t synth_num_rows(int32_t N, int32_t s0, int32_t L) {
    int64_t P = 0;
    for (int l = 0; l < L; ++l) P += level_rows(N, s0, l);
    return P;
}

/* Visit footprint (level stride s, centre (i,j)) with integer weights:
 * acc[key[v*N+u]] += wx[p] * wy[q]. */
static void footprint_accumulate(int32_t N, const uint16_t* key, int32_t s, int32_t qmin, int32_t Wf,
                                 const uint32_t* w, int64_t i, int64_t j, uint64_t* acc) {
    int64_t bu = (((i * s + qmin) % N) + N) % N, bv = (((j * s + qmin) % N) + N) % N;
    for (int32_t q = 0; q < Wf; ++q) {
        int64_t v = bv + q;
        if (v >= N) v -= N;
        const uint16_t* row = key + v * N;
        uint64_t wy = w[q];
        int64_t u = bu;
        for (int32_t p = 0; p < Wf; ++p) {
            acc[row[u]] += wy * (uint64_t)w[p];
            if (++u == N) u = 0;
        }
    }
}

/* Exact-rank positional factors: Z[z][k] = footprint-weighted fraction of
 * texels whose snapped normal is atom k (z = level offset + j*n_l + i).
 * With X_k, Y_k the atom's 1-D angular profiles this gives D = sum_k X_k Y_k Z_k
 * exactly (Eq. 5 with R = #atoms).  rows [z0, z1) only (z1 <= P). */
EXPORT void synth_build_z_exact(int32_t N, const uint16_t* atom_map, int32_t R, int32_t s0, int32_t L, int64_t z0,
                                int64_t z1, float* Z /* [(z1-z0)][R] */) {
    uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * N);
    int64_t off = 0;
    for (int32_t l = 0; l < L; ++l) {
        int32_t s = s0 << l, n = N / s;
        int64_t rows = (int64_t)n * n;
        int64_t a = off > z0 ? off : z0, b = (off + rows) < z1 ? (off + rows) : z1;
        if (a < b) {
            int32_t qmin;
            int32_t Wf = synth_footprint_table(s, N, &qmin, w);
            uint64_t sw = 0;
            for (int p = 0; p < Wf; ++p) sw += w[p];
            double tot = (double)sw * (double)sw;
#pragma omp parallel
            {
                uint64_t* acc = (uint64_t*)malloc(sizeof(uint64_t) * R);
#pragma omp for schedule(dynamic, 16)
                for (int64_t z = a; z < b; ++z) {
                    int64_t c = z - off, i = c % n, j = c / n;
                    memset(acc, 0, sizeof(uint64_t) * R);
                    footprint_accumulate(N, atom_map, s, qmin, Wf, w, i, j, acc);
                    float* out = Z + (z - z0) * R;
                    for (int k = 0; k < R; ++k) out[k] = (float)((double)acc[k] / tot);
                }
                free(acc);
            }
        }
        off += rows;
    }
    free(w);
}

/* Same values as synth_build_z_exact for an arbitrary list of rows (the rows
 * a sampled parity / baseline set touches); out[k][R] for rows[k]. */
EXPORT void synth_build_z_rows(int32_t N, const uint16_t* atom_map, int32_t R, int32_t s0, int32_t L,
                               const int64_t* rows, int64_t nrows, float* out) {
    int64_t offs[64];
    int64_t off = 0;
    for (int32_t l = 0; l < L; ++l) { offs[l] = off; off += level_rows(N, s0, l); }
    offs[L] = off;
    uint32_t* tabs = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)N * L);
    int32_t qmins[64], wfs[64];
    double tots[64];
    for (int32_t l = 0; l < L; ++l) {
        wfs[l] = synth_footprint_table(s0 << l, N, &qmins[l], tabs + (size_t)l * N);
        uint64_t sw = 0;
        for (int p = 0; p < wfs[l]; ++p) sw += tabs[(size_t)l * N + p];
        tots[l] = (double)sw * (double)sw;
    }
#pragma omp parallel
    {
        uint64_t* acc = (uint64_t*)malloc(sizeof(uint64_t) * R);
#pragma omp for schedule(dynamic, 1)
        for (int64_t k = 0; k < nrows; ++k) {
            int64_t z = rows[k];
            int32_t l = 0;
            while (l + 1 < L && z >= offs[l + 1]) ++l;
            int32_t s = s0 << l, n = N / s;
            int64_t c = z - offs[l];
            memset(acc, 0, sizeof(uint64_t) * R);
            footprint_accumulate(N, atom_map, s, qmins[l], wfs[l], tabs + (size_t)l * N, c % n, c / n, acc);
            for (int r = 0; r < R; ++r) out[k * R + r] = (float)((double)acc[r] / tots[l]);
        }
        free(acc);
    }
    free(tabs);
}

/* Full footprint NDF tensor (pure normal histogram, Eq. 2 with sigma_r -> 0,
 * bin masses summing to 1 per footprint): D[z][x][y], x = n_x bin, y = n_y bin. */
EXPORT void synth_hist_tensor(int32_t N, const uint16_t* bins, int32_t A, int32_t s0, int32_t L, double* D) {
    uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * N);
    int64_t NB = (int64_t)A * A, off = 0;
    for (int32_t l = 0; l < L; ++l) {
        int32_t s = s0 << l, n = N / s;
        int32_t qmin;
        int32_t Wf = synth_footprint_table(s, N, &qmin, w);
        uint64_t sw = 0;
        for (int p = 0; p < Wf; ++p) sw += w[p];
        double tot = (double)sw * (double)sw;
#pragma omp parallel
        {
            uint64_t* acc = (uint64_t*)malloc(sizeof(uint64_t) * NB);
#pragma omp for schedule(dynamic, 4)
            for (int64_t c = 0; c < (int64_t)n * n; ++c) {
                memset(acc, 0, sizeof(uint64_t) * NB);
                footprint_accumulate(N, bins, s, qmin, Wf, w, c % n, c / n, acc);
                double* out = D + (off + c) * NB;
                for (int64_t b = 0; b < NB; ++b) {
                    int64_t bx = b % A, by = b / A;
                    out[bx * A + by] = (double)acc[b] / tot;
                }
            }
            free(acc);
        }
        off += (int64_t)n * n;
    }
    free(w);
}

/* 1-D angular profile of an atom at bin c: the bin-integrated Gaussian of
 * std sigma_b bins centred at c+1/2 (intrinsic roughness G_r of Eq. 2,
 * separable, so each atom stays rank-1), truncated at +-ceil(4 sigma_b) bins
 * and renormalised to sum 1 over the grid.  sigma_b = 0 gives a one-hot. */
EXPORT void synth_atom_profiles(int32_t A, int32_t R, const int32_t* atom_bins, double sigma_b, float* X /*[A][R]*/,
                                float* Y /*[A][R]*/) {
    double* col = (double*)malloc(sizeof(double) * A);
    for (int axis = 0; axis < 2; ++axis) {
        float* F = axis ? Y : X;
        for (int r = 0; r < R; ++r) {
            int c = axis ? atom_bins[r] / A : atom_bins[r] % A;
            double sum = 0.0;
            for (int x = 0; x < A; ++x) col[x] = 0.0;
            if (sigma_b <= 0.0) {
                col[c] = 1.0;
                sum = 1.0;
            } else {
                int T = (int)ceil(4.0 * sigma_b);
                for (int x = c - T; x <= c + T; ++x) {
                    if (x < 0 || x >= A) continue;
                    double lo = ((double)x - (c + 0.5)) / sigma_b, hi = ((double)x + 1.0 - (c + 0.5)) / sigma_b;
                    col[x] = 0.5 * (erfc(-hi / M_SQRT2) - erfc(-lo / M_SQRT2));
                    sum += col[x];
                }
            }
            for (int x = 0; x < A; ++x) F[(int64_t)x * R + r] = (float)(col[x] / sum);
        }
    }
    free(col);
}

/* ------------------------------------------------------------ queries -- */
typedef struct {
    int32_t N, A;
    int32_t size_mix;        /* 0: log2 S ~ U[lg_lo, lg_hi]; 1: 50/50 of [lg_lo,lg_hi] and [lg_lo2,lg_hi2] */
    int32_t side_mode;       /* 0: sides ~ U{side_lo..side_hi}; 1: half-width w ~ U[w_lo,w_hi], side = max(1, floor(2w+1/2)) */
    int32_t side_lo, side_hi;
    int32_t centre_mode;     /* 0: uniform placement; 1: centred w.p. p_texel on the bin of the texel under the footprint centre (+-jitter);
                                2: centred on the bin of a Beckmann(alpha_h) half vector */
    int32_t jitter;
    double lg_lo, lg_hi, lg_lo2, lg_hi2;
    double w_lo, w_hi;
    double p_texel, alpha_h;
} synth_qdist;

/* 16-byte record: float u, v, size; uint32 rect = x1 | x2<<8 | y1<<16 | y2<<24 (inclusive). */
typedef struct { float u, v, size; uint32_t rect; } synth_qrec;

static inline int uniform_int(uint64_t seed, uint32_t stream, uint64_t idx, int lo, int hi) {
    int v = lo + (int)floor(rng_unit(seed, stream, idx) * (double)(hi - lo + 1));
    return v > hi ? hi : v;
}
static inline void place(int c, int side, int A, int* x1, int* x2) {
    int a = c - (side - 1) / 2;
    if (a > A - side) a = A - side;
    if (a < 0) a = 0;
    *x1 = a;
    *x2 = a + side - 1;
}

EXPORT void synth_gen_queries(const synth_qdist* q, uint64_t seed, int64_t i0, int64_t i1, const uint16_t* bins,
                              synth_qrec* out) {
    const int N = q->N, A = q->A;
    const float fN = (float)N, below = nextafterf(fN, 0.0f);
#pragma omp parallel for schedule(static)
    for (int64_t i = i0; i < i1; ++i) {
        uint64_t g = (uint64_t)i;
        synth_qrec r;
        float u = (float)(N * rng_unit(seed, 0, g)), v = (float)(N * rng_unit(seed, 1, g));
        r.u = u < fN ? u : below;
        r.v = v < fN ? v : below;
        double lo = q->lg_lo, hi = q->lg_hi;
        if (q->size_mix && rng_unit(seed, 2, g) >= 0.5) { lo = q->lg_lo2; hi = q->lg_hi2; }
        r.size = (float)exp2(lo + (hi - lo) * rng_unit(seed, 3, g));
        int sx, sy;
        if (q->side_mode == 0) {
            sx = uniform_int(seed, 4, g, q->side_lo, q->side_hi);
            sy = uniform_int(seed, 5, g, q->side_lo, q->side_hi);
        } else {
            double wx = q->w_lo + (q->w_hi - q->w_lo) * rng_unit(seed, 4, g);
            double wy = q->w_lo + (q->w_hi - q->w_lo) * rng_unit(seed, 5, g);
            sx = (int)floor(2.0 * wx + 0.5); sy = (int)floor(2.0 * wy + 0.5);
            if (sx < 1) sx = 1;
            if (sy < 1) sy = 1;
        }
        if (sx > A) sx = A;
        if (sy > A) sy = A;
        int x1, x2, y1, y2;
        int centred = 0, cx = 0, cy = 0;
        if (q->centre_mode == 1 && bins && rng_unit(seed, 6, g) < q->p_texel) {
            /* the normal of the texel under the footprint centre: the footprint's NDF holds it with
               positive weight, so the rectangle sits on the footprint's own NDF support (glint queries) */
            const int64_t t = (int64_t)r.v * N + (int64_t)r.u;
            cx = bins[t] % A; cy = bins[t] / A;
            if (q->jitter) {
                cx += uniform_int(seed, 9, g, -q->jitter, q->jitter);
                cy += uniform_int(seed, 10, g, -q->jitter, q->jitter);
            }
            centred = 1;
        } else if (q->centre_mode == 2) {
            float hx, hy;
            beckmann_nxy(q->alpha_h, rng_unit(seed, 11, g), rng_unit(seed, 12, g), &hx, &hy);
            cx = bin1(hx, A); cy = bin1(hy, A);
            centred = 1;
        }
        if (centred) {
            place(cx, sx, A, &x1, &x2);
            place(cy, sy, A, &y1, &y2);
        } else {
            x1 = uniform_int(seed, 7, g, 0, A - sx); x2 = x1 + sx - 1;
            y1 = uniform_int(seed, 8, g, 0, A - sy); y2 = y1 + sy - 1;
        }
        r.rect = (uint32_t)x1 | ((uint32_t)x2 << 8) | ((uint32_t)y1 << 16) | ((uint32_t)y2 << 24);
        out[i - i0] = r;
    }
}

/* Spherical-Gaussian light samples for environment prefiltering (Sec. 5.4):
 * footprint (u, v, S) as the config's query stream, the half vector of the
 * sampled lobe direction ~ Beckmann(alpha_h) projected, bandwidth lambda
 * log-uniform in [lam_lo, lam_hi], amplitude U[amp_lo, amp_hi]. */
typedef struct { float u, v, size, hx, hy, lambda, amplitude, pad; } synth_sgrec;

EXPORT void synth_gen_sg_lights(const synth_qdist* q, uint64_t seed, int64_t i0, int64_t i1, double alpha_h,
                                double lam_lo, double lam_hi, double amp_lo, double amp_hi, synth_sgrec* out) {
    const int N = q->N;
    const float fN = (float)N, below = nextafterf(fN, 0.0f);
#pragma omp parallel for schedule(static)
    for (int64_t i = i0; i < i1; ++i) {
        uint64_t g = (uint64_t)i;
        synth_sgrec r;
        float u = (float)(N * rng_unit(seed, 0, g)), v = (float)(N * rng_unit(seed, 1, g));
        r.u = u < fN ? u : below;
        r.v = v < fN ? v : below;
        r.size = (float)exp2(q->lg_lo + (q->lg_hi - q->lg_lo) * rng_unit(seed, 3, g));
        beckmann_nxy(alpha_h, rng_unit(seed, 30, g), rng_unit(seed, 31, g), &r.hx, &r.hy);
        r.lambda = (float)exp(log(lam_lo) + (log(lam_hi) - log(lam_lo)) * rng_unit(seed, 32, g));
        r.amplitude = (float)(amp_lo + (amp_hi - amp_lo) * rng_unit(seed, 33, g));
        r.pad = 0.0f;
        out[i - i0] = r;
    }
}

/* ------------------------------------------------------------ Wang tiles --
 * 16 edge-coloured tiles (2 colours for horizontal edges, 2 for vertical edges,
 * tile id = N | E<<1 | S<<2 | W<<3), each T x T texels of Voronoi flakes
 * ("16 Wang tiles ... tile size as 512 x 512").  Seeds live on a
 * jittered grid of cells of side ~spacing; a grid cell in the band along an
 * edge draws its seed from (edge orientation, edge colour, position along the
 * edge), interior cells from the tile id, so tiles sharing an edge colour have
 * the same seeds along it (near-seamless; corners are not constrained, as in
 * the paper).  nxy: [16][T][T][2]. */
EXPORT void synth_wang_tiles(int32_t T, uint64_t seed, double spacing, double alpha, float* nxy) {
    int nc = (int)floor((double)T / spacing + 0.5);
    if (nc < 3) nc = 3;
    const double cs = (double)T / nc;
    for (int tile = 0; tile < 16; ++tile) {
        const int cn = tile & 1, ce = (tile >> 1) & 1, csouth = (tile >> 2) & 1, cw = (tile >> 3) & 1;
        const int64_t NF = (int64_t)nc * nc;
        double* sx = (double*)malloc(sizeof(double) * NF);
        double* sy = (double*)malloc(sizeof(double) * NF);
        float* fnx = (float*)malloc(sizeof(float) * NF);
        float* fny = (float*)malloc(sizeof(float) * NF);
        for (int64_t f = 0; f < NF; ++f) {
            const int ci = (int)(f % nc), cj = (int)(f / nc);
            uint64_t key;
            if (cj == 0 && ci > 0 && ci < nc - 1) key = 0x1000 + (uint64_t)cn * 0x100 + ci;                /* N */
            else if (cj == nc - 1 && ci > 0 && ci < nc - 1) key = 0x1000 + (uint64_t)csouth * 0x100 + ci;  /* S */
            else if (ci == 0 && cj > 0 && cj < nc - 1) key = 0x2000 + (uint64_t)cw * 0x100 + cj;           /* W */
            else if (ci == nc - 1 && cj > 0 && cj < nc - 1) key = 0x2000 + (uint64_t)ce * 0x100 + cj;      /* E */
            else if ((ci == 0 || ci == nc - 1) && (cj == 0 || cj == nc - 1)) key = 0x3000;                 /* corner */
            else key = 0x4000 + (uint64_t)tile * 0x10000 + (uint64_t)f;                                    /* interior */
            /* band seeds sit on the edge-normal axis symmetric for the two tiles sharing the edge */
            double jx = rng_unit(seed, 40, key), jy = rng_unit(seed, 41, key);
            if (cj == 0) jy = 0.5 * jy;               /* keep N-band seeds near the edge */
            if (cj == nc - 1) jy = 1.0 - 0.5 * jy;
            if (ci == 0) jx = 0.5 * jx;
            if (ci == nc - 1) jx = 1.0 - 0.5 * jx;
            sx[f] = (ci + jx) * cs;
            sy[f] = (cj + jy) * cs;
            beckmann_nxy(alpha, rng_unit(seed, 42, key), rng_unit(seed, 43, key), &fnx[f], &fny[f]);
        }
        float* out = nxy + (int64_t)tile * T * T * 2;
#pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < (int64_t)T * T; ++t) {
            const double px = (double)(t % T) + 0.5, py = (double)(t / T) + 0.5;
            const int ci = (int)floor(px / cs), cj = (int)floor(py / cs);
            double best = 1e300;
            int64_t bf = 0;
            for (int dj = -2; dj <= 2; ++dj)
                for (int di = -2; di <= 2; ++di) {
                    const int ii = ci + di, jj = cj + dj;
                    if (ii < 0 || jj < 0 || ii >= nc || jj >= nc) continue;
                    const int64_t f = (int64_t)jj * nc + ii;
                    const double dx = px - sx[f], dy = py - sy[f], d2 = dx * dx + dy * dy;
                    if (d2 < best || (d2 == best && f < bf)) { best = d2; bf = f; }
                }
            out[2 * t] = fnx[bf];
            out[2 * t + 1] = fny[bf];
        }
        free(sx); free(sy); free(fnx); free(fny);
    }
}

/* Extended per-tile positional factors for Wang-tile stores (P:438-442:
 * "the sampled centers could locate outside the Wang tiles").  Level l of a tile
 * has n = T/(s0 2^l) cells plus `margin` cells on each side; row
 * z = off_l + (j + m) (n + 2m) + (i + m) for local cells i, j in [-m, n + m).
 * Z[t][z][k] = sum over the tile's OWN texels u of G_p(u - c) [atom(u) = k] /
 * W_total, with W_total the footprint's full weight (sum w)^2: a footprint that
 * straddles tiles is the SUM of the tiles' partial NDFs (linearity of Eq. 2).
 * atom_map: [16][T][T]; Z: [16][P_ext][R]. */
EXPORT int64_t synth_wang_rows(int32_t T, int32_t s0, int32_t L, int32_t margin) {
    int64_t P = 0;
    for (int l = 0; l < L; ++l) {
        const int64_t n = T / ((int64_t)s0 << l) + 2 * margin;
        P += n * n;
    }
    return P;
}

EXPORT void synth_wang_z(int32_t T, const uint16_t* atom_map, int32_t R, int32_t s0, int32_t L, int32_t margin,
                         float* Z) {
    const int64_t Pext = synth_wang_rows(T, s0, L, margin);
    for (int tile = 0; tile < 16; ++tile) {
        const uint16_t* am = atom_map + (int64_t)tile * T * T;
        int64_t off = 0;
        for (int32_t l = 0; l < L; ++l) {
            const int32_t s = s0 << l, n = T / s, ne = n + 2 * margin;
            /* unfolded window table over a virtual line much longer than the tile */
            const double sigma = 1.5 * (double)s / sqrt(12.0), c = 0.5 * (1.0 - (double)s);
            const int64_t qmin = (int64_t)ceil(-4.0 * sigma - c), qmax = (int64_t)floor(4.0 * sigma - c);
            const int64_t W = qmax - qmin + 1;
            uint32_t* wt = (uint32_t*)malloc(sizeof(uint32_t) * W);
            uint64_t sw = 0;
            for (int64_t q = qmin; q <= qmax; ++q) {
                const double d = (double)q + c;
                wt[q - qmin] = (uint32_t)llround(65536.0 * exp(-d * d / (2.0 * sigma * sigma)));
                sw += wt[q - qmin];
            }
            const double tot = (double)sw * (double)sw;
#pragma omp parallel
            {
                uint64_t* acc = (uint64_t*)malloc(sizeof(uint64_t) * R);
#pragma omp for schedule(dynamic, 16)
                for (int64_t cidx = 0; cidx < (int64_t)ne * ne; ++cidx) {
                    const int64_t i = cidx % ne - margin, j = cidx / ne - margin;
                    memset(acc, 0, sizeof(uint64_t) * R);
                    /* texels x = i*s + q for q in [qmin, qmax], clipped to the tile */
                    const int64_t qy0 = qmin > -j * s ? qmin : -j * s, qy1 = qmax < T - 1 - j * s ? qmax : T - 1 - j * s;
                    const int64_t qx0 = qmin > -i * s ? qmin : -i * s, qx1 = qmax < T - 1 - i * s ? qmax : T - 1 - i * s;
                    for (int64_t qy = qy0; qy <= qy1; ++qy) {
                        const uint64_t wy = wt[qy - qmin];
                        const uint16_t* row = am + (j * s + qy) * T + i * s;
                        for (int64_t qx = qx0; qx <= qx1; ++qx) acc[row[qx]] += wy * (uint64_t)wt[qx - qmin];
                    }
                    float* out = Z + ((int64_t)tile * Pext + off + cidx) * R;
                    for (int k = 0; k < R; ++k) out[k] = (float)((double)acc[k] / tot);
                }
                free(acc);
            }
            free(wt);
            off += (int64_t)ne * ne;
        }
    }
}

EXPORT int32_t synth_max_threads(void) { return omp_get_max_threads(); }
