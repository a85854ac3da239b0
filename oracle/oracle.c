/*
 * oracle.c -- plain fp64 CPU oracle of the batched NDF range query.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code with the CUDA path (paper_2109_14807_b200/) and includes none
 * of its headers: the 16-byte query record and the descriptor are restated
 * here from the paper's statement of the query.
 *
 * What it computes (P:n = line n of /root/reference/PAPER.md), per record
 * (u, v, S, [x1,x2] x [y1,y2]):
 *   1. footprint level (Sec. 4.1, "trilinear interpolation between different
 *      samples in the same level and between different levels", P:276, P:327;
 *      clamp above the top level):
 *        l* = clamp(log2(S/s0), 0, L-1), l0 = min(floor(l*), L-2), t = l* - l0
 *   2. the 4 spatial neighbours on each of levels l0 (weight 1-t), l0+1
 *      (weight t): centres at ((i+1/2)s_l, (j+1/2)s_l) on a grid of stride
 *      s_l = s0 2^l, f = u/s_l - 1/2, i0 = floor(f), a = f - i0,
 *      bilinear weights (1-a)(1-b), a(1-b), (1-a)b, ab; indices wrap modulo
 *      n_l for tileable maps, clamp to [0, n_l-1] otherwise;
 *   3. per neighbour z_k, Eq. 6 as a SUM over the rectangle:
 *        D_k = sum_r C_r (sum_{x=x1..x2} X_r(x)) (sum_{y=y1..y2} Y_r(y)) Z_r(z_k)
 *      -- the 1-D segment sums are written out directly (the plain definition
 *      of X-bar times the segment length M, P:345 and Appendix), not
 *      through a prefix table;
 *   4. SUM = sum_k w_k D_k ("Eqn. 5 will simply be called multiple times",
 *      P:327); MEAN = SUM / ((x2-x1+1)(y2-y1+1)) (Eq. 6 is an average).
 * Everything is accumulated in double from the fp32 factor inputs.
 *
 * Invalid records (non-finite or |u|,|v| > 2^22, S <= 0, x1 > x2, x2 >= A,
 * y1 > y2, y2 >= A) produce NaN (SPEC "invalid range").
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <omp.h>

#define EXPORT __attribute__((visibility("default")))

typedef struct {
    int32_t N;    /* map side (texels), power of two              */
    int32_t s0;   /* base stride, power of two dividing N         */
    int32_t L;    /* number of levels, 2 <= L <= log2(N/s0) + 1   */
    int32_t A;    /* angular grid side                            */
    int32_t R;    /* rank                                         */
    int32_t wrap; /* 1: periodic neighbours, 0: clamp to edge     */
} oracle_desc;

typedef struct { float u, v, size; uint32_t rect; } oracle_rec; /* 16 B */

/* Step 1. */
static void oracle_level(const oracle_desc* d, double S, int* l0, double* t) {
    double ls = log2(S / (double)d->s0);
    if (ls < 0.0) ls = 0.0;                 /* below the base level: clamp */
    if (ls > d->L - 1) ls = d->L - 1;       /* above the top level: "directly clamp" */
    int f = (int)floor(ls);
    if (f > d->L - 2) f = d->L - 2;
    *l0 = f;
    *t = ls - f;
}

/* Step 2: neighbour indices and bilinear fraction along one axis. */
static void oracle_axis(const oracle_desc* d, int l, double u, int64_t* i0, int64_t* i1, double* a) {
    int64_t s = (int64_t)d->s0 << l, n = d->N / s;
    double f = u / (double)s - 0.5;
    double fl = floor(f);
    *a = f - fl;
    int64_t i = (int64_t)fl, j = i + 1;
    if (d->wrap) {
        i = ((i % n) + n) % n;
        j = ((j % n) + n) % n;
    } else {
        i = i < 0 ? 0 : (i > n - 1 ? n - 1 : i);
        j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
    }
    *i0 = i;
    *i1 = j;
}

static int64_t oracle_level_offset(const oracle_desc* d, int l) {
    int64_t off = 0;
    for (int m = 0; m < l; ++m) {
        int64_t n = d->N / ((int64_t)d->s0 << m);
        off += n * n;
    }
    return off;
}

/* Step 3: Eq. 6 sum over the rectangle for one positional index z. */
static double oracle_range_sum(const oracle_desc* d, const float* C, const double* xs, const double* ys,
                               const float* zrow) {
    double acc = 0.0;
    for (int r = 0; r < d->R; ++r) acc += (double)C[r] * xs[r] * ys[r] * (double)zrow[r];
    return acc;
}

static int oracle_valid(const oracle_desc* d, const oracle_rec* q, int* x1, int* x2, int* y1, int* y2) {
    *x1 = (int)(q->rect & 255u);
    *x2 = (int)((q->rect >> 8) & 255u);
    *y1 = (int)((q->rect >> 16) & 255u);
    *y2 = (int)((q->rect >> 24) & 255u);
    if (!isfinite(q->u) || !isfinite(q->v) || !isfinite(q->size)) return 0;
    if (fabs((double)q->u) > 4194304.0 || fabs((double)q->v) > 4194304.0) return 0;
    if (!(q->size > 0.0f)) return 0;
    if (*x1 > *x2 || *x2 >= d->A || *y1 > *y2 || *y2 >= d->A) return 0;
    return 1;
}

/* One query.  zmap (optional) maps a global row index z to its row in Z
 * (sparse storage of only the rows a sample touches); NULL = dense [P][R]. */
static double oracle_query_one(const oracle_desc* d, const float* C, const float* X, const float* Y, const float* Z,
                               const int64_t* zmap, const oracle_rec* q, int mean, double* xs, double* ys) {
    int x1, x2, y1, y2;
    if (!oracle_valid(d, q, &x1, &x2, &y1, &y2)) return NAN;
    const int R = d->R;
    /* 1-D segment sums, the numerators of X-bar and Y-bar. */
    for (int r = 0; r < R; ++r) { xs[r] = 0.0; ys[r] = 0.0; }
    for (int x = x1; x <= x2; ++x)
        for (int r = 0; r < R; ++r) xs[r] += (double)X[(int64_t)x * R + r];
    for (int y = y1; y <= y2; ++y)
        for (int r = 0; r < R; ++r) ys[r] += (double)Y[(int64_t)y * R + r];

    int l0;
    double t;
    oracle_level(d, (double)q->size, &l0, &t);
    double sum = 0.0;
    for (int dl = 0; dl < 2; ++dl) {
        int l = l0 + dl;
        double wl = dl ? t : 1.0 - t;
        int64_t n = d->N / ((int64_t)d->s0 << l), off = oracle_level_offset(d, l);
        int64_t i0, i1, j0, j1;
        double a, b;
        oracle_axis(d, l, (double)q->u, &i0, &i1, &a);
        oracle_axis(d, l, (double)q->v, &j0, &j1, &b);
        const int64_t zk[4] = {off + j0 * n + i0, off + j0 * n + i1, off + j1 * n + i0, off + j1 * n + i1};
        const double wk[4] = {(1 - a) * (1 - b), a * (1 - b), (1 - a) * b, a * b};
        for (int k = 0; k < 4; ++k) {
            int64_t z = zmap ? zmap[zk[k]] : zk[k];
            if (z < 0) return NAN; /* a row the sparse sample did not provide */
            sum += wl * wk[k] * oracle_range_sum(d, C, xs, ys, Z + z * (int64_t)R);
        }
    }
    if (mean) sum /= (double)(x2 - x1 + 1) * (double)(y2 - y1 + 1);
    return sum;
}

EXPORT void oracle_query_batch(const oracle_desc* d, const float* C, const float* X, const float* Y, const float* Z,
                               const int64_t* zmap, const oracle_rec* q, int64_t n, int mean, double* out,
                               int nthreads) {
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
    {
        double xs[4096], ys[4096]; /* R <= 4096 */
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) out[i] = oracle_query_one(d, C, X, Y, Z, zmap, &q[i], mean, xs, ys);
    }
}

/* The 8 (row, weight) pairs of one record, for tests that need the touched
 * rows (sparse Z samples) -- same steps 1-2 as above. Returns 0 if invalid. */
EXPORT int oracle_neighbours(const oracle_desc* d, const oracle_rec* q, int64_t* rows, double* w) {
    int x1, x2, y1, y2;
    if (!oracle_valid(d, q, &x1, &x2, &y1, &y2)) return 0;
    int l0;
    double t;
    oracle_level(d, (double)q->size, &l0, &t);
    for (int dl = 0; dl < 2; ++dl) {
        int l = l0 + dl;
        double wl = dl ? t : 1.0 - t;
        int64_t n = d->N / ((int64_t)d->s0 << l), off = oracle_level_offset(d, l);
        int64_t i0, i1, j0, j1;
        double a, b;
        oracle_axis(d, l, (double)q->u, &i0, &i1, &a);
        oracle_axis(d, l, (double)q->v, &j0, &j1, &b);
        rows[4 * dl + 0] = off + j0 * n + i0; w[4 * dl + 0] = wl * (1 - a) * (1 - b);
        rows[4 * dl + 1] = off + j0 * n + i1; w[4 * dl + 1] = wl * a * (1 - b);
        rows[4 * dl + 2] = off + j1 * n + i0; w[4 * dl + 2] = wl * (1 - a) * b;
        rows[4 * dl + 3] = off + j1 * n + i1; w[4 * dl + 3] = wl * a * b;
    }
    return 1;
}

EXPORT void oracle_neighbours_batch(const oracle_desc* d, const oracle_rec* q, int64_t n, int64_t* rows, double* w) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        if (!oracle_neighbours(d, &q[i], rows + 8 * i, w + 8 * i))
            for (int k = 0; k < 8; ++k) { rows[8 * i + k] = -1; w[8 * i + k] = NAN; }
}

/* ------------------------------------------------------------------------
 * Hierarchical importance sampling (Sec. 5.2), one global group.
 * "We start from the entire NDF image, and subdivide it evenly into four
 * quads ... acquire the average values in these four quads ... use the four
 * average values as relative probabilities, and randomly choose one quad to
 * proceed ... until reaching the bottom level, i.e. a pixel"; "when we
 * reach a pixel, we uniformly perturb the sample location inside it".
 * Readings: the descent starts from the record's rectangle (the
 * whole A x A image for plain sampling -- with one global group there is no
 * separate block choice); a range of width w splits into ceil(w/2) | floor(w/2)
 * (equal halves for the power-of-two grids of the configs); the relative
 * probabilities are the quads' SUMS (= averages x area, identical to the
 * paper's averages for equal quads, and exact for unequal ones); quad order
 * (x-low,y-low), (x-high,y-low), (x-low,y-high), (x-high,y-high); one variate
 * per level, xi[l] in [0,1), t = xi[l] * total, first quad with t < cumulative
 * sum (a zero quad is never chosen; if rounding leaves t >= all sums, the last
 * nonzero quad); xi[8], xi[9] jitter the pixel.  Outputs the pixel, its
 * probability mass / domain mass (the sampling pmf: "the PDF ... is
 * exactly the same as the evaluated NDF value") and the smallest relative
 * distance of a variate to a decision boundary (for tests).
 */
typedef struct {
    double xs[4096], ys[4096];
} oracle_scratch;

/* Eq. 6 SUM over [xa, xb) x [ya, yb) blended over the 8 neighbours */
static double oracle_rect_sum(const oracle_desc* d, const float* C, const float* X, const float* Y, const float* Z,
                              const int64_t* zmap, const int64_t* zk, const double* wk, int xa, int xb, int ya,
                              int yb, oracle_scratch* sc) {
    if (xb <= xa || yb <= ya) return 0.0;
    const int R = d->R;
    for (int r = 0; r < R; ++r) { sc->xs[r] = 0.0; sc->ys[r] = 0.0; }
    for (int x = xa; x < xb; ++x)
        for (int r = 0; r < R; ++r) sc->xs[r] += (double)X[(int64_t)x * R + r];
    for (int y = ya; y < yb; ++y)
        for (int r = 0; r < R; ++r) sc->ys[r] += (double)Y[(int64_t)y * R + r];
    double sum = 0.0;
    for (int k = 0; k < 8; ++k) {
        int64_t z = zmap ? zmap[zk[k]] : zk[k];
        if (z < 0) return NAN;
        sum += wk[k] * oracle_range_sum(d, C, sc->xs, sc->ys, Z + z * (int64_t)R);
    }
    return sum;
}

EXPORT void oracle_sample_batch(const oracle_desc* d, const float* C, const float* X, const float* Y, const float* Z,
                                const int64_t* zmap, const oracle_rec* q, const float* xi /* [n][10] */, int64_t n,
                                int32_t* pixel /* [n][2] */, double* prob, double* hxy /* [n][2] */,
                                double* margin) {
#pragma omp parallel
    {
        oracle_scratch* sc = (oracle_scratch*)malloc(sizeof(oracle_scratch));
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            int64_t zk[8];
            double wk[8];
            pixel[2 * i] = pixel[2 * i + 1] = -1;
            prob[i] = NAN;
            hxy[2 * i] = hxy[2 * i + 1] = NAN;
            margin[i] = INFINITY;
            if (!oracle_neighbours(d, &q[i], zk, wk)) continue;
            int xa = (int)(q[i].rect & 255u), xb = (int)((q[i].rect >> 8) & 255u) + 1;
            int ya = (int)((q[i].rect >> 16) & 255u), yb = (int)(q[i].rect >> 24) + 1;
            const double root = oracle_rect_sum(d, C, X, Y, Z, zmap, zk, wk, xa, xb, ya, yb, sc);
            if (!(root > 0.0)) { prob[i] = 0.0; continue; }
            double last = root, mg = INFINITY;
            for (int l = 0; xb - xa > 1 || yb - ya > 1; ++l) {
                const int xm = xa + (xb - xa + 1) / 2, ym = ya + (yb - ya + 1) / 2;
                const double Q[4] = {oracle_rect_sum(d, C, X, Y, Z, zmap, zk, wk, xa, xm, ya, ym, sc),
                                     oracle_rect_sum(d, C, X, Y, Z, zmap, zk, wk, xm, xb, ya, ym, sc),
                                     oracle_rect_sum(d, C, X, Y, Z, zmap, zk, wk, xa, xm, ym, yb, sc),
                                     oracle_rect_sum(d, C, X, Y, Z, zmap, zk, wk, xm, xb, ym, yb, sc)};
                const double tot = ((Q[0] + Q[1]) + Q[2]) + Q[3];
                const double t = (double)xi[10 * i + l] * tot;
                double c = 0.0;
                int k = -1;
                for (int j = 0; j < 4; ++j) {
                    if (Q[j] > 0.0) {
                        const double dist = fabs(t - c) / tot;  /* distance to this quad's lower edge */
                        if (c > 0.0 && dist < mg) mg = dist;
                    }
                    c += Q[j];
                    if (k < 0 && t < c) k = j;
                }
                if (k < 0) for (int j = 3; j >= 0; --j) if (Q[j] > 0.0) { k = j; break; }
                if (k & 1) xa = xm; else xb = xm;
                if (k & 2) ya = ym; else yb = ym;
                last = Q[k];
            }
            pixel[2 * i] = xa;
            pixel[2 * i + 1] = ya;
            prob[i] = last / root;
            hxy[2 * i] = ((double)xa + (double)xi[10 * i + 8]) * 2.0 / d->A - 1.0;
            hxy[2 * i + 1] = ((double)ya + (double)xi[10 * i + 9]) * 2.0 / d->A - 1.0;
            margin[i] = mg;
        }
        free(sc);
    }
}

/* ------------------------------------------------------------------------
 * Environment prefiltering (Sec. 5.4).  A spherical Gaussian with
 * amplitude A and bandwidth lambda has compact-eps support
 *     theta = arccos((ln eps - ln A) / lambda + 1)           (eps = 0.3)
 * and the NDF is blurred over a square of side
 *     Q = 256 (theta/2)/pi * 2 = 256 theta / pi             (P:426-428, 256 = NDF resolution)
 * Readings: the resolution is the store's A (Q = A theta/pi); an
 * arccos argument below -1 gives theta = pi, above 1 gives theta = 0;
 * the side is floor(Q + 1/2) clamped to [1, A]; the square is centred on the bin
 * of the projected half vector (bin = min(floor((h+1)A/2), A-1)) and shifted to
 * stay inside the grid (x1 = clamp(c - (side-1)/2, 0, A - side)).
 * Outputs theta, Q and the packed rectangle; q_margin is the distance of Q from
 * the nearest rounding boundary (x.5), used by tests to accept either side there.
 */
typedef struct { float u, v, size, hx, hy, lambda, amplitude, pad; } oracle_sgrec;

static int oracle_bin(double h, int A) {
    int b = (int)floor((h + 1.0) * 0.5 * A);
    return b < 0 ? 0 : (b > A - 1 ? A - 1 : b);
}

EXPORT void oracle_sg_rects(const oracle_sgrec* in, int64_t n, double eps, int A, double* theta, double* Q,
                            uint32_t* rect, double* q_margin) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double arg = (log(eps) - log((double)in[i].amplitude)) / (double)in[i].lambda + 1.0;
        double th = arg <= -1.0 ? M_PI : (arg >= 1.0 ? 0.0 : acos(arg));
        double q = (double)A * th / M_PI;
        int side = (int)floor(q + 0.5);
        if (side < 1) side = 1;
        if (side > A) side = A;
        double fr = q + 0.5 - floor(q + 0.5);
        q_margin[i] = fr < 1.0 - fr ? fr : 1.0 - fr;
        int cx = oracle_bin((double)in[i].hx, A), cy = oracle_bin((double)in[i].hy, A);
        int x1 = cx - (side - 1) / 2, y1 = cy - (side - 1) / 2;
        if (x1 > A - side) x1 = A - side;
        if (x1 < 0) x1 = 0;
        if (y1 > A - side) y1 = A - side;
        if (y1 < 0) y1 = 0;
        theta[i] = th;
        Q[i] = q;
        rect[i] = (uint32_t)x1 | ((uint32_t)(x1 + side - 1) << 8) | ((uint32_t)y1 << 16) |
                  ((uint32_t)(y1 + side - 1) << 24);
    }
}

/* ------------------------------------------------------------------------
 * Implicit Wang tiling (Sec. 5.5).  The world is an infinite grid
 * of T x T cells; each lattice vertex hashes to two random bits -- the colours
 * of its right (horizontal) and bottom (vertical) edges ("we
 * generate two random numbers with the vertex index as seed ... set to edges
 * e_ah and e_av, which are the right and bottom edges of vertex A") -- and a
 * cell's four edge colours pick one of the 16 tiles (edge-to-tile map:
 * id = N | E<<1 | S<<2 | W<<3).  Each tile has its own CP store over an
 * extended centre grid ("the sampled centers could locate outside the Wang
 * tiles") holding the tile's PARTIAL footprint NDF (its own texels,
 * normalised by the whole footprint's weight), so "the NDF image for a query
 * that crosses the borders between different Wang tiles is ... computed by
 * combining the precomputed NDF images from all overlapping Wang tiles":
 *     D(c) = sum over tiles t overlapping the footprint of D_t(c - origin_t).
 * Readings: the hash is splitmix64 of (seed, vx, vy) (any fixed
 * hash; the paper's "hash table" maps bits to colours one to one); the world is
 * not periodic; level select, neighbours and weights as in the plain query, with
 * world cell indices; tile t's extended grid has `margin` cells on each side.
 */
typedef struct {
    int32_t T, s0, L, margin, A, R;
    uint64_t seed;
} oracle_tiles;

static uint64_t oracle_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* bit 0: colour of the vertex's right edge, bit 1: of its bottom edge */
static uint64_t oracle_vertex(uint64_t seed, int64_t vx, int64_t vy) {
    return oracle_mix(oracle_mix(seed) ^ ((uint64_t)(uint32_t)vx | ((uint64_t)(uint32_t)vy << 32)));
}
EXPORT int oracle_tile_id(uint64_t seed, int64_t cx, int64_t cy) {
    const int n = (int)(oracle_vertex(seed, cx, cy) & 1u);            /* top edge: right edge of (cx, cy)   */
    const int sth = (int)(oracle_vertex(seed, cx, cy + 1) & 1u);      /* bottom edge: of (cx, cy+1)        */
    const int w = (int)((oracle_vertex(seed, cx, cy) >> 1) & 1u);     /* left edge: bottom edge of (cx, cy) */
    const int e = (int)((oracle_vertex(seed, cx + 1, cy) >> 1) & 1u); /* right edge: of (cx+1, cy)          */
    return n | (e << 1) | (sth << 2) | (w << 3);
}

static int64_t oracle_tile_rows(const oracle_tiles* d) {
    int64_t P = 0;
    for (int l = 0; l < d->L; ++l) {
        const int64_t ne = d->T / ((int64_t)d->s0 << l) + 2 * d->margin;
        P += ne * ne;
    }
    return P;
}

EXPORT void oracle_tiled_query_batch(const oracle_tiles* d, const float* C, const float* X, const float* Y,
                                     const float* Z /* [16][P_ext][R] */, const oracle_rec* q, int64_t n, int mean,
                                     double* out) {
    const int64_t Pext = oracle_tile_rows(d);
    const oracle_desc pd = {d->T, d->s0, d->L, d->A, d->R, 0};
#pragma omp parallel
    {
        double xs[4096], ys[4096];
#pragma omp for schedule(dynamic, 64)
        for (int64_t qi = 0; qi < n; ++qi) {
            int x1, x2, y1, y2;
            if (!oracle_valid(&pd, &q[qi], &x1, &x2, &y1, &y2) || fabs((double)q[qi].u) > 1073741824.0) {
                out[qi] = NAN;
                continue;
            }
            const int R = d->R;
            for (int r = 0; r < R; ++r) { xs[r] = 0.0; ys[r] = 0.0; }
            for (int x = x1; x <= x2; ++x)
                for (int r = 0; r < R; ++r) xs[r] += (double)X[(int64_t)x * R + r];
            for (int y = y1; y <= y2; ++y)
                for (int r = 0; r < R; ++r) ys[r] += (double)Y[(int64_t)y * R + r];
            int l0;
            double t;
            oracle_level(&pd, (double)q[qi].size, &l0, &t);
            double sum = 0.0;
            for (int dl = 0; dl < 2; ++dl) {
                const int l = l0 + dl;
                const double wl = dl ? t : 1.0 - t;
                const int64_t s = (int64_t)d->s0 << l, nn = d->T / s, ne = nn + 2 * d->margin;
                int64_t off = 0;
                for (int m = 0; m < l; ++m) {
                    const int64_t e2 = d->T / ((int64_t)d->s0 << m) + 2 * d->margin;
                    off += e2 * e2;
                }
                const double fu = (double)q[qi].u / (double)s - 0.5, fv = (double)q[qi].v / (double)s - 0.5;
                const int64_t iu = (int64_t)floor(fu), iv = (int64_t)floor(fv);
                const double a = fu - floor(fu), b = fv - floor(fv);
                for (int k = 0; k < 4; ++k) {
                    const int64_t iw = iu + (k & 1), jw = iv + (k >> 1);
                    const double wk = wl * ((k & 1) ? a : 1.0 - a) * ((k >> 1) ? b : 1.0 - b);
                    /* every tile whose extended grid contains this world centre */
                    const int64_t tx0 = (int64_t)floor((double)(iw - (nn + d->margin) + 1) / (double)nn);
                    const int64_t tx1 = (int64_t)floor((double)(iw + d->margin) / (double)nn);
                    const int64_t ty0 = (int64_t)floor((double)(jw - (nn + d->margin) + 1) / (double)nn);
                    const int64_t ty1 = (int64_t)floor((double)(jw + d->margin) / (double)nn);
                    for (int64_t ty = ty0; ty <= ty1; ++ty)
                        for (int64_t tx = tx0; tx <= tx1; ++tx) {
                            const int64_t il = iw - tx * nn, jl = jw - ty * nn;
                            if (il < -d->margin || il >= nn + d->margin || jl < -d->margin || jl >= nn + d->margin)
                                continue;
                            const int tile = oracle_tile_id(d->seed, tx, ty);
                            const int64_t z = (int64_t)tile * Pext + off + (jl + d->margin) * ne + (il + d->margin);
                            sum += wk * oracle_range_sum(&pd, C, xs, ys, Z + z * R);
                        }
                }
            }
            if (mean) sum /= (double)(x2 - x1 + 1) * (double)(y2 - y1 + 1);
            out[qi] = sum;
        }
    }
}

/* ------------------------------------------------------------------------
 * Blocked / clustered store (Sec. 4.2; range splitting P:353).
 * Each NDF image is cut into t x t angular blocks; blocks of footprints centred
 * in the same spatial region (side `region` texels) form a group with its own
 * CP factors (Eq. 5 per group); all-blank blocks are dropped
 * (P:294).  A query evaluates, for each of its 8 trilinear neighbours,
 * every block the rectangle overlaps -- "when the angular range happen to
 * overlap multiple image blocks, we subdivide it into smaller ones according to
 * the boundary of the image blocks" -- with that block's group factors
 * (Eq. 6 on the sub-rectangle), and sums.  Readings: a centre
 * ((i+1/2)s, (j+1/2)s) belongs to region (floor(cx/region), floor(cy/region));
 * group g = region * nb^2 + block; group_set[g] names the group's factor set
 * (C, X, Y), slab_ptr[z][block] its slab (-1 = blank).  The sum over the
 * sub-rectangles is the SUM over the whole rectangle; MEAN divides by its area.
 */
typedef struct {
    int32_t N, s0, L, A, t, region, R, wrap;
} oracle_blocked;

/* ------------------------------------------------------------------------
 * Importance sampling over implicit Wang tiles (Sec. 5.5): "we first
 * choose one Wang tile from all the Wang tiles covered by the pixel footprint
 * with equal probability.  Then, we sample a direction from the chosen Wang
 * tile, similar to Sec. 5.2.  After getting the sampled direction, we computed
 * the NDF value, which is the same as BRDF evaluation.  The PDF is set the
 * same as NDF value."
 * Readings (reading 25):
 *   - a tile instance (world cell (tx, ty)) is covered by the footprint when
 *     it holds texels of the footprint: its partial NDF has positive mass over
 *     the whole angular domain, sum_k w_k sum_r C_r (sum_x X_r)(sum_y Y_r) Z_r(z_k)
 *     > 0 over the rows z_k of the instance that the query reads;
 *   - the covered instances are ordered by (ty, tx); the chosen one is the
 *     c-th, c = floor(xi[10] * count) taken in fp32 (a float decision made in
 *     the same precision as the GPU), clamped to count - 1;
 *   - "sample a direction from the chosen Wang tile": the hierarchical descent
 *     of oracle_sample_batch on that instance's partial NDF (its rows only);
 *   - "the PDF is set the same as NDF value": the full (all-tile) NDF mass of
 *     the sampled pixel over the full mass of the record's rectangle, i.e. the
 *     plain sampler's pmf definition evaluated on the combined NDF.
 * Outputs per sample: pixel (-1 = none), prob (full pixel mass / full domain
 * mass), prob_tile (the chosen tile's pixel mass / its domain mass), h,
 * margin (as oracle_sample_batch), tile (tx, ty), count, and the domain masses
 * of the chosen tile's partial NDF and of the full NDF (for tests).
 */
#define TILE_MAX_ROWS 4096

typedef struct { int64_t tx, ty, z; double w; } oracle_tile_row;

/* every (tile instance, row, weight) the query reads with positive weight */
static int oracle_tile_rows_of(const oracle_tiles* d, const oracle_rec* q, int64_t Pext, oracle_tile_row* rows) {
    const oracle_desc pd = {d->T, d->s0, d->L, d->A, d->R, 0};
    int l0, nrow = 0;
    double t;
    oracle_level(&pd, (double)q->size, &l0, &t);
    for (int dl = 0; dl < 2; ++dl) {
        const int l = l0 + dl;
        const double wl = dl ? t : 1.0 - t;
        const int64_t s = (int64_t)d->s0 << l, nn = d->T / s, ne = nn + 2 * d->margin;
        int64_t off = 0;
        for (int m = 0; m < l; ++m) {
            const int64_t e2 = d->T / ((int64_t)d->s0 << m) + 2 * d->margin;
            off += e2 * e2;
        }
        const double fu = (double)q->u / (double)s - 0.5, fv = (double)q->v / (double)s - 0.5;
        const int64_t iu = (int64_t)floor(fu), iv = (int64_t)floor(fv);
        const double a = fu - floor(fu), b = fv - floor(fv);
        for (int k = 0; k < 4; ++k) {
            const int64_t iw = iu + (k & 1), jw = iv + (k >> 1);
            const double wk = wl * ((k & 1) ? a : 1.0 - a) * ((k >> 1) ? b : 1.0 - b);
            if (!(wk > 0.0)) continue;
            /* brute force over nearby tile instances: every extended grid that holds this centre */
            const int64_t cx = (int64_t)floor((double)iw / (double)nn), cy = (int64_t)floor((double)jw / (double)nn);
            const int64_t B = d->margin + 1;
            for (int64_t ty = cy - B; ty <= cy + B; ++ty)
                for (int64_t tx = cx - B; tx <= cx + B; ++tx) {
                    const int64_t il = iw - tx * nn, jl = jw - ty * nn;
                    if (il < -d->margin || il >= nn + d->margin || jl < -d->margin || jl >= nn + d->margin)
                        continue;
                    if (nrow >= TILE_MAX_ROWS) return -1;
                    const int tile = oracle_tile_id(d->seed, tx, ty);
                    rows[nrow].tx = tx;
                    rows[nrow].ty = ty;
                    rows[nrow].z = (int64_t)tile * Pext + off + (jl + d->margin) * ne + (il + d->margin);
                    rows[nrow].w = wk;
                    ++nrow;
                }
        }
    }
    return nrow;
}

/* Eq. 6 SUM over [xa, xb) x [ya, yb) of the rows of instance (tx, ty) (all instances if all != 0) */
static double oracle_tile_rect_sum(const oracle_tiles* d, const float* C, const float* X, const float* Y,
                                   const float* Z, const oracle_tile_row* rows, int nrow, int all, int64_t tx,
                                   int64_t ty, int xa, int xb, int ya, int yb, oracle_scratch* sc) {
    if (xb <= xa || yb <= ya) return 0.0;
    const int R = d->R;
    const oracle_desc pd = {d->T, d->s0, d->L, d->A, d->R, 0};
    for (int r = 0; r < R; ++r) { sc->xs[r] = 0.0; sc->ys[r] = 0.0; }
    for (int x = xa; x < xb; ++x)
        for (int r = 0; r < R; ++r) sc->xs[r] += (double)X[(int64_t)x * R + r];
    for (int y = ya; y < yb; ++y)
        for (int r = 0; r < R; ++r) sc->ys[r] += (double)Y[(int64_t)y * R + r];
    double sum = 0.0;
    for (int k = 0; k < nrow; ++k)
        if (all || (rows[k].tx == tx && rows[k].ty == ty))
            sum += rows[k].w * oracle_range_sum(&pd, C, sc->xs, sc->ys, Z + rows[k].z * R);
    return sum;
}

EXPORT void oracle_tiled_sample_batch(const oracle_tiles* d, const float* C, const float* X, const float* Y,
                                      const float* Z, const oracle_rec* q, const float* xi /* [n][11] */, int64_t n,
                                      int32_t* pixel /* [n][2] */, double* prob, double* prob_tile,
                                      double* hxy /* [n][2] */, double* margin, int64_t* tile /* [n][2] */,
                                      int32_t* count, double* mass_tile, double* mass_all) {
    const int64_t Pext = oracle_tile_rows(d);
    const oracle_desc pd = {d->T, d->s0, d->L, d->A, d->R, 0};
#pragma omp parallel
    {
        oracle_scratch* sc = (oracle_scratch*)malloc(sizeof(oracle_scratch));
        oracle_tile_row* rows = (oracle_tile_row*)malloc(sizeof(oracle_tile_row) * TILE_MAX_ROWS);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < n; ++i) {
            int x1, x2, y1, y2;
            pixel[2 * i] = pixel[2 * i + 1] = -1;
            prob[i] = prob_tile[i] = NAN;
            hxy[2 * i] = hxy[2 * i + 1] = NAN;
            margin[i] = INFINITY;
            tile[2 * i] = tile[2 * i + 1] = 0;
            count[i] = 0;
            mass_tile[i] = mass_all[i] = NAN;
            if (!oracle_valid(&pd, &q[i], &x1, &x2, &y1, &y2)) continue;
            const int nrow = oracle_tile_rows_of(d, &q[i], Pext, rows);
            if (nrow <= 0) continue;
            /* distinct covered instances (positive full-domain mass), ordered by (ty, tx) */
            int64_t inst[TILE_MAX_ROWS][2];
            int ni = 0;
            for (int k = 0; k < nrow; ++k) {
                int seen = 0;
                for (int j = 0; j < ni; ++j) seen |= (inst[j][0] == rows[k].tx && inst[j][1] == rows[k].ty);
                if (seen) continue;
                const double m = oracle_tile_rect_sum(d, C, X, Y, Z, rows, nrow, 0, rows[k].tx, rows[k].ty, 0, d->A,
                                                      0, d->A, sc);
                if (m > 0.0) { inst[ni][0] = rows[k].tx; inst[ni][1] = rows[k].ty; ++ni; }
            }
            if (ni == 0) { prob[i] = prob_tile[i] = 0.0; continue; }
            for (int a = 1; a < ni; ++a)  /* insertion sort by (ty, tx) */
                for (int b = a; b > 0 && (inst[b][1] < inst[b - 1][1] ||
                                          (inst[b][1] == inst[b - 1][1] && inst[b][0] < inst[b - 1][0])); --b) {
                    int64_t t0 = inst[b][0], t1 = inst[b][1];
                    inst[b][0] = inst[b - 1][0]; inst[b][1] = inst[b - 1][1];
                    inst[b - 1][0] = t0; inst[b - 1][1] = t1;
                }
            const float cf = xi[11 * i + 10] * (float)ni;  /* fp32 decision (reading 25) */
            int c = (int)floorf(cf);
            if (c > ni - 1) c = ni - 1;
            const int64_t tx = inst[c][0], ty = inst[c][1];
            tile[2 * i] = tx;
            tile[2 * i + 1] = ty;
            count[i] = ni;
            int xa = x1, xb = x2 + 1, ya = y1, yb = y2 + 1;
            const double root_all = oracle_tile_rect_sum(d, C, X, Y, Z, rows, nrow, 1, 0, 0, xa, xb, ya, yb, sc);
            const double root = oracle_tile_rect_sum(d, C, X, Y, Z, rows, nrow, 0, tx, ty, xa, xb, ya, yb, sc);
            mass_tile[i] = root;
            mass_all[i] = root_all;
            if (!(root > 0.0)) { prob[i] = prob_tile[i] = 0.0; continue; }
            double last = root, mg = INFINITY;
            for (int l = 0; xb - xa > 1 || yb - ya > 1; ++l) {
                const int xm = xa + (xb - xa + 1) / 2, ym = ya + (yb - ya + 1) / 2;
                const double Q[4] = {
                    oracle_tile_rect_sum(d, C, X, Y, Z, rows, nrow, 0, tx, ty, xa, xm, ya, ym, sc),
                    oracle_tile_rect_sum(d, C, X, Y, Z, rows, nrow, 0, tx, ty, xm, xb, ya, ym, sc),
                    oracle_tile_rect_sum(d, C, X, Y, Z, rows, nrow, 0, tx, ty, xa, xm, ym, yb, sc),
                    oracle_tile_rect_sum(d, C, X, Y, Z, rows, nrow, 0, tx, ty, xm, xb, ym, yb, sc)};
                const double tot = ((Q[0] + Q[1]) + Q[2]) + Q[3];
                const double tt = (double)xi[11 * i + l] * tot;
                double cum = 0.0;
                int k = -1;
                for (int j = 0; j < 4; ++j) {
                    if (Q[j] > 0.0) {
                        const double dist = fabs(tt - cum) / tot;
                        if (cum > 0.0 && dist < mg) mg = dist;
                    }
                    cum += Q[j];
                    if (k < 0 && tt < cum) k = j;
                }
                if (k < 0) for (int j = 3; j >= 0; --j) if (Q[j] > 0.0) { k = j; break; }
                if (k & 1) xa = xm; else xb = xm;
                if (k & 2) ya = ym; else yb = ym;
                last = Q[k];
            }
            pixel[2 * i] = xa;
            pixel[2 * i + 1] = ya;
            prob_tile[i] = last / root;
            prob[i] = oracle_tile_rect_sum(d, C, X, Y, Z, rows, nrow, 1, 0, 0, xa, xb, ya, yb, sc) / root_all;
            hxy[2 * i] = ((double)xa + (double)xi[11 * i + 8]) * 2.0 / d->A - 1.0;
            hxy[2 * i + 1] = ((double)ya + (double)xi[11 * i + 9]) * 2.0 / d->A - 1.0;
            margin[i] = mg;
        }
        free(rows);
        free(sc);
    }
}

EXPORT void oracle_blocked_query_batch(const oracle_blocked* d, const float* C, const float* X, const float* Y,
                                       const int32_t* group_set, const int64_t* slab_ptr, const float* Z,
                                       const oracle_rec* q, int64_t n, int mean, double* out) {
    const oracle_desc pd = {d->N, d->s0, d->L, d->A, d->R, d->wrap};
    const int t = d->t, nb = d->A / d->t, R = d->R;
    const int64_t nr = d->N / d->region;
#pragma omp parallel
    {
        double xs[4096], ys[4096];
#pragma omp for schedule(dynamic, 64)
        for (int64_t qi = 0; qi < n; ++qi) {
            int64_t rows[8];
            double w[8];
            int x1, x2, y1, y2;
            if (!oracle_valid(&pd, &q[qi], &x1, &x2, &y1, &y2) || !oracle_neighbours(&pd, &q[qi], rows, w)) {
                out[qi] = NAN;
                continue;
            }
            double sum = 0.0;
            for (int k = 0; k < 8; ++k) {
                /* level, cell and region of row z */
                int64_t z = rows[k], off = 0;
                int l = 0;
                for (;; ++l) {
                    const int64_t nn = d->N / ((int64_t)d->s0 << l);
                    if (z < off + nn * nn) break;
                    off += nn * nn;
                }
                const int64_t s = (int64_t)d->s0 << l, nn = d->N / s, c = z - off, i = c % nn, j = c / nn;
                const int64_t reg = (((2 * j + 1) * s) / (2 * d->region)) * nr + ((2 * i + 1) * s) / (2 * d->region);
                for (int byb = y1 / t; byb <= y2 / t; ++byb)
                    for (int bxb = x1 / t; bxb <= x2 / t; ++bxb) {
                        const int b = byb * nb + bxb;
                        const int64_t slab = slab_ptr[z * nb * nb + b];
                        if (slab < 0) continue; /* blank block */
                        const int set = group_set[reg * nb * nb + b];
                        if (set < 0) continue;
                        const int lx1 = (x1 > bxb * t ? x1 : bxb * t) - bxb * t;
                        const int lx2 = (x2 < bxb * t + t - 1 ? x2 : bxb * t + t - 1) - bxb * t;
                        const int ly1 = (y1 > byb * t ? y1 : byb * t) - byb * t;
                        const int ly2 = (y2 < byb * t + t - 1 ? y2 : byb * t + t - 1) - byb * t;
                        for (int r = 0; r < R; ++r) { xs[r] = 0.0; ys[r] = 0.0; }
                        for (int x = lx1; x <= lx2; ++x)
                            for (int r = 0; r < R; ++r) xs[r] += (double)X[((int64_t)set * t + x) * R + r];
                        for (int y = ly1; y <= ly2; ++y)
                            for (int r = 0; r < R; ++r) ys[r] += (double)Y[((int64_t)set * t + y) * R + r];
                        sum += w[k] * oracle_range_sum(&pd, C + (int64_t)set * R, xs, ys, Z + slab * R);
                    }
            }
            if (mean) sum /= (double)(x2 - x1 + 1) * (double)(y2 - y1 + 1);
            out[qi] = sum;
        }
    }
}

/* ------------------------------------------------------------------------
 * Importance sampling on the blocked / clustered store (Sec. 5.2):
 * "we first choose an image block to start, again according to their averaged
 * NDF values", then the hierarchical quad descent of oracle_sample_batch
 * inside the chosen block.  Readings (reading 26): the blocks are
 * the store's t x t angular blocks that the record's rectangle overlaps, in
 * order b = by * nb + bx; a block's weight is its Eq. 6 SUM over the part of
 * the rectangle inside it, blended over the footprint's 8 neighbours (= its
 * average x area: the paper's averages for the equal full blocks of a
 * whole-image rectangle); xi[10] picks the block (first block with
 * xi * total < cumulative weight; zero blocks never; rounding fallback = the
 * last nonzero block); xi[0..] drive the descent levels inside it, xi[8], xi[9]
 * jitter.  prob = the pixel's SUM / the rectangle's SUM (block pmf x descent
 * pmf), margin = the smallest relative distance of any variate (block choice
 * included) to its decision boundary; block[i] = the chosen block (-1 none).
 */
typedef struct {
    int64_t rows[8];
    double w[8];
    int64_t reg[8];
} oracle_bfoot;

/* Eq. 6 SUM over [xa, xb) x [ya, yb) (global bins) restricted to angular block (bx, by), blended over the 8
 * neighbours of the footprint */
static double oracle_block_rect_sum(const oracle_blocked* d, const float* C, const float* X, const float* Y,
                                    const int32_t* group_set, const int64_t* slab_ptr, const float* Z,
                                    const oracle_bfoot* f, int bx, int by, int xa, int xb, int ya, int yb,
                                    double* xs, double* ys) {
    const oracle_desc pd = {d->N, d->s0, d->L, d->A, d->R, d->wrap};
    const int t = d->t, nb = d->A / d->t, R = d->R;
    const int lx1 = (xa > bx * t ? xa : bx * t) - bx * t, lx2 = (xb < bx * t + t ? xb : bx * t + t) - bx * t;
    const int ly1 = (ya > by * t ? ya : by * t) - by * t, ly2 = (yb < by * t + t ? yb : by * t + t) - by * t;
    if (lx2 <= lx1 || ly2 <= ly1) return 0.0;
    const int b = by * nb + bx;
    double sum = 0.0;
    for (int k = 0; k < 8; ++k) {
        const int64_t slab = slab_ptr[f->rows[k] * nb * nb + b];
        if (slab < 0) continue; /* blank block */
        const int set = group_set[f->reg[k] * nb * nb + b];
        if (set < 0) continue;
        for (int r = 0; r < R; ++r) { xs[r] = 0.0; ys[r] = 0.0; }
        for (int x = lx1; x < lx2; ++x)
            for (int r = 0; r < R; ++r) xs[r] += (double)X[((int64_t)set * t + x) * R + r];
        for (int y = ly1; y < ly2; ++y)
            for (int r = 0; r < R; ++r) ys[r] += (double)Y[((int64_t)set * t + y) * R + r];
        sum += f->w[k] * oracle_range_sum(&pd, C + (int64_t)set * R, xs, ys, Z + slab * R);
    }
    return sum;
}

EXPORT void oracle_blocked_sample_batch(const oracle_blocked* d, const float* C, const float* X, const float* Y,
                                        const int32_t* group_set, const int64_t* slab_ptr, const float* Z,
                                        const oracle_rec* q, const float* xi /* [n][11] */, int64_t n,
                                        int32_t* pixel /* [n][2] */, double* prob, double* hxy /* [n][2] */,
                                        double* margin, int32_t* block) {
    const oracle_desc pd = {d->N, d->s0, d->L, d->A, d->R, d->wrap};
    const int t = d->t, nb = d->A / d->t;
    const int64_t nr = d->N / d->region;
#pragma omp parallel
    {
        double xs[4096], ys[4096];
        double Sb[256];
#pragma omp for schedule(dynamic, 64)
        for (int64_t i = 0; i < n; ++i) {
            oracle_bfoot f;
            int x1, x2, y1, y2;
            pixel[2 * i] = pixel[2 * i + 1] = -1;
            prob[i] = NAN;
            hxy[2 * i] = hxy[2 * i + 1] = NAN;
            margin[i] = INFINITY;
            block[i] = -1;
            if (!oracle_valid(&pd, &q[i], &x1, &x2, &y1, &y2) || !oracle_neighbours(&pd, &q[i], f.rows, f.w)) continue;
            for (int k = 0; k < 8; ++k) { /* region of the neighbour's centre (as oracle_blocked_query_batch) */
                int64_t z = f.rows[k], off = 0;
                int l = 0;
                for (;; ++l) {
                    const int64_t nn = d->N / ((int64_t)d->s0 << l);
                    if (z < off + nn * nn) break;
                    off += nn * nn;
                }
                const int64_t s = (int64_t)d->s0 << l, nn = d->N / s, c = z - off, ii = c % nn, jj = c / nn;
                f.reg[k] = (((2 * jj + 1) * s) / (2 * d->region)) * nr + ((2 * ii + 1) * s) / (2 * d->region);
            }
            /* 1. block choice by the blocks' weights over the rectangle */
            const int bx0 = x1 / t, bx1 = x2 / t, by0 = y1 / t, by1 = y2 / t;
            double total = 0.0;
            int nbk = 0;
            for (int by = by0; by <= by1; ++by)
                for (int bx = bx0; bx <= bx1; ++bx) {
                    Sb[nbk] = oracle_block_rect_sum(d, C, X, Y, group_set, slab_ptr, Z, &f, bx, by, x1, x2 + 1, y1,
                                                    y2 + 1, xs, ys);
                    total += Sb[nbk++];
                }
            if (!(total > 0.0)) { prob[i] = 0.0; continue; }
            double mg = INFINITY, cum = 0.0;
            const double tb = (double)xi[11 * i + 10] * total;
            int kb = -1;
            for (int j = 0; j < nbk; ++j) {
                if (Sb[j] > 0.0) {
                    const double dist = fabs(tb - cum) / total;
                    if (cum > 0.0 && dist < mg) mg = dist;
                }
                cum += Sb[j];
                if (kb < 0 && tb < cum) kb = j;
            }
            if (kb < 0) for (int j = nbk - 1; j >= 0; --j) if (Sb[j] > 0.0) { kb = j; break; }
            const int bx = bx0 + kb % (bx1 - bx0 + 1), by = by0 + kb / (bx1 - bx0 + 1);
            block[i] = by * nb + bx;
            /* 2. quad descent inside the chosen block (as oracle_sample_batch) */
            int xa = x1 > bx * t ? x1 : bx * t, xb = (x2 + 1 < bx * t + t ? x2 + 1 : bx * t + t);
            int ya = y1 > by * t ? y1 : by * t, yb = (y2 + 1 < by * t + t ? y2 + 1 : by * t + t);
            const double root = Sb[kb];
            double last = root;
            for (int l = 0; xb - xa > 1 || yb - ya > 1; ++l) {
                const int xm = xa + (xb - xa + 1) / 2, ym = ya + (yb - ya + 1) / 2;
                const double Q[4] = {
                    oracle_block_rect_sum(d, C, X, Y, group_set, slab_ptr, Z, &f, bx, by, xa, xm, ya, ym, xs, ys),
                    oracle_block_rect_sum(d, C, X, Y, group_set, slab_ptr, Z, &f, bx, by, xm, xb, ya, ym, xs, ys),
                    oracle_block_rect_sum(d, C, X, Y, group_set, slab_ptr, Z, &f, bx, by, xa, xm, ym, yb, xs, ys),
                    oracle_block_rect_sum(d, C, X, Y, group_set, slab_ptr, Z, &f, bx, by, xm, xb, ym, yb, xs, ys)};
                const double tot = ((Q[0] + Q[1]) + Q[2]) + Q[3];
                const double tt = (double)xi[11 * i + l] * tot;
                double c = 0.0;
                int k = -1;
                for (int j = 0; j < 4; ++j) {
                    if (Q[j] > 0.0) {
                        const double dist = fabs(tt - c) / tot;
                        if (c > 0.0 && dist < mg) mg = dist;
                    }
                    c += Q[j];
                    if (k < 0 && tt < c) k = j;
                }
                if (k < 0) for (int j = 3; j >= 0; --j) if (Q[j] > 0.0) { k = j; break; }
                if (k & 1) xa = xm; else xb = xm;
                if (k & 2) ya = ym; else yb = ym;
                last = Q[k];
            }
            pixel[2 * i] = xa;
            pixel[2 * i + 1] = ya;
            prob[i] = last / total;
            hxy[2 * i] = ((double)xa + (double)xi[11 * i + 8]) * 2.0 / d->A - 1.0;
            hxy[2 * i + 1] = ((double)ya + (double)xi[11 * i + 9]) * 2.0 / d->A - 1.0;
            margin[i] = mg;
        }
    }
}

EXPORT int oracle_max_threads(void) { return omp_get_max_threads(); }
