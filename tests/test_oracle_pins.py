"""Pins of the fp64 oracle to what the paper and the mathematics fix (CPU only).

Each test names the passage it follows (P:n = /root/reference/PAPER.md line n).
A plausible slip anywhere in the oracle -- a dropped term, a wrong sign or
index, a transposed operand, a wrong centre phase, level offset or level
weight -- fails at least one of these (see DESIGN.md §4 for the mapping).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_worked.json")


def _store_desc(N, s0, L, A, R, wrap):
    return oracle.make_desc(N, s0, L, A, R, wrap)


def _rand_records(rng, n, N, A, lg_lo, lg_hi, span=(-1.0, 2.0)):
    u = rng.uniform(span[0] * N, span[1] * N, n)
    v = rng.uniform(span[0] * N, span[1] * N, n)
    S = np.exp2(rng.uniform(lg_lo, lg_hi, n))
    x1 = rng.integers(0, A, n)
    x2 = np.minimum(A - 1, x1 + rng.integers(0, A, n))
    y1 = rng.integers(0, A, n)
    y2 = np.minimum(A - 1, y1 + rng.integers(0, A, n))
    return synth.make_records(u, v, S, x1, x2, y1, y2)


# ---------------------------------------------------------------- golden --
def test_golden_appendix_rank1():
    """Appendix proposition on hand-worked values, through the oracle."""
    g = json.load(open(GOLDEN))["appendix_rank1"]
    X = np.array(g["X"], np.float32)[:, None]
    Y = np.array(g["Y"], np.float32)[:, None]
    A = max(len(X), len(Y))
    Xp = np.zeros((A, 1), np.float32); Xp[:len(X)] = X
    Yp = np.zeros((A, 1), np.float32); Yp[:len(Y)] = Y
    d = _store_desc(2, 1, 2, A, 1, True)
    Z = np.ones((5, 1), np.float32)
    for c in g["cases"]:
        rec = synth.make_records(0.7, 1.3, 1.5, c["x1"], c["x2"], c["y1"], c["y2"])
        got = oracle.query_batch(d, np.ones(1, np.float32), Xp, Yp, Z, rec, mean=True)[0]
        assert got == pytest.approx(c["mean"], rel=1e-15)


def test_golden_trilinear_store():
    """Hand-worked trilinear + Eq. 6 values."""
    g = json.load(open(GOLDEN))["trilinear_store"]
    N, s0, L, A, R = g["N"], g["s0"], g["L"], g["A"], g["R"]
    Z = np.zeros((21, 1), np.float32)
    for j in range(4):
        for i in range(4):
            Z[j * 4 + i] = 1 + i + 4 * j
    for j in range(2):
        for i in range(2):
            Z[16 + j * 2 + i] = 100 + i + 2 * j
    Z[20] = 1000
    d = _store_desc(N, s0, L, A, R, g["wrap"])
    x1, x2, y1, y2 = g["rect"]
    for c in g["cases"]:
        rec = synth.make_records(c["u"], c["v"], c["size"], x1, x2, y1, y2)
        for mean, key in ((False, "sum"), (True, "mean")):
            got = oracle.query_batch(d, np.array(g["C"], np.float32), np.array(g["X"], np.float32),
                                     np.array(g["Y"], np.float32), Z, rec, mean=mean)[0]
            assert got == pytest.approx(c[key], rel=1e-12), (c, key)
            # the brute-force twin reaches the same hand value
            b = brute.query(N, s0, L, g["wrap"], np.array(g["C"]), np.array(g["X"]), np.array(g["Y"]), Z, rec[0],
                            mean=mean)
            assert b == pytest.approx(c[key], rel=1e-12)


# ------------------------------------------------------- Appendix / Eq. 6 --
def test_appendix_rank1_identity_random():
    """10^4 random rank-1 slabs: oracle range mean == brute-force mean of X (x) Y."""
    rng = np.random.default_rng(7)
    C1 = np.ones(1, np.float32)
    Z = np.ones((5, 1), np.float32)
    worst = 0.0
    for trial in range(10_000):
        A = int(rng.integers(1, 40))
        X = rng.random((A, 1)).astype(np.float32)
        Y = rng.random((A, 1)).astype(np.float32)
        x1, y1 = rng.integers(0, A, 2)
        x2 = int(rng.integers(x1, A)); y2 = int(rng.integers(y1, A))
        slab = np.outer(X[:, 0].astype(np.float64), Y[:, 0].astype(np.float64))
        ref = slab[x1:x2 + 1, y1:y2 + 1].mean()
        d = _store_desc(2, 1, 2, A, 1, True)
        got = oracle.query_batch(d, C1, X, Y, Z, synth.make_records(1.0, 1.0, 1.0, x1, x2, y1, y2))[0]
        worst = max(worst, abs(got - ref) / max(abs(ref), 1e-300))
    assert worst < 1e-12


@pytest.mark.parametrize("wrap", [True, False])
@pytest.mark.parametrize("mean", [True, False])
def test_oracle_equals_bruteforce_reconstruction(wrap, mean):
    """BASELINE check 1: CP query == brute-force sum of the reconstructed tensor (Eq. 5) over the range,
    blended over the 8 neighbours."""
    N, s0, L, A, R = 16, 1, 5, 9, 6
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=3, sparsity=0.3)
    d = _store_desc(N, s0, L, A, R, wrap)
    rng = np.random.default_rng(11)
    recs = _rand_records(rng, 400, N, A, -2.0, 6.0)
    got = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs, mean=mean)
    ref = np.array([brute.query(N, s0, L, wrap, f.C, f.X, f.Y, f.Z, r, mean=mean) for r in recs])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0)


def test_base_stride_and_partial_levels():
    """s0 > 1 and L < log2(N/s0)+1: level strides s0*2^l and offsets."""
    N, s0, L, A, R = 32, 4, 3, 5, 3
    P = sum((N // (s0 << l)) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=5)
    rng = np.random.default_rng(12)
    recs = _rand_records(rng, 300, N, A, 0.0, 7.0)
    for wrap in (True, False):
        d = _store_desc(N, s0, L, A, R, wrap)
        got = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs, mean=False)
        ref = np.array([brute.query(N, s0, L, wrap, f.C, f.X, f.Y, f.Z, r, mean=False) for r in recs])
        np.testing.assert_allclose(got, ref, rtol=1e-12)


# ------------------------------------------------------- interpolation pins --
@pytest.mark.parametrize("level", [0, 1, 2, 3, 4])
def test_bilinear_reproduces_affine_fields(level):
    """Bilinear interpolation over centres ((i+1/2)s, (j+1/2)s) reproduces an affine
    field exactly: Z(i,j) = 5 + 0.25 cx(i) + 0.5 cy(j)  =>  query(u, v) = 5 + 0.25 u + 0.5 v.
    Other levels hold 1e6 so a wrong level offset, centre phase, axis swap or weight flip shows."""
    N, s0, L = 32, 1, 6
    offs = np.cumsum([0] + [(N >> l) ** 2 for l in range(L)])
    Z = np.full((offs[-1], 1), 1e6, np.float32)
    s = s0 << level
    n = N // s
    for j in range(n):
        for i in range(n):
            Z[offs[level] + j * n + i] = 5 + 0.25 * (i + 0.5) * s + 0.5 * (j + 0.5) * s
    rng = np.random.default_rng(level)
    u = rng.uniform(0.5 * s, N - 0.5 * s, 200)
    v = rng.uniform(0.5 * s, N - 0.5 * s, 200)
    u = u.astype(np.float32); v = v.astype(np.float32)
    size = float(s0 << level) if level < L - 1 else 1e9
    recs = synth.make_records(u, v, size, 0, 0, 0, 0)
    one = np.ones((1, 1), np.float32)
    for wrap in (True, False):
        got = oracle.query_batch(_store_desc(N, s0, L, 1, 1, wrap), np.ones(1, np.float32), one, one, Z, recs)
        np.testing.assert_allclose(got, 5 + 0.25 * u.astype(np.float64) + 0.5 * v.astype(np.float64), rtol=1e-12)


def test_level_interpolation_linear_in_log2_size():
    """Level blend is linear in log2 S (reading of "trilinear"): with Z = l+1 on
    level l the query returns clamp(log2(S/s0), 0, L-1) + 1, and clamps outside."""
    N, s0, L = 64, 2, 6
    offs = np.cumsum([0] + [(N // (s0 << l)) ** 2 for l in range(L)])
    Z = np.zeros((offs[-1], 1), np.float32)
    for l in range(L):
        Z[offs[l]:offs[l + 1]] = l + 1
    rng = np.random.default_rng(3)
    lg = rng.uniform(-3, L + 3, 500)
    S = np.exp2(lg).astype(np.float32)
    recs = synth.make_records(rng.uniform(0, N, 500), rng.uniform(0, N, 500), S, 0, 0, 0, 0)
    one = np.ones((1, 1), np.float32)
    got = oracle.query_batch(_store_desc(N, s0, L, 1, 1, True), np.ones(1, np.float32), one, one, Z, recs)
    ref = np.clip(np.log2(S.astype(np.float64) / s0), 0, L - 1) + 1
    np.testing.assert_allclose(got, ref, rtol=1e-12)


def test_exact_centre_returns_stored_sample():
    """A query at a sample centre with S = s_l reads exactly that precomputed sample (the
    pyramid stores NDFs at those footprints; SPEC S:345 'single point query, weights (1,0,...)')."""
    N, s0, L, A, R = 16, 1, 5, 4, 3
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=9)
    d = _store_desc(N, s0, L, A, R, False)
    offs = np.cumsum([0] + [(N >> l) ** 2 for l in range(L)])
    for l in range(L - 1):
        s = 1 << l; n = N // s
        for (i, j) in ((0, 0), (n - 1, 0), (n // 2, n - 1)):
            rec = synth.make_records((i + 0.5) * s, (j + 0.5) * s, float(s), 1, 2, 0, 3)
            got = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, rec, mean=False)[0]
            z = offs[l] + j * n + i
            img = brute.reconstruct(f.C, f.X, f.Y, f.Z[z])
            assert got == pytest.approx(img[1:3, 0:4].sum(), rel=1e-12)


def test_periodicity_wrap():
    """Tileable maps: q(u + N, v) = q(u, v - N) = q(u, v)."""
    N, s0, L, A, R = 32, 1, 6, 6, 4
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=2)
    d = _store_desc(N, s0, L, A, R, True)
    rng = np.random.default_rng(5)
    r0 = _rand_records(rng, 300, N, A, 0, 6, span=(0.0, 1.0))
    r0["u"] = np.round(r0["u"] * 1024) / 1024  # dyadic, so u + N and v - N are exact in fp32
    r0["v"] = np.round(r0["v"] * 1024) / 1024
    r1 = r0.copy(); r1["u"] = r0["u"] + N
    r2 = r0.copy(); r2["v"] = r0["v"] - N
    q0, q1, q2 = (oracle.query_batch(d, f.C, f.X, f.Y, f.Z, r) for r in (r0, r1, r2))
    np.testing.assert_allclose(q1, q0, rtol=1e-12)
    np.testing.assert_allclose(q2, q0, rtol=1e-12)


def test_clamp_outside_pyramid():
    """Above the top level the footprint "directly clamp[s]" to the largest precomputed; below the
    base it clamps to level 0 (DESIGN reading: the Yan 2016 fallback is out of scope)."""
    N, s0, L, A, R = 16, 1, 5, 4, 3
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=4)
    d = _store_desc(N, s0, L, A, R, True)
    rng = np.random.default_rng(8)
    base = _rand_records(rng, 100, N, A, 0, 1, span=(0, 1))
    hi_a = base.copy(); hi_a["size"] = 16.0
    hi_b = base.copy(); hi_b["size"] = 1e6
    lo_a = base.copy(); lo_a["size"] = 1.0
    lo_b = base.copy(); lo_b["size"] = 1e-3
    q = [oracle.query_batch(d, f.C, f.X, f.Y, f.Z, r) for r in (hi_a, hi_b, lo_a, lo_b)]
    np.testing.assert_array_equal(q[0], q[1])
    np.testing.assert_array_equal(q[2], q[3])


# ------------------------------------------------------ invariants (BJ checks) --
def test_disjoint_ranges_add():
    """BASELINE check 4: SUM(R1) + SUM(R2) = SUM(R1 u R2) for splits along x and y."""
    N, s0, L, A, R = 16, 1, 5, 12, 5
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=6)
    d = _store_desc(N, s0, L, A, R, True)
    rng = np.random.default_rng(9)
    n = 300
    u, v = rng.uniform(0, N, n), rng.uniform(0, N, n)
    S = np.exp2(rng.uniform(0, 4, n))
    x1 = rng.integers(0, A - 1, n); x2 = rng.integers(x1 + 1, A)
    xm = rng.integers(x1, x2)  # split: [x1, xm] u [xm+1, x2]
    y1 = rng.integers(0, A, n); y2 = rng.integers(y1, A)
    whole = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, synth.make_records(u, v, S, x1, x2, y1, y2), mean=False)
    left = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, synth.make_records(u, v, S, x1, xm, y1, y2), mean=False)
    right = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, synth.make_records(u, v, S, xm + 1, x2, y1, y2), mean=False)
    np.testing.assert_allclose(left + right, whole, rtol=1e-12)
    # and along y, using the transposed roles
    ym = np.minimum(y2, y1 + rng.integers(0, A, n))
    ok = ym < y2
    a = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, synth.make_records(u, v, S, x1, x2, y1, ym), mean=False)
    b = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, synth.make_records(u, v, S, x1, x2, np.minimum(ym + 1, y2), y2),
                           mean=False)
    w = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, synth.make_records(u, v, S, x1, x2, y1, y2), mean=False)
    np.testing.assert_allclose((a + b)[ok], w[ok], rtol=1e-12)


def test_linearity_in_factors():
    """Eq. 5 is linear: doubling Z doubles results; splitting the ranks into two stores adds."""
    N, s0, L, A, R = 16, 1, 5, 7, 6
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=10)
    rng = np.random.default_rng(10)
    recs = _rand_records(rng, 200, N, A, 0, 5)
    d = _store_desc(N, s0, L, A, R, True)
    q = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs)
    q2 = oracle.query_batch(d, f.C, f.X, f.Y, 2 * f.Z, recs)
    np.testing.assert_allclose(q2, 2 * q, rtol=1e-12)
    k = 2
    da, db = _store_desc(N, s0, L, A, k, True), _store_desc(N, s0, L, A, R - k, True)
    qa = oracle.query_batch(da, f.C[:k], f.X[:, :k], f.Y[:, :k], f.Z[:, :k], recs)
    qb = oracle.query_batch(db, f.C[k:], f.X[:, k:], f.Y[:, k:], f.Z[:, k:], recs)
    np.testing.assert_allclose(qa + qb, q, rtol=1e-12)


def test_point_and_range_identical():
    """"identical results generated using our range query once and our point query repeatedly"
    (S:698): range mean == mean of the 1x1 queries over its pixels."""
    N, s0, L, A, R = 16, 1, 5, 10, 4
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=12)
    d = _store_desc(N, s0, L, A, R, True)
    rng = np.random.default_rng(13)
    for _ in range(50):
        u, v, S = rng.uniform(0, N), rng.uniform(0, N), 2 ** rng.uniform(0, 4)
        x1, y1 = rng.integers(0, A, 2); x2 = rng.integers(x1, A); y2 = rng.integers(y1, A)
        rng_q = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, synth.make_records(u, v, S, x1, x2, y1, y2))[0]
        xs, ys = np.meshgrid(np.arange(x1, x2 + 1), np.arange(y1, y2 + 1), indexing="ij")
        pts = oracle.query_batch(d, f.C, f.X, f.Y, f.Z,
                                 synth.make_records(np.full(xs.size, u), np.full(xs.size, v), np.full(xs.size, S),
                                                    xs.ravel(), xs.ravel(), ys.ravel(), ys.ravel()))
        assert rng_q == pytest.approx(pts.mean(), rel=1e-12)


def test_invalid_records_are_nan():
    """SPEC "invalid range" / "invalid indices" -> NaN per record."""
    d = _store_desc(8, 1, 4, 4, 2, True)
    P = 64 + 16 + 4 + 1
    f = synth.random_factors(4, 2, P, seed=1)
    recs = synth.make_records([1, 1, 1, np.nan, 1, 1, 1, 1, 5e6],
                              [1, 1, 1, 1, np.inf, 1, 1, 1, 1],
                              [1, 0, -1, 1, 1, np.nan, 1, 1, 1],
                              [0, 0, 0, 0, 0, 0, 2, 0, 0], [3, 3, 3, 3, 3, 3, 1, 4, 3],
                              [0, 0, 0, 0, 0, 0, 0, 0, 0], [3, 3, 3, 3, 3, 3, 3, 3, 3])
    q = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs)
    assert np.isfinite(q[0])
    assert np.isnan(q[1:]).all()


# ----------------------------------------------- exact-rank histogram check --
def _brute_histogram(nxy_bins_x, nxy_bins_y, N, s, i, j, A, table):
    """Brute-force footprint NDF of Eq. 2 with sigma_r -> 0 (a normal histogram):
    splat every texel of the footprint window into its (x, y) bin with weight G_p(u)."""
    qmin, w = table
    img = np.zeros((A, A))
    tot = float(w.sum()) ** 2
    for q in range(w.shape[0]):
        vv = (j * s + qmin + q) % N
        for p in range(w.shape[0]):
            uu = (i * s + qmin + p) % N
            img[nxy_bins_x[vv, uu], nxy_bins_y[vv, uu]] += float(w[p]) * float(w[q])
    return img / tot


@pytest.mark.parametrize("snap", [False, True])
def test_exact_rank_equals_bruteforce_histogram(snap):
    """BASELINE check 2: for exact-rank synthetic tensors the CP query equals brute-force normal-histogram
    NDFs (Eq. 2) of the (snapped) normal map, summed over the rectangle."""
    base = synth.Config(0, "pin", N=32, A=12, R=1, n_queries=0, map_kind="flakes",
                        map_params=dict(spacing=3.0, alpha=0.35), sigma_r=0.0)
    nxy = synth.make_map(base)
    bins = synth.bin_map(base, nxy)
    npop = len(np.unique(bins))
    R = max(2, npop // 2) if snap else npop
    cfg = base.scaled(R=R)
    f = synth.build_factors(cfg, nxy, bins)
    ab, am = f.info["atom_bins"], f.info["atom_map"]
    # per-texel (x, y) bin of the texel's (snapped) normal
    tb = ab[am] if snap else bins.astype(np.int64)
    bx, by = tb % cfg.A, tb // cfg.A
    d = oracle.desc_of(cfg)
    offs = synth.level_offsets(cfg)
    rng = np.random.default_rng(21)
    checked = 0
    for l in range(cfg.L):
        s = 1 << l; n = cfg.N // s
        table = synth.footprint_table(s, cfg.N)
        for _ in range(3 if l < 3 else 1):
            i, j = rng.integers(0, n, 2)
            img = _brute_histogram(bx, by, cfg.N, s, i, j, cfg.A, table)
            assert img.sum() == pytest.approx(1.0, abs=1e-12)
            x1, y1 = rng.integers(0, cfg.A, 2); x2 = rng.integers(x1, cfg.A); y2 = rng.integers(y1, cfg.A)
            size = float(s) if l < cfg.L - 1 else 1e6
            rec = synth.make_records((i + 0.5) * s, (j + 0.5) * s, size, x1, x2, y1, y2)
            got = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, rec, mean=False)[0]
            # Z is the fp32 rounding of the exact fraction: allow fp32 factor rounding only
            assert got == pytest.approx(img[x1:x2 + 1, y1:y2 + 1].sum(), rel=2e-6, abs=1e-7)
            full = oracle.query_batch(d, f.C, f.X, f.Y, f.Z,
                                      synth.make_records((i + 0.5) * s, (j + 0.5) * s, size, 0, cfg.A - 1, 0,
                                                         cfg.A - 1), mean=False)[0]
            assert full == pytest.approx(1.0, abs=2e-6)
            checked += 1
    assert checked >= 10


def test_exact_rank_with_intrinsic_roughness():
    """sigma_r > 0: Eq. 2's G_r is separable, so each atom stays rank-1; the query equals the
    brute-force splat of each texel's bin-integrated Gaussian (computed here with scipy)."""
    from scipy.stats import norm
    cfg = synth.Config(0, "pin", N=16, A=10, R=1, n_queries=0, map_kind="flakes",
                       map_params=dict(spacing=3.0, alpha=0.3), sigma_r=0.15)
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    cfg = cfg.scaled(R=len(np.unique(bins)))
    f = synth.build_factors(cfg, nxy, bins)
    sb = cfg.sigma_r * cfg.A / 2.0
    T = math.ceil(4 * sb)

    def prof(c):
        x = np.arange(cfg.A)
        p = norm.cdf((x + 1 - (c + 0.5)) / sb) - norm.cdf((x - (c + 0.5)) / sb)
        p[np.abs(x - c) > T] = 0.0
        return p / p.sum()

    d = oracle.desc_of(cfg)
    s, n = 2, cfg.N // 2
    table = synth.footprint_table(s, cfg.N)
    qmin, w = table
    i, j = 3, 5
    img = np.zeros((cfg.A, cfg.A))
    tot = float(w.sum()) ** 2
    for q in range(w.shape[0]):
        vv = (j * s + qmin + q) % cfg.N
        for p in range(w.shape[0]):
            uu = (i * s + qmin + p) % cfg.N
            b = int(bins[vv, uu])
            img += float(w[p]) * float(w[q]) / tot * np.outer(prof(b % cfg.A), prof(b // cfg.A))
    for (x1, x2, y1, y2) in ((0, 9, 0, 9), (2, 4, 3, 7), (5, 5, 5, 5), (0, 0, 0, 9)):
        rec = synth.make_records((i + 0.5) * s, (j + 0.5) * s, float(s), x1, x2, y1, y2)
        got = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, rec, mean=False)[0]
        assert got == pytest.approx(img[x1:x2 + 1, y1:y2 + 1].sum(), rel=1e-5, abs=1e-8)


def test_constant_map_is_rank1_and_position_independent():
    """All-up (or constant-tilt) normal map: every footprint NDF is the same blob, so the
    query is independent of u, v, S and the full-domain integral is 1."""
    cfg = synth.Config(0, "const", N=32, A=8, R=1, n_queries=0, map_kind="constant",
                       map_params=dict(nx=0.3, ny=-0.2), sigma_r=0.0)
    f = synth.build_factors(cfg)
    bx = int(math.floor((0.3 + 1) * 4)); by = int(math.floor((-0.2 + 1) * 4))
    d = oracle.desc_of(cfg)
    rng = np.random.default_rng(1)
    n = 100
    recs = synth.make_records(rng.uniform(0, 32, n), rng.uniform(0, 32, n), np.exp2(rng.uniform(0, 5, n)),
                              bx, bx, by, by)
    q = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs, mean=False)
    np.testing.assert_allclose(q, 1.0, rtol=1e-6)
    recs["rect"] = synth.pack_rect(0, bx - 1, 0, 7)
    assert np.all(oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs, mean=False) == 0.0)


def test_full_domain_normalisation_config1_als():
    """BASELINE check 3: the full-angular-domain integral is the footprint's normalisation (1 for the
    mass-renormalised config-1 ALS store), for any centre and size."""
    cfg = synth.CONFIGS[1]
    f = synth.build_factors(cfg)
    rng = np.random.default_rng(2)
    n = 500
    recs = synth.make_records(rng.uniform(0, 64, n), rng.uniform(0, 64, n), np.exp2(rng.uniform(-1, 7, n)),
                              0, cfg.A - 1, 0, cfg.A - 1)
    q = oracle.query_batch(oracle.desc_of(cfg), f.C, f.X, f.Y, f.Z, recs, mean=False)
    np.testing.assert_allclose(q, 1.0, rtol=3e-6)


# ----------------------------------------------------- helper-path pins --
@pytest.mark.parametrize("wrap", [True, False])
def test_neighbours_reproduce_position_and_level(wrap):
    """oracle.neighbours (steps 1-2 on their own, used to pick the rows of sparse samples): the 8 weights
    are a partition of unity split (1-t, t) between the two levels (t linear in log2 S, P:276/P:327,
    clamped at the pyramid ends); each row lies in its level's range; and bilinear weights have
    linear precision: at each level, sum_k w_k centre_k = (u, v) for interior points, with
    centre (i+1/2, j+1/2) s_l decoded from the row index (so a wrong offset, axis swap or phase fails)."""
    N, s0, L = 64, 2, 6
    d = _store_desc(N, s0, L, 4, 1, wrap)
    offs = np.cumsum([0] + [(N // s0 >> l) ** 2 for l in range(L)])
    rng = np.random.default_rng(11)
    n = 4000
    lgS = rng.uniform(-1.0, L + 1.0, n)
    S = np.exp2(lgS).astype(np.float32)
    lstar = np.clip(np.log2(S.astype(np.float64) / s0), 0, L - 1)
    l0 = np.minimum(np.floor(lstar), L - 2).astype(np.int64)
    t = lstar - l0
    s_hi = (s0 << (l0 + 1)).astype(np.float64)  # interior margin at the coarser level
    u = (rng.uniform(0, 1, n) * np.maximum(N - 2 * s_hi, 0) + np.minimum(s_hi, N / 2)).astype(np.float32)
    v = (rng.uniform(0, 1, n) * np.maximum(N - 2 * s_hi, 0) + np.minimum(s_hi, N / 2)).astype(np.float32)
    recs = synth.make_records(u, v, S, 0, 0, 0, 0)
    rows, w = oracle.neighbours(d, recs)
    np.testing.assert_allclose(w.sum(1), 1.0, rtol=0, atol=1e-12)
    np.testing.assert_allclose(w[:, :4].sum(1), 1.0 - t, rtol=0, atol=1e-12)
    for dl in (0, 1):
        l = l0 + dl
        r = rows[:, 4 * dl:4 * dl + 4]
        assert ((r >= offs[l][:, None]) & (r < offs[l + 1][:, None])).all()
        n_l = (N // s0) >> l
        k = r - offs[l][:, None]
        ci = (k % n_l[:, None] + 0.5) * (s0 << l)[:, None]
        cj = (k // n_l[:, None] + 0.5) * (s0 << l)[:, None]
        ww = w[:, 4 * dl:4 * dl + 4]
        tot = ww.sum(1)
        m = (tot > 1e-9) & (N - 2 * s_hi > 0)  # interior points exist below the top level
        np.testing.assert_allclose((ww * ci).sum(1)[m] / tot[m], u[m].astype(np.float64), rtol=0, atol=1e-9)
        np.testing.assert_allclose((ww * cj).sum(1)[m] / tot[m], v[m].astype(np.float64), rtol=0, atol=1e-9)
    bad = synth.make_records([np.nan], [1.0], [1.0], 0, 0, 0, 0)
    rb, wb = oracle.neighbours(d, bad)
    assert (rb == -1).all() and np.isnan(wb).all()


def test_sparse_z_path_equals_dense():
    """The sparse-Z path (zmap: only the rows a sample touches, used by the config-5 parity and bench
    samples) returns the dense path's bits, for rows gathered by oracle.neighbours; a record needing a row
    the sample lacks is NaN (never a silent zero)."""
    cfg, bins = synth.CONFIGS[2], None
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    f = synth.build_factors(cfg, nxy, bins)
    recs = synth.gen_queries(cfg, bins, 0, 30_000)
    d = oracle.desc_of(cfg)
    dense = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs)
    rows, _ = oracle.neighbours(d, recs)
    Zs, zmap = oracle.sparse_z(rows.ravel(), cfg.P, lambda u: f.Z[u])
    assert Zs.shape[0] < cfg.P // 2
    sparse = oracle.query_batch(d, f.C, f.X, f.Y, Zs, recs, zmap=zmap)
    assert sparse.tobytes() == dense.tobytes()
    # drop one needed row: exactly the records that use it become NaN
    drop = rows[0, 0]
    zmap2 = zmap.copy()
    zmap2[drop] = -1
    got = oracle.query_batch(d, f.C, f.X, f.Y, Zs, recs, zmap=zmap2)
    uses = (rows == drop).any(1)
    assert np.isnan(got[uses]).all() and got[~uses].tobytes() == dense[~uses].tobytes()


def test_rectangles_mostly_on_the_footprint_support():
    """parity must not be dominated by trivially zero blank-region queries.  On configs 1-4
    (oracle on 20K queries of each stream) at least 45% of the results are nonzero."""
    for k in (1, 2, 3, 4):
        cfg = synth.CONFIGS[k]
        if k >= 3:
            cfg = cfg.scaled(N=512)
        nxy = synth.make_map(cfg)
        bins = synth.bin_map(cfg, nxy)
        f = synth.build_factors(cfg, nxy, bins)
        recs = synth.gen_queries(cfg, bins, 0, 20_000)
        ref = oracle.query_batch(oracle.desc_of(cfg), f.C, f.X, f.Y, f.Z, recs)
        assert (ref > 0).mean() >= 0.45, (k, (ref > 0).mean())
