"""Pins of the factor-builder oracle (oracle/als.py) -- CPU only.

Each pin ties a function to something other than itself: an independent implementation of Eq. 2, a closed
form, a textbook property of (nonnegative) ALS, or exact arithmetic.  A dropped weight, a transposed
Khatri-Rao operand, a wrong mode order or a sign slip in the HALS step fails at least one of them.
"""
import math

import numpy as np
import pytest

import synth
from oracle import als


def _small_cfg(N=32, A=8):
    return synth.CONFIGS[1].scaled(N=N, A=A)


# ------------------------------------------------------------------------- histogram --
def test_hist_matches_independent_c_builder():
    """Eq. 2 (sigma_r -> 0) histogram: the numpy oracle equals synth.c's integer-accumulating builder exactly."""
    cfg = _small_cfg(32, 8)
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    D = als.hist_tensor(cfg.N, cfg.s0, cfg.L, cfg.A, bins)
    Dc = synth.hist_tensor(cfg, bins)
    assert D.shape == Dc.shape
    assert np.array_equal(D, Dc)


def test_hist_rows_are_normalised_and_constant_map_is_one_hot():
    """Every footprint histogram is a distribution over the A x A grid (P:211 normalised G_p); a constant map
    puts all mass in one bin at every level and position."""
    N, A = 16, 4
    bins = np.full((N, N), 1 + A * 2, np.uint16)  # x = 1, y = 2
    D = als.hist_tensor(N, 1, 5, A, bins)
    assert np.allclose(D.sum((1, 2)), 1.0, atol=1e-15, rtol=0)
    assert np.all(D[:, 1, 2] == 1.0)
    rng = np.random.default_rng(3)
    bins = rng.integers(0, A * A, (N, N)).astype(np.uint16)
    D = als.hist_tensor(N, 1, 5, A, bins)
    assert np.allclose(D.sum((1, 2)), 1.0, atol=1e-12, rtol=0)
    # level 0 at s = 1: sigma = 0.433, the footprint is dominated by its own texel
    assert D[0].max() > 0.5
    # top level (one footprint, window folded over the whole map): all texels, nearly equal weights
    b = bins.astype(int).ravel()
    cnt = np.bincount((b % A) * A + b // A, minlength=A * A) / (N * N)
    assert np.abs(D[-1].ravel() - cnt).max() < 0.05


def test_tf32_round_exact_values():
    """Round-to-nearest-even to 11 significant bits."""
    one = 1.0
    u = 2.0 ** -10  # spacing at 1
    vals = np.array([one, one + u / 2, one + 3 * u / 2, one + u / 4, one + 3 * u / 4, 3.0, 2.0 ** -40 * (1 + u / 2)])
    want = np.array([one, one, one + 2 * u, one, one + u, 3.0, 2.0 ** -40], np.float32)
    got = als.tf32_round(vals)
    assert np.array_equal(got, want)
    x = np.random.default_rng(1).random(10000) * 10.0 ** np.random.default_rng(2).integers(-12, 3, 10000)
    r = als.tf32_round(x)
    assert np.all((r.view(np.uint32) & 0x1FFF) == 0)
    assert np.abs(r.astype(np.float64) / x - 1).max() <= 2.0 ** -11


# ---------------------------------------------------------------------------- MTTKRP --
def test_mttkrp_rank1_closed_form():
    """D = z o x o y  =>  M_z = z (x'X * y'Y), M_x = x (z'Z * y'Y), M_y = y (z'Z * x'X)."""
    rng = np.random.default_rng(4)
    P, A1, A2, R = 7, 5, 6, 3
    z, x, y = rng.random(P), rng.random(A1), rng.random(A2)
    D = np.einsum("z,x,y->zxy", z, x, y)
    Z, X, Y = rng.random((P, R)), rng.random((A1, R)), rng.random((A2, R))
    assert np.allclose(als.mttkrp(D, Z, X, Y, "z"), np.outer(z, (x @ X) * (y @ Y)), rtol=1e-13)
    assert np.allclose(als.mttkrp(D, Z, X, Y, "x"), np.outer(x, (z @ Z) * (y @ Y)), rtol=1e-13)
    assert np.allclose(als.mttkrp(D, Z, X, Y, "y"), np.outer(y, (z @ Z) * (x @ X)), rtol=1e-13)


def test_mttkrp_elementwise_triple_loop():
    """M_z[z, r] = sum_{x,y} D[z,x,y] X[x,r] Y[y,r] etc., by explicit loops on a tiny tensor."""
    rng = np.random.default_rng(5)
    P, A1, A2, R = 3, 4, 2, 2
    D = rng.random((P, A1, A2))
    Z, X, Y = rng.random((P, R)), rng.random((A1, R)), rng.random((A2, R))
    Mz, Mx, My = np.zeros((P, R)), np.zeros((A1, R)), np.zeros((A2, R))
    for a in range(P):
        for b in range(A1):
            for c in range(A2):
                for r in range(R):
                    Mz[a, r] += D[a, b, c] * X[b, r] * Y[c, r]
                    Mx[b, r] += D[a, b, c] * Z[a, r] * Y[c, r]
                    My[c, r] += D[a, b, c] * Z[a, r] * X[b, r]
    assert np.allclose(als.mttkrp(D, Z, X, Y, "z"), Mz, rtol=1e-13)
    assert np.allclose(als.mttkrp(D, Z, X, Y, "x"), Mx, rtol=1e-13)
    assert np.allclose(als.mttkrp(D, Z, X, Y, "y"), My, rtol=1e-13)


# ---------------------------------------------------------------------------- HALS --
def _lowrank(rng, P, A, R):
    Z, X, Y = rng.random((P, R)), rng.random((A, R)), rng.random((A, R))
    return np.einsum("zr,xr,yr->zxy", Z, X, Y)


def test_hals_update_solves_unconstrained_least_squares_when_interior():
    """If the exact least-squares solution is positive, repeated HALS column passes converge to it
    (block coordinate descent on a strictly convex quadratic)."""
    rng = np.random.default_rng(6)
    K = rng.random((40, 3)) + 0.1
    Ftrue = rng.random((5, 3)) + 0.5
    T = Ftrue @ K.T
    F = rng.random((5, 3)) + 0.5
    for _ in range(400):
        F = als.hals_update(F, T @ K, K.T @ K)
    assert np.allclose(F, Ftrue, rtol=1e-8)


def test_hals_objective_is_monotone_and_recovers_exact_low_rank():
    """Each HALS block update cannot increase ||D - D_hat||; on an exactly rank-R nonnegative tensor the fit
    error goes to ~0 (Eq. 5 exact)."""
    rng = np.random.default_rng(7)
    P, A, R = 30, 6, 3
    D = _lowrank(rng, P, A, R)
    Z, X, Y, hist = als.cp_als(D, rng.random((P, R)), rng.random((A, R)), rng.random((A, R)), tol=1e-12,
                               max_sweeps=3000)
    assert all(b <= a * (1 + 1e-12) + 1e-15 for a, b in zip(hist, hist[1:]))
    assert hist[-1] < 1e-4
    Dh = np.einsum("zr,xr,yr->zxy", Z, X, Y)
    # the inner-product form of the error cancels: err^2 is exact to ~1e-14 (fp64 ulps of ||D||^2)
    assert abs((np.linalg.norm(D - Dh) / np.linalg.norm(D)) ** 2 - hist[-1] ** 2) < 1e-13


def test_fit_error_identity():
    """The fit error from inner products equals the directly computed relative residual."""
    rng = np.random.default_rng(8)
    D = rng.random((9, 4, 5))
    Z, X, Y = rng.random((9, 2)), rng.random((4, 2)), rng.random((5, 2))
    My = als.mttkrp(D, Z, X, Y, "y")
    direct = np.linalg.norm(D - np.einsum("zr,xr,yr->zxy", Z, X, Y)) / np.linalg.norm(D)
    assert math.isclose(als.fit_error(float((D * D).sum()), My, Y, Z, X), direct, rel_tol=1e-12)


def test_hals_kkt_at_convergence():
    """Nonnegative least squares optimality of each block at convergence: F >= 0, gradient
    F G - M >= 0 where F ~ 0, and ~0 where F > 0 (complementarity)."""
    rng = np.random.default_rng(9)
    cfg = _small_cfg(16, 4)
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    D = als.hist_tensor(cfg.N, cfg.s0, cfg.L, cfg.A, bins)
    P, R = D.shape[0], 3
    Z, X, Y, hist = als.cp_als(D, rng.random((P, R)), rng.random((4, R)), rng.random((4, R)), tol=1e-13,
                               max_sweeps=5000)
    for F, M, G in ((Z, als.mttkrp(D, Z, X, Y, "z"), (X.T @ X) * (Y.T @ Y)),
                    (X, als.mttkrp(D, Z, X, Y, "x"), (Z.T @ Z) * (Y.T @ Y)),
                    (Y, als.mttkrp(D, Z, X, Y, "y"), (Z.T @ Z) * (X.T @ X))):
        g = F @ G - M
        scale = np.abs(M).max()
        assert (F >= 0).all()
        assert (g > -1e-5 * scale).all()
        assert (np.abs(F * g) < 1e-5 * scale * np.abs(F).max()).all()


def test_stopping_rule_and_sweep_cap():
    """stop at relative fit-error change < tol, or at the sweep cap."""
    rng = np.random.default_rng(10)
    D = rng.random((12, 4, 4))
    init = (rng.random((12, 2)), rng.random((4, 2)), rng.random((4, 2)))
    *_, h = als.cp_als(D, *init, tol=1e-4, max_sweeps=500)
    assert len(h) < 500 and abs(h[-2] - h[-1]) < 1e-4 * h[-2]
    assert all(abs(a - b) >= 1e-4 * a for a, b in zip(h[:-2], h[1:-1]))
    *_, h3 = als.cp_als(D, *init, tol=0.0, max_sweeps=3)
    assert len(h3) == 3 and h3 == h[:3]


def test_normalise_preserves_tensor_and_masses():
    """Normalisation moves scale between factors (same D_hat); with renormalise each row's mass is 1."""
    rng = np.random.default_rng(11)
    Z, X, Y = rng.random((10, 3)), rng.random((5, 3)), rng.random((5, 3))
    C, Xn, Yn, Zn = als.normalise(Z, X, Y, renormalise=False)
    assert np.allclose(als.reconstruct(C, Xn, Yn, Zn), np.einsum("zr,xr,yr->zxy", Z, X, Y), rtol=1e-13)
    assert np.allclose(Xn.sum(0), 1) and np.allclose(Yn.sum(0), 1) and np.allclose(Zn.max(0), 1)
    C, Xn, Yn, Zn = als.normalise(Z, X, Y)
    assert np.allclose(als.reconstruct(C, Xn, Yn, Zn).sum((1, 2)), 1.0, rtol=1e-13)
