"""GPU parity of the map-domain factor builder (pndf_mttkrp_map, pndf_cp_als_map; SURVEY §8(f) row 3 at
configs 3-4 scale) vs the fp64 oracle (oracle/als.py), which forms the dense tensor D explicitly.

The map path contracts over texels in fp64 and never forms D, so it factors the EXACT histogram (no tf32
rounding): its MTTKRPs match the oracle's dense MTTKRP of the exact D to ~1e-12 relative (fp64 reordering) --
asserted at 1e-9.  ||D||^2 comes from exact integer bin counts: relative 1e-12.  At config-3 size (where D
would be 366 GB) sampled Z-mode rows are checked against the oracle's rows, and the X / Y modes against the
identity sum_x M_X[x, r] X[x, r] = sum_z M_Z[z, r] Z[z, r] = <D, X_r o Y_r o Z_r> (both are the same full
contraction, computed along different passes).
"""
import numpy as np
import pytest

import synth
from oracle import als

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _pndf():
    from paper_2109_14807_b200 import pndf
    return pndf


def _inputs(N, A, R, kind=1):
    cfg = synth.CONFIGS[kind].scaled(N=N, A=A, R=R)
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    return cfg, bins


def _init(P, A, R, seed=1):
    rng = np.random.default_rng(seed)
    return rng.random((P, R)).astype(np.float32), rng.random((A, R)).astype(np.float32), \
        rng.random((A, R)).astype(np.float32)


def _run_mttkrp(cfg, bins, R, Z, X, Y, mode):
    pndf = _pndf()
    d_bins = torch.from_numpy(bins.astype(np.int16).view(np.int16)).cuda()
    M = torch.full((cfg.P if mode == 0 else cfg.A, R), float("nan"), dtype=torch.float64, device="cuda")
    nD2 = pndf.mttkrp_map(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, R, True), d_bins,
                          torch.from_numpy(Z).cuda(), torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(),
                          mode, M)
    return M.cpu().numpy(), nD2


@pytest.mark.parametrize("N,A,R,kind", [(64, 32, 8, 1), (64, 32, 40, 1), (128, 64, 32, 2), (32, 256, 16, 2),
                                        (16, 32, 8, 1)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_mttkrp_map_matches_dense_oracle(N, A, R, kind, mode):
    """Every level, ragged rank chunks (R = 40), A = 256 (slabbed bin counts), a map smaller than the top
    levels' footprint windows (N = 16: windows fold modulo N)."""
    cfg, bins = _inputs(N, A, R, kind)
    Z, X, Y = _init(cfg.P, cfg.A, R, seed=R + mode)
    got, nD2 = _run_mttkrp(cfg, bins, R, Z, X, Y, mode)
    D = als.hist_tensor(cfg.N, cfg.s0, cfg.L, cfg.A, bins)
    ref = als.mttkrp(D, Z.astype(np.float64), X.astype(np.float64), Y.astype(np.float64), "zxy"[mode])
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=0)
    assert nD2 == pytest.approx(float((D * D).sum()), rel=1e-12)


def test_mttkrp_map_config3_full_size():
    """Config 3 (2048^2 map, A = 128, R = 64, P = 5.6M; D would be 366 GB): sampled Z rows of every level vs
    the oracle's rows of D, and the three modes agree on <D, X_r o Y_r o Z_r>."""
    cfg = synth.CONFIGS[3]
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    R = cfg.R
    Z, X, Y = _init(cfg.P, cfg.A, R, seed=9)
    Mz, nD2 = _run_mttkrp(cfg, bins, R, Z, X, Y, 0)
    off = np.cumsum([0] + [(cfg.N >> l) ** 2 for l in range(cfg.L)])
    rng = np.random.default_rng(4)
    rows = np.unique(np.concatenate([rng.integers(off[l], off[l + 1], 6) for l in range(cfg.L)]))
    Dr = als.hist_rows(cfg.N, cfg.s0, cfg.L, cfg.A, bins, rows)
    ref = Dr.reshape(rows.shape[0], -1) @ als.khatri_rao(X.astype(np.float64), Y.astype(np.float64))
    np.testing.assert_allclose(Mz[rows], ref, rtol=1e-9, atol=0)
    Mx, _ = _run_mttkrp(cfg, bins, R, Z, X, Y, 1)
    My, _ = _run_mttkrp(cfg, bins, R, Z, X, Y, 2)
    tz = (Mz * Z.astype(np.float64)).sum(0)
    np.testing.assert_allclose((Mx * X.astype(np.float64)).sum(0), tz, rtol=1e-9)
    np.testing.assert_allclose((My * Y.astype(np.float64)).sum(0), tz, rtol=1e-9)
    assert nD2 > 0


@pytest.mark.parametrize("N,A,R,kind", [(64, 32, 8, 1), (64, 64, 16, 2)])
def test_cp_als_map_sweeps_match_oracle(N, A, R, kind):
    """Three sweeps from a warm start agree with the oracle's three on the exact D (as test_gpu_als does for
    the tensor path, which factors tf32(D))."""
    pndf = _pndf()
    cfg, bins = _inputs(N, A, R, kind)
    D = als.hist_tensor(cfg.N, cfg.s0, cfg.L, cfg.A, bins)
    Zi, Xi, Yi = _init(cfg.P, cfg.A, R, seed=11)
    Zw, Xw, Yw, _ = als.cp_als(D, Zi, Xi, Yi, tol=0.0, max_sweeps=30)
    Z0, X0, Y0 = (a.astype(np.float32) for a in (Zw, Xw, Yw))
    dZ, dX, dY = (torch.from_numpy(a.copy()).cuda() for a in (Z0, X0, Y0))
    d_bins = torch.from_numpy(bins.astype(np.int16).view(np.int16)).cuda()
    err = pndf.cp_als_map(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, R, True), d_bins, dZ, dX, dY,
                          max_sweeps=3, tol=0.0)
    Z, X, Y, hist = als.cp_als(D, Z0, X0, Y0, tol=0.0, max_sweeps=3)
    assert len(err) == 3
    np.testing.assert_allclose(err, hist, rtol=1e-7, atol=1e-8)
    for got, ref, what in ((dZ, Z, "Z"), (dX, X, "X"), (dY, Y, "Y")):
        scale = np.abs(ref).max(0, keepdims=True)
        rel = (np.abs(got.cpu().numpy() - ref) / scale).max()
        assert rel <= 1e-5, f"{what}: {rel:.3e}"


def test_cp_als_map_config3_runs_at_paper_settings():
    """Config 3 on one B200 (the row's 'done when'): P:308 settings capped at a few sweeps for test time;
    the fit error decreases and the normalised factors are valid store input."""
    pndf = _pndf()
    cfg = synth.CONFIGS[3]
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    Z0, X0, Y0 = _init(cfg.P, cfg.A, cfg.R, seed=1)
    dZ, dX, dY = (torch.from_numpy(a.copy()).cuda() for a in (Z0, X0, Y0))
    dC = torch.empty(cfg.R, dtype=torch.float32, device="cuda")
    d_bins = torch.from_numpy(bins.astype(np.int16).view(np.int16)).cuda()
    err = pndf.cp_als_map(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, True), d_bins, dZ, dX, dY, dC,
                          max_sweeps=6, tol=1e-4, normalise=True)
    assert len(err) >= 2 and np.all(np.diff(err) <= 1e-9)
    C, X, Y, Z = (t.cpu().numpy().astype(np.float64) for t in (dC, dX, dY, dZ))
    assert np.all(np.isfinite(Z)) and (Z >= 0).all()
    assert np.allclose(X.sum(0), 1, atol=1e-6) and np.allclose(Y.sum(0), 1, atol=1e-6)
    st = pndf.load_factors(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, True), dC.cpu().numpy(),
                           dX.cpu().numpy(), dY.cpu().numpy(), dZ)
    st.free()


def test_cp_als_map_rejects_bad_inputs():
    pndf = _pndf()
    cfg, bins = _inputs(64, 32, 8, 1)
    Z0, X0, Y0 = _init(cfg.P, cfg.A, 8)
    X0[3, 2] = -1.0
    dZ, dX, dY = (torch.from_numpy(a.copy()).cuda() for a in (Z0, X0, Y0))
    d_bins = torch.from_numpy(bins.astype(np.int16).view(np.int16)).cuda()
    with pytest.raises(pndf.PndfError):
        pndf.cp_als_map(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, 8, True), d_bins, dZ, dX, dY, max_sweeps=2)
    with pytest.raises(pndf.PndfError):  # clamped (non-periodic) maps are outside the builder's definition
        pndf.cp_als_map(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, 8, False), d_bins, dZ, dX, dY, max_sweeps=2)
