"""GPU parity of the factor builder (pndf_hist_tensor, pndf_mttkrp, pndf_cp_als) vs the
fp64 oracle (oracle/als.py).

Tolerances (DESIGN.md §5 "Factor builder"): the histogram is integer work rounded once -> bit-exact.  Every
MTTKRP term is a product of nonnegative numbers, so there is no cancellation: the tensor-core result (D exact in
tf32, factor operand split hi + lo, fp32 accumulation over K <= 2^14 terms) is within 1e-4 relative of the
fp64 oracle, element by element.  ALS sweeps compound those errors through the HALS divisions; three sweeps
from the same warm start agree column-normwise to 1e-4 and in the fit-error history to 1e-6 relative.
"""
import numpy as np
import pytest

import synth
from oracle import als
from tests._util import assert_parity

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _pndf():
    from paper_2109_14807_b200 import pndf
    return pndf


def _inputs(N, A, R, kind=1):
    cfg = synth.CONFIGS[kind].scaled(N=N, A=A, R=R)
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    return cfg, bins


def _gpu_hist(cfg, bins):
    pndf = _pndf()
    P = cfg.P
    d_bins = torch.from_numpy(bins.astype(np.int16).view(np.int16)).cuda()
    D = torch.empty((P, cfg.A, cfg.A), dtype=torch.float32, device="cuda")
    Dt = torch.empty_like(D)
    pndf.hist_tensor(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, True), d_bins, D, Dt)
    torch.cuda.synchronize()
    return D, Dt


def _init(P, A, R, seed=1):
    rng = np.random.default_rng(seed)
    return rng.random((P, R)).astype(np.float32), rng.random((A, R)).astype(np.float32), \
        rng.random((A, R)).astype(np.float32)


@pytest.mark.parametrize("N,A,kind", [(64, 32, 1), (128, 64, 2)])
def test_hist_tensor_bit_exact(N, A, kind):
    cfg, bins = _inputs(N, A, 8, kind)
    D, Dt = _gpu_hist(cfg, bins)
    ref = als.tf32_round(als.hist_tensor(cfg.N, cfg.s0, cfg.L, cfg.A, bins))
    got = D.cpu().numpy()
    assert got.tobytes() == ref.tobytes()
    assert Dt.cpu().numpy().tobytes() == np.ascontiguousarray(ref.transpose(0, 2, 1)).tobytes()


def test_hist_tensor_full_config2_sampled_rows():
    """Config 2 at full size (P = 349525 rows, 5.7 GB): sampled rows of every level bit-exact."""
    cfg, bins = _inputs(512, 64, 32, 2)
    D, _ = _gpu_hist(cfg, bins)
    off = np.cumsum([0] + [(cfg.N >> l) ** 2 for l in range(cfg.L)])
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([rng.integers(off[l], off[l + 1], 8) for l in range(cfg.L)] + [off[1:] - 1]))
    ref = als.tf32_round(als.hist_rows(cfg.N, cfg.s0, cfg.L, cfg.A, bins, rows))
    got = D[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert got.tobytes() == ref.tobytes()


@pytest.mark.parametrize("N,A,R", [(64, 32, 8), (64, 32, 32), (64, 32, 100), (64, 32, 128), (32, 128, 16)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_mttkrp_parity(N, A, R, mode):
    """Every operand width (Rp = 16..128, TMEM double buffers up to 256 columns), ragged last tiles
    (P = 5461 / 1365 rows), A = 32 .. 128 (K = A^2 up to 16384 for mode Z)."""
    pndf = _pndf()
    cfg, bins = _inputs(N, A, R, 1)
    D, Dt = _gpu_hist(cfg, bins)
    Z, X, Y = _init(cfg.P, cfg.A, R, seed=R + mode)
    out_rows = cfg.P if mode == 0 else cfg.A
    M = torch.full((out_rows, R), float("nan"), dtype=torch.float64, device="cuda")
    pndf.mttkrp(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, R, True), D, Dt, torch.from_numpy(Z).cuda(),
                torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), mode, M)
    torch.cuda.synchronize()
    Dref = D.cpu().numpy().astype(np.float64)  # bit-exact to the oracle's tf32 tensor (test above)
    ref = als.mttkrp(Dref, Z.astype(np.float64), X.astype(np.float64), Y.astype(np.float64), "zxy"[mode])
    assert_parity(M.cpu().numpy(), ref, f"mttkrp mode {'zxy'[mode]}")


def test_mttkrp_z_full_config2_sampled_rows():
    """Mode Z at config 2's full size (GEMM 349525 x 4096 x 32): sampled rows vs the oracle's rows."""
    pndf = _pndf()
    cfg, bins = _inputs(512, 64, 32, 2)
    D, Dt = _gpu_hist(cfg, bins)
    Z, X, Y = _init(cfg.P, cfg.A, 32, seed=5)
    M = torch.empty((cfg.P, 32), dtype=torch.float64, device="cuda")
    pndf.mttkrp(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, 32, True), D, Dt, torch.from_numpy(Z).cuda(),
                torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), 0, M)
    torch.cuda.synchronize()
    rows = np.unique(np.random.default_rng(6).integers(0, cfg.P, 300))
    Dr = als.tf32_round(als.hist_rows(cfg.N, cfg.s0, cfg.L, cfg.A, bins, rows)).astype(np.float64)
    ref = Dr.reshape(rows.shape[0], -1) @ als.khatri_rao(X.astype(np.float64), Y.astype(np.float64))
    assert_parity(M[torch.from_numpy(rows).cuda()].cpu().numpy(), ref, "mttkrp z (config 2 rows)")


def _cmp_factors(got, ref, what):
    """Column-normwise: |g - o| <= 1e-4 max|o[:, r]| (entries far below their column's scale come out of
    cancellations in the HALS step and carry no relative accuracy in either precision)."""
    scale = np.abs(ref).max(0, keepdims=True)
    rel = (np.abs(got - ref) / scale).max()
    assert rel <= 1e-4, f"{what}: max |g - o| / column max = {rel:.3e}"


@pytest.mark.parametrize("N,A,R,kind", [(64, 32, 8, 1), (64, 64, 16, 2), (32, 32, 96, 1)])
def test_cp_als_sweeps_match_oracle(N, A, R, kind):
    """Three sweeps from a warm start (30 oracle sweeps from a seeded init) agree with the oracle's three.
    From a cold random init the first sweeps are chaotic: rounding M_Z to fp32 alone moves the oracle's own
    fit error by 0.5% within two sweeps, so the trajectory is compared where ALS contracts."""
    pndf = _pndf()
    cfg, bins = _inputs(N, A, R, kind)
    D, Dt = _gpu_hist(cfg, bins)
    Dref = D.cpu().numpy().astype(np.float64)
    Zi, Xi, Yi = _init(cfg.P, cfg.A, R, seed=11)
    Zw, Xw, Yw, _ = als.cp_als(Dref, Zi, Xi, Yi, tol=0.0, max_sweeps=30)
    Z0, X0, Y0 = (a.astype(np.float32) for a in (Zw, Xw, Yw))
    dZ, dX, dY = (torch.from_numpy(a.copy()).cuda() for a in (Z0, X0, Y0))
    err = pndf.cp_als(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, R, True), D, Dt, dZ, dX, dY,
                      max_sweeps=3, tol=0.0)
    Z, X, Y, hist = als.cp_als(Dref, Z0, X0, Y0, tol=0.0, max_sweeps=3)
    assert len(err) == 3
    # (the error formula's cancellation leaves ~1e-8 of ||D||^2 in err^2: atol guards near-exact fits)
    np.testing.assert_allclose(err, hist, rtol=1e-6, atol=1e-6)
    _cmp_factors(dZ.cpu().numpy(), Z, "Z")
    _cmp_factors(dX.cpu().numpy(), X, "X")
    _cmp_factors(dY.cpu().numpy(), Y, "Y")


def test_cp_als_paper_settings_and_normalise():
    """P:308 (tol 1e-4, <= 500 sweeps) on config 1: converges, the error history decreases, it tracks the
    oracle's, and the normalised factors (reading 16) feed the query path: unit-sum X_r, Y_r, row masses 1."""
    pndf = _pndf()
    cfg, bins = _inputs(64, 32, 8, 1)
    D, Dt = _gpu_hist(cfg, bins)
    Z0, X0, Y0 = _init(cfg.P, cfg.A, 8, seed=1)
    dZ, dX, dY = (torch.from_numpy(a.copy()).cuda() for a in (Z0, X0, Y0))
    dC = torch.empty(8, dtype=torch.float32, device="cuda")
    err = pndf.cp_als(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, 8, True), D, Dt, dZ, dX, dY, dC,
                      max_sweeps=500, tol=1e-4, normalise=True)
    assert 2 <= len(err) < 500
    assert np.all(np.diff(err) <= 1e-7 * err[:-1])
    Dref = D.cpu().numpy().astype(np.float64)
    *_, hist = als.cp_als(Dref, Z0, X0, Y0, tol=1e-4, max_sweeps=500)
    k = min(len(err), len(hist))
    np.testing.assert_allclose(err[:k], hist[:k], rtol=1e-4)
    assert abs(err[-1] - hist[-1]) <= 1e-3 * hist[-1]
    C, X, Y, Z = (t.cpu().numpy().astype(np.float64) for t in (dC, dX, dY, dZ))
    assert np.allclose(X.sum(0), 1, atol=1e-6) and np.allclose(Y.sum(0), 1, atol=1e-6)
    assert np.allclose(Z @ C, 1, atol=1e-5)
    # the built store answers range queries like the oracle on the same factors
    f = synth.Factors(C=dC.cpu().numpy(), X=dX.cpu().numpy(), Y=dY.cpu().numpy(), Z=dZ.cpu().numpy())
    from tests._util import oracle_on, torch_records
    recs = synth.gen_queries(cfg, bins, 0, 4000)
    st = pndf.load_factors(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, 8, True), f.C, f.X, f.Y, f.Z)
    out = torch.empty(recs.shape[0], dtype=torch.float32, device="cuda")
    st.query_batch(torch_records(recs), out, 0)
    st.sync()
    st.free()
    assert_parity(out.cpu().numpy(), oracle_on(cfg, f, recs), "queries on the GPU-built store")


def test_builder_rejects_bad_inputs():
    pndf = _pndf()
    cfg, bins = _inputs(64, 32, 8, 1)
    D, Dt = _gpu_hist(cfg, bins)
    Z0, X0, Y0 = _init(cfg.P, cfg.A, 8)
    X0[3, 2] = -1.0
    dZ, dX, dY = (torch.from_numpy(a.copy()).cuda() for a in (Z0, X0, Y0))
    with pytest.raises(pndf.PndfError):
        pndf.cp_als(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, 8, True), D, Dt, dZ, dX, dY, max_sweeps=2)
    with pytest.raises(pndf.PndfError):  # A = 16 is below the builder's range
        pndf.hist_tensor(pndf.make_desc(64, 1, 7, 16, 8, True), torch.zeros((64, 64), dtype=torch.int16,
                                                                          device="cuda"), D)
