"""GPU parity of the batched hierarchical importance sampler (pndf_sample_batch) vs the fp64 oracle.

Both sides consume the same caller-supplied variates.  A quad decision is a floating-point
comparison (t = xi * total vs cumulative quad sums), taken in fp32 on the GPU and in fp64 in
the oracle, so the sampled pixel is compared exactly wherever the oracle's decision margin
exceeds 1e-4 (relative); elsewhere (either neighbouring quad is a correct outcome) the GPU's
pixel is checked to be valid and its pdf to equal the oracle's NDF value of that pixel.
"""
import numpy as np
import pytest

import oracle
import synth
from tests._util import assert_parity, config_inputs, desc_args, torch_records

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _pndf():
    from paper_2109_14807_b200 import pndf
    return pndf


def _run(d_args, f, recs, xi, opts=0, prefix=0):
    pndf = _pndf()
    st = pndf.load_factors(pndf.make_desc(**d_args, prefix=prefix), f.C, f.X, f.Y, f.Z)
    out = torch.full((recs.shape[0], 4), float("nan"), dtype=torch.float32, device="cuda")
    st.sample_batch(torch_records(recs), torch.from_numpy(xi).cuda(), out, opts)
    status = st.sync(raise_on_query_error=False)
    o = out.cpu().numpy()
    st.free()
    res = np.empty(recs.shape[0], pndf.SAMPLE_DTYPE)
    res["hx"], res["hy"], res["pdf"] = o[:, 0], o[:, 1], o[:, 2]
    res["pixel"] = o[:, 3].view(np.uint32)
    return res, status


def _check(cfg_like, f, recs, xi, got):
    d = oracle.make_desc(cfg_like["N"], cfg_like["s0"], cfg_like["L"], cfg_like["A"], cfg_like["R"], cfg_like["wrap"])
    A = cfg_like["A"]
    ref = oracle.sample_batch(d, f.C, f.X, f.Y, f.Z, recs, xi)
    gx = (got["pixel"] & 0xffff).astype(np.int64)
    gy = (got["pixel"] >> 16).astype(np.int64)
    none_g = got["pixel"] == 0xffffffff
    none_o = ref["pixel"][:, 0] < 0
    assert np.array_equal(none_g, none_o)
    ok = ~none_o
    firm = ok & (ref["margin"] > 1e-4)
    assert np.array_equal(gx[firm], ref["pixel"][firm, 0]) and np.array_equal(gy[firm], ref["pixel"][firm, 1])
    # jittered half vector of the GPU's own pixel
    hx = (gx + xi[:, 8].astype(np.float64)) * 2.0 / A - 1.0
    hy = (gy + xi[:, 9].astype(np.float64)) * 2.0 / A - 1.0
    np.testing.assert_allclose(got["hx"][ok], hx[ok], atol=2e-6)
    np.testing.assert_allclose(got["hy"][ok], hy[ok], atol=2e-6)
    # pdf = pixel mass / domain mass / (2/A)^2, evaluated by the oracle at the GPU's pixel
    pix = recs[ok].copy()
    pix["rect"] = synth.pack_rect(gx[ok], gx[ok], gy[ok], gy[ok])
    num = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, pix, mean=False)
    den = oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs[ok], mean=False)
    assert (num > 0).all()
    assert_parity(got["pdf"][ok], num / den * (A * A / 4.0), "sampler pdf")
    return int(firm.sum()), int(ok.sum() - firm.sum())


@pytest.mark.parametrize("shape", [(16, 1, 5, 16, 5, True), (32, 1, 6, 64, 40, False), (16, 1, 5, 256, 256, True),
                                   (64, 2, 5, 37, 9, True)])
@pytest.mark.parametrize("prefix", [0, 2])
def test_sampler_parity_random_stores(shape, prefix):
    N, s0, L, A, R, wrap = shape
    P = sum((N // (s0 << l)) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=A + R, sparsity=0.4)
    rng = np.random.default_rng(A * R)
    n = 2000
    x1 = rng.integers(0, A, n); x2 = np.minimum(A - 1, x1 + rng.integers(0, A, n))
    y1 = rng.integers(0, A, n); y2 = np.minimum(A - 1, y1 + rng.integers(0, A, n))
    recs = synth.make_records(rng.uniform(-N, 2 * N, n), rng.uniform(-N, 2 * N, n),
                              np.exp2(rng.uniform(-1, L + 1, n)), x1, x2, y1, y2)
    recs["rect"][: n // 2] = synth.pack_rect(0, A - 1, 0, A - 1)  # half of them sample the whole image
    xi = rng.random((n, 10)).astype(np.float32)
    args = dict(N=N, s0=s0, L=L, A=A, R=R, wrap=wrap)
    got, st = _run(args, f, recs, xi, prefix=prefix)
    assert st == 0
    firm, soft = _check(args, f, recs, xi, got)
    assert firm > 0.99 * (firm + soft)
    got_b, _ = _run(args, f, recs, xi, opts=2, prefix=prefix)
    assert got_b.tobytes() == got.tobytes()  # binning never changes a bit


@pytest.mark.parametrize("k", [2, 5])
def test_sampler_parity_configs(k):
    if k == 5:
        cfg = synth.CONFIGS[5].scaled(N=512)
        nxy = synth.make_map(cfg)
        bins = synth.bin_map(cfg, nxy)
        f = synth.build_factors(cfg, nxy, bins)
    else:
        cfg, bins, f = config_inputs(k)
    recs = synth.gen_queries(cfg, bins, 0, 20_000)
    recs["rect"] = synth.pack_rect(0, cfg.A - 1, 0, cfg.A - 1)
    xi = np.random.default_rng(k).random((recs.shape[0], 10)).astype(np.float32)
    got, st = _run(desc_args(cfg), f, recs, xi)
    assert st == 0
    _check(desc_args(cfg), f, recs, xi, got)


def test_sampler_histogram_matches_ndf():
    """Fig. 10 / P:389: the histogram of samples equals the evaluated NDF image (1M samples, config 2)."""
    cfg, bins, f = config_inputs(2)
    A = cfg.A
    n = 1_000_000
    rec = synth.make_records(100.3, 200.7, 24.0, 0, A - 1, 0, A - 1)
    recs = np.repeat(rec, n)
    xi = np.random.default_rng(9).random((n, 10)).astype(np.float32)
    got, _ = _run(desc_args(cfg), f, recs, xi)
    h = np.zeros((A, A))
    np.add.at(h, (got["pixel"] & 0xffff, got["pixel"] >> 16), 1)
    xs, ys = np.meshgrid(np.arange(A), np.arange(A), indexing="ij")
    pix = np.repeat(rec, A * A)
    pix["rect"] = synth.pack_rect(xs.ravel(), xs.ravel(), ys.ravel(), ys.ravel())
    img = oracle.query_batch(oracle.desc_of(cfg), f.C, f.X, f.Y, f.Z, pix, mean=False).reshape(A, A)
    p = img / img.sum()
    assert h[p == 0].sum() == 0
    assert np.abs(h / n - p).sum() < 0.02


def test_sampler_blank_and_invalid():
    pndf = _pndf()
    N, s0, L, A, R = 16, 1, 5, 8, 2
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=2)
    f.X[:4] = 0.0
    recs = synth.make_records([3.0, 3.0, np.nan], [3.0, 3.0, 1.0], [2.0, 2.0, 1.0], [0, 0, 0], [3, 7, 7],
                              [0, 0, 0], [7, 7, 7])
    got, st = _run(dict(N=N, s0=s0, L=L, A=A, R=R, wrap=True), f, recs, np.full((3, 10), 0.5, np.float32))
    assert st == pndf.EQUERY
    assert got["pixel"][0] == 0xffffffff and got["pdf"][0] == 0 and np.isnan(got["hx"][0])
    assert got["pixel"][1] != 0xffffffff and got["pdf"][1] > 0
    assert got["pixel"][2] == 0xffffffff and np.isnan(got["pdf"][2])
