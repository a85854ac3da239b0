"""GPU parity of implicit Wang-tiled queries (pndf_load_tiles + pndf_query_batch) vs the fp64 oracle."""
import numpy as np
import pytest

import oracle
import synth
from tests._util import assert_parity, torch_records

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _pndf():
    from paper_2109_14807_b200 import pndf
    return pndf


def _tile_queries(tc, n, seed):
    rng = np.random.default_rng(seed)
    A = tc.A
    w = rng.uniform(0.5, 4.0, (n, 2))
    side = np.maximum(1, np.floor(2 * w + 0.5)).astype(np.int64)
    x1 = rng.integers(0, A - side[:, 0] + 1)
    y1 = rng.integers(0, A - side[:, 1] + 1)
    return synth.make_records(rng.uniform(0, tc.world, n), rng.uniform(0, tc.world, n),
                              np.exp2(rng.uniform(0, np.log2(tc.T), n)), x1, x1 + side[:, 0] - 1, y1,
                              y1 + side[:, 1] - 1)


@pytest.mark.parametrize("prefix", [0, 2])
def test_tiled_query_parity(prefix):
    pndf = _pndf()
    tc = synth.TileConfig(T=128)
    tiles = synth.wang_tiles(tc)
    f = synth.wang_factors(tc, tiles)
    recs = _tile_queries(tc, 100_000, 1)
    recs[:100]["u"] = np.arange(100, dtype=np.float32) * tc.T  # exactly on tile borders
    td_o = oracle.TilesDesc(T=tc.T, s0=tc.s0, L=tc.L, margin=tc.margin, A=tc.A, R=tc.R, seed=tc.seed)
    ref = oracle.tiled_query_batch(td_o, f.C, f.X, f.Y, f.Z, recs)
    st = pndf.load_tiles(pndf.make_tile_desc(tc.T, tc.s0, tc.L, tc.margin, tc.A, tc.R, tc.seed, prefix=prefix),
                         f.C, f.X, f.Y, f.Z)
    out = torch.full((recs.shape[0],), float("nan"), dtype=torch.float32, device="cuda")
    st.query_batch(torch_records(recs), out, 0)
    st.sync()
    assert_parity(out.cpu().numpy(), ref, "wang tiled")
    # full angular domain: the footprint's total mass, 1 for any world footprint (tiles' partials add up)
    full = recs[:5000].copy()
    full["rect"] = synth.pack_rect(0, tc.A - 1, 0, tc.A - 1)
    o2 = torch.empty(5000, dtype=torch.float32, device="cuda")
    st.query_batch(torch_records(full), o2, 1)  # PNDF_SUM
    st.sync()
    np.testing.assert_allclose(o2.cpu().numpy(), 1.0, atol=2e-5)
    xi = torch.zeros((4, 10), dtype=torch.float32, device="cuda")
    with pytest.raises(pndf.PndfError):
        st.sample_batch(torch_records(recs[:4]), xi, torch.empty((4, 4), dtype=torch.float32, device="cuda"))
    st.free()


@pytest.mark.parametrize("prefix", [0, 2])
def test_tiled_sample_parity(prefix):
    """pndf_sample_tiles vs oracle.tiled_sample_batch (Sec. 5.5; reading 25).  The tile
    choice is an integer decision from exact inputs (covered = positive mass; c = floor(xi * count) in fp32
    on both sides): compared exactly.  Quad decisions are fp32 vs fp64 comparisons: pixels compared exactly
    where the oracle's margin exceeds 1e-4, otherwise checked for validity; the pdf is the full NDF value of
    the GPU's own pixel (oracle tiled query)."""
    pndf = _pndf()
    tc = synth.TileConfig(T=128)
    f = synth.wang_factors(tc, synth.wang_tiles(tc))
    n = 20_000
    recs = _tile_queries(tc, n, 3)
    recs["rect"][::2] = synth.pack_rect(0, tc.A - 1, 0, tc.A - 1)  # half: the whole image
    recs[:64]["u"] = np.arange(64, dtype=np.float32) * tc.T          # exactly on tile borders
    xi = np.random.default_rng(4).random((n, 11), dtype=np.float32)
    td_o = oracle.TilesDesc(T=tc.T, s0=tc.s0, L=tc.L, margin=tc.margin, A=tc.A, R=tc.R, seed=tc.seed)
    ref = oracle.tiled_sample_batch(td_o, f.C, f.X, f.Y, f.Z, recs, xi)
    st = pndf.load_tiles(pndf.make_tile_desc(tc.T, tc.s0, tc.L, tc.margin, tc.A, tc.R, tc.seed, prefix=prefix),
                         f.C, f.X, f.Y, f.Z)
    out = torch.full((n, 4), float("nan"), dtype=torch.float32, device="cuda")
    tile = torch.full((n, 2), -99, dtype=torch.int32, device="cuda")
    st.sample_tiles(torch_records(recs), torch.from_numpy(xi).cuda(), out, tile)
    st.sync()
    o = out.cpu().numpy()
    gt = tile.cpu().numpy()
    pixel = o[:, 3].view(np.uint32)
    np.testing.assert_array_equal(gt, ref["tile"])
    assert (ref["count"] > 1).sum() > n // 4  # many footprints straddle tiles
    none_g = pixel == 0xffffffff
    none_o = ref["pixel"][:, 0] < 0
    assert np.array_equal(none_g, none_o)
    assert not none_o[::2].any()  # a covered tile has mass on the whole image
    ok = ~none_o
    gx = (pixel & 0xffff).astype(np.int64)
    gy = (pixel >> 16).astype(np.int64)
    firm = ok & (ref["margin"] > 1e-4)
    assert firm.sum() > 0.9 * ok.sum()
    assert np.array_equal(gx[firm], ref["pixel"][firm, 0]) and np.array_equal(gy[firm], ref["pixel"][firm, 1])
    A = tc.A
    np.testing.assert_allclose(o[ok, 0], (gx[ok] + xi[ok, 8].astype(np.float64)) * 2.0 / A - 1.0, atol=2e-6)
    np.testing.assert_allclose(o[ok, 1], (gy[ok] + xi[ok, 9].astype(np.float64)) * 2.0 / A - 1.0, atol=2e-6)
    pix = recs[ok].copy()
    pix["rect"] = synth.pack_rect(gx[ok], gx[ok], gy[ok], gy[ok])
    num = oracle.tiled_query_batch(td_o, f.C, f.X, f.Y, f.Z, pix, mean=False)
    den = oracle.tiled_query_batch(td_o, f.C, f.X, f.Y, f.Z, recs[ok], mean=False)
    assert (num > 0).all()
    assert_parity(o[ok, 2].astype(np.float64), num / den * (A * A / 4.0), "tiled sampler pdf")
    # invalid record -> NaN pdf + sticky PNDF_EQUERY; plain stores reject pndf_sample_tiles
    bad = recs[:2].copy()
    bad["size"][0] = -1.0
    st.sample_tiles(torch_records(bad), torch.from_numpy(xi[:2]).cuda(), out[:2])
    assert st.sync(raise_on_query_error=False) == pndf.EQUERY
    assert np.isnan(out[0, 2].item())
    st.free()


def test_tiled_sample_level_sort_is_bitwise_neutral():
    """Batches >= 65536 are sampled in footprint-level order (pndf_sample_tiles' level sort): every
    record's sample, pdf and chosen tile must be bitwise those of the unsorted (PNDF_BIN_OFF) run."""
    pndf = _pndf()
    tc = synth.TileConfig(T=128)
    f = synth.wang_factors(tc, synth.wang_tiles(tc))
    n = 200_000
    recs = _tile_queries(tc, n, 9)
    recs["rect"][::3] = synth.pack_rect(0, tc.A - 1, 0, tc.A - 1)
    recs["size"][5] = float("nan")  # one invalid record: NaN wherever it lands in the sorted order
    xi = torch.from_numpy(np.random.default_rng(10).random((n, 11), dtype=np.float32)).cuda()
    st = pndf.load_tiles(pndf.make_tile_desc(tc.T, tc.s0, tc.L, tc.margin, tc.A, tc.R, tc.seed), f.C, f.X, f.Y, f.Z)
    outs = []
    for opts in (0, pndf.BIN_OFF):
        out = torch.full((n, 4), -1.0, dtype=torch.float32, device="cuda")
        tile = torch.full((n, 2), -99, dtype=torch.int32, device="cuda")
        st.sample_tiles(torch_records(recs), xi, out, tile, opts)
        assert st.sync(raise_on_query_error=False) == pndf.EQUERY
        outs.append((out.cpu().numpy(), tile.cpu().numpy()))
        if opts == 0:
            assert st.stats()["last_binned"] == 1
    assert outs[0][0].tobytes() == outs[1][0].tobytes()
    assert np.array_equal(outs[0][1], outs[1][1])
    assert np.isnan(outs[0][0][5, 2]) and (outs[0][0][:, 3].view(np.uint32) != 0xffffffff).sum() > n // 4
    st.free()


def test_tiled_query_level_sort_is_bitwise_neutral():
    """Tiled query batches >= 65536 run in footprint-level order; results must be bitwise those of the
    caller's-order run (PNDF_BIN_OFF), including the NaN of an invalid record."""
    pndf = _pndf()
    tc = synth.TileConfig(T=128)
    f = synth.wang_factors(tc, synth.wang_tiles(tc))
    n = 200_000
    recs = _tile_queries(tc, n, 11)
    recs["size"][7] = -2.0
    st = pndf.load_tiles(pndf.make_tile_desc(tc.T, tc.s0, tc.L, tc.margin, tc.A, tc.R, tc.seed), f.C, f.X, f.Y, f.Z)
    res = []
    for opts in (0, pndf.BIN_OFF):
        out = torch.full((n,), -1.0, dtype=torch.float32, device="cuda")
        st.query_batch(torch_records(recs), out, opts)
        assert st.sync(raise_on_query_error=False) == pndf.EQUERY
        assert st.stats()["last_binned"] == (1 if opts == 0 else 0)
        res.append(out.cpu().numpy())
    assert res[0].tobytes() == res[1].tobytes() and np.isnan(res[0][7])
    st.free()


def _random_tile_store(T, s0, L, margin, A, R, seed, outer_zero_beyond=None):
    """Random nonnegative tiled factors whose rows are nonzero out to the whole margin (or, with
    outer_zero_beyond = d, zero beyond d cells past the tile)."""
    P_ext = sum(((T // s0 >> l) + 2 * margin) ** 2 for l in range(L))
    f = synth.random_factors(A, R, 16 * P_ext, seed=seed, sparsity=0.3)
    if outer_zero_beyond is not None:
        Z = f.Z.reshape(16, P_ext, R)
        off = 0
        for l in range(L):
            nl = T // s0 >> l
            ne = nl + 2 * margin
            jl, il = np.divmod(np.arange(ne * ne), ne)
            il, jl = il - margin, jl - margin
            d = np.maximum(np.maximum(np.maximum(-il, il - (nl - 1)), np.maximum(-jl, jl - (nl - 1))), 0)
            Z[:, off + np.flatnonzero(d > outer_zero_beyond), :] = 0
            off += ne * ne
    return f


@pytest.mark.parametrize("margin,zero_beyond", [(3, None), (4, None), (4, 1), (6, None)])
def test_tiled_store_full_margin(margin, zero_beyond):
    """pndf.h: a tiled query sums every tile whose extended grid holds each neighbour ("all
    overlapping Wang tiles").  A random store with nonzero rows out to the whole margin (the synthetic
    flake tiles stop at 2 cells) must match the oracle, which sums every margin row; the measured reach
    is the margin (or the zeroed ring's inner edge).  The sampler covers reach <= 4 and rejects larger."""
    pndf = _pndf()
    T, s0, L, A, R, seed = 8, 1, 4, 16, 8, 5
    f = _random_tile_store(T, s0, L, margin, A, R, seed=margin, outer_zero_beyond=zero_beyond)
    want_reach = margin if zero_beyond is None else zero_beyond
    rng = np.random.default_rng(margin)
    n = 6000
    world = 40 * T
    x1 = rng.integers(0, A, n)
    y1 = rng.integers(0, A, n)
    recs = synth.make_records(rng.uniform(0, world, n), rng.uniform(0, world, n), np.exp2(rng.uniform(0, L + 1, n)),
                              x1, np.minimum(A - 1, x1 + rng.integers(0, 5, n)), y1,
                              np.minimum(A - 1, y1 + rng.integers(0, 5, n)))
    td_o = oracle.TilesDesc(T=T, s0=s0, L=L, margin=margin, A=A, R=R, seed=seed)
    ref = oracle.tiled_query_batch(td_o, f.C, f.X, f.Y, f.Z, recs)
    for prefix in (0, 2):
        st = pndf.load_tiles(pndf.make_tile_desc(T, s0, L, margin, A, R, seed, prefix=prefix), f.C, f.X, f.Y, f.Z)
        assert st.stats()["tile_reach"] == want_reach
        out = torch.full((n,), float("nan"), dtype=torch.float32, device="cuda")
        st.query_batch(torch_records(recs), out, 0)
        st.sync()
        assert_parity(out.cpu().numpy(), ref, f"tiled margin={margin} prefix={prefix}")
        xi_np = np.random.default_rng(margin + 1).random((n, 11), dtype=np.float32)
        xi = torch.from_numpy(xi_np).cuda()
        so = torch.full((n, 4), float("nan"), dtype=torch.float32, device="cuda")
        tile = torch.full((n, 2), -99, dtype=torch.int32, device="cuda")
        if want_reach > 4:
            with pytest.raises(pndf.PndfError):
                st.sample_tiles(torch_records(recs), xi, so, tile)
            st.free()
            continue
        st.sample_tiles(torch_records(recs), xi, so, tile)
        st.sync()
        st.free()
        sref = oracle.tiled_sample_batch(td_o, f.C, f.X, f.Y, f.Z, recs, xi_np)
        np.testing.assert_array_equal(tile.cpu().numpy(), sref["tile"])  # tile choice: exact
        o = so.cpu().numpy()
        pixel = o[:, 3].view(np.uint32)
        ok = pixel != 0xffffffff
        assert np.array_equal(~ok, sref["pixel"][:, 0] < 0)
        gx, gy = (pixel & 0xffff).astype(np.int64), (pixel >> 16).astype(np.int64)
        firm = ok & (sref["margin"] > 1e-4)
        assert firm.sum() > 0.9 * ok.sum()
        assert np.array_equal(gx[firm], sref["pixel"][firm, 0]) and np.array_equal(gy[firm], sref["pixel"][firm, 1])
        pix = recs[ok].copy()
        pix["rect"] = synth.pack_rect(gx[ok], gx[ok], gy[ok], gy[ok])
        num = oracle.tiled_query_batch(td_o, f.C, f.X, f.Y, f.Z, pix, mean=False)
        den = oracle.tiled_query_batch(td_o, f.C, f.X, f.Y, f.Z, recs[ok], mean=False)
        assert_parity(o[ok, 2].astype(np.float64), num / den * (A * A / 4.0), f"tiled pdf margin={margin}")


def test_tiled_capture_without_scratch_runs_unsorted():
    """A tiled batch >= 65536 captured into a CUDA graph before the store has sort scratch runs in the
    caller's order (no allocation during capture) and gives the same bits as the sorted run."""
    pndf = _pndf()
    tc = synth.TileConfig(T=128)
    f = synth.wang_factors(tc, synth.wang_tiles(tc))
    n = 100_000
    recs = _tile_queries(tc, n, 21)
    st = pndf.load_tiles(pndf.make_tile_desc(tc.T, tc.s0, tc.L, tc.margin, tc.A, tc.R, tc.seed), f.C, f.X, f.Y, f.Z)
    assert st.stats()["tile_reach"] == 2
    q = torch_records(recs)
    out = torch.zeros(n, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            st.query_batch(q, out, 0, stream=s)
        g.replay()
        s.synchronize()
    captured = out.cpu().numpy().copy()
    out2 = torch.zeros(n, dtype=torch.float32, device="cuda")
    st.query_batch(q, out2, 0)
    st.sync()
    assert st.stats()["last_binned"] == 1
    assert captured.tobytes() == out2.cpu().numpy().tobytes()
    st.free()
