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
