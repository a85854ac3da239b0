"""GPU parity of the blocked / clustered store (pndf_load_blocked + pndf_query_batch) vs the fp64 oracle."""
import numpy as np
import pytest

import oracle
import synth
from tests._util import assert_parity, torch_records

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("region,wrap", [(8, True), (32, False)])
def test_blocked_store_parity(region, wrap):
    from paper_2109_14807_b200 import pndf
    cfg = synth.CONFIGS[2].scaled(wrap=wrap)
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    bs, _ = synth.build_blocked(cfg, nxy, bins, t=16, region=region)
    recs = synth.gen_queries(cfg, bins, 0, 300_000)
    rng = np.random.default_rng(2)
    m = 20_000
    x1 = rng.integers(0, cfg.A, m); x2 = np.minimum(cfg.A - 1, x1 + rng.integers(0, 40, m))
    y1 = rng.integers(0, cfg.A, m); y2 = np.minimum(cfg.A - 1, y1 + rng.integers(0, 40, m))
    recs["rect"][:m] = synth.pack_rect(x1, x2, y1, y2)  # rectangles crossing block borders
    ref = oracle.blocked_query_batch(cfg, bs, recs)
    st = pndf.load_blocked(cfg.N, cfg.s0, cfg.L, cfg.A, wrap, bs)
    out = torch.full((recs.shape[0],), float("nan"), dtype=torch.float32, device="cuda")
    st.query_batch(torch_records(recs), out, 0)
    st.sync()
    assert_parity(out.cpu().numpy(), ref, "blocked store")
    st.free()


@pytest.mark.parametrize("region,wrap,whole", [(8, True, True), (32, False, True), (8, True, False)])
def test_blocked_sampling_parity(region, wrap, whole):
    """pndf_sample_blocked vs oracle.blocked_sample_batch on the same variates: the chosen block and
    pixel agree wherever every decision (block choice and each descent level) is firm (margin > 1e-4 relative:
    the GPU takes them in fp32), and the pdf matches the oracle's pixel share of the rectangle's mass."""
    from paper_2109_14807_b200 import pndf
    cfg = synth.CONFIGS[2].scaled(wrap=wrap)
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    bs, _ = synth.build_blocked(cfg, nxy, bins, t=16, region=region)
    n = 20_000
    recs = synth.gen_queries(cfg, bins, 0, n)
    if whole:
        recs["rect"] = synth.pack_rect(0, cfg.A - 1, 0, cfg.A - 1)
    else:
        rng = np.random.default_rng(3)
        x1 = rng.integers(0, cfg.A - 30, n); y1 = rng.integers(0, cfg.A - 30, n)
        recs["rect"] = synth.pack_rect(x1, x1 + rng.integers(8, 30, n), y1, y1 + rng.integers(8, 30, n))
    recs["rect"][7] = synth.pack_rect(5, 2, 0, 0)  # invalid record -> NaN + sticky error
    xi = np.random.default_rng(11).random((n, 11), dtype=np.float32)
    ref = oracle.blocked_sample_batch(cfg, bs, recs, xi)
    st = pndf.load_blocked(cfg.N, cfg.s0, cfg.L, cfg.A, wrap, bs)
    out = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    blk = torch.empty(n, dtype=torch.int32, device="cuda")
    st.sample_blocked(torch_records(recs), torch.from_numpy(xi).cuda(), out, blk)
    assert st.sync(raise_on_query_error=False) == pndf.EQUERY
    o = out.cpu().numpy()
    pix = o[:, 3].view(np.uint32)
    b = blk.cpu().numpy()
    assert np.isnan(o[7, 2]) and pix[7] == 0xffffffff
    valid = np.arange(n) != 7
    none = valid & (ref["pixel"][:, 0] < 0)
    assert np.all(pix[none] == 0xffffffff) and np.all(o[none, 2] == 0.0) and np.all(b[none] == -1)
    firm = valid & (ref["pixel"][:, 0] >= 0) & (ref["margin"] > 1e-4)
    assert firm.sum() > 0.5 * (valid & (ref["pixel"][:, 0] >= 0)).sum()
    assert np.array_equal(b[firm], ref["block"][firm])
    assert np.array_equal((pix[firm] & 0xffff).astype(np.int64), ref["pixel"][firm, 0])
    assert np.array_equal((pix[firm] >> 16).astype(np.int64), ref["pixel"][firm, 1])
    pdf_ref = ref["prob"][firm] * cfg.A * cfg.A / 4.0
    np.testing.assert_allclose(o[firm, 2], pdf_ref, rtol=1e-4)
    h_ref = ref["h"][firm]
    np.testing.assert_allclose(o[firm, 0], h_ref[:, 0], atol=1e-6)
    np.testing.assert_allclose(o[firm, 1], h_ref[:, 1], atol=1e-6)
    st.free()
