"""GPU parity of environment-light prefiltering (pndf_sg_queries -> pndf_query_batch) vs the oracle.

The rectangle's side is floor(Q + 1/2) and its centre a bin index: both integer decisions taken from
fp32 arithmetic on the GPU and fp64 in the oracle.  They are compared exactly unless the oracle's Q
is within 1e-4 of a rounding boundary or h within 1e-5 bins of a bin edge (either neighbour is then
a correct outcome); the prefiltered NDF value is compared with the oracle's query on the GPU's rectangle.
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


@pytest.mark.parametrize("k", [2, 5])
def test_sg_rects_and_prefiltered_query(k):
    pndf = _pndf()
    if k == 5:
        cfg = synth.CONFIGS[5].scaled(N=512)
        nxy = synth.make_map(cfg)
        bins = synth.bin_map(cfg, nxy)
        f = synth.build_factors(cfg, nxy, bins)
    else:
        cfg, bins, f = config_inputs(k)
    n = 200_000
    sg = synth.gen_sg_lights(cfg, 0, n, lam=(2.0, 5000.0), amp=(0.2, 3.0))
    sg["amp"][:10] = [0.0, -1.0, np.nan, 1, 1, 1, 1, 1, 1, 1]   # invalid amplitudes
    sg["lam"][3] = 0.0
    d_sg = torch.from_numpy(sg.view(np.float32).reshape(-1, 8).copy()).cuda()
    d_q = torch.empty((n, 4), dtype=torch.int32, device="cuda")
    pndf.sg_queries(d_sg, d_q, cfg.A, eps=0.3)
    torch.cuda.synchronize()
    q = d_q.cpu().numpy().view(synth.QREC).reshape(-1)
    ref = oracle.sg_rects(sg, cfg.A, eps=0.3)
    x1, x2, y1, y2 = synth.unpack_rect(q["rect"])
    bad = ~((sg["lam"] > 0) & (sg["amp"] > 0))
    assert (x1[bad] > x2[bad]).all()                       # invalid lights -> invalid rectangles
    ok = ~bad
    assert np.array_equal(q["u"], sg["u"]) and np.array_equal(q["size"], sg["size"])
    fx = ((sg["hx"].astype(np.float64) + 1) * cfg.A / 2) % 1.0
    fy = ((sg["hy"].astype(np.float64) + 1) * cfg.A / 2) % 1.0
    edge = (np.minimum(fx, 1 - fx) < 1e-5) | (np.minimum(fy, 1 - fy) < 1e-5)
    firm = ok & (ref["q_margin"] > 1e-4) & ~edge
    assert firm.mean() > 0.99
    assert np.array_equal(q["rect"][firm], ref["rect"][firm])
    # soft cases: side within 1 of the oracle's
    rx1, rx2, _, _ = synth.unpack_rect(ref["rect"])
    assert (np.abs((x2 - x1).astype(int) - (rx2 - rx1).astype(int))[ok] <= 1).all()
    # the prefiltered query on those rectangles
    st = pndf.load_factors(pndf.make_desc(**desc_args(cfg)), f.C, f.X, f.Y, f.Z)
    out = torch.full((n,), float("nan"), dtype=torch.float32, device="cuda")
    st.query_batch(d_q, out, 0)
    assert st.sync(raise_on_query_error=False) == pndf.EQUERY  # the invalid lights
    got = out.cpu().numpy()
    exp = oracle.query_batch(oracle.desc_of(cfg), f.C, f.X, f.Y, f.Z, q, mean=True)
    assert np.isnan(got[bad]).all()
    assert_parity(got[ok], exp[ok], "sg prefiltered")
    st.free()
