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
