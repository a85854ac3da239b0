"""Pins of the oracle's blocked / clustered store query (Sec. 4.2), CPU only.

The blocked store built by synth.build_blocked holds exactly the same tensor as a single global CP store of
rank nb^2 R (each block's atoms embedded in the full grid), so every query -- including rectangles that cross
block boundaries (split per P:353) and blank blocks (pruned) -- must agree with the plain oracle on the
global store, which is itself pinned in test_oracle_pins.py."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("region", [8, 32])
def test_blocked_equals_global_store(region):
    cfg = synth.CONFIGS[2].scaled(N=128)
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    bs, glob = synth.build_blocked(cfg, nxy, bins, t=16, region=region)
    assert 0.5 < bs.info["blank_fraction"] < 1.0
    recs = synth.gen_queries(cfg, bins, 0, 20000)
    # also rectangles spanning several blocks and the whole grid
    rng = np.random.default_rng(1)
    x1 = rng.integers(0, cfg.A, 2000); x2 = np.minimum(cfg.A - 1, x1 + rng.integers(0, 40, 2000))
    y1 = rng.integers(0, cfg.A, 2000); y2 = np.minimum(cfg.A - 1, y1 + rng.integers(0, 40, 2000))
    recs["rect"][:2000] = synth.pack_rect(x1, x2, y1, y2)
    recs["rect"][2000:2100] = synth.pack_rect(0, cfg.A - 1, 0, cfg.A - 1)
    got = oracle.blocked_query_batch(cfg, bs, recs, mean=False)
    d = oracle.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, glob.C.shape[0], cfg.wrap)
    ref = oracle.query_batch(d, glob.C, glob.X, glob.Y, glob.Z, recs, mean=False)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(got[2000:2100], 1.0, atol=3e-6)  # full-domain mass


def test_blank_blocks_are_pruned():
    cfg = synth.CONFIGS[2].scaled(N=64)
    bs, glob = synth.build_blocked(cfg, t=16, region=8)
    nb = cfg.A // 16
    mass = glob.Z.reshape(cfg.P, nb * nb, -1).sum(axis=2)
    assert np.array_equal(bs.slab_ptr >= 0, mass > 0)
    assert bs.Z.shape[0] == int((mass > 0).sum())
