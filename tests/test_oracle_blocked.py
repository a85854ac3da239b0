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


def _blocked_fixture(N=128, t=16, region=8):
    cfg = synth.CONFIGS[2].scaled(N=N)
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    bs, glob = synth.build_blocked(cfg, nxy, bins, t=t, region=region)
    return cfg, bins, bs, glob


def _global_sum(cfg, glob, recs, x1, x2, y1, y2):
    r = recs.copy()
    r["rect"] = synth.pack_rect(x1, x2, y1, y2)
    d = oracle.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, glob.C.shape[0], cfg.wrap)
    return oracle.query_batch(d, glob.C, glob.X, glob.Y, glob.Z, r, mean=False)


@pytest.mark.parametrize("whole", [True, False])
def test_blocked_sampler_pdf_is_the_pixel_mass(whole):
    """P:389 ("the PDF ... is exactly the same as the evaluated NDF value"): prob = the sampled pixel's mass over
    the rectangle's mass, evaluated independently on the equivalent global store (block-first or not, the pmf
    of a pixel is its share of the mass).  Also: the pixel lies in the rectangle and in the chosen block."""
    cfg, bins, bs, glob = _blocked_fixture()
    n = 3000
    recs = synth.gen_queries(cfg, bins, 0, n)
    if whole:
        recs["rect"] = synth.pack_rect(0, cfg.A - 1, 0, cfg.A - 1)
    else:  # rectangles crossing block borders
        rng = np.random.default_rng(2)
        x1 = rng.integers(0, cfg.A - 30, n); y1 = rng.integers(0, cfg.A - 30, n)
        recs["rect"] = synth.pack_rect(x1, x1 + rng.integers(8, 30, n), y1, y1 + rng.integers(8, 30, n))
    xi = np.random.default_rng(5).random((n, 11), dtype=np.float32)
    res = oracle.blocked_sample_batch(cfg, bs, recs, xi)
    ok = res["pixel"][:, 0] >= 0
    assert ok.mean() > (0.9 if whole else 0.3)
    r0 = recs["rect"][~ok]  # no sample exactly where the rectangle holds no mass
    assert np.all(_global_sum(cfg, glob, recs[~ok], r0 & 255, (r0 >> 8) & 255, (r0 >> 16) & 255, r0 >> 24) <= 1e-15)
    assert np.all(res["prob"][~ok] == 0.0)
    px, py = res["pixel"][ok, 0], res["pixel"][ok, 1]
    r = recs["rect"][ok]
    assert np.all((px >= (r & 255)) & (px <= ((r >> 8) & 255)) & (py >= ((r >> 16) & 255)) & (py <= (r >> 24)))
    nb = cfg.A // bs.t
    assert np.array_equal(res["block"][ok], (py // bs.t) * nb + px // bs.t)
    pix_mass = _global_sum(cfg, glob, recs[ok], px, px, py, py)
    rect_mass = _global_sum(cfg, glob, recs[ok], r & 255, (r >> 8) & 255, (r >> 16) & 255, r >> 24)
    np.testing.assert_allclose(res["prob"][ok], pix_mass / rect_mass, rtol=1e-9)


def test_blocked_sampler_frequencies():
    """One footprint, 60000 samples: every block is chosen with frequency ~ its mass share and every pixel
    with frequency ~ its pmf (binomial 5-sigma bounds)."""
    cfg, bins, bs, glob = _blocked_fixture(N=64)
    m = 60000
    rec = synth.gen_queries(cfg, bins, 7, 8)
    rec["rect"] = synth.pack_rect(0, cfg.A - 1, 0, cfg.A - 1)
    recs = np.repeat(rec, m)
    xi = np.random.default_rng(9).random((m, 11), dtype=np.float32)
    res = oracle.blocked_sample_batch(cfg, bs, recs, xi)
    assert (res["pixel"][:, 0] >= 0).all()
    t, nb = bs.t, cfg.A // bs.t
    tot = _global_sum(cfg, glob, rec, 0, cfg.A - 1, 0, cfg.A - 1)[0]
    freq = np.bincount(res["block"], minlength=nb * nb) / m
    for b in range(nb * nb):
        bx, by = b % nb, b // nb
        p = _global_sum(cfg, glob, rec, bx * t, bx * t + t - 1, by * t, by * t + t - 1)[0] / tot
        assert abs(freq[b] - p) <= 5 * np.sqrt(max(p * (1 - p), 1e-12) / m) + 1e-12, (b, freq[b], p)
    key = res["pixel"][:, 1] * cfg.A + res["pixel"][:, 0]
    u, cnt = np.unique(key, return_counts=True)
    pm = {k: res["prob"][np.argmax(key == k)] for k in u}
    for k, c in zip(u, cnt):
        p = pm[k]
        assert abs(c / m - p) <= 5 * np.sqrt(p * (1 - p) / m) + 1e-12
