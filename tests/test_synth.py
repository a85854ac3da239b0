"""Input generators: determinism, shard independence, basic statistics (CPU only).

The generators are stand-ins for the paper's maps; their *values* are
"parity unpinned" -- only determinism and structure are checked here.
"""
import numpy as np
import pytest

import synth


def test_maps_deterministic_and_unit():
    for k in (1, 2):
        cfg = synth.CONFIGS[k]
        a, b = synth.make_map(cfg), synth.make_map(cfg)
        assert np.array_equal(a, b)
        assert (a[..., 0] ** 2 + a[..., 1] ** 2 < 1).all()


def test_scratch_map_has_tilted_texels():
    cfg = synth.CONFIGS[4].scaled(N=256, map_params=dict(n_scr=50, width=2.0, max_tilt_deg=30.0, alpha_base=0.02))
    m = synth.make_map(cfg)
    r = np.hypot(m[..., 0], m[..., 1])
    assert (r > 0.2).mean() > 0.01 and r.max() <= np.sin(np.radians(30)) + 1e-6 + 0.2


def test_flake_count_matches_spacing():
    cfg = synth.CONFIGS[2]
    ids = synth.flake_ids(cfg)
    nc = round(cfg.N / cfg.map_params["spacing"])
    assert len(np.unique(ids)) == pytest.approx(nc * nc, rel=0.05)


def test_query_shards_are_split_independent():
    cfg = synth.CONFIGS[2]
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    full = synth.gen_queries(cfg, bins, 0, 10000)
    parts = np.concatenate([synth.gen_queries(cfg, bins, a, b) for a, b in ((0, 3333), (3333, 7001), (7001, 10000))])
    assert full.tobytes() == parts.tobytes()


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_query_records_valid(k):
    cfg = synth.CONFIGS[k]
    bins = synth.bin_map(cfg.scaled(N=64), synth.make_map(cfg.scaled(N=64))) if cfg.qdist.get("centre_mode") == 1 \
        else None
    c = cfg.scaled(N=64) if bins is not None else cfg
    q = synth.gen_queries(c, bins, 0, 20000)
    x1, x2, y1, y2 = synth.unpack_rect(q["rect"])
    assert (x1 <= x2).all() and (x2 < cfg.A).all() and (y1 <= y2).all() and (y2 < cfg.A).all()
    assert (q["u"] >= 0).all() and (q["u"] < c.N).all() and (q["size"] >= 1).all()


def test_footprint_tables():
    # level 0 (s=1): sigma = 1.5/sqrt(12) = 0.433, window |d| <= 1.73 -> 3 taps, centre 65536
    qmin, w = synth.footprint_table(1, 64)
    assert qmin == -1 and w.tolist() == [round(65536 * np.exp(-1 / (2 * 0.1875))), 65536,
                                         round(65536 * np.exp(-1 / (2 * 0.1875)))]
    # a window longer than the map folds onto N entries
    qmin, w = synth.footprint_table(64, 64)
    assert w.shape[0] == 64


def test_exact_rank_mass_is_one():
    cfg = synth.CONFIGS[2].scaled(N=128)
    f = synth.build_factors(cfg)
    assert np.allclose(f.Z.sum(1), 1.0, atol=2e-6)
    assert np.allclose(f.X.sum(0), 1.0, atol=1e-6) and np.allclose(f.Y.sum(0), 1.0, atol=1e-6)


def test_als_recovers_exact_low_rank_tensor():
    """CP-ALS (builder): an exact nonnegative rank-3 tensor is recovered (relative error < 1e-6)."""
    from synth import als
    rng = np.random.default_rng(0)
    Z, X, Y = rng.random((40, 3)), rng.random((10, 3)), rng.random((12, 3))
    D = np.einsum("zr,xr,yr->zxy", Z, X, Y)
    _, _, _, hist = als.nncp_hals(D, 3, seed=1, tol=1e-12, max_iter=3000)
    assert hist[-1] < 1e-6
    assert all(b <= a * (1 + 1e-9) for a, b in zip(hist, hist[1:]))
