"""Pins of the oracle's hierarchical importance sampler (Sec. 5.2), CPU only.

* the returned probability is the pixel's mass over the domain's mass, read off a brute-force
  reconstruction of the blended NDF image ("the PDF ... is exactly the same as the
  evaluated NDF value" -- the descent telescopes: prod_l Q_chosen / Q_parent = pixel / root);
* Monte Carlo: the histogram of samples matches image / total (chi-square), the paper's Fig. 10
  check ("converged histogram of 10M sampled half vector directions ... exactly identical");
* with all variates at 0 the descent always takes the first nonzero quad -- checked against a
  descent on the brute-force image;
* the jittered half vector lies inside its pixel; a blank domain yields no sample.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import brute


def _store(seed=0, A=16, R=5, N=16, L=5, sparsity=0.3):
    P = sum((N >> l) ** 2 for l in range(L))
    f = synth.random_factors(A, R, P, seed=seed, sparsity=sparsity)
    return f, oracle.make_desc(N, 1, L, A, R, True)


def _image(f, d, rec):
    return brute.blended_image(d.N, d.s0, d.L, bool(d.wrap), f.C, f.X, f.Y, f.Z, rec["u"], rec["v"], rec["size"])


def test_probability_is_pixel_mass_over_domain_mass():
    f, d = _store()
    rng = np.random.default_rng(0)
    n = 300
    recs = synth.make_records(rng.uniform(0, 16, n), rng.uniform(0, 16, n), np.exp2(rng.uniform(0, 4, n)),
                              0, 15, 0, 15)
    # also sub-rectangles of odd sizes (unequal halves)
    x1 = rng.integers(0, 8, n); x2 = x1 + rng.integers(0, 8, n)
    y1 = rng.integers(0, 8, n); y2 = y1 + rng.integers(0, 8, n)
    recs[n // 2:]["rect"] = synth.pack_rect(x1, x2, y1, y2)[n // 2:]
    xi = rng.random((n, 10)).astype(np.float32)
    out = oracle.sample_batch(d, f.C, f.X, f.Y, f.Z, recs, xi)
    for i in range(n):
        img = _image(f, d, recs[i])
        r = int(recs[i]["rect"])
        a, b, c, e = r & 255, (r >> 8) & 255, (r >> 16) & 255, r >> 24
        dom = img[a:b + 1, c:e + 1]
        px, py = out["pixel"][i]
        assert a <= px <= b and c <= py <= e
        assert img[px, py] > 0
        assert out["prob"][i] == pytest.approx(img[px, py] / dom.sum(), rel=1e-10)
        hx, hy = out["h"][i]
        assert px * 2 / 16 - 1 <= hx < (px + 1) * 2 / 16 - 1
        assert py * 2 / 16 - 1 <= hy < (py + 1) * 2 / 16 - 1


def test_histogram_matches_ndf_image():
    f, d = _store(seed=3, A=8, R=4, sparsity=0.5)
    rec = synth.make_records(5.3, 9.7, 3.0, 0, 7, 0, 7)
    img = _image(f, d, rec[0])
    p = img / img.sum()
    n = 200_000
    rng = np.random.default_rng(1)
    recs = np.repeat(rec, n)
    out = oracle.sample_batch(d, f.C, f.X, f.Y, f.Z, recs, rng.random((n, 10)).astype(np.float32))
    h = np.zeros((8, 8))
    np.add.at(h, (out["pixel"][:, 0], out["pixel"][:, 1]), 1)
    assert h[p == 0].sum() == 0  # blank pixels are never sampled
    m = p > 0
    chi2 = (((h[m] - n * p[m]) ** 2) / (n * p[m])).sum()
    dof = int(m.sum()) - 1
    assert chi2 < dof + 5 * np.sqrt(2 * dof)  # ~5 sigma
    assert np.abs(h / n - p).sum() < 0.02   # relative L1 < 2% (SPEC acceptance #3)


def test_zero_variates_take_first_nonzero_quads():
    f, d = _store(seed=5, A=16, R=3, sparsity=0.6)
    rng = np.random.default_rng(4)
    n = 50
    recs = synth.make_records(rng.uniform(0, 16, n), rng.uniform(0, 16, n), np.exp2(rng.uniform(0, 4, n)),
                              0, 15, 0, 15)
    out = oracle.sample_batch(d, f.C, f.X, f.Y, f.Z, recs, np.zeros((n, 10), np.float32))
    for i in range(n):
        img = _image(f, d, recs[i])
        xa, xb, ya, yb = 0, 16, 0, 16
        while xb - xa > 1 or yb - ya > 1:  # descent on the brute-force image
            xm, ym = xa + (xb - xa + 1) // 2, ya + (yb - ya + 1) // 2
            quads = [(xa, xm, ya, ym), (xm, xb, ya, ym), (xa, xm, ym, yb), (xm, xb, ym, yb)]
            for (a, b, c, e) in quads:
                if b > a and e > c and img[a:b, c:e].sum() > 0:
                    xa, xb, ya, yb = a, b, c, e
                    break
        assert tuple(out["pixel"][i]) == (xa, ya)


def test_blank_domain_yields_no_sample():
    f, d = _store(seed=2, A=8, R=2, sparsity=0.0)
    f.X[:4] = 0.0  # x bins 0..3 carry no mass
    rec = synth.make_records(3.0, 3.0, 2.0, 0, 3, 0, 7)
    out = oracle.sample_batch(d, f.C, f.X, f.Y, f.Z, rec, np.full((1, 10), 0.5, np.float32))
    assert out["prob"][0] == 0.0 and tuple(out["pixel"][0]) == (-1, -1)
