"""Pins of the oracle's environment-prefiltering rectangle (Sec. 5.4), CPU only."""
import math

import numpy as np
import pytest

import oracle
import synth


def _sg(lam, amp, hx=0.0, hy=0.0):
    lam = np.atleast_1d(np.asarray(lam, np.float32))
    out = np.zeros(lam.shape[0], synth.SGREC)
    out["lam"] = lam
    out["amp"] = amp
    out["hx"] = hx
    out["hy"] = hy
    out["size"] = 1.0
    return out


def test_compact_support_angle_inverts_the_formula():
    """cos(theta) = 1 + (ln eps - ln A)/lambda, checked through the cosine."""
    rng = np.random.default_rng(0)
    lam = np.exp(rng.uniform(np.log(2.0), np.log(5000.0), 1000)).astype(np.float32)
    amp = rng.uniform(0.4, 3.0, 1000).astype(np.float32)
    r = oracle.sg_rects(_sg(lam, amp), 256, eps=0.3)
    rhs = 1.0 + (math.log(0.3) - np.log(amp.astype(np.float64))) / lam.astype(np.float64)
    inside = (rhs > -1) & (rhs < 1)
    np.testing.assert_allclose(np.cos(r["theta"][inside]), rhs[inside], atol=1e-12)
    assert (r["theta"][rhs >= 1] == 0).all() and (r["theta"][rhs <= -1] == np.pi).all()


def test_spec_example_and_side_length():
    """A=1, lambda=25, eps=0.3 -> theta = arccos(0.95184) = 0.3116 rad, Q = 256 theta / pi = 25.39 (
    P:426: Q = 256 (theta/2)/pi * 2)."""
    r = oracle.sg_rects(_sg(25.0, 1.0), 256, eps=0.3)
    assert r["theta"][0] == pytest.approx(0.31161, abs=2e-5)
    assert r["Q"][0] == pytest.approx(25.392, abs=2e-3)
    x1, x2, y1, y2 = synth.unpack_rect(r["rect"])
    assert x2[0] - x1[0] + 1 == 25 and y2[0] - y1[0] + 1 == 25
    # centred on the bin of h = (0, 0): bin 128, side 25 -> [116, 140]
    assert (x1[0], x2[0]) == (116, 140)


def test_limits_monotonicity_and_clipping():
    # theta decreases with lambda (fixed A, eps)
    lam = np.exp(np.linspace(np.log(1.0), np.log(1e6), 50)).astype(np.float32)
    th = oracle.sg_rects(_sg(lam, 1.0), 64)["theta"]
    assert (np.diff(th) <= 0).all()
    # a very narrow lobe is a point query, a very wide one covers the image (clamps S:465-483)
    r = oracle.sg_rects(_sg([1e9, 0.05], 1.0), 64)
    x1, x2, y1, y2 = synth.unpack_rect(r["rect"])
    assert x2[0] == x1[0] and y2[0] == y1[0]
    assert (x1[1], x2[1], y1[1], y2[1]) == (0, 63, 0, 63)
    # near the grid edge the square shifts inside, keeping its side
    r = oracle.sg_rects(_sg(40.0, 1.0, hx=0.999, hy=-0.999), 64)
    x1, x2, y1, y2 = synth.unpack_rect(r["rect"])
    side = int(math.floor(r["Q"][0] + 0.5))
    assert x2[0] == 63 and y1[0] == 0 and x2[0] - x1[0] + 1 == side and y2[0] - y1[0] + 1 == side
