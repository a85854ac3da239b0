"""numpy brute-force twin of the oracle, for tiny inputs only.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Independent of oracle.c:
it never forms segment sums of the factors.  Instead it
  1. reconstructs the dense tensor  D-hat(x, y, z) = sum_r C_r X_r(x) Y_r(y) Z_r(z)
     (Eq. 5) for the rows a query touches,
  2. blends the 8 neighbouring NDF images with their trilinear weights
     ("trilinearly blending the specific NDF values"), and
  3. sums / averages the blended image over the inclusive rectangle by an
     explicit double loop over its pixels ("perform multiple point queries at
     different pixels ... and average them").
This is BASELINE.json check 1: "the CP query equals a brute-force sum of the
reconstructed tensor over the range".
"""
from __future__ import annotations

import math

import numpy as np


def level_select(S: float, s0: int, L: int):
    """l* = clamp(log2(S/s0), 0, L-1), l0 = min(floor(l*), L-2), t = l* - l0."""
    ls = min(max(math.log2(S / s0), 0.0), L - 1.0)
    l0 = min(int(math.floor(ls)), L - 2)
    return l0, ls - l0


def axis(u: float, s: int, n: int, wrap: bool):
    f = u / s - 0.5
    i = math.floor(f)
    a = f - i
    if wrap:
        return i % n, (i + 1) % n, a
    c = lambda k: min(max(k, 0), n - 1)
    return c(i), c(i + 1), a


def reconstruct(C, X, Y, Zrow) -> np.ndarray:
    """Dense A x A NDF image of one positional index: sum_r C_r X_r (x) Y_r Z_r(z)."""
    C = np.asarray(C, np.float64)
    X = np.asarray(X, np.float64)
    Y = np.asarray(Y, np.float64)
    Zr = np.asarray(Zrow, np.float64)
    img = np.zeros((X.shape[0], Y.shape[0]))
    for r in range(C.shape[0]):
        img += C[r] * Zr[r] * np.outer(X[:, r], Y[:, r])
    return img


def blended_image(N, s0, L, wrap, C, X, Y, Z, u, v, S) -> np.ndarray:
    l0, t = level_select(float(S), s0, L)
    img = np.zeros((X.shape[0], Y.shape[0]))
    off = 0
    offs = []
    for l in range(L):
        offs.append(off)
        off += (N // (s0 << l)) ** 2
    for dl, wl in ((0, 1.0 - t), (1, t)):
        l = l0 + dl
        s = s0 << l
        n = N // s
        i0, i1, a = axis(float(u), s, n, wrap)
        j0, j1, b = axis(float(v), s, n, wrap)
        for (i, j, w) in ((i0, j0, (1 - a) * (1 - b)), (i1, j0, a * (1 - b)), (i0, j1, (1 - a) * b),
                          (i1, j1, a * b)):
            if wl * w != 0.0:
                img += wl * w * reconstruct(C, X, Y, Z[offs[l] + j * n + i])
    return img


def query(N, s0, L, wrap, C, X, Y, Z, rec, mean=True) -> float:
    r = int(rec["rect"])
    x1, x2, y1, y2 = r & 255, (r >> 8) & 255, (r >> 16) & 255, (r >> 24) & 255
    img = blended_image(N, s0, L, wrap, C, X, Y, Z, rec["u"], rec["v"], rec["size"])
    acc = 0.0
    for x in range(x1, x2 + 1):          # explicit pixel loop: repeated point queries
        for y in range(y1, y2 + 1):
            acc += img[x, y]
    if mean:
        acc /= (x2 - x1 + 1) * (y2 - y1 + 1)
    return acc
