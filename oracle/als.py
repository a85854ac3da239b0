"""fp64 oracle of the GPU factor builder: footprint NDF histograms and nonnegative CP-ALS.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and bench.py's cpu_baseline leg; shares no
code with the CUDA path and never imports it.  Plain numpy, fp64, small inputs.

What it computes, in the paper's order:
  * ``hist_tensor``  -- the tensor to be factored: for every pixel footprint of every level (centre
    ((i+1/2)s, (j+1/2)s), Gaussian G_p with sigma = 1.5 s / sqrt(12)) the footprint-weighted
    histogram of the texel normals over the A x A angular grid (Eq. 2 with sigma_r -> 0), one row per
    footprint, level-major rows z = off_l + j n_l + i ("stacking all these image blocks").  Weights are the
    16-bit integer Gaussian of DESIGN.md reading 11; counts accumulate exactly; D = count / total.
  * ``tf32_round``   -- round-to-nearest-even to 11 significant bits (reading 23: the builder factors
    the tf32-representable histogram).
  * ``mttkrp``       -- the matricised-tensor-times-Khatri-Rao product of each ALS sub-problem, written with the
    Khatri-Rao matrix formed explicitly (the textbook definition).
  * ``cp_als``       -- CP decomposition by alternating least squares (Eq. 5: "maximum error
    1e-4, maximum iteration count 500"), nonnegative via HALS column updates, mode order Z, X, Y, each sweep
    ending with a per-rank norm balance; the stopping rule and init follow DESIGN.md reading 15 (relative change
    of the fit error < tol; init is an INPUT).
  * ``normalise``    -- unit-sum X_r, Y_r, weight into C_r (Z_r max = 1), per-row mass renormalisation
    (reading 16).
Pins: tests/test_oracle_als.py.
"""
from __future__ import annotations

import math

import numpy as np

HALS_EPS = 1e-30  # floor of a HALS update (keeps factors strictly positive; fp32-representable)


# ------------------------------------------------------------------ histogram tensor (Eq. 2) --
def footprint_weights(s: int, N: int):
    """1-D integer footprint weights of a level with stride s: texel k = i s + q has distance
    d = q + (1 - s)/2 to the centre (i+1/2)s; w = round(65536 exp(-d^2 / 2 sigma^2)), |d| <= 4 sigma;
    a window longer than the periodic map folds modulo N.  Returns (qmin, w[Wf])."""
    sigma = 1.5 * s / math.sqrt(12.0)
    c = 0.5 * (1.0 - s)
    qmin = math.ceil(-4.0 * sigma - c)
    qmax = math.floor(4.0 * sigma - c)
    W = qmax - qmin + 1
    Wf = min(W, N)
    w = np.zeros(Wf, np.int64)
    for q in range(qmin, qmax + 1):
        d = q + c
        w[(q - qmin) % Wf] += int(math.floor(65536.0 * math.exp(-d * d / (2.0 * sigma * sigma)) + 0.5))
    return qmin, w


def hist_tensor(N: int, s0: int, L: int, A: int, bins: np.ndarray) -> np.ndarray:
    """D[z, x, y] (fp64) for a periodic map; bins[v, u] = x + A*y (uint16) is the angular bin of texel (u, v)."""
    P = sum((N // (s0 << l)) ** 2 for l in range(L))
    return hist_rows(N, s0, L, A, bins, np.arange(P))


def hist_rows(N: int, s0: int, L: int, A: int, bins: np.ndarray, rows) -> np.ndarray:
    """The rows z of hist_tensor (for sampled checks at full size): D[k] = histogram of footprint rows[k]."""
    rows = np.asarray(rows, np.int64)
    bx = (bins.astype(np.int64) % A)
    by = (bins.astype(np.int64) // A)
    flat = (bx * A + by)  # [v, u] -> x*A + y
    off = np.cumsum([0] + [(N // (s0 << l)) ** 2 for l in range(L)])
    out = np.zeros((rows.shape[0], A, A))
    tabs = [footprint_weights(s0 << l, N) for l in range(L)]
    for k, z in enumerate(rows):
        l = int(np.searchsorted(off, z, side="right") - 1)
        s = s0 << l
        n = N // s
        c = int(z - off[l])
        i, j = c % n, c // n
        qmin, w = tabs[l]
        Wf = w.shape[0]
        tot = float(w.sum()) ** 2
        vs = (j * s + qmin + np.arange(Wf)) % N
        us = (i * s + qmin + np.arange(Wf)) % N
        win = flat[np.ix_(vs, us)]                       # [q (v), p (u)]
        ww = np.outer(w, w).astype(np.float64)           # w_y[q] * w_x[p], exact integers
        cnt = np.bincount(win.ravel(), weights=ww.ravel(), minlength=A * A)
        out[k] = (cnt / tot).reshape(A, A)
    return out


def tf32_round(x: np.ndarray) -> np.ndarray:
    """Nearest value with 11 significant bits (ties to even), returned as float32 (exact)."""
    x = np.asarray(x, np.float64)
    m, e = np.frexp(x)                      # x = m 2^e, 0.5 <= |m| < 1
    r = np.ldexp(np.rint(np.ldexp(m, 11)), e - 11)
    return r.astype(np.float32)


# --------------------------------------------------------------------------------- CP-ALS --
def khatri_rao(B: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Rows (b, c) -> B[b, :] * C[c, :] (b major)."""
    return np.einsum("br,cr->bcr", B, C).reshape(-1, B.shape[1])


def mttkrp(D: np.ndarray, Z: np.ndarray, X: np.ndarray, Y: np.ndarray, mode: str) -> np.ndarray:
    """M = D_(mode) (Khatri-Rao of the other two factors), D[z, x, y]."""
    P, A1, A2 = D.shape
    if mode == "z":
        return D.reshape(P, A1 * A2) @ khatri_rao(X, Y)
    if mode == "x":
        return D.transpose(1, 0, 2).reshape(A1, P * A2) @ khatri_rao(Z, Y)
    if mode == "y":
        return D.transpose(2, 0, 1).reshape(A2, P * A1) @ khatri_rao(Z, X)
    raise ValueError(mode)


def hals_update(F: np.ndarray, M: np.ndarray, G: np.ndarray) -> np.ndarray:
    """One HALS pass over the columns of F for min ||D_(n) - F K^T||, K^T K = G, D_(n) K = M, F >= 0:
    F[:, r] <- max(eps, F[:, r] + (M[:, r] - F G[:, r]) / G[r, r]), r = 0..R-1 in order."""
    F = F.copy()
    for r in range(F.shape[1]):
        if G[r, r] <= 0:
            continue
        F[:, r] = np.maximum(HALS_EPS, F[:, r] + (M[:, r] - F @ G[:, r]) / G[r, r])
    return F


def fit_error(nD2: float, My: np.ndarray, Y: np.ndarray, Z: np.ndarray, X: np.ndarray) -> float:
    """||D - D_hat|| / ||D|| from <D, D_hat> = sum(My * Y) and ||D_hat||^2 = sum((Z'Z)*(X'X)*(Y'Y))."""
    inner = float((My * Y).sum())
    nDh2 = float(((Z.T @ Z) * (X.T @ X) * (Y.T @ Y)).sum())
    return math.sqrt(max(0.0, nD2 - 2.0 * inner + nDh2) / nD2)


def hals_sweep(D: np.ndarray, Z: np.ndarray, X: np.ndarray, Y: np.ndarray, nD2: float):
    """One ALS sweep (modes Z, X, Y); returns the new factors and the fit error after it."""
    Z = hals_update(Z, mttkrp(D, Z, X, Y, "z"), (X.T @ X) * (Y.T @ Y))
    X = hals_update(X, mttkrp(D, Z, X, Y, "x"), (Z.T @ Z) * (Y.T @ Y))
    My = mttkrp(D, Z, X, Y, "y")
    Y = hals_update(Y, My, (Z.T @ Z) * (X.T @ X))
    err = fit_error(nD2, My, Y, Z, X)
    Z, X, Y = balance(Z, X, Y)
    return Z, X, Y, err


def balance(Z: np.ndarray, X: np.ndarray, Y: np.ndarray):
    """Rescale each rank's three columns to the geometric mean of their 2-norms (D_hat unchanged; DESIGN.md
    reading 23: keeps HALS away from the scaling drift in which one factor's column decays to the floor while
    another grows without bound)."""
    nz, nx, ny = (np.sqrt((F * F).sum(0)) for F in (Z, X, Y))
    ok = (nz > 0) & (nx > 0) & (ny > 0)
    g = np.cbrt(np.where(ok, nz * nx * ny, 1.0))
    one = np.ones_like(g)
    return (Z * np.where(ok, g / np.where(ok, nz, 1.0), one), X * np.where(ok, g / np.where(ok, nx, 1.0), one),
            Y * np.where(ok, g / np.where(ok, ny, 1.0), one))


def cp_als(D: np.ndarray, Z0: np.ndarray, X0: np.ndarray, Y0: np.ndarray, tol: float = 1e-4,
           max_sweeps: int = 500):
    """Nonnegative CP-ALS from the given init.  Stops after the first sweep whose fit error changed by
    less than tol relative to the previous sweep's, or after max_sweeps.  Returns (Z, X, Y, history)."""
    D = np.asarray(D, np.float64)
    Z, X, Y = (np.array(F, np.float64) for F in (Z0, X0, Y0))
    nD2 = float((D * D).sum())
    hist = []
    for _ in range(max_sweeps):
        Z, X, Y, err = hals_sweep(D, Z, X, Y, nD2)
        if hist and abs(hist[-1] - err) < tol * max(hist[-1], 1e-300):
            hist.append(err)
            break
        hist.append(err)
    return Z, X, Y, hist


def normalise(Z: np.ndarray, X: np.ndarray, Y: np.ndarray, renormalise: bool = True):
    """(C, X, Y, Z) with unit-sum X_r, Y_r, max_z Z_r = 1 (all-zero ranks keep C_r = 1) and, with renormalise,
    every row's reconstructed mass sum_r C_r Z_r(z) = 1 (rows of zero mass untouched)."""
    sx = X.sum(0)
    sy = Y.sum(0)
    sx = np.where(sx > 0, sx, 1.0)
    sy = np.where(sy > 0, sy, 1.0)
    X = X / sx
    Y = Y / sy
    Z = Z * (sx * sy)
    C = Z.max(0)
    C = np.where(C > 0, C, 1.0)
    Z = Z / C
    if renormalise:
        M = Z @ C
        M = np.where(M > 0, M, 1.0)
        Z = Z / M[:, None]
    return C, X, Y, Z


def reconstruct(C, X, Y, Z) -> np.ndarray:
    """D_hat[z, x, y] = sum_r C_r X_r(x) Y_r(y) Z_r(z) (Eq. 5)."""
    return np.einsum("r,xr,yr,zr->zxy", C, X, Y, Z)
