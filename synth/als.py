"""Nonnegative CP-ALS (HALS updates) for the config-1 factors.

BASELINE.json configs[0]: "CP rank R=8 factors fp32, nonnegative, from CPU CP-ALS".
Paper: CP decomposition by alternating least squares, "maximum error set as
10^-4 and maximum iteration count set as 500".  Readings:
  * "maximum error 1e-4" = relative change of the fit error per sweep;
  * init: seeded uniform [0,1); nonnegativity by HALS column updates;
  * post-fit: X_r, Y_r scaled to unit sum, scale moved into C_r (Z_r max = 1),
    then each row Z[z,:] renormalised so every footprint's reconstructed mass
    sum_r C_r sum X_r sum Y_r Z_r(z) is 1.
This is the factor *builder* (an input generator), not the query path.
"""
from __future__ import annotations

import numpy as np


def _kr(B: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Khatri-Rao product: rows (b, c) -> B[b] * C[c]."""
    return (B[:, None, :] * C[None, :, :]).reshape(-1, B.shape[1])


def _hals(F: np.ndarray, M: np.ndarray, G: np.ndarray) -> np.ndarray:
    for r in range(F.shape[1]):
        if G[r, r] <= 0:
            continue
        F[:, r] = np.maximum(1e-300, F[:, r] + (M[:, r] - F @ G[:, r]) / G[r, r])
    return F


def nncp_hals(D: np.ndarray, R: int, seed: int = 1, tol: float = 1e-4, max_iter: int = 500):
    """Nonnegative CP of a 3-way tensor D[z, x, y]. Returns (Z, X, Y, history)."""
    P, A1, A2 = D.shape
    rng = np.random.default_rng(seed)
    X = rng.random((A1, R))
    Y = rng.random((A2, R))
    Z = rng.random((P, R))
    D_z = D.reshape(P, A1 * A2)                       # [z, (x,y)]
    D_x = D.transpose(1, 0, 2).reshape(A1, P * A2)    # [x, (z,y)]
    D_y = D.transpose(2, 0, 1).reshape(A2, P * A1)    # [y, (z,x)]
    nD2 = float((D * D).sum())
    hist = []
    prev = None
    for it in range(max_iter):
        Z = _hals(Z, D_z @ _kr(X, Y), (X.T @ X) * (Y.T @ Y))
        X = _hals(X, D_x @ _kr(Z, Y), (Z.T @ Z) * (Y.T @ Y))
        My = D_y @ _kr(Z, X)
        Y = _hals(Y, My, (Z.T @ Z) * (X.T @ X))
        inner = float((My * Y).sum())
        nDh2 = float(((Z.T @ Z) * (X.T @ X) * (Y.T @ Y)).sum())
        err = np.sqrt(max(0.0, nD2 - 2.0 * inner + nDh2) / nD2)
        hist.append(err)
        if prev is not None and abs(prev - err) < tol * max(prev, 1e-300):
            break
        prev = err
    return Z, X, Y, hist


def factors_from_tensor(D: np.ndarray, R: int, seed: int = 1, tol: float = 1e-4, max_iter: int = 500,
                        renormalise: bool = True):
    from . import Factors
    Z, X, Y, hist = nncp_hals(D, R, seed=seed, tol=tol, max_iter=max_iter)
    sx = X.sum(0)
    sy = Y.sum(0)
    X = X / sx
    Y = Y / sy
    Z = Z * (sx * sy)
    C = Z.max(0)
    C[C <= 0] = 1.0
    Z = Z / C
    if renormalise:
        M = Z @ C                                    # sum_r C_r * 1 * 1 * Z_r(z)
        M[M <= 0] = 1.0
        Z = Z / M[:, None]
    return Factors(C=C.astype(np.float32), X=np.ascontiguousarray(X, np.float32),
                   Y=np.ascontiguousarray(Y, np.float32), Z=np.ascontiguousarray(Z, np.float32),
                   info=dict(als_history=hist, als_sweeps=len(hist), als_rel_err=hist[-1]))
