"""fp64 CPU oracle of the batched NDF range query (Deng et al., arXiv 2109.14807).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares no
code with the CUDA path (``paper_2109_14807_b200``) and never imports it.

Two independent implementations:
  * ``query_batch``  -- oracle.c, the plain definition written out in fp64
    (Eq. 6 per neighbour; trilinear blend; clamp);
  * ``brute.py``     -- numpy brute force for tiny inputs: reconstruct the
    tensor D-hat of Eq. 5 and sum it over the rectangle.
Both take the RAW factors (C, X, Y, Z) -- not the CUDA path's store image.

Parity pins (tests/test_oracle_pins.py) tie both to what the paper and the
mathematics fix; DESIGN.md §4 lists them.  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "_liboracle.so")
_lib = None


class Desc(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("s0", ctypes.c_int32), ("L", ctypes.c_int32),
                ("A", ctypes.c_int32), ("R", ctypes.c_int32), ("wrap", ctypes.c_int32)]


class TilesDesc(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int32), ("s0", ctypes.c_int32), ("L", ctypes.c_int32), ("margin", ctypes.c_int32),
                ("A", ctypes.c_int32), ("R", ctypes.c_int32), ("seed", ctypes.c_uint64)]


class BlockedDesc(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("s0", ctypes.c_int32), ("L", ctypes.c_int32), ("A", ctypes.c_int32),
                ("t", ctypes.c_int32), ("region", ctypes.c_int32), ("R", ctypes.c_int32), ("wrap", ctypes.c_int32)]


def build_lib(force: bool = False) -> str:
    """gcc -O2 -fopenmp (no -ffast-math, no hand SIMD)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.oracle_query_batch.argtypes = [ctypes.POINTER(Desc), P, P, P, P, P, P, ctypes.c_int64, ctypes.c_int, P,
                                         ctypes.c_int]
        L.oracle_neighbours_batch.argtypes = [ctypes.POINTER(Desc), P, ctypes.c_int64, P, P]
        L.oracle_sample_batch.argtypes = [ctypes.POINTER(Desc), P, P, P, P, P, P, P, ctypes.c_int64, P, P, P, P]
        L.oracle_sg_rects.argtypes = [P, ctypes.c_int64, ctypes.c_double, ctypes.c_int, P, P, P, P]
        L.oracle_tile_id.restype = ctypes.c_int
        L.oracle_tile_id.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64]
        L.oracle_tiled_query_batch.argtypes = [ctypes.POINTER(TilesDesc), P, P, P, P, P, ctypes.c_int64, ctypes.c_int, P]
        L.oracle_tiled_sample_batch.argtypes = [ctypes.POINTER(TilesDesc), P, P, P, P, P, P, ctypes.c_int64, P, P, P,
                                                P, P, P, P, P, P]
        L.oracle_blocked_query_batch.argtypes = [ctypes.POINTER(BlockedDesc), P, P, P, P, P, P, P, ctypes.c_int64,
                                                 ctypes.c_int, P]
        L.oracle_blocked_sample_batch.argtypes = [ctypes.POINTER(BlockedDesc), P, P, P, P, P, P, P, P,
                                                  ctypes.c_int64, P, P, P, P, P]
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return lib().oracle_max_threads()


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def make_desc(N, s0, L, A, R, wrap=True) -> Desc:
    return Desc(N=N, s0=s0, L=L, A=A, R=R, wrap=1 if wrap else 0)


def desc_of(cfg) -> Desc:
    return make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, cfg.wrap)


def query_batch(desc: Desc, C, X, Y, Z, records: np.ndarray, mean: bool = True, zmap=None,
                threads: int = 0) -> np.ndarray:
    """fp64 results for 16-byte records (u, v, size, rect)."""
    assert desc.R <= 4096
    C = np.ascontiguousarray(C, np.float32)
    X = np.ascontiguousarray(X, np.float32)
    Y = np.ascontiguousarray(Y, np.float32)
    Z = np.ascontiguousarray(Z, np.float32)
    assert C.shape == (desc.R,) and X.shape == (desc.A, desc.R) and Y.shape == (desc.A, desc.R)
    assert Z.ndim == 2 and Z.shape[1] == desc.R
    recs = np.ascontiguousarray(records)
    assert recs.dtype.itemsize == 16
    if zmap is not None:
        zmap = np.ascontiguousarray(zmap, np.int64)
    out = np.empty(recs.shape[0], np.float64)
    lib().oracle_query_batch(ctypes.byref(desc), _ptr(C), _ptr(X), _ptr(Y), _ptr(Z), _ptr(zmap), _ptr(recs),
                             recs.shape[0], 1 if mean else 0, _ptr(out), threads)
    return out


def sample_batch(desc: Desc, C, X, Y, Z, records: np.ndarray, xi: np.ndarray, zmap=None):
    """Hierarchical importance sampling (Sec. 5.2), fp64.
    xi: float32 [n, 10] variates (8 descent levels + 2 jitter).  Returns dict of
    pixel int32 [n, 2] (-1 = no sample), prob float64 [n] (pixel mass / domain mass),
    h float64 [n, 2] (projected half vector), margin float64 [n] (min relative distance
    of a variate to a decision boundary)."""
    C = np.ascontiguousarray(C, np.float32)
    X = np.ascontiguousarray(X, np.float32)
    Y = np.ascontiguousarray(Y, np.float32)
    Z = np.ascontiguousarray(Z, np.float32)
    recs = np.ascontiguousarray(records)
    xi = np.ascontiguousarray(xi, np.float32)
    n = recs.shape[0]
    assert xi.shape == (n, 10)
    if zmap is not None:
        zmap = np.ascontiguousarray(zmap, np.int64)
    pix = np.empty((n, 2), np.int32)
    prob = np.empty(n, np.float64)
    h = np.empty((n, 2), np.float64)
    mg = np.empty(n, np.float64)
    lib().oracle_sample_batch(ctypes.byref(desc), _ptr(C), _ptr(X), _ptr(Y), _ptr(Z), _ptr(zmap), _ptr(recs),
                              _ptr(xi), n, _ptr(pix), _ptr(prob), _ptr(h), _ptr(mg))
    return dict(pixel=pix, prob=prob, h=h, margin=mg)


def sg_rects(sg: np.ndarray, A: int, eps: float = 0.3):
    """Environment prefiltering (Sec. 5.4): compact-eps support angle theta, square side Q and the
    angular rectangle of each 32-byte SG-light record (u, v, size, hx, hy, lambda, amplitude, pad).
    Returns dict(theta, Q, rect uint32, q_margin)."""
    sg = np.ascontiguousarray(sg)
    assert sg.dtype.itemsize == 32
    n = sg.shape[0]
    th = np.empty(n, np.float64)
    Q = np.empty(n, np.float64)
    rect = np.empty(n, np.uint32)
    mg = np.empty(n, np.float64)
    lib().oracle_sg_rects(_ptr(sg), n, eps, A, _ptr(th), _ptr(Q), _ptr(rect), _ptr(mg))
    return dict(theta=th, Q=Q, rect=rect, q_margin=mg)


def tile_id(seed: int, cx: int, cy: int) -> int:
    """Wang tile of world cell (cx, cy) from the vertex-hash edge colours."""
    return lib().oracle_tile_id(seed, cx, cy)


def tiled_query_batch(td: TilesDesc, C, X, Y, Z, records: np.ndarray, mean: bool = True) -> np.ndarray:
    """Implicit Wang-tiled range query (Sec. 5.5): sum of the overlapped tiles' partial NDFs. Z: [16*P_ext, R]."""
    C = np.ascontiguousarray(C, np.float32)
    X = np.ascontiguousarray(X, np.float32)
    Y = np.ascontiguousarray(Y, np.float32)
    Z = np.ascontiguousarray(Z, np.float32)
    recs = np.ascontiguousarray(records)
    out = np.empty(recs.shape[0], np.float64)
    lib().oracle_tiled_query_batch(ctypes.byref(td), _ptr(C), _ptr(X), _ptr(Y), _ptr(Z), _ptr(recs),
                                   recs.shape[0], 1 if mean else 0, _ptr(out))
    return out


def tiled_sample_batch(td: TilesDesc, C, X, Y, Z, records: np.ndarray, xi: np.ndarray):
    """Importance sampling over implicit Wang tiles (Sec. 5.5), fp64: one covered tile instance
    chosen with equal probability (xi[:, 10]), the hierarchical descent of sample_batch on its partial
    NDF (xi[:, 0:8], jitter xi[:, 8:10]), pdf from the full NDF.  Returns dict of pixel int32 [n, 2]
    (-1 = none), prob (full pixel mass / full domain mass), prob_tile (the chosen tile's pmf), h,
    margin, tile int64 [n, 2] (tx, ty), count int32 [n] (covered instances), mass_tile / mass_all (domain
    mass of the chosen tile's partial NDF / of the full NDF)."""
    C = np.ascontiguousarray(C, np.float32)
    X = np.ascontiguousarray(X, np.float32)
    Y = np.ascontiguousarray(Y, np.float32)
    Z = np.ascontiguousarray(Z, np.float32)
    recs = np.ascontiguousarray(records)
    xi = np.ascontiguousarray(xi, np.float32)
    n = recs.shape[0]
    assert xi.shape == (n, 11)
    pix = np.empty((n, 2), np.int32)
    prob = np.empty(n, np.float64)
    prob_t = np.empty(n, np.float64)
    h = np.empty((n, 2), np.float64)
    mg = np.empty(n, np.float64)
    tile = np.empty((n, 2), np.int64)
    cnt = np.empty(n, np.int32)
    mt = np.empty(n, np.float64)
    ma = np.empty(n, np.float64)
    lib().oracle_tiled_sample_batch(ctypes.byref(td), _ptr(C), _ptr(X), _ptr(Y), _ptr(Z), _ptr(recs), _ptr(xi), n,
                                    _ptr(pix), _ptr(prob), _ptr(prob_t), _ptr(h), _ptr(mg), _ptr(tile), _ptr(cnt),
                                    _ptr(mt), _ptr(ma))
    return dict(pixel=pix, prob=prob, prob_tile=prob_t, h=h, margin=mg, tile=tile, count=cnt, mass_tile=mt,
                mass_all=ma)


def blocked_query_batch(cfg, bs, records: np.ndarray, mean: bool = True) -> np.ndarray:
    """Blocked / clustered store query (Sec. 4.2 + P:353): per neighbour, per overlapped angular block, the
    group's Eq. 6 on the sub-rectangle.  cfg: pyramid geometry (N, s0, L, A, wrap); bs: synth.BlockedStore."""
    d = BlockedDesc(N=cfg.N, s0=cfg.s0, L=cfg.L, A=cfg.A, t=bs.t, region=bs.region, R=bs.R,
                    wrap=1 if cfg.wrap else 0)
    recs = np.ascontiguousarray(records)
    out = np.empty(recs.shape[0], np.float64)
    arr = [np.ascontiguousarray(a, dt) for a, dt in ((bs.C, np.float32), (bs.X, np.float32), (bs.Y, np.float32),
                                                    (bs.group_set, np.int32), (bs.slab_ptr, np.int64),
                                                    (bs.Z, np.float32))]
    lib().oracle_blocked_query_batch(ctypes.byref(d), *[_ptr(a) for a in arr], _ptr(recs), recs.shape[0],
                                     1 if mean else 0, _ptr(out))
    return out


def blocked_sample_batch(cfg, bs, records: np.ndarray, xi: np.ndarray):
    """Importance sampling on the blocked store (Sec. 5.2), fp64: an angular block of the record's
    rectangle chosen by the blocks' blended sums (xi[:, 10]), then the quad descent of sample_batch inside it
    (xi[:, 0:8], jitter xi[:, 8:10]).  Returns dict of pixel int32 [n, 2] (-1 = none), prob (pixel SUM /
    rectangle SUM), h, margin, block int32 [n] (chosen block, -1 = none)."""
    d = BlockedDesc(N=cfg.N, s0=cfg.s0, L=cfg.L, A=cfg.A, t=bs.t, region=bs.region, R=bs.R,
                    wrap=1 if cfg.wrap else 0)
    recs = np.ascontiguousarray(records)
    xi = np.ascontiguousarray(xi, np.float32)
    n = recs.shape[0]
    assert xi.shape == (n, 11)
    arr = [np.ascontiguousarray(a, dt) for a, dt in ((bs.C, np.float32), (bs.X, np.float32), (bs.Y, np.float32),
                                                    (bs.group_set, np.int32), (bs.slab_ptr, np.int64),
                                                    (bs.Z, np.float32))]
    pix = np.empty((n, 2), np.int32)
    prob = np.empty(n, np.float64)
    h = np.empty((n, 2), np.float64)
    mg = np.empty(n, np.float64)
    blk = np.empty(n, np.int32)
    lib().oracle_blocked_sample_batch(ctypes.byref(d), *[_ptr(a) for a in arr], _ptr(recs), _ptr(xi), n,
                                      _ptr(pix), _ptr(prob), _ptr(h), _ptr(mg), _ptr(blk))
    return dict(pixel=pix, prob=prob, h=h, margin=mg, block=blk)


def neighbours(desc: Desc, records: np.ndarray):
    """(rows int64 [n,8], weights float64 [n,8]) -- steps 1-2 of the oracle."""
    recs = np.ascontiguousarray(records)
    n = recs.shape[0]
    rows = np.empty((n, 8), np.int64)
    w = np.empty((n, 8), np.float64)
    lib().oracle_neighbours_batch(ctypes.byref(desc), _ptr(recs), n, _ptr(rows), _ptr(w))
    return rows, w


def sparse_z(rows_needed: np.ndarray, P: int, row_fn):
    """Build (Zsub, zmap) holding only the given rows; row_fn(sorted_rows) -> [k, R]."""
    u = np.unique(rows_needed[rows_needed >= 0])
    zmap = np.full(P, -1, np.int64)
    zmap[u] = np.arange(u.shape[0])
    return np.ascontiguousarray(row_fn(u), np.float32), zmap
