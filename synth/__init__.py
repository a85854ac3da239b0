"""Seeded synthetic inputs for the NDF range-query path (maps, CP factors, queries).

Shared by the oracle (``oracle/``) and the CUDA product path; holds none of the
query arithmetic.  The workload recipe follows BASELINE.json ``configs`` and
SURVEY.md §8(d) ("Common synthetic construction"); DESIGN.md §3 restates it.

Everything here is a pure function of (config, seed):
  * map seed 0 for every map, factor/ALS seed 1, query seed 100+k;
  * queries come from a counter-based RNG, so shard [i0, i1) is identical no
    matter how the index range is split across ranks.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "synth.c")
_LIB_PATH = os.path.join(_HERE, "_libsynth.so")
_lib = None

QREC = np.dtype([("u", "<f4"), ("v", "<f4"), ("size", "<f4"), ("rect", "<u4")])
assert QREC.itemsize == 16


def build_lib(force: bool = False) -> str:
    """Compile csrc/synth.c -> _libsynth.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _QDist(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int32), ("A", ctypes.c_int32),
        ("size_mix", ctypes.c_int32), ("side_mode", ctypes.c_int32),
        ("side_lo", ctypes.c_int32), ("side_hi", ctypes.c_int32),
        ("centre_mode", ctypes.c_int32), ("jitter", ctypes.c_int32),
        ("lg_lo", ctypes.c_double), ("lg_hi", ctypes.c_double),
        ("lg_lo2", ctypes.c_double), ("lg_hi2", ctypes.c_double),
        ("w_lo", ctypes.c_double), ("w_hi", ctypes.c_double),
        ("p_texel", ctypes.c_double), ("alpha_h", ctypes.c_double),
    ]


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, u64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.synth_rng64.restype = u64
        L.synth_rng64.argtypes = [u64, ctypes.c_uint32, u64]
        L.synth_map_gaussian_slopes.argtypes = [i32, u64, f64, P]
        L.synth_map_flakes.argtypes = [i32, u64, f64, f64, P, P]
        L.synth_map_scratches.argtypes = [i32, u64, i32, f64, f64, f64, P]
        L.synth_bin_map.argtypes = [i32, P, i32, P]
        L.synth_select_atoms.restype = i32
        L.synth_select_atoms.argtypes = [i32, P, i32, i32, P, P]
        L.synth_footprint_table.restype = i32
        L.synth_footprint_table.argtypes = [i32, i32, P, P]
        L.synth_num_rows.restype = i64
        L.synth_num_rows.argtypes = [i32, i32, i32]
        L.synth_build_z_exact.argtypes = [i32, P, i32, i32, i32, i64, i64, P]
        L.synth_build_z_rows.argtypes = [i32, P, i32, i32, i32, P, i64, P]
        L.synth_hist_tensor.argtypes = [i32, P, i32, i32, i32, P]
        L.synth_atom_profiles.argtypes = [i32, i32, P, f64, P, P]
        L.synth_gen_queries.argtypes = [ctypes.POINTER(_QDist), u64, i64, i64, P, P]
        L.synth_gen_sg_lights.argtypes = [ctypes.POINTER(_QDist), u64, i64, i64, f64, f64, f64, f64, f64, P]
        L.synth_wang_tiles.argtypes = [i32, u64, f64, f64, P]
        L.synth_wang_rows.restype = i64
        L.synth_wang_rows.argtypes = [i32, i32, i32, i32]
        L.synth_wang_z.argtypes = [i32, P, i32, i32, i32, i32, P]
        L.synth_max_threads.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


# --------------------------------------------------------------- configs --
@dataclass(frozen=True)
class Config:
    """One workload of BASELINE.json ``configs`` (1-based ``idx``)."""
    idx: int
    name: str
    N: int                      # map side (texels), power of two
    A: int                      # angular grid side
    R: int                      # CP rank
    n_queries: int
    map_kind: str               # "slopes" | "flakes" | "scratches"
    map_params: dict = field(default_factory=dict)
    factor_kind: str = "exact"  # "als" (config 1) | "exact" (exact-rank normal quantisation)
    sigma_r: float = 0.005      # intrinsic roughness in projected units (S:133 default) for "exact"
    s0: int = 1                 # base stride (configs use 1: sizes "1,2,4,...")
    wrap: bool = True           # periodic maps -> wrapped neighbours
    qdist: dict = field(default_factory=dict)
    map_seed: int = 0
    factor_seed: int = 1

    @property
    def L(self) -> int:
        return int(round(math.log2(self.N // self.s0))) + 1

    @property
    def P(self) -> int:
        return sum((self.N // (self.s0 << l)) ** 2 for l in range(self.L))

    @property
    def query_seed(self) -> int:
        return 100 + self.idx

    def scaled(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    1: Config(1, "tiny", N=64, A=32, R=8, n_queries=10**4, map_kind="slopes", map_params=dict(sigma=0.2),
              factor_kind="als",
              qdist=dict(lg_lo=0.0, lg_hi=6.0, side_mode=0, side_lo=1, side_hi=8, centre_mode=0)),
    2: Config(2, "flakes", N=512, A=64, R=32, n_queries=10**6, map_kind="flakes",
              map_params=dict(spacing=12.0, alpha=0.1),
              qdist=dict(lg_lo=0.0, lg_hi=9.0, side_mode=1, w_lo=0.5, w_hi=4.0, centre_mode=1, p_texel=0.5)),
    3: Config(3, "tileable", N=2048, A=128, R=64, n_queries=10**7, map_kind="flakes",
              map_params=dict(spacing=8.0, alpha=0.05),
              qdist=dict(lg_lo=0.0, lg_hi=11.0, side_mode=0, side_lo=1, side_hi=16, centre_mode=1, p_texel=0.5)),
    4: Config(4, "scratches", N=2048, A=128, R=128, n_queries=10**8, map_kind="scratches",
              map_params=dict(n_scr=1000, width=2.0, max_tilt_deg=30.0, alpha_base=0.02),
              qdist=dict(size_mix=1, lg_lo=0.0, lg_hi=2.0, lg_lo2=8.0, lg_hi2=11.0, side_mode=0, side_lo=1,
                         side_hi=3, centre_mode=1, p_texel=0.75, jitter=1)),
    5: Config(5, "scaling", N=4096, A=256, R=256, n_queries=10**9, map_kind="flakes",
              map_params=dict(spacing=12.0, alpha=0.08),
              qdist=dict(lg_lo=0.0, lg_hi=12.0, side_mode=0, side_lo=1, side_hi=16, centre_mode=2, alpha_h=0.3)),
}


# ------------------------------------------------------------------ maps --
def make_map(cfg: Config) -> np.ndarray:
    """Normal map as projected normals (n_x, n_y): float32 [N, N, 2], row v, column u."""
    L = lib()
    out = np.empty((cfg.N, cfg.N, 2), np.float32)
    mp = cfg.map_params
    if cfg.map_kind == "slopes":
        L.synth_map_gaussian_slopes(cfg.N, cfg.map_seed, mp["sigma"], _p(out))
    elif cfg.map_kind == "flakes":
        L.synth_map_flakes(cfg.N, cfg.map_seed, mp["spacing"], mp["alpha"], _p(out), None)
    elif cfg.map_kind == "scratches":
        L.synth_map_scratches(cfg.N, cfg.map_seed, mp["n_scr"], mp["width"], mp["max_tilt_deg"], mp["alpha_base"],
                              _p(out))
    elif cfg.map_kind == "constant":
        out[..., 0] = mp.get("nx", 0.0)
        out[..., 1] = mp.get("ny", 0.0)
    else:
        raise ValueError(cfg.map_kind)
    return out


def flake_ids(cfg: Config) -> np.ndarray:
    assert cfg.map_kind == "flakes"
    nxy = np.empty((cfg.N, cfg.N, 2), np.float32)
    ids = np.empty((cfg.N, cfg.N), np.int32)
    lib().synth_map_flakes(cfg.N, cfg.map_seed, cfg.map_params["spacing"], cfg.map_params["alpha"], _p(nxy), _p(ids))
    return ids


def bin_map(cfg: Config, nxy: np.ndarray) -> np.ndarray:
    """Angular bin id (by*A + bx) per texel, uint16 [N, N]; bin = min(floor((n+1)A/2), A-1)."""
    out = np.empty((cfg.N, cfg.N), np.uint16)
    lib().synth_bin_map(cfg.N, _p(np.ascontiguousarray(nxy, np.float32)), cfg.A, _p(out))
    return out


def select_atoms(cfg: Config, bins: np.ndarray):
    """(atom_bins int32 [R], atom_map uint16 [N,N], #populated bins)."""
    ab = np.empty(cfg.R, np.int32)
    am = np.empty((cfg.N, cfg.N), np.uint16)
    npop = lib().synth_select_atoms(cfg.N, _p(bins), cfg.A, cfg.R, _p(ab), _p(am))
    return ab, am, npop


def footprint_table(s: int, N: int):
    """Integer footprint weights of a level with stride s: (qmin, w uint32[Wf])."""
    w = np.zeros(N, np.uint32)
    qmin = np.zeros(1, np.int32)
    Wf = lib().synth_footprint_table(s, N, _p(qmin), _p(w))
    return int(qmin[0]), w[:Wf].copy()


def level_offsets(cfg: Config):
    offs, o = [], 0
    for l in range(cfg.L):
        offs.append(o)
        o += (cfg.N // (cfg.s0 << l)) ** 2
    return offs


def build_z_exact(cfg: Config, atom_map: np.ndarray, z0: int = 0, z1: int | None = None) -> np.ndarray:
    z1 = cfg.P if z1 is None else z1
    Z = np.empty((z1 - z0, cfg.R), np.float32)
    lib().synth_build_z_exact(cfg.N, _p(atom_map), cfg.R, cfg.s0, cfg.L, z0, z1, _p(Z))
    return Z


def build_z_rows(cfg: Config, atom_map: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Rows `rows` of the exact-rank Z (same bits as build_z_exact)."""
    rows = np.ascontiguousarray(rows, np.int64)
    out = np.empty((rows.shape[0], cfg.R), np.float32)
    lib().synth_build_z_rows(cfg.N, _p(atom_map), cfg.R, cfg.s0, cfg.L, _p(rows), rows.shape[0], _p(out))
    return out


_CUDA_SRC = os.path.join(_HERE, "csrc", "synth_cuda.cu")
_CUDA_LIB = os.path.join(_HERE, "_libsynth_cuda.so")
_cuda_lib = None


def build_cuda_lib(force: bool = False) -> str:
    """nvcc -> _libsynth_cuda.so (the GPU twin of the exact-rank Z builder)."""
    if force or not os.path.exists(_CUDA_LIB) or os.path.getmtime(_CUDA_LIB) < os.path.getmtime(_CUDA_SRC):
        tmp = _CUDA_LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["nvcc", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-O3", "-lineinfo", _CUDA_SRC, "-o", tmp])
        os.replace(tmp, _CUDA_LIB)
    return _CUDA_LIB


def build_z_exact_cuda(cfg: Config, atom_map: np.ndarray, device: int = 0):
    """Exact-rank Z built on the GPU (bit-identical to build_z_exact): torch float32 [P, R] on cuda:device."""
    import torch
    global _cuda_lib
    if _cuda_lib is None:
        if not os.path.exists(_CUDA_LIB):
            build_cuda_lib()
        _cuda_lib = ctypes.CDLL(_CUDA_LIB)
        P_ = ctypes.c_void_p
        _cuda_lib.synth_cuda_build_z_exact.restype = ctypes.c_int
        _cuda_lib.synth_cuda_build_z_exact.argtypes = [ctypes.c_int, P_, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                       P_, P_, P_, P_, P_, P_, P_]
    dev = torch.device("cuda", device)
    tabs, offs, lens, qmins, tots = [], [], [], [], []
    o = 0
    for l in range(cfg.L):
        qmin, w = footprint_table(cfg.s0 << l, cfg.N)
        tabs.append(w)
        offs.append(o)
        lens.append(w.shape[0])
        qmins.append(qmin)
        sw = int(w.astype(np.uint64).sum())
        tots.append(float(sw) * float(sw))
        o += w.shape[0]
    tab_dev = torch.from_numpy(np.concatenate(tabs).view(np.int32)).to(dev)
    am_dev = torch.from_numpy(atom_map.view(np.int16)).to(dev)
    Z = torch.empty((cfg.P, cfg.R), dtype=torch.float32, device=dev)
    offs = np.array(offs, np.int64); lens = np.array(lens, np.int32)
    qmins = np.array(qmins, np.int32); tots = np.array(tots, np.float64)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev)
        rc = _cuda_lib.synth_cuda_build_z_exact(cfg.N, ctypes.c_void_p(am_dev.data_ptr()), cfg.R, cfg.s0, cfg.L,
                                                ctypes.c_void_p(tab_dev.data_ptr()), _p(offs), _p(lens), _p(qmins),
                                                _p(tots), ctypes.c_void_p(Z.data_ptr()),
                                                ctypes.c_void_p(st.cuda_stream))
        if rc != 0:
            raise RuntimeError(f"synth_cuda_build_z_exact failed: cudaError {rc}")
        st.synchronize()
    return Z


def hist_tensor(cfg: Config, bins: np.ndarray) -> np.ndarray:
    """Footprint NDF tensor D[z, x, y] (bin masses, each footprint sums to 1)."""
    D = np.empty((cfg.P, cfg.A, cfg.A), np.float64)
    lib().synth_hist_tensor(cfg.N, _p(bins), cfg.A, cfg.s0, cfg.L, _p(D))
    return D


def atom_profiles(cfg: Config, atom_bins: np.ndarray, sigma_b: float | None = None):
    if sigma_b is None:
        sigma_b = cfg.sigma_r * cfg.A / 2.0
    X = np.empty((cfg.A, cfg.R), np.float32)
    Y = np.empty((cfg.A, cfg.R), np.float32)
    lib().synth_atom_profiles(cfg.A, cfg.R, _p(np.ascontiguousarray(atom_bins, np.int32)), float(sigma_b), _p(X),
                              _p(Y))
    return X, Y


@dataclass
class Factors:
    """Raw CP factors of Eq. 5: C [R], X [A][R], Y [A][R], Z [P][R] (fp32, nonnegative)."""
    C: np.ndarray
    X: np.ndarray
    Y: np.ndarray
    Z: np.ndarray | None          # None when Z lives only on the device (GPU twin builder)
    info: dict = field(default_factory=dict)


def build_factors(cfg: Config, nxy: np.ndarray | None = None, bins: np.ndarray | None = None,
                  with_z: bool = True) -> Factors:
    if nxy is None and bins is None:
        nxy = make_map(cfg)
    if bins is None:
        bins = bin_map(cfg, nxy)
    if cfg.factor_kind == "als":
        from . import als
        D = hist_tensor(cfg, bins)
        return als.factors_from_tensor(D, cfg.R, seed=cfg.factor_seed)
    ab, am, npop = select_atoms(cfg, bins)
    X, Y = atom_profiles(cfg, ab)
    Z = build_z_exact(cfg, am) if with_z else None
    return Factors(C=np.ones(cfg.R, np.float32), X=X, Y=Y, Z=Z,
                   info=dict(atom_bins=ab, atom_map=am, populated_bins=npop))


# --------------------------------------------------------------- queries --
def qdist_struct(cfg: Config) -> _QDist:
    q = dict(size_mix=0, lg_lo2=0.0, lg_hi2=0.0, side_mode=0, side_lo=1, side_hi=1, w_lo=0.5, w_hi=0.5,
             centre_mode=0, p_texel=0.0, jitter=0, alpha_h=0.1)
    q.update(cfg.qdist)
    return _QDist(N=cfg.N, A=cfg.A, **q)


def gen_queries(cfg: Config, bins: np.ndarray | None, i0: int = 0, i1: int | None = None,
                seed: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Query records [i0, i1) of the config's stream (structured dtype QREC)."""
    i1 = cfg.n_queries if i1 is None else i1
    seed = cfg.query_seed if seed is None else seed
    qd = qdist_struct(cfg)
    if qd.centre_mode == 1 and bins is None:
        raise ValueError("texel-centred rectangles need the bin map")
    if out is None:
        out = np.empty(i1 - i0, QREC)
    assert out.dtype == QREC and out.shape[0] == i1 - i0
    lib().synth_gen_queries(ctypes.byref(qd), seed, i0, i1,
                            None if bins is None else _p(np.ascontiguousarray(bins)), _p(out))
    return out


SGREC = np.dtype([("u", "<f4"), ("v", "<f4"), ("size", "<f4"), ("hx", "<f4"), ("hy", "<f4"),
                  ("lam", "<f4"), ("amp", "<f4"), ("pad", "<f4")])


def gen_sg_lights(cfg: Config, i0: int = 0, i1: int | None = None, seed: int | None = None, alpha_h: float = 0.3,
                  lam=(10.0, 1000.0), amp=(0.5, 2.0), out: np.ndarray | None = None) -> np.ndarray:
    """SG-light query inputs for environment prefiltering (Sec. 5.4): footprint as the config's queries,
    half vector ~ Beckmann(alpha_h), lambda log-uniform in `lam`, amplitude uniform in `amp`."""
    i1 = cfg.n_queries if i1 is None else i1
    seed = cfg.query_seed + 1000 if seed is None else seed
    if out is None:
        out = np.empty(i1 - i0, SGREC)
    assert out.dtype == SGREC and out.shape[0] == i1 - i0
    qd = qdist_struct(cfg)
    lib().synth_gen_sg_lights(ctypes.byref(qd), seed, i0, i1, alpha_h, lam[0], lam[1], amp[0], amp[1], _p(out))
    return out


@dataclass(frozen=True)
class TileConfig:
    """Wang-tile workload (16 tiles of 512^2: a 100K^2 synthesized map)."""
    T: int = 512
    A: int = 64
    R: int = 32
    s0: int = 1
    margin: int = 3
    spacing: float = 12.0
    alpha: float = 0.1
    sigma_r: float = 0.005
    seed: int = 7
    world: int = 102400
    n_queries: int = 10**7

    @property
    def L(self) -> int:
        return int(round(math.log2(self.T // self.s0))) + 1


def wang_tiles(tc: TileConfig) -> np.ndarray:
    """16 edge-coloured flake tiles: float32 [16, T, T, 2] projected normals."""
    out = np.empty((16, tc.T, tc.T, 2), np.float32)
    lib().synth_wang_tiles(tc.T, 0, tc.spacing, tc.alpha, _p(out))
    return out


def wang_rows(tc: TileConfig) -> int:
    return lib().synth_wang_rows(tc.T, tc.s0, tc.L, tc.margin)


def wang_factors(tc: TileConfig, tiles: np.ndarray):
    """Exact-rank factors shared by the 16 tiles (atoms from all tiles), extended per-tile Z [16*P_ext, R]."""
    cfg = Config(0, "wang", N=tc.T, A=tc.A, R=tc.R, n_queries=0, map_kind="flakes", sigma_r=tc.sigma_r, s0=tc.s0)
    allbins = np.concatenate([bin_map(cfg, tiles[t]) for t in range(16)], axis=0)  # [16T, T]
    # atoms = the R most populated bins over all tiles (ties -> lower bin id); nearest-atom snapping
    cnt = np.bincount(allbins.ravel().astype(np.int64), minlength=tc.A * tc.A)
    order = np.lexsort((np.arange(cnt.size), -cnt))[: tc.R]
    ab = order.astype(np.int32)
    bx, by = ab % tc.A, ab // tc.A
    pop = np.nonzero(cnt)[0]
    px, py = pop % tc.A, pop // tc.A
    d2 = (px[:, None] - bx[None, :]) ** 2 + (py[:, None] - by[None, :]) ** 2
    lut = np.full(tc.A * tc.A, 0, np.int64)
    lut[pop] = np.argmin(d2, axis=1)  # ties -> lower atom index
    am = lut[allbins.astype(np.int64)].astype(np.uint16).reshape(16, tc.T, tc.T)
    X, Y = atom_profiles(cfg, ab)
    P = wang_rows(tc)
    Z = np.empty((16 * P, tc.R), np.float32)
    lib().synth_wang_z(tc.T, _p(np.ascontiguousarray(am)), tc.R, tc.s0, tc.L, tc.margin, _p(Z))
    return Factors(C=np.ones(tc.R, np.float32), X=X, Y=Y, Z=Z, info=dict(atom_bins=ab, atom_map=am, rows=P))


@dataclass
class BlockedStore:
    """Paper-faithful blocked / clustered store inputs."""
    t: int                    # angular block side
    region: int               # spatial region side (texels) of the footprint centres
    R: int                    # rank per group
    C: np.ndarray             # [n_sets, R]
    X: np.ndarray             # [n_sets, t, R]
    Y: np.ndarray             # [n_sets, t, R]
    group_set: np.ndarray     # [n_groups] int32 factor set of the group (-1 = empty group)
    slab_ptr: np.ndarray      # [P, nb*nb] int64 global slab index or -1 (blank block)
    Z: np.ndarray             # [n_slabs, R]
    info: dict = field(default_factory=dict)


def _block_profiles(A, t, R, atom_bins_local, sigma_b):
    """Atom profiles truncated to the atom's block and renormalised (so the block holds all the mass)."""
    Xb = np.zeros((t, R), np.float32)
    Yb = np.zeros((t, R), np.float32)
    from math import erf, sqrt
    for k, (cx, cy) in enumerate(atom_bins_local):
        if cx < 0:
            continue
        for F, c in ((Xb, cx), (Yb, cy)):
            col = np.zeros(t)
            if sigma_b <= 0:
                col[c] = 1.0
            else:
                T = int(np.ceil(4 * sigma_b))
                for x in range(max(0, c - T), min(t, c + T + 1)):
                    lo, hi = (x - (c + 0.5)) / sigma_b, (x + 1 - (c + 0.5)) / sigma_b
                    col[x] = 0.5 * (erf(hi / sqrt(2)) - erf(lo / sqrt(2)))
            F[:, k] = (col / col.sum()).astype(np.float32)
    return Xb, Yb


def build_blocked(cfg: Config, nxy: np.ndarray | None = None, bins: np.ndarray | None = None, t: int = 16,
                  region: int = 8, sigma_b: float | None = None) -> tuple:
    """Exact-rank blocked store: per angular block b the R most populated bins of b are its atoms, every texel
    snaps to the nearest atom of its own block, and group (region, b) holds the slabs of all footprints centred
    in the region whose block b is not blank (blank blocks pruned).  Returns (BlockedStore,
    global_factors) -- the second is the same tensor as ONE global CP store (rank nb^2 R) for cross-checks."""
    assert cfg.A % t == 0
    if bins is None:
        bins = bin_map(cfg, make_map(cfg) if nxy is None else nxy)
    A, R, nb = cfg.A, cfg.R, cfg.A // t
    sigma_b = cfg.sigma_r * A / 2.0 if sigma_b is None else sigma_b
    bx, by = bins.astype(np.int64) % A, bins.astype(np.int64) // A
    blk = (by // t) * nb + (bx // t)
    cnt = np.bincount(bins.ravel().astype(np.int64), minlength=A * A)
    atom_local = -np.ones((nb * nb, R, 2), np.int64)
    lut = np.zeros(A * A, np.int64)  # bin -> global atom id b*R + k
    for b in range(nb * nb):
        ox, oy = (b % nb) * t, (b // nb) * t
        ids = np.array([(oy + y) * A + ox + x for y in range(t) for x in range(t)])
        c = cnt[ids]
        pop = ids[c > 0]
        if pop.size == 0:
            continue
        order = np.lexsort((pop, -cnt[pop]))[:R]
        ab = pop[order]
        atom_local[b, :ab.size, 0] = ab % A - ox
        atom_local[b, :ab.size, 1] = ab // A - oy
        axx, ayy = ab % A, ab // A
        px, py = pop % A, pop // A
        d2 = (px[:, None] - axx[None, :]) ** 2 + (py[:, None] - ayy[None, :]) ** 2
        lut[pop] = b * R + np.argmin(d2, axis=1)
    am = lut[bins.astype(np.int64)].astype(np.uint16)
    Rt = nb * nb * R
    assert Rt <= 65535
    gcfg = cfg.scaled(R=Rt)
    Zg = build_z_exact(gcfg, np.ascontiguousarray(am))            # [P, nb^2 R]
    sets_X = np.zeros((nb * nb, t, R), np.float32)
    sets_Y = np.zeros((nb * nb, t, R), np.float32)
    for b in range(nb * nb):
        sets_X[b], sets_Y[b] = _block_profiles(A, t, R, atom_local[b], sigma_b)
    # groups: (region of the footprint centre, block)
    nr = cfg.N // region
    P = cfg.P
    zr = np.zeros(P, np.int64)
    off = 0
    for l in range(cfg.L):
        s = cfg.s0 << l
        n = cfg.N // s
        j, i = np.divmod(np.arange(n * n), n)
        rx = ((2 * i + 1) * s) // (2 * region)
        ry = ((2 * j + 1) * s) // (2 * region)
        zr[off:off + n * n] = ry * nr + rx
        off += n * n
    mass = Zg.reshape(P, nb * nb, R).sum(axis=2)                  # per (row, block)
    nonblank = mass > 0
    slab_ptr = -np.ones((P, nb * nb), np.int64)
    # slabs grouped by (region, block): sort (group, row) pairs
    rows, blocks = np.nonzero(nonblank)
    groups = zr[rows] * (nb * nb) + blocks
    order = np.lexsort((rows, groups))
    rows, blocks = rows[order], blocks[order]
    slab_ptr[rows, blocks] = np.arange(rows.size)
    Zs = Zg.reshape(P, nb * nb, R)[rows, blocks]                  # [S, R]
    group_set = -np.ones(nr * nr * nb * nb, np.int32)
    group_set[np.unique(groups)] = (np.unique(groups) % (nb * nb)).astype(np.int32)
    store = BlockedStore(t=t, region=region, R=R, C=np.ones((nb * nb, R), np.float32), X=sets_X, Y=sets_Y,
                         group_set=group_set, slab_ptr=slab_ptr, Z=np.ascontiguousarray(Zs, np.float32),
                         info=dict(n_slabs=int(rows.size), blank_fraction=float(1 - nonblank.mean()),
                                   n_groups=int(np.unique(groups).size)))
    # the same tensor as one global CP store: profiles embedded in the full grid
    Xg = np.zeros((A, Rt), np.float32)
    Yg = np.zeros((A, Rt), np.float32)
    for b in range(nb * nb):
        ox, oy = (b % nb) * t, (b // nb) * t
        Xg[ox:ox + t, b * R:(b + 1) * R] = sets_X[b]
        Yg[oy:oy + t, b * R:(b + 1) * R] = sets_Y[b]
    glob = Factors(C=np.ones(Rt, np.float32), X=Xg, Y=Yg, Z=Zg, info=dict(R=Rt))
    return store, glob


def pack_rect(x1, x2, y1, y2):
    x1, x2, y1, y2 = (np.asarray(a, np.uint32) for a in (x1, x2, y1, y2))
    return x1 | (x2 << 8) | (y1 << 16) | (y2 << 24)


def unpack_rect(rect):
    r = np.asarray(rect, np.uint32)
    return r & 255, (r >> 8) & 255, (r >> 16) & 255, (r >> 24) & 255


def make_records(u, v, size, x1, x2, y1, y2) -> np.ndarray:
    u = np.atleast_1d(np.asarray(u, np.float32))
    out = np.empty(u.shape[0], QREC)
    out["u"] = u
    out["v"] = np.asarray(v, np.float32)
    out["size"] = np.asarray(size, np.float32)
    out["rect"] = pack_rect(x1, x2, y1, y2)
    return out


def random_factors(A: int, R: int, P: int, seed: int, sparsity: float = 0.0):
    """Random nonnegative fp32 factors for property tests (not a workload)."""
    rng = np.random.default_rng(seed)
    C = rng.uniform(0.25, 2.0, R).astype(np.float32)
    X = rng.random((A, R)).astype(np.float32)
    Y = rng.random((A, R)).astype(np.float32)
    Z = rng.random((P, R)).astype(np.float32)
    if sparsity > 0:
        X[rng.random((A, R)) < sparsity] = 0
        Y[rng.random((A, R)) < sparsity] = 0
        Z[rng.random((P, R)) < sparsity] = 0
    return Factors(C=C, X=X, Y=Y, Z=Z)
