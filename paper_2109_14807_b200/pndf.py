"""Thin ctypes binding of libpndf (include/pndf.h): argument marshalling only.

Every step of the query runs in the CUDA kernels of csrc/; nothing here
computes.  Names follow the C ABI: ``load_factors`` -> ``pndf_load_factors``,
``Store.query_batch`` -> ``pndf_query_batch``, ``Store.sync`` -> ``pndf_sync``,
``Store.query_batch_host`` -> ``pndf_query_batch_host``.  PyTorch (optional)
supplies device memory and streams; numpy arrays are accepted for host data.
If the shared library is missing this module raises -- there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PNDF_LIB") or os.path.join(_PKG, "libpndf.so")  # PNDF_LIB: tuning variants

ABI_VERSION = 1
OK, EINVAL, ENOMEM, ECUDA, EFORMAT, EQUERY = 0, -1, -2, -3, -4, -5
CLAMP, WRAP = 0, 1
PREFIX_AUTO, PREFIX_HILO, PREFIX_U32 = 0, 2, 4
MEAN, SUM, BIN_AUTO, BIN_ON, BIN_OFF, TIMING = 0, 1, 0, 2, 4, 8

QUERY_DTYPE = np.dtype([("u", "<f4"), ("v", "<f4"), ("size", "<f4"), ("rect", "<u4")])


class PndfError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        msg = f"{what}: {error_string(status)} ({status})"
        if status == ECUDA or status == ENOMEM:
            msg += f" [{last_cuda_error()}]"
        super().__init__(msg)


class Desc(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("map_size", ctypes.c_int32), ("base_stride", ctypes.c_int32),
                ("num_levels", ctypes.c_int32), ("ang_res", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


class TileDesc(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("tile_size", ctypes.c_int32), ("base_stride", ctypes.c_int32),
                ("num_levels", ctypes.c_int32), ("margin", ctypes.c_int32), ("ang_res", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("flags", ctypes.c_uint32), ("seed", ctypes.c_uint64)]


class BlockDesc(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("map_size", ctypes.c_int32), ("base_stride", ctypes.c_int32),
                ("num_levels", ctypes.c_int32), ("ang_res", ctypes.c_int32), ("block", ctypes.c_int32),
                ("region", ctypes.c_int32), ("rank", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("num_sets", ctypes.c_int32), ("num_slabs", ctypes.c_int64)]


class StoreStats(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("rank_padded", ctypes.c_int32), ("lanes_per_query", ctypes.c_int32),
                ("zc_bytes", ctypes.c_int64), ("prefix_bytes", ctypes.c_int64),
                ("kernel_launches", ctypes.c_uint64), ("timed_batches", ctypes.c_uint64),
                ("query_ms", ctypes.c_double), ("bin_ms", ctypes.c_double), ("last_binned", ctypes.c_int32),
                ("prefix_format", ctypes.c_int32),
                ("range_table_bytes", ctypes.c_int64), ("range_table_width", ctypes.c_int32), ("tile_reach", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


SAMPLE_DTYPE = np.dtype([("hx", "<f4"), ("hy", "<f4"), ("pdf", "<f4"), ("pixel", "<u4")])

EXPORTS = ("pndf_load_factors", "pndf_query_batch", "pndf_sample_batch", "pndf_sample_tiles", "pndf_sync", "pndf_query_batch_host",
           "pndf_free",
           "pndf_error_string", "pndf_last_cuda_error", "pndf_abi_version", "pndf_store_stats_get",
           "pndf_store_stats_reset", "pndf_store_image", "pndf_set_lanes", "pndf_bin_permutation",
           "pndf_sg_queries", "pndf_load_tiles", "pndf_load_blocked", "pndf_hist_tensor", "pndf_cp_als",
           "pndf_mttkrp", "pndf_rows_touched", "pndf_cp_als_map", "pndf_mttkrp_map",
           "pndf_sample_blocked")

ALS_NORMALISE = 1


class AlsOpts(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("max_sweeps", ctypes.c_int32), ("tol", ctypes.c_double),
                ("flags", ctypes.c_uint32)]

SG_DTYPE = np.dtype([("u", "<f4"), ("v", "<f4"), ("size", "<f4"), ("hx", "<f4"), ("hy", "<f4"),
                     ("lam", "<f4"), ("amp", "<f4"), ("pad", "<f4")])

_lib = None


def lib():
    """Load libpndf.so (raises if it has not been built -- no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2109_14807_b200.build` "
                               "(the CUDA extension is required; there is no fallback path)")
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        L.pndf_load_factors.restype = i32
        L.pndf_load_factors.argtypes = [ctypes.POINTER(Desc), P, P, P, P, ctypes.c_int, P, ctypes.POINTER(P)]
        L.pndf_query_batch.restype = i32
        L.pndf_query_batch.argtypes = [P, P, i64, P, u32, P]
        L.pndf_sample_batch.restype = i32
        L.pndf_sample_batch.argtypes = [P, P, P, i64, P, u32, P]
        L.pndf_sample_tiles.restype = i32
        L.pndf_sample_tiles.argtypes = [P, P, P, i64, P, P, u32, P]
        L.pndf_sample_blocked.restype = i32
        L.pndf_sample_blocked.argtypes = [P, P, P, i64, P, P, u32, P]
        L.pndf_sync.restype = i32
        L.pndf_sync.argtypes = [P, P]
        L.pndf_query_batch_host.restype = i32
        L.pndf_query_batch_host.argtypes = [P, P, i64, P, u32]
        L.pndf_free.restype = i32
        L.pndf_free.argtypes = [P]
        L.pndf_error_string.restype = ctypes.c_char_p
        L.pndf_error_string.argtypes = [i32]
        L.pndf_last_cuda_error.restype = ctypes.c_char_p
        L.pndf_abi_version.restype = u32
        L.pndf_store_stats_get.restype = i32
        L.pndf_store_stats_get.argtypes = [P, ctypes.POINTER(StoreStats)]
        L.pndf_store_stats_reset.restype = i32
        L.pndf_store_stats_reset.argtypes = [P]
        L.pndf_store_image.restype = i32
        L.pndf_store_image.argtypes = [P, P, P, i64, i64]
        L.pndf_bin_permutation.restype = i32
        L.pndf_bin_permutation.argtypes = [P, P, i64, P, P]
        L.pndf_load_tiles.restype = i32
        L.pndf_load_tiles.argtypes = [ctypes.POINTER(TileDesc), P, P, P, P, ctypes.c_int, P, ctypes.POINTER(P)]
        L.pndf_load_blocked.restype = i32
        L.pndf_load_blocked.argtypes = [ctypes.POINTER(BlockDesc), P, P, P, P, P, P, ctypes.c_int, P,
                                        ctypes.POINTER(P)]
        L.pndf_sg_queries.restype = i32
        L.pndf_sg_queries.argtypes = [P, i64, ctypes.c_float, i32, P, P]
        L.pndf_rows_touched.restype = i32
        L.pndf_rows_touched.argtypes = [P, P, i64, P]
        L.pndf_set_lanes.restype = i32
        L.pndf_set_lanes.argtypes = [P, i32]
        L.pndf_hist_tensor.restype = i32
        L.pndf_hist_tensor.argtypes = [ctypes.POINTER(Desc), P, P, P, P]
        L.pndf_cp_als.restype = i32
        L.pndf_cp_als.argtypes = [ctypes.POINTER(Desc), P, P, P, P, P, P, ctypes.POINTER(AlsOpts), P,
                                  ctypes.POINTER(i32), P]
        L.pndf_cp_als_map.restype = i32
        L.pndf_cp_als_map.argtypes = [ctypes.POINTER(Desc), P, P, P, P, P, ctypes.POINTER(AlsOpts), P,
                                      ctypes.POINTER(i32), P]
        L.pndf_mttkrp_map.restype = i32
        L.pndf_mttkrp_map.argtypes = [ctypes.POINTER(Desc), P, P, P, P, i32, P, P, P]
        L.pndf_mttkrp.restype = i32
        L.pndf_mttkrp.argtypes = [ctypes.POINTER(Desc), P, P, P, P, P, i32, P, P]
        _lib = L
    return _lib


def error_string(status: int) -> str:
    return lib().pndf_error_string(status).decode()


def last_cuda_error() -> str:
    return lib().pndf_last_cuda_error().decode()


def _check(status: int, what: str):
    if status != OK:
        raise PndfError(status, what)


def _ptr(x):
    """Raw address of a numpy array or torch tensor (host or device); None -> NULL."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
        return ctypes.c_void_p(x.ctypes.data)
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensors must be contiguous"
        return ctypes.c_void_p(x.data_ptr())
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    raise TypeError(type(x))


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def sg_queries(d_lights, d_queries, ang_res: int, eps: float = 0.3, stream=None, n: int | None = None):
    """pndf_sg_queries: device SG-light records (32 B) -> device query records (16 B) for pndf_query_batch."""
    n = d_queries.shape[0] if n is None else n
    _check(lib().pndf_sg_queries(_ptr(d_lights), n, eps, ang_res, _ptr(d_queries), _stream(stream)),
           "pndf_sg_queries")


def make_desc(N: int, s0: int, L: int, A: int, R: int, wrap: bool = True, prefix: int = PREFIX_AUTO) -> Desc:
    return Desc(abi_version=ABI_VERSION, map_size=N, base_stride=s0, num_levels=L, ang_res=A, rank=R,
                flags=(WRAP if wrap else CLAMP) | prefix)


class Store:
    """A device factor store (opaque pndf_store handle)."""

    def __init__(self, handle: ctypes.c_void_p, desc: Desc):
        self._h = handle
        self.desc = desc

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("store freed")
        return self._h

    def query_batch(self, queries, out, opts: int = 0, stream=None, n: int | None = None):
        """Enqueue pndf_query_batch on ``stream``: queries = device tensor of 16-byte records
        (e.g. int32 [n, 4]), out = device float32 [n]."""
        n = out.shape[0] if n is None else n
        _check(lib().pndf_query_batch(self.handle, _ptr(queries), n, _ptr(out), opts, _stream(stream)),
               "pndf_query_batch")

    def sample_batch(self, queries, xi, out, opts: int = 0, stream=None, n: int | None = None):
        """Enqueue pndf_sample_batch: queries = device records (rect = sampling domain), xi = device
        float32 [n, 10] variates in [0,1), out = device buffer of n 16-byte pndf_sample records
        (e.g. int32/float32 [n, 4])."""
        n = xi.shape[0] if n is None else n
        _check(lib().pndf_sample_batch(self.handle, _ptr(queries), _ptr(xi), n, _ptr(out), opts, _stream(stream)),
               "pndf_sample_batch")

    def sample_tiles(self, queries, xi, out, tile=None, opts: int = 0, stream=None, n: int | None = None):
        """Enqueue pndf_sample_tiles on a tiled store (Sec. 5.5): xi = device float32 [n, 11]
        (8 descent levels, 2 jitter, 1 tile choice), out = n 16-byte pndf_sample records, tile =
        optional device int32 [n, 2] receiving the chosen tile instance (tx, ty)."""
        n = xi.shape[0] if n is None else n
        _check(lib().pndf_sample_tiles(self.handle, _ptr(queries), _ptr(xi), n, _ptr(out), _ptr(tile), opts,
                                       _stream(stream)), "pndf_sample_tiles")

    def sample_blocked(self, queries, xi, out, block=None, opts: int = 0, stream=None, n: int | None = None):
        """pndf_sample_blocked: block choice + quad descent on a blocked store; xi [n, 11] fp32 (device)."""
        n = queries.shape[0] if n is None else n
        _check(lib().pndf_sample_blocked(self.handle, _ptr(queries), _ptr(xi), n, _ptr(out), _ptr(block), opts,
                                         _stream(stream)), "pndf_sample_blocked")

    def sync(self, stream=None, raise_on_query_error: bool = True) -> int:
        st = lib().pndf_sync(self.handle, _stream(stream))
        if st == EQUERY and not raise_on_query_error:
            return st
        _check(st, "pndf_sync")
        return st

    def query_batch_host(self, h_queries, h_out, opts: int = 0, raise_on_query_error: bool = True) -> int:
        n = h_out.shape[0]
        st = lib().pndf_query_batch_host(self.handle, _ptr(h_queries), n, _ptr(h_out), opts)
        if st == EQUERY and not raise_on_query_error:
            return st
        _check(st, "pndf_query_batch_host")
        return st

    def stats(self) -> dict:
        s = StoreStats()
        _check(lib().pndf_store_stats_get(self.handle, ctypes.byref(s)), "pndf_store_stats_get")
        return s.as_dict()

    def reset_stats(self):
        _check(lib().pndf_store_stats_reset(self.handle), "pndf_store_stats_reset")

    def image(self, z0: int = 0, z1: int | None = None, prefix: bool = True):
        st = self.stats()
        Rp, A = st["rank_padded"], self.desc.ang_res
        z1 = st["rows"] if z1 is None else z1
        if not prefix:
            pxy = None
        elif st["prefix_format"] == 1:
            pxy = np.empty((2, A + 1, Rp), np.uint32)
        else:
            pxy = np.empty((2, A + 1, 2, Rp), np.float32)
        zc = np.empty((z1 - z0, Rp), np.float32)
        _check(lib().pndf_store_image(self.handle, _ptr(pxy), _ptr(zc), z0, z1), "pndf_store_image")
        return pxy, zc

    def bin_permutation(self, queries, perm, keys=None):
        """Test support: binning pass only -> permutation (and sorted keys) in device buffers."""
        _check(lib().pndf_bin_permutation(self.handle, _ptr(queries), perm.shape[0], _ptr(perm), _ptr(keys)),
               "pndf_bin_permutation")

    def rows_touched(self, queries, out, n: int | None = None):
        """Measurement support: distinct Zc rows the query kernel reads for these records -> out (device int64 [1])."""
        n = queries.shape[0] if n is None else n
        _check(lib().pndf_rows_touched(self.handle, _ptr(queries), n, _ptr(out)), "pndf_rows_touched")

    def set_lanes(self, lanes: int):
        _check(lib().pndf_set_lanes(self.handle, lanes), "pndf_set_lanes")

    def free(self):
        if self._h is not None:
            lib().pndf_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def load_factors(desc: Desc, C, X, Y, Z, device: int = 0, stream=None) -> Store:
    """pndf_load_factors: raw fp32 factors (host numpy or device tensors) -> device store."""
    h = ctypes.c_void_p()
    _check(lib().pndf_load_factors(ctypes.byref(desc), _ptr(C), _ptr(X), _ptr(Y), _ptr(Z), device, _stream(stream),
                                   ctypes.byref(h)), "pndf_load_factors")
    return Store(h, desc)


def make_tile_desc(T: int, s0: int, L: int, margin: int, A: int, R: int, seed: int, prefix: int = PREFIX_AUTO):
    return TileDesc(abi_version=ABI_VERSION, tile_size=T, base_stride=s0, num_levels=L, margin=margin, ang_res=A,
                    rank=R, flags=prefix, seed=seed)


def load_tiles(td: TileDesc, C, X, Y, Z, device: int = 0, stream=None) -> Store:
    """pndf_load_tiles: 16 Wang tiles sharing X, Y; Z = [16 * P_ext, R] extended per-tile factors."""
    h = ctypes.c_void_p()
    _check(lib().pndf_load_tiles(ctypes.byref(td), _ptr(C), _ptr(X), _ptr(Y), _ptr(Z), device, _stream(stream),
                                 ctypes.byref(h)), "pndf_load_tiles")
    d = make_desc(td.tile_size, td.base_stride, td.num_levels, td.ang_res, td.rank, False)
    return Store(h, d)


def load_blocked(N: int, s0: int, L: int, A: int, wrap: bool, bs, device: int = 0, stream=None) -> Store:
    """pndf_load_blocked from a synth.BlockedStore-like object (t, region, R, C, X, Y, group_set, slab_ptr, Z)."""
    arr = dict(C=np.ascontiguousarray(bs.C, np.float32), X=np.ascontiguousarray(bs.X, np.float32),
               Y=np.ascontiguousarray(bs.Y, np.float32), G=np.ascontiguousarray(bs.group_set, np.int32),
               S=np.ascontiguousarray(bs.slab_ptr, np.int64), Z=np.ascontiguousarray(bs.Z, np.float32))
    bd = BlockDesc(abi_version=ABI_VERSION, map_size=N, base_stride=s0, num_levels=L, ang_res=A, block=bs.t,
                   region=bs.region, rank=bs.R, flags=WRAP if wrap else CLAMP, num_sets=arr["C"].shape[0],
                   num_slabs=arr["Z"].shape[0])
    h = ctypes.c_void_p()
    _check(lib().pndf_load_blocked(ctypes.byref(bd), _ptr(arr["C"]), _ptr(arr["X"]), _ptr(arr["Y"]),
                                   _ptr(arr["G"]), _ptr(arr["S"]), _ptr(arr["Z"]), device, _stream(stream),
                                   ctypes.byref(h)), "pndf_load_blocked")
    return Store(h, make_desc(N, s0, L, A, bs.R, wrap))


# ---- GPU factor builder ---------------------------------------------------------
def hist_tensor(desc: Desc, d_bins, d_D, d_Dt=None, stream=None):
    """pndf_hist_tensor: D[z][x][y] (and Dt[z][y][x]) = tf32-rounded footprint histograms, device buffers."""
    _check(lib().pndf_hist_tensor(ctypes.byref(desc), _ptr(d_bins), _ptr(d_D), _ptr(d_Dt), _stream(stream)),
           "pndf_hist_tensor")


def mttkrp(desc: Desc, d_D, d_Dt, d_Z, d_X, d_Y, mode: int, d_M, stream=None):
    """pndf_mttkrp (test support): mode 0 = Z, 1 = X, 2 = Y, into d_M (fp64, device)."""
    _check(lib().pndf_mttkrp(ctypes.byref(desc), _ptr(d_D), _ptr(d_Dt), _ptr(d_Z), _ptr(d_X), _ptr(d_Y), mode,
                             _ptr(d_M), _stream(stream)), "pndf_mttkrp")


def cp_als(desc: Desc, d_D, d_Dt, d_Z, d_X, d_Y, d_C=None, max_sweeps: int = 500, tol: float = 1e-4,
           normalise: bool = False, stream=None):
    """pndf_cp_als: factors updated in place (device fp32); returns the fit-error history (numpy)."""
    o = AlsOpts(abi_version=ABI_VERSION, max_sweeps=max_sweeps, tol=tol, flags=ALS_NORMALISE if normalise else 0)
    err = np.zeros(max_sweeps, np.float64)
    n = ctypes.c_int32(0)
    _check(lib().pndf_cp_als(ctypes.byref(desc), _ptr(d_D), _ptr(d_Dt), _ptr(d_C), _ptr(d_X), _ptr(d_Y),
                             _ptr(d_Z), ctypes.byref(o), _ptr(err), ctypes.byref(n), _stream(stream)), "pndf_cp_als")
    return err[:n.value].copy()


def cp_als_map(desc: Desc, d_bins, d_Z, d_X, d_Y, d_C=None, max_sweeps: int = 500, tol: float = 1e-4,
               normalise: bool = False, stream=None):
    """pndf_cp_als_map: CP-ALS of the exact footprint tensor without forming it (device bins [N][N] uint16);
    factors updated in place (device fp32); returns the fit-error history (numpy)."""
    o = AlsOpts(abi_version=ABI_VERSION, max_sweeps=max_sweeps, tol=tol, flags=ALS_NORMALISE if normalise else 0)
    err = np.zeros(max_sweeps, np.float64)
    n = ctypes.c_int32(0)
    _check(lib().pndf_cp_als_map(ctypes.byref(desc), _ptr(d_bins), _ptr(d_C), _ptr(d_X), _ptr(d_Y), _ptr(d_Z),
                                 ctypes.byref(o), _ptr(err), ctypes.byref(n), _stream(stream)), "pndf_cp_als_map")
    return err[:n.value].copy()


def mttkrp_map(desc: Desc, d_bins, d_Z, d_X, d_Y, mode: int, d_M, stream=None) -> float:
    """pndf_mttkrp_map (test support): one map-domain MTTKRP into d_M (fp64, device); returns ||D||^2."""
    v = ctypes.c_double(0.0)
    _check(lib().pndf_mttkrp_map(ctypes.byref(desc), _ptr(d_bins), _ptr(d_Z), _ptr(d_X), _ptr(d_Y), mode,
                                 _ptr(d_M), ctypes.byref(v), _stream(stream)), "pndf_mttkrp_map")
    return v.value
