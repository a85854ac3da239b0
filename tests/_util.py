"""Shared helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import functools

import numpy as np

import oracle
import synth

# BASELINE.json north_star: "within 1e-4 relative (or 1e-7 absolute on near-zero values) in fp32"
RTOL = 1e-4
ATOL = 1e-7


def assert_parity(gpu: np.ndarray, ref: np.ndarray, what: str = ""):
    """|g - o| <= 1e-4 |o|  or  |g - o| <= 1e-7, element by element; NaN only where the oracle is NaN."""
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape
    nan_o, nan_g = np.isnan(ref), np.isnan(gpu)
    assert np.array_equal(nan_o, nan_g), f"{what}: NaN pattern differs ({nan_o.sum()} vs {nan_g.sum()})"
    m = ~nan_o
    err = np.abs(gpu[m] - ref[m])
    ok = (err <= RTOL * np.abs(ref[m])) | (err <= ATOL)
    if not ok.all():
        bad = np.flatnonzero(~ok)[:5]
        raise AssertionError(f"{what}: {int((~ok).sum())}/{ok.size} outside tolerance; e.g. gpu={gpu[m][bad]} "
                             f"oracle={ref[m][bad]}")
    rel = err / np.maximum(np.abs(ref[m]), 1e-300)
    # the 1e-7 floor is for near-zero values: above 1e-6 the relative bound must hold on its own (a 1e-5
    # result may not hide a 1% error behind the absolute floor)
    big = np.abs(ref[m]) > 1e-6
    if big.any() and rel[big].max() > RTOL:
        i = np.flatnonzero(big)[np.argmax(rel[big])]
        raise AssertionError(f"{what}: relative error {rel[i]:.3g} on a non-negligible value "
                             f"(gpu={gpu[m][i]}, oracle={ref[m][i]})")
    return dict(n=int(m.sum()), max_abs=float(err.max(initial=0)), max_rel_nonzero=float(
        rel[np.abs(ref[m]) > 1e-6].max(initial=0)), zeros=int((ref[m] == 0).sum()))


def torch_records(recs: np.ndarray, device="cuda"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(recs).view(np.int32).reshape(-1, 4)).to(device)


def run_gpu(desc_args: dict, f, recs: np.ndarray, opts: int = 0, lanes: int = 0, prefix: int = 0,
            want_format: int | None = None):
    """Load a store from raw factors, run one batch through the C ABI, return fp32 results + sticky status."""
    import torch
    from paper_2109_14807_b200 import pndf
    d = pndf.make_desc(**desc_args, prefix=prefix)
    st = pndf.load_factors(d, f.C, f.X, f.Y, f.Z)
    if want_format is not None:
        assert st.stats()["prefix_format"] == want_format
    if lanes:
        st.set_lanes(lanes)
    q = torch_records(recs)
    # NaN-filled so a permutation that skips a query cannot pass off a stale value
    out = torch.full((recs.shape[0],), float("nan"), dtype=torch.float32, device="cuda")
    st.query_batch(q, out, opts)
    status = st.sync(raise_on_query_error=False)
    res = out.cpu().numpy()
    st.free()
    return res, status


def desc_args(cfg) -> dict:
    return dict(N=cfg.N, s0=cfg.s0, L=cfg.L, A=cfg.A, R=cfg.R, wrap=cfg.wrap)


@functools.lru_cache(maxsize=None)
def config_inputs(k: int, host_z: bool = True):
    """(cfg, nxy-free bins, factors) for BASELINE config k (cached per process)."""
    cfg = synth.CONFIGS[k]
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    f = synth.build_factors(cfg, nxy, bins, with_z=host_z)
    return cfg, bins, f


def oracle_on(cfg, f, recs, mean=True, zsparse=None):
    d = oracle.desc_of(cfg)
    if zsparse is None:
        return oracle.query_batch(d, f.C, f.X, f.Y, f.Z, recs, mean=mean)
    Zs, zmap = zsparse
    return oracle.query_batch(d, f.C, f.X, f.Y, Zs, recs, mean=mean, zmap=zmap)


def expected_prefix_format(f) -> int:
    """The AUTO rule restated in numpy: U32 (1) iff for every rank of X and Y the fixed-point step
    2^-e (e = largest with total*2^e <= 2^32-2) is <= 2^-15 of the smallest nonzero entry."""
    import math
    for F in (f.X, f.Y):
        F = np.asarray(F, np.float64)
        for r in range(F.shape[1]):
            T = float(F[:, r].sum())
            if T <= 0:
                continue
            e = math.floor(math.log2(4294967294.0 / T))
            while math.ldexp(T, e) > 4294967294.0:
                e -= 1
            nz = F[:, r][F[:, r] > 0]
            if math.ldexp(1.0, -e) > math.ldexp(float(nz.min()), -15):
                return 0
    return 1
