#!/usr/bin/env python
"""bench.py -- batched NDF range queries/s on B200 (BASELINE.json "metric").

One step = one pndf_query_batch over this rank's shard of the workload's query
batch: binning (row a1) + the query kernel (rows a2-a6), inputs resident in HBM.
Default workload: BASELINE.json configs[4] ("Scaling": 4096^2 flake map, A=R=256,
10^9 queries sharded over the ranks; factors replicated) -- the config the
metric's "1/2/4/8 B200" numbers are quoted on, and it fits one GPU.

Launch: python bench.py [--gpus N --steps K --warmup W]; for N > 1 under
torchrun (one process per GPU, NCCL only for the max-time / checksum reductions
after the timed region -- the path has no exchange step).
``--impl reference`` times the fp64 CPU oracle on a bounded sample instead.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (seeded inputs; no query arithmetic)

METRIC = "NDF range queries/sec at 1/2/4/8 B200 and % of gather (HBM/L2) roofline"
UNIT = "queries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--op", default="query", choices=["query", "sample", "sg", "wang", "wang_sample", "blocked", "als",
                                                      "als_map", "blocked_sample",
                                                      "sweep"],
                    help="query: the range-query path (default); sample: SURVEY §8(f) row 1, hierarchical "
                         "importance sampling over the whole A x A image; sg: §8(f) row 4, environment-light "
                         "prefiltering (SG rectangle generation + range query)")
    ap.add_argument("--queries", type=int, default=0, help="override the config's total query count")
    ap.add_argument("--s0", type=int, default=0, help="override the base stride (SURVEY §8(d): config 3 at s0=4 "
                                                       "is the ~L2-resident variant, Zc 89.5 MB)")
    ap.add_argument("--as-shard", default="", help="K/W: one GPU runs rank K's shard of a W-GPU job "
                                                    "(per-GPU cost of the multi-GPU run on a one-GPU box)")
    ap.add_argument("--shard", default="spatial", choices=["spatial", "index"],
                    help="N > 1: spatial = rank k answers the stream's queries centred in the k-th vertical "
                         "strip of the map; index = the k-th contiguous index range (identical at N = 1)")
    ap.add_argument("--bin", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--lanes", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the sampled oracle check of the timed batch")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU work of the oracle sample")
    return ap.parse_args()


def workload_name(cfg) -> str:
    s0 = f", base stride s0={cfg.s0}" if cfg.s0 != 1 else ""
    return (f"config{cfg.idx}-{cfg.name}: {cfg.N}^2 {cfg.map_kind} map, A={cfg.A}, R={cfg.R}, "
            f"L={cfg.L} levels (P={cfg.P} rows){s0}, {cfg.n_queries:.0e} queries")


def max_side(cfg) -> int:
    """Widest query rectangle side of the config's generator."""
    return {1: 8, 2: 8, 3: 16, 4: 3, 5: 16}.get(cfg.idx, cfg.A)


def bytes_per_query(R: int) -> int:
    """record 16 B + result 4 B + 8 Z rows + 4 prefix rows of R fp32 = 20 + 48 R."""
    return 20 + 48 * R


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)), "measured"
    return {"hbm_gbs": 6650.0}, "fallback"


FLOP_RANK_QUERY = 19  # a4 8 FMA (16 flop) + a6 dx*dy (1) + FMA into the rank sum (2), per rank and query


def fp32_peak_tflops():
    """FP32 ceiling of the SMs: SMs x 128 FP32 lanes x 2 flop (FMA) x max SM clock.  On B200:
    148 x 128 x 2 x 1965 MHz = 74.4 TFLOP/s (unit counts and clock from B200_PROFILING.md / MEASURED_PEAKS.json;
    packed FFMA2 issues 2 FMAs per lane every 2 cycles, B300_MICROARCH.md 'pipe rates', so it reaches it)."""
    import torch
    peaks, _ = measured_peaks()
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return sms * 128 * 2 * mhz * 1e6 / 1e12


def issue_ceiling(inst_per_unit):
    """Units/s at one warp instruction per cycle on each of the 4 SMSPs of every SM (max SM clock)."""
    import torch
    peaks, _ = measured_peaks()
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return sms * 4 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / inst_per_unit if inst_per_unit else None


def query_kernel_name(st):
    """The query kernel a store's batches launch (csrc/query_kernel.cuh launch_q): 32 lanes per query, at most
    2 float4 per lane and a range table -> query_g5_kernel (unless PNDF_NOG5 / PNDF_NOG4), else query_kernel."""
    g32 = st["lanes_per_query"] == 32 and st["rank_padded"] <= 256 and st.get("range_table_width", 0) > 0
    if g32 and not int(os.environ.get("PNDF_NOG5", "0") or 0):
        return "pndf::query_g5_kernel"
    if g32 and not int(os.environ.get("PNDF_NOG4", "0") or 0):
        return "pndf::query_g4_kernel"
    return "pndf::query_kernel"


def alu_roof(flop_per_unit, units, k_ms, kernel, unit_name, **extra):
    """`roofline` object against the FP32 ALU ceiling (the binding roof of these gather-and-reduce kernels
    once binning keeps the Zc rows on chip: DESIGN.md §5)."""
    peak = fp32_peak_tflops()
    achieved = flop_per_unit * units / (k_ms * 1e-3) / 1e12
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": None, "kernel": kernel, "kernel_ms": k_ms, f"flop_per_{unit_name}": flop_per_unit,
            "peak_source": "derived: SMs x 128 FP32 lanes x 2 flop x sm_max_mhz (MEASURED_PEAKS.json), "
                           "DESIGN.md §5"}
    roof.update(extra)
    return roof


def ncu_traffic(cfg_idx: int):
    """DRAM bytes per query of the query kernel from the committed ncu --set full summary, if any
    (profiles/ncu_traffic.json, written from a capture of the same launch configuration)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"config{cfg_idx}")


def l2_read_gbs():
    """Measured L2-resident read bandwidth of this GPU (tools/membw.cu, float4 loads, 48 MB set)."""
    import ctypes
    src = os.path.join(ROOT, "tools", "membw.cu")
    so = os.path.join(ROOT, "tools", "libmembw.so")
    try:
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            subprocess.check_call(["nvcc", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                                   "arch=compute_100a,code=sm_100a", "-O3", "-o", so, src])
        lib = ctypes.CDLL(so)
        lib.membw_l2_read_gbs.restype = ctypes.c_double
        lib.membw_l2_read_gbs.argtypes = [ctypes.c_int]
        v = lib.membw_l2_read_gbs(48)
        return v if v > 0 else None
    except Exception:
        return None


def parity_sample(cfg, f, h_q, d_out, k=4096, seed=7):
    """Check k sampled outputs of the timed batch against the fp64 oracle (BJ tolerance)."""
    import oracle
    import torch
    n = d_out.shape[0]
    rng = np.random.default_rng(seed)
    idx = np.unique(rng.integers(0, n, min(k, n)))
    recs = np.ascontiguousarray(h_q[torch.from_numpy(idx)].numpy()).view(synth.QREC).reshape(-1)
    got = d_out[torch.from_numpy(idx).to(d_out.device)].cpu().numpy().astype(np.float64)
    d = oracle.desc_of(cfg)
    rows, _ = oracle.neighbours(d, recs)
    Zs, zmap = oracle.sparse_z(rows, cfg.P, lambda u: z_rows_for(cfg, f, u))
    ref = oracle.query_batch(d, f.C, f.X, f.Y, Zs, recs, mean=True, zmap=zmap)
    err = np.abs(got - ref)
    ok = (err <= 1e-4 * np.abs(ref)) | (err <= 1e-7)
    nz = np.abs(ref) > 1e-6
    return {"checked": int(idx.shape[0]), "pass": bool(ok.all()), "max_abs_err": float(err.max()),
            "max_rel_err_nonzero": float((err[nz] / np.abs(ref[nz])).max()) if nz.any() else 0.0,
            "tolerance": "1e-4 rel or 1e-7 abs (BASELINE.json north_star)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, bus_id: str | None):
        self.bus_id = bus_id
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200"]
            if self.bus_id:
                cmd += ["-i", self.bus_id]
            self.proc = subprocess.Popen(cmd, stdout=self.f, stderr=subprocess.DEVNULL)
            # wait (<= 3 s) until the sampler is live, so even a timed region of a few ms is covered
            t0 = time.time()
            while time.time() - t0 < 3.0 and self.proc.poll() is None and os.path.getsize(self.f.name) == 0:
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)  # one more sample at the end of the region (short regions)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = [r.split(", ") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax = max(smax, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip() == "Active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


def bus_id_of(dev) -> str | None:
    try:
        import torch
        p = torch.cuda.get_device_properties(dev)
        return f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
    except Exception:
        return None


# ---------------------------------------------------------------- inputs --
def host_inputs(cfg):
    """Map -> angular bins -> factors (C, X, Y on host; Z stays None for exact-rank configs)."""
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    del nxy
    if cfg.factor_kind == "als":
        f = synth.build_factors(cfg, None, bins)
    else:
        f = synth.build_factors(cfg, None, bins, with_z=False)
    return bins, f


def z_rows_for(cfg, f, rows):
    if f.Z is not None:
        return f.Z[rows]
    return synth.build_z_rows(cfg, f.info["atom_map"], rows)


MAX_SAMPLE = 1_000_000  # bounds the host RAM of the pre-gathered Z rows


def oracle_sample_rate(cfg, f, recs, threads=0, min_seconds=0.0):
    """Time the fp64 oracle (as it stands) on recs, repeating passes until min_seconds of work;
    the Z rows it reads are gathered (untimed) before the timed region."""
    import oracle
    d = oracle.desc_of(cfg)
    rows, _ = oracle.neighbours(d, recs)
    Zs, zmap = oracle.sparse_z(rows, cfg.P, lambda u: z_rows_for(cfg, f, u))
    passes, dt = 0, 0.0
    t0 = time.perf_counter()
    while True:
        out = oracle.query_batch(d, f.C, f.X, f.Y, Zs, recs, mean=True, zmap=zmap, threads=threads)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    return recs.shape[0] * passes / dt, dt, out, passes


def spatial_shard(cfg, bins, n_total: int, rank: int, world: int):
    """The stream's queries [0, n_total) whose centre lies in this rank's strip (shard.spatial_owner),
    generated chunk by chunk (untimed setup), in stream order, as a pinned [n, 4] int32 tensor."""
    import torch
    from paper_2109_14807_b200.shard import spatial_owner
    keep = []
    chunk = 1 << 26
    for a in range(0, n_total, chunk):
        recs = synth.gen_queries(cfg, bins, a, min(n_total, a + chunk))
        keep.append(recs[spatial_owner(recs["u"], cfg.N, world) == rank])
    mine = np.concatenate(keep) if keep else np.empty(0, synth.QREC)
    h_q = torch.empty((mine.shape[0], 4), dtype=torch.int32, pin_memory=torch.cuda.is_available())
    h_q.numpy().view(synth.QREC).reshape(-1)[:] = mine
    return h_q


def cpu_baseline(cfg, f, bins, shard0: int, seconds: float):
    """Oracle on a bounded sample of the same workload (first m queries of the stream), all host cores."""
    import oracle
    probe = synth.gen_queries(cfg, bins, shard0, shard0 + 2000)
    r0 = oracle_sample_rate(cfg, f, probe)[0]
    m = int(max(2000, min(cfg.n_queries, MAX_SAMPLE, r0 * seconds)))
    recs = synth.gen_queries(cfg, bins, shard0, shard0 + m)
    rate, dt, _, passes = oracle_sample_rate(cfg, f, recs, min_seconds=seconds)
    return {"value": rate, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
            "sample": f"queries [{shard0}, {shard0 + m}) of the {cfg.n_queries:.0e}-query stream x {passes} "
                      f"pass(es), {dt:.1f} s; fp64, OpenMP over queries, Z rows pre-gathered"}


# --------------------------------------------------------------- ref arm --
def run_reference(args, cfg, rank, world):
    if rank != 0:
        return 0
    import oracle
    bins, f = host_inputs(cfg)
    n_total = args.queries or cfg.n_queries
    probe = synth.gen_queries(cfg, bins, 0, 2000)
    r0 = oracle_sample_rate(cfg, f, probe)[0]
    per_step = max(2000, int(r0 * min(20.0, args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup))))
    per_step = min(per_step, n_total, MAX_SAMPLE)
    times = []
    for s in range(args.warmup + args.steps):
        a = (s * per_step) % max(1, n_total - per_step + 1)
        recs = synth.gen_queries(cfg, bins, a, a + per_step)
        rate, dt, _, _ = oracle_sample_rate(cfg, f, recs)
        if s >= args.warmup:
            times.append(dt)
    t = float(np.mean(times))
    value = per_step / t
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "sample_queries_per_step": per_step},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
                             "sample": f"{per_step} queries per step from the config's stream"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm --
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2109_14807_b200 import pndf
    from paper_2109_14807_b200.shard import reduce_times_and_checksum, shard_range

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n_total = args.queries or cfg.n_queries
    i0, i1 = shard_range(n_total, rank, world)
    n = i1 - i0

    # ---- store (untimed): map on host, exact-rank Z built on this GPU (synth CUDA twin)
    t_setup = time.perf_counter()
    bins, f = host_inputs(cfg)
    if f.Z is None:
        Z = synth.build_z_exact_cuda(cfg, f.info["atom_map"], local_rank)
    else:
        Z = f.Z
    prefix = {"auto": pndf.PREFIX_AUTO, "hilo": pndf.PREFIX_HILO, "u32": pndf.PREFIX_U32}[
        os.environ.get("PNDF_PREFIX", "auto")]  # SAT storage format (experiments); AUTO by default
    desc = pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, cfg.wrap, prefix=prefix)
    store = pndf.load_factors(desc, f.C, f.X, f.Y, Z, device=local_rank)
    del Z
    torch.cuda.empty_cache()
    if args.lanes:
        store.set_lanes(args.lanes)

    # ---- this rank's query shard: pinned host copy (for e2e) + resident device copy
    sim_rank, sim_world = (int(x) for x in args.as_shard.split("/")) if args.as_shard else (rank, world)
    if sim_world > 1 and args.shard == "spatial":
        h_q = spatial_shard(cfg, bins, n_total, sim_rank, sim_world)
        n = h_q.shape[0]
    elif sim_world > 1:
        i0, i1 = shard_range(n_total, sim_rank, sim_world)
        n = i1 - i0
        h_q = torch.empty((n, 4), dtype=torch.int32, pin_memory=True)
        synth.gen_queries(cfg, bins, i0, i1, out=h_q.numpy().view(synth.QREC).reshape(-1))
    else:
        h_q = torch.empty((n, 4), dtype=torch.int32, pin_memory=True)
        synth.gen_queries(cfg, bins, i0, i1, out=h_q.numpy().view(synth.QREC).reshape(-1))
    d_q = h_q.to(dev, non_blocking=False)
    d_out = torch.empty(n, dtype=torch.float32, device=dev)
    opts = {"auto": pndf.BIN_AUTO, "on": pndf.BIN_ON, "off": pndf.BIN_OFF}[args.bin]
    setup_s = time.perf_counter() - t_setup

    l2_gbs = l2_read_gbs() if rank == 0 else None

    # ---- warm-up
    for _ in range(args.warmup):
        store.query_batch(d_q, d_out, opts)
        store.sync()
    store.reset_stats()
    launches0 = store.stats()["kernel_launches"]

    # ---- timed region: K steps, CUDA events on the launching stream, barrier + sync both sides
    clocks = ClockSampler(bus_id_of(dev))
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        store.query_batch(d_q, d_out, opts | pndf.TIMING)
        store.sync()
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    st = store.stats()
    launches = st["kernel_launches"] - launches0
    q_ms = st["query_ms"] / max(1, st["timed_batches"])
    b_ms = st["bin_ms"] / max(1, st["timed_batches"])

    checksum = float(d_out.double().sum().item())
    d_out_ref = d_out.clone() if n <= 1_000_000 else None
    (ms_step, q_ms_max, b_ms_max), checksum = reduce_times_and_checksum([ms_rank, q_ms, b_ms], checksum, dev)
    value = (n if args.as_shard else n_total) / (ms_step * 1e-3)  # --as-shard: this shard's own rate

    # ---- N > 1: the same job index-sharded too (rank k answers the k-th contiguous range of the stream)
    index_sh = None
    if world > 1 and args.shard == "spatial" and not args.as_shard:
        j0, j1 = shard_range(n_total, rank, world)
        h_qi = torch.empty((j1 - j0, 4), dtype=torch.int32, pin_memory=True)
        synth.gen_queries(cfg, bins, j0, j1, out=h_qi.numpy().view(synth.QREC).reshape(-1))
        d_qi = h_qi.to(dev)
        d_oi = torch.empty(j1 - j0, dtype=torch.float32, device=dev)
        for _ in range(args.warmup):
            store.query_batch(d_qi, d_oi, opts)
            store.sync()
        dist.barrier()
        torch.cuda.synchronize()
        ia, ib = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ia.record()
        for _ in range(args.steps):
            store.query_batch(d_qi, d_oi, opts)
            store.sync()
        ib.record()
        torch.cuda.synchronize()
        dist.barrier()
        (ims,), ichk = reduce_times_and_checksum([ia.elapsed_time(ib) / args.steps],
                                                 float(d_oi.double().sum().item()), dev)
        index_sh = {"value": n_total / (ims * 1e-3), "unit": UNIT, "ms_per_step": ims, "checksum": ichk,
                    "note": "rank k answers queries [k n/N, (k+1) n/N) of the stream: no partition step, but each "
                            "rank's batch is 1/N as dense per Zc row, so binning finds less reuse"}
        del d_qi, d_oi, h_qi

    # ---- launch-bound small batches: steady state of GRAPH_BATCHES back-to-back
    # batches captured in one CUDA graph, beside the single-batch step time above
    graph = None
    if world == 1 and n <= 1_000_000 and not store.stats()["last_binned"]:
        try:
            gs = torch.cuda.Stream()
            gs.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(gs):
                store.query_batch(d_q, d_out, opts, stream=gs)  # warm on the capture stream
                gs.synchronize()
                with torch.cuda.graph(g, stream=gs):
                    for _ in range(GRAPH_BATCHES):
                        store.query_batch(d_q, d_out, opts, stream=gs)
            torch.cuda.current_stream().wait_stream(gs)
            g.replay()
            torch.cuda.synchronize()
            reps = 10
            ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ga.record()
            for _ in range(reps):
                g.replay()
            gb.record()
            torch.cuda.synchronize()
            store.sync()
            gms = ga.elapsed_time(gb) / (reps * GRAPH_BATCHES)
            graph = {"batches_per_graph": GRAPH_BATCHES, "us_per_batch": gms * 1e3,
                     "value": n / (gms * 1e-3), "unit": UNIT,
                     "single_batch_us": ms_step * 1e3,
                     "bitwise_equal_to_step": bool(torch.equal(d_out, d_out_ref))}
            del g
        except Exception as e:  # report, do not hide
            graph = {"error": repr(e)[:200]}

    # ---- end to end through the public API with HOST buffers (H2D + kernels + D2H inside)
    e2e = None
    if not args.no_e2e:
        h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
        store.query_batch_host(h_q, h_out, opts)  # warm the host pipeline buffers
        times = []
        for _ in range(max(1, args.e2e_steps)):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            store.query_batch_host(h_q, h_out, opts)
            times.append(time.perf_counter() - t0)
        (te,), _ = reduce_times_and_checksum([float(np.mean(times))], 0.0, dev)
        e2e = {"value": n_total / te, "unit": UNIT, "h2d_bytes_per_step": int(h_q.numel() * 4),
               "d2h_bytes_per_step": int(h_out.numel() * 4),
               "bitwise_equal_to_device_path": bool(torch.equal(h_out.to(dev), d_out))}

    if rank != 0:
        store.free()
        return 0

    peaks, peak_src = measured_peaks()
    hbm = peaks["hbm_gbs"]
    tr = ncu_traffic(cfg.idx)
    traffic = None if tr is None else int(tr["dram_bytes_per_query"] * n)
    # compulsory HBM bytes of the batch: every distinct Zc row once + record and result (+ permutation)
    d_rows = torch.zeros(1, dtype=torch.int64, device=dev)
    store.rows_touched(d_q, d_rows)
    rows_u = int(d_rows.item())
    comp = rows_u * st["rank_padded"] * 4 + n * (20 + (4 if st["last_binned"] else 0))
    Rp = st["rank_padded"]
    ang_rows = 2 if max_side(cfg) <= min(48, cfg.A) else 4  # range-table rows (sides <= 48 bins) else SAT rows
    ceil = {"fp32_alu": fp32_peak_tflops() * 1e12 / (FLOP_RANK_QUERY * cfg.R),
            "l2_angular_rows": (l2_gbs * 1e9 / (ang_rows * 4 * Rp)) if l2_gbs else None,
            "hbm_compulsory": hbm * 1e9 / (comp / n),
            "issue": issue_ceiling(tr.get("warp_instructions_per_query")) if tr else None,
            # query_g5_kernel: both range rows cross the SM's shared-memory path twice (gather4 in, LDS.128
            # out) at 128 B per cycle, + ~6 wavefronts of descriptors, weights and partials
            "smem_path": (issue_ceiling(4.0 * (2 * ang_rows * 4 * Rp / 128 + 6)))
            if query_kernel_name(st) == "pndf::query_g5_kernel" else None}
    roof = alu_roof(FLOP_RANK_QUERY * cfg.R, n, q_ms, query_kernel_name(st), "query",
                    traffic=traffic, traffic_source=None if tr is None else tr.get("source"),
                    ceilings_queries_per_s=ceil, achieved_queries_per_s=n / (q_ms * 1e-3),
                    hbm_compulsory={"bytes": comp, "distinct_zc_rows": rows_u, "gbs": comp / (q_ms * 1e-3) / 1e9,
                                    "frac_of_hbm": comp / (q_ms * 1e-3) / 1e9 / hbm,
                                    "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs"},
                    l2={"peak_gbs_measured": l2_gbs, "angular_row_bytes_per_query": ang_rows * 4 * Rp,
                        "frac": (n * ang_rows * 4 * Rp / (q_ms * 1e-3) / 1e9 / l2_gbs) if l2_gbs else None,
                        "ncu_l2_read_bytes_per_query": tr.get("l2_read_bytes_per_query") if tr else None},
                    touched_bytes_per_query=bytes_per_query(cfg.R),
                    note="frac = FP32 work (19 flop per rank and query) over the FP32 ceiling; the other ceilings "
                         "beside it; touched_bytes_per_query (20 + 48R, the method's 12 look-ups) is not a roof: "
                         "binned queries reuse Zc rows from registers",
                    binning_ms=b_ms, query_share_of_step=q_ms / ms_rank if ms_rank else None)
    # the ceiling the kernel sits closest to (frac above stays the FP32 one the contract names)
    fr = {k: (n / (q_ms * 1e-3)) / v for k, v in ceil.items() if v}
    near = max(fr, key=fr.get)
    roof["closest_ceiling"] = {"name": near, "frac": fr[near]}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, f, bins, i0, args.cpu_seconds)
    parity = parity_sample(cfg, f, h_q, d_out) if not args.no_parity else None
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "queries_total": n_total, "queries_per_rank": n,
                       "parallelism": f"query-sharded x{world} ({args.shard if world > 1 else 'whole stream'}), "
                                      "factors replicated",
                       "stream": ("pre-partitioned by vertical map strip (screen-space tiles of a renderer); the "
                                  "partition is untimed setup" if world > 1 and args.shard == "spatial" else
                                  "index-sharded" if world > 1 else "whole stream on one GPU"),
                       "binning": args.bin, "binned": bool(st["last_binned"]),
                       "lanes_per_query": st["lanes_per_query"], "rank_padded": st["rank_padded"],
                       "sat_format": ["fp32 hi/lo", "u32 fixed point"][st["prefix_format"]],
                       "l2": ("inputs larger than L2 (Zc %.1f GB, records %.1f GB vs 126 MB L2); no flush" % (
                           st["zc_bytes"] / 1e9, n * 16 / 1e9)) if st["zc_bytes"] + n * 16 > 126e6 else
                       ("L2-resident by design (Zc %.1f MB + records %.1f MB < 126 MB L2; SURVEY §8(d) bounds "
                        "this config by L2); no flush" % (st["zc_bytes"] / 1e6, n * 16 / 1e6)),
                       "setup_s": round(setup_s, 1)},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "graph_steady_state": graph, "index_sharding": index_sh,
            "parity_sample": parity,
            "clocks": clk, "checksum": checksum}
    print(json.dumps(line), flush=True)
    store.free()
    return 0


SWEEP_METRIC = "NDF range queries/sec across footprint size x rectangle side (constant cost, P:118)"
SWEEP_S = (1, 16, 256, 2048)
SWEEP_SIDE = (1, 16, 128)


def run_sweep_op(args, cfg, rank, world, local_rank):
    """--op sweep (SURVEY §8(d) secondary sweep): config 3's store, each cell a batch of queries with the
    footprint size S fixed in {1, 16, 256, 2048} and square rectangles of side fixed in {1, 16, 128},
    centres uniform over the map, rectangles uniform over the grid.  The method's claim is constant cost
    per query ("achieving both constant performance and constant storage, a.k.a. constant cost"): q/s
    may vary with cache residency (S picks the level: S = 2048 touches 43 KB of Zc, S = 1 the whole 1.1
    GB level 0) and with the a5 path (sides <= 48 read one range-table row per axis, side 128 two SAT
    rows), never with rectangle area.  `value` = the slowest cell; each cell is parity-sampled."""
    import torch
    from paper_2109_14807_b200 import pndf
    if world > 1 and rank != 0:
        return 0  # replicas only: one GPU measures the sweep
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n = args.queries or cfg.n_queries
    bins, f = host_inputs(cfg)
    Z = synth.build_z_exact_cuda(cfg, f.info["atom_map"], local_rank) if f.Z is None else f.Z
    store = pndf.load_factors(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, cfg.wrap), f.C, f.X, f.Y, Z,
                              device=local_rank)
    del Z
    torch.cuda.empty_cache()
    rng = np.random.default_rng(700)
    h_q = torch.empty((n, 4), dtype=torch.int32, pin_memory=True)
    d_q = torch.empty((n, 4), dtype=torch.int32, device=dev)
    d_out = torch.empty(n, dtype=torch.float32, device=dev)
    cells, worst, all_pass = [], None, True
    clocks = ClockSampler(bus_id_of(dev))
    clocks.start()
    for S in SWEEP_S:
        for side in SWEEP_SIDE:
            x1 = rng.integers(0, cfg.A - side + 1, n)
            y1 = rng.integers(0, cfg.A - side + 1, n)
            recs = synth.make_records(rng.uniform(0, cfg.N, n), rng.uniform(0, cfg.N, n), np.full(n, float(S)),
                                      x1, x1 + side - 1, y1, y1 + side - 1)
            h_q.numpy().view(synth.QREC).reshape(-1)[:] = recs
            d_q.copy_(h_q)
            for _ in range(args.warmup):
                store.query_batch(d_q, d_out, pndf.BIN_AUTO)
                store.sync()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                store.query_batch(d_q, d_out, pndf.BIN_AUTO)
                store.sync()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            par = parity_sample(cfg, f, h_q, d_out, k=1024) if not args.no_parity else None
            all_pass = all_pass and (par is None or par["pass"])
            qps = n / (ms * 1e-3)
            cells.append({"S": S, "side": side, "queries_per_s": qps, "ms": ms,
                          "binned": bool(store.stats()["last_binned"]), "parity_pass": None if par is None
                          else par["pass"]})
            worst = qps if worst is None else min(worst, qps)
    clk = clocks.stop()
    by_s = {S: [c["queries_per_s"] for c in cells if c["S"] == S] for S in SWEEP_S}
    line = {"metric": SWEEP_METRIC, "value": worst, "unit": "queries/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max(c["ms"] for c in cells), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg) + f", {n} queries per cell, S fixed x square side fixed",
                       "S": list(SWEEP_S), "side": list(SWEEP_SIDE)},
            "sweep": cells,
            "side_spread_at_fixed_S": {str(S): max(v) / min(v) for S, v in by_s.items()},
            "roofline": None, "cpu_baseline": None, "e2e": None,
            "gpu_launches": None, "parity_sample": {"pass": all_pass, "checked_per_cell": 1024},
            "clocks": clk}
    print(json.dumps(line), flush=True)
    store.free()
    return 0


GRAPH_BATCHES = 100

SAMPLE_METRIC = "NDF importance samples/sec (hierarchical quad descent, Sec. 5.2)"


def sample_bytes(R: int, A: int) -> int:
    """Per sample: record 16 + variates 40 + result 16 B, 8 Zc rows, 4 corner + 2 per level SAT rows of R fp32."""
    levels = max(1, (A - 1).bit_length())
    return 72 + 4 * R * (8 + 4 + 2 * levels)


def sample_flop(R: int, A: int) -> int:
    """Method flops per sample: Z-hat interpolation 16R, the root range query 3R (dx*dy, FMA), then per level of
    the quad descent 4 quadrant range queries of 3R each."""
    levels = max(1, (A - 1).bit_length())
    return 16 * R + 3 * R + levels * 4 * 3 * R


def run_sample_op(args, cfg, rank, world, local_rank):
    """--op sample: pndf_sample_batch over the shard (domain = whole image), same timing rules."""
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2109_14807_b200 import pndf
    from paper_2109_14807_b200.shard import reduce_times_and_checksum, shard_range
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n_total = args.queries or min(cfg.n_queries, 10**8)
    i0, i1 = shard_range(n_total, rank, world)
    n = i1 - i0
    bins, f = host_inputs(cfg)
    Z = synth.build_z_exact_cuda(cfg, f.info["atom_map"], local_rank) if f.Z is None else f.Z
    store = pndf.load_factors(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, cfg.wrap), f.C, f.X, f.Y, Z,
                              device=local_rank)
    if args.lanes:
        store.set_lanes(args.lanes)
    del Z
    torch.cuda.empty_cache()
    h_q = torch.empty((n, 4), dtype=torch.int32)
    recs = h_q.numpy().view(synth.QREC).reshape(-1)
    synth.gen_queries(cfg, bins, i0, i1, out=recs)
    recs["rect"] = synth.pack_rect(0, cfg.A - 1, 0, cfg.A - 1)
    d_q = h_q.to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    d_xi = torch.rand((n, 10), generator=g, device=dev, dtype=torch.float32)
    d_out = torch.empty((n, 4), dtype=torch.float32, device=dev)
    opts = {"auto": pndf.BIN_AUTO, "on": pndf.BIN_ON, "off": pndf.BIN_OFF}[args.bin]
    for _ in range(args.warmup):
        store.sample_batch(d_q, d_xi, d_out, opts)
        store.sync()
    store.reset_stats()
    l0 = store.stats()["kernel_launches"]
    clocks = ClockSampler(bus_id_of(dev))
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        store.sample_batch(d_q, d_xi, d_out, opts | pndf.TIMING)
        store.sync()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    st = store.stats()
    ms_rank = e0.elapsed_time(e1) / args.steps
    k_ms = st["query_ms"] / max(1, st["timed_batches"])
    (ms_step, k_ms_max), _ = reduce_times_and_checksum([ms_rank, k_ms], 0.0, dev)
    if rank != 0:
        store.free()
        return 0
    Bs = sample_bytes(cfg.R, cfg.A)
    # parity on a sample of the timed batch (oracle sampler on the same variates)
    idx = np.unique(np.random.default_rng(3).integers(0, n, min(n, 2000)))
    rs = recs[idx]
    xi = d_xi[torch.from_numpy(idx).to(dev)].cpu().numpy()
    o = d_out[torch.from_numpy(idx).to(dev)].cpu().numpy()
    pix = o[:, 3].view(np.uint32)
    d = oracle.desc_of(cfg)
    rows, _ = oracle.neighbours(d, rs)
    Zs, zmap = oracle.sparse_z(rows, cfg.P, lambda u: z_rows_for(cfg, f, u))
    ref = oracle.sample_batch(d, f.C, f.X, f.Y, Zs, rs, xi, zmap=zmap)
    firm = ref["margin"] > 1e-4
    same = (pix & 0xffff == ref["pixel"][:, 0]) & (pix >> 16 == ref["pixel"][:, 1])
    pdf_ref = ref["prob"] * cfg.A * cfg.A / 4.0
    rel = np.abs(o[:, 2] - pdf_ref) / np.maximum(pdf_ref, 1e-30)
    t0 = time.perf_counter()
    ref2 = oracle.sample_batch(d, f.C, f.X, f.Y, Zs, rs, xi, zmap=zmap)
    cpu_rate = rs.shape[0] / (time.perf_counter() - t0)
    line = {"metric": SAMPLE_METRIC, "value": n_total / (ms_step * 1e-3), "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg) + "; importance sampling over the whole A x A image",
                       "samples_total": n_total, "binned": bool(st["last_binned"]),
                       "sat_format": ["fp32 hi/lo", "u32 fixed point"][st["prefix_format"]]},
            "roofline": alu_roof(sample_flop(cfg.R, cfg.A), n, k_ms, "pndf::sample_kernel", "sample",
                                 touched_bytes_per_sample=Bs,
                                 note="flop = Z-hat (16R) + root range query (3R) + 4 quadrant range queries "
                                      "(3R each) per descent level (P:385-389); touched bytes are not a roof"),
            "cpu_baseline": {"value": cpu_rate, "unit": "samples/s", "cores": oracle.max_threads(),
                             "kind": "oracle", "sample": f"{rs.shape[0]} samples of the timed batch"},
            "gpu_launches": int(st["kernel_launches"] - l0), "clocks": clk,
            "parity_sample": {"checked": int(rs.shape[0]), "pixel_match_where_firm": bool(same[firm].all()),
                              "firm": int(firm.sum()), "pdf_max_rel_err_firm": float(rel[firm].max())},
            "e2e": None}
    print(json.dumps(line), flush=True)
    store.free()
    return 0


SG_METRIC = "SG-prefiltered NDF range queries/sec (Sec. 5.4: rectangle generation + range query)"


def run_sg_op(args, cfg, rank, world, local_rank):
    """--op sg: per step pndf_sg_queries (SG light -> rectangle) + pndf_query_batch, same timing rules."""
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2109_14807_b200 import pndf
    from paper_2109_14807_b200.shard import reduce_times_and_checksum, shard_range
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n_total = args.queries or min(cfg.n_queries, 2 * 10**8)
    i0, i1 = shard_range(n_total, rank, world)
    n = i1 - i0
    bins, f = host_inputs(cfg)
    Z = synth.build_z_exact_cuda(cfg, f.info["atom_map"], local_rank) if f.Z is None else f.Z
    store = pndf.load_factors(pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, cfg.wrap), f.C, f.X, f.Y, Z,
                              device=local_rank)
    del Z
    torch.cuda.empty_cache()
    sg = synth.gen_sg_lights(cfg, i0, i1)
    d_sg = torch.from_numpy(sg.view(np.float32).reshape(-1, 8)).to(dev)
    d_q = torch.empty((n, 4), dtype=torch.int32, device=dev)
    d_out = torch.empty(n, dtype=torch.float32, device=dev)
    opts = {"auto": pndf.BIN_AUTO, "on": pndf.BIN_ON, "off": pndf.BIN_OFF}[args.bin]
    for _ in range(args.warmup):
        pndf.sg_queries(d_sg, d_q, cfg.A)
        store.query_batch(d_q, d_out, opts)
        store.sync()
    store.reset_stats()
    l0 = store.stats()["kernel_launches"]
    clocks = ClockSampler(bus_id_of(dev))
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        pndf.sg_queries(d_sg, d_q, cfg.A)
        store.query_batch(d_q, d_out, opts | pndf.TIMING)
        store.sync()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    st = store.stats()
    ms_rank = e0.elapsed_time(e1) / args.steps
    q_ms = st["query_ms"] / max(1, st["timed_batches"])
    (ms_step,), _ = reduce_times_and_checksum([ms_rank], 0.0, dev)
    if rank != 0:
        store.free()
        return 0
    Bq = bytes_per_query(cfg.R) + 32 + 16  # + SG record read, generated record write
    h_q = d_q.cpu().numpy().view(synth.QREC).reshape(-1)
    idx = np.unique(np.random.default_rng(4).integers(0, n, min(n, 4096)))
    ref_r = oracle.sg_rects(sg[idx], cfg.A)
    rect_ok = float(np.mean(h_q["rect"][idx] == ref_r["rect"]))
    d = oracle.desc_of(cfg)
    rows, _ = oracle.neighbours(d, h_q[idx])
    Zs, zmap = oracle.sparse_z(rows, cfg.P, lambda u: z_rows_for(cfg, f, u))
    t0 = time.perf_counter()
    ref = oracle.query_batch(d, f.C, f.X, f.Y, Zs, h_q[idx], mean=True, zmap=zmap)
    cpu_rate = idx.shape[0] / (time.perf_counter() - t0)
    got = d_out[torch.from_numpy(idx).to(dev)].cpu().numpy().astype(np.float64)
    err = np.abs(got - ref)
    line = {"metric": SG_METRIC, "value": n_total / (ms_step * 1e-3), "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg) + "; SG lights: lambda log-U[10,1000], A U[0.5,2], "
                                                         "half vector Beckmann 0.3, eps 0.3",
                       "queries_total": n_total, "binned": bool(st["last_binned"])},
            "roofline": alu_roof(FLOP_RANK_QUERY * cfg.R, n, q_ms, query_kernel_name(st) + " (after sg_rect_kernel)",
                                 "query", touched_bytes_per_query=Bq, step_ms=ms_rank),
            "cpu_baseline": {"value": cpu_rate, "unit": "queries/s", "cores": oracle.max_threads(),
                             "kind": "oracle", "sample": f"{idx.shape[0]} queries of the timed batch"},
            "gpu_launches": int(st["kernel_launches"] - l0) + args.steps, "clocks": clk,
            "parity_sample": {"checked": int(idx.shape[0]), "rect_identical_frac": rect_ok,
                              "query_pass": bool(((err <= 1e-4 * np.abs(ref)) | (err <= 1e-7)).all())},
            "e2e": None}
    print(json.dumps(line), flush=True)
    store.free()
    return 0


WANG_METRIC = "Wang-tiled NDF range queries/sec (Sec. 5.5: implicit 16-tile map, 100K^2 texels)"
WANG_SAMPLE_METRIC = "Wang-tiled NDF importance samples/sec (Sec. 5.5, P:454: equal-probability covered tile + hierarchical descent)"


def wang_rows_touched(tc, recs) -> np.ndarray:
    """Zc rows the tiled kernels read per record (reading 21/25): for each level of positive weight and each
    neighbour of positive weight, the tiles whose stored rows (within 2 cells of the tile) hold it."""
    S = recs["size"].astype(np.float64)
    ls = np.clip(np.log2(S / tc.s0), 0.0, tc.L - 1)
    l0 = np.minimum(np.floor(ls), tc.L - 2).astype(np.int64)
    t = ls - l0
    rows = np.zeros(recs.shape[0], np.int64)
    for dl in (0, 1):
        l = l0 + dl
        wl = t if dl else 1.0 - t
        s = (tc.s0 << l).astype(np.float64)
        nl = (tc.T // (tc.s0 << l)).astype(np.int64)
        cnt = []
        for c in ("u", "v"):
            f = recs[c].astype(np.float64) / s - 0.5
            i0 = np.floor(f).astype(np.int64)
            a = f - i0
            per = [(i0 + k + 2) // nl - (i0 + k - 2) // nl + 1 for k in (0, 1)]
            cnt.append((per[0], per[1] * (a > 0)))
        tot = (cnt[0][0] + cnt[0][1]) * (cnt[1][0] + cnt[1][1])
        rows += np.where(wl > 0, tot, 0)
    return rows


def run_wang_op(args, cfg, rank, world, local_rank):
    """--op wang: range queries on an implicitly Wang-tiled 102400^2 map (16 tiles of 512^2, A=64, R=32)."""
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2109_14807_b200 import pndf
    from paper_2109_14807_b200.shard import reduce_times_and_checksum, shard_range
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    tc = synth.TileConfig()
    n_total = args.queries or tc.n_queries
    i0, i1 = shard_range(n_total, rank, world)
    n = i1 - i0
    tiles = synth.wang_tiles(tc)
    f = synth.wang_factors(tc, tiles)
    store = pndf.load_tiles(pndf.make_tile_desc(tc.T, tc.s0, tc.L, tc.margin, tc.A, tc.R, tc.seed), f.C, f.X, f.Y,
                            f.Z, device=local_rank)
    if args.lanes:
        store.set_lanes(args.lanes)
    # queries: world positions uniform, sizes log-uniform in [1, T], config-2-like rectangles
    rng = np.random.default_rng(500 + rank)
    A = tc.A
    w = rng.uniform(0.5, 4.0, (n, 2))
    side = np.maximum(1, np.floor(2 * w + 0.5)).astype(np.int64)
    x1 = rng.integers(0, A - side[:, 0] + 1)
    y1 = rng.integers(0, A - side[:, 1] + 1)
    recs = synth.make_records(rng.uniform(0, tc.world, n), rng.uniform(0, tc.world, n),
                              np.exp2(rng.uniform(0, np.log2(tc.T), n)), x1, x1 + side[:, 0] - 1, y1,
                              y1 + side[:, 1] - 1)
    sample = args.op == "wang_sample"
    if sample:  # plain NDF sampling over the whole image (Sec. 5.5)
        recs["rect"] = synth.pack_rect(0, A - 1, 0, A - 1)
        xi_h = np.random.default_rng(600 + rank).random((n, 11), dtype=np.float32)
        d_xi = torch.from_numpy(xi_h).to(dev)
    d_q = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).to(dev)
    d_out = torch.empty((n, 4) if sample else n, dtype=torch.float32, device=dev)

    def step(opts):
        if sample:
            store.sample_tiles(d_q, d_xi, d_out, None, opts)
        else:
            store.query_batch(d_q, d_out, opts)
        store.sync()

    for _ in range(args.warmup):
        step(0)
    store.reset_stats()
    clocks = ClockSampler(bus_id_of(dev))
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step(pndf.TIMING)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    st = store.stats()
    ms_rank = e0.elapsed_time(e1) / args.steps
    (ms_step,), _ = reduce_times_and_checksum([ms_rank], 0.0, dev)
    if rank != 0:
        store.free()
        return 0
    td_o = oracle.TilesDesc(T=tc.T, s0=tc.s0, L=tc.L, margin=tc.margin, A=tc.A, R=tc.R, seed=tc.seed)
    if sample:
        idx = np.unique(np.random.default_rng(5).integers(0, n, min(n, 4000)))
        t0 = time.perf_counter()
        ref = oracle.tiled_sample_batch(td_o, f.C, f.X, f.Y, f.Z, recs[idx], xi_h[idx])
        cpu_rate = idx.shape[0] / (time.perf_counter() - t0)
        o = d_out[torch.from_numpy(idx).to(dev)].cpu().numpy()
        pix = o[:, 3].view(np.uint32)
        firm = (ref["pixel"][:, 0] >= 0) & (ref["margin"] > 1e-4)
        passed = bool(np.array_equal((pix[firm] & 0xffff).astype(np.int64), ref["pixel"][firm, 0]) and
                      np.array_equal((pix[firm] >> 16).astype(np.int64), ref["pixel"][firm, 1]) and
                      np.array_equal(pix == 0xffffffff, ref["pixel"][:, 0] < 0))
        unit, kern = "samples/s", "pndf::tiled_sample_kernel"
    else:
        idx = np.unique(np.random.default_rng(5).integers(0, n, min(n, 20000)))
        t0 = time.perf_counter()
        ref = oracle.tiled_query_batch(td_o, f.C, f.X, f.Y, f.Z, recs[idx])
        cpu_rate = idx.shape[0] / (time.perf_counter() - t0)
        got = d_out[torch.from_numpy(idx).to(dev)].cpu().numpy().astype(np.float64)
        err = np.abs(got - ref)
        passed = bool(((err <= 1e-4 * np.abs(ref)) | (err <= 1e-7)).all())
        unit, kern = "queries/s", "pndf::tiled_query_kernel"
    # algorithmic bytes: record + result, the Zc rows of every overlapped tile, and the angular rows
    # (one range-table row per axis for the narrow query rectangles; for whole-image sampling the 4
    # domain-corner SAT rows plus 2 midpoint rows per descent level)
    rows_mean = float(wang_rows_touched(tc, recs[idx]).mean())
    Rp, levels = st["rank_padded"], int(round(math.log2(tc.A)))
    Bq = (32 + 4 * Rp * (rows_mean + 4 + 2 * levels)) if sample else (20 + 4 * Rp * (rows_mean + 2))
    k_ms = st["query_ms"] / max(1, st["timed_batches"])
    # method flops per record: 2R per positive-weight (tile, neighbour) Zc row into Z-hat, then the rank
    # product 3R (query) or the descent's root + 4 quadrant queries per level (sampling)
    R = tc.R
    fl = 2 * R * rows_mean + (3 * R + levels * 12 * R if sample else 3 * R)
    wang_roof = alu_roof(fl, n, k_ms, kern, "record", touched_bytes_per_record=Bq, zc_rows_per_query_mean=rows_mean,
                         level_sort_ms=st["bin_ms"] / max(1, st["timed_batches"]),
                         note="16 tiles' Zc %.0f MB (> L2); rows per record = the positive-weight Zc rows of all "
                              "overlapped tiles, measured on the parity sample" % (st["zc_bytes"] / 1e6))
    line = {"metric": WANG_SAMPLE_METRIC if sample else WANG_METRIC, "value": n_total / (ms_step * 1e-3),
            "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"16 Wang tiles of {tc.T}^2 flakes (spacing {tc.spacing}, alpha {tc.alpha}), "
                                   f"A={tc.A}, R={tc.R}, margin {tc.margin}, world {tc.world}^2, S log-U[1,{tc.T}]"
                                   + (", whole-image sampling domain" if sample else ""),
                       "queries_total": n_total, "rows": int(st["rows"]),
                       "sat_format": ["fp32 hi/lo", "u32 fixed point"][st["prefix_format"]]},
            "roofline": wang_roof,
            "cpu_baseline": {"value": cpu_rate, "unit": unit, "cores": oracle.max_threads(),
                             "kind": "oracle", "sample": f"{idx.shape[0]} records of the timed batch"},
            "gpu_launches": int(st["kernel_launches"]), "clocks": clk,
            "parity_sample": {"checked": int(idx.shape[0]), "pass": passed},
            "e2e": None}
    print(json.dumps(line), flush=True)
    store.free()
    return 0


BLOCKED_METRIC = "NDF range queries/sec on the blocked/clustered store (Sec. 4.2: t=16 blocks, 8x8-texel regions)"
BLOCKED_SAMPLE_METRIC = ("NDF importance samples/sec on the blocked/clustered store (Sec. 5.2, P:387: block chosen by "
                         "its averaged NDF, then the quad descent)")


def blocked_roofline(cfg, n, k_ms):
    """Algorithmic bytes of the blocked query: record + result, and per bilinear neighbour of both levels one
    block's slab pointer + group set (8 B), its Zc row (4R) and 8 HILO prefix rows (32R).  Counts one
    non-blank block per neighbour: rectangles that cross block borders read more, blank blocks less."""
    Bq = 20 + 8 * (8 + 36 * cfg.R)
    # per neighbour (8): its block's X-bar, Y-bar from hi/lo prefix rows (2 x 3 FADD per rank), the rank
    # product dx*dy*z (3 flop per rank), then the weighted blend
    return alu_roof(8 * 9 * cfg.R + 16, n, k_ms, "pndf::blocked_query_kernel", "query", touched_bytes_per_query=Bq,
                    note=blocked_roofline.__doc__.split("\n")[0].strip())


ALS_METRIC = "CP-ALS sweeps/sec of the GPU factor builder (P:308; footprint NDF tensor P x A x A, rank R)"


def run_als_op(args, cfg, rank, world, local_rank):
    """--op als: footprint histogram tensor of the config's map on the GPU, then HALS CP-ALS
    sweeps (tcgen05 MTTKRP).  A step = one sweep; `e2e` = the whole builder at the paper's settings (tol 1e-4,
    <= 500 sweeps) from host bins to host factors.  Replicas only (one map per GPU)."""
    import torch
    import torch.distributed as dist
    from paper_2109_14807_b200 import pndf
    from paper_2109_14807_b200.shard import reduce_times_and_checksum
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    desc = pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, True)
    d_bins = torch.from_numpy(bins.view(np.int16)).to(dev)
    D = torch.empty((cfg.P, cfg.A, cfg.A), dtype=torch.float32, device=dev)
    Dt = torch.empty_like(D)
    rng = np.random.default_rng(1)
    init = [rng.random((cfg.P, cfg.R)).astype(np.float32), rng.random((cfg.A, cfg.R)).astype(np.float32),
            rng.random((cfg.A, cfg.R)).astype(np.float32)]
    fz, fx, fy = (torch.from_numpy(a).to(dev) for a in init)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pndf.hist_tensor(desc, d_bins, D, Dt)
    torch.cuda.synchronize()
    e0.record()
    pndf.hist_tensor(desc, d_bins, D, Dt)
    e1.record()
    torch.cuda.synchronize()
    hist_ms = e0.elapsed_time(e1)
    pndf.cp_als(desc, D, Dt, fz, fx, fy, max_sweeps=max(3, args.warmup), tol=0.0)
    clocks = ClockSampler(bus_id_of(dev))
    clocks.start()
    # the sampler's start leaves the GPU idle for a moment: re-warm so the short timed region runs at clock
    pndf.cp_als(desc, D, Dt, fz, fx, fy, max_sweeps=max(3, args.warmup), tol=0.0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    err = pndf.cp_als(desc, D, Dt, fz, fx, fy, max_sweeps=args.steps, tol=0.0)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_rank = e0.elapsed_time(e1) / args.steps
    (ms_step,), _ = reduce_times_and_checksum([ms_rank], float(err[-1]), dev)
    # end to end at the paper's settings: host bins -> D -> ALS (tol 1e-4, <= 500 sweeps) -> host factors
    t0 = time.perf_counter()
    d_b2 = torch.from_numpy(bins.view(np.int16)).to(dev)
    pndf.hist_tensor(desc, d_b2, D, Dt)
    gz, gx, gy = (torch.from_numpy(a).to(dev) for a in init)
    gc = torch.empty(cfg.R, dtype=torch.float32, device=dev)
    hist_e2e = pndf.cp_als(desc, D, Dt, gz, gx, gy, gc, max_sweeps=500, tol=1e-4, normalise=True)
    out = [t.cpu() for t in (gc, gx, gy, gz)]
    e2e_s = time.perf_counter() - t0
    if rank != 0:
        return 0
    peaks, src = measured_peaks()
    dbytes = cfg.P * cfg.A * cfg.A * 4
    mttkrp_flop = 3 * 2 * cfg.P * cfg.A * cfg.A * cfg.R  # three MTTKRPs of the full tensor per sweep
    tf32_peak = peaks.get("bf16_tflops", 2250.0) * (1.1 / 2.25)  # measured bf16 x nominal tf32/bf16 (B200_PROFILING)
    achieved = mttkrp_flop / (ms_step * 1e-3) / 1e12
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        from oracle import als as oals
        small = cfg.scaled(N=max(64, cfg.N // 4))
        sb = synth.bin_map(small, synth.make_map(small))
        Dc = oals.tf32_round(oals.hist_tensor(small.N, small.s0, small.L, small.A, sb)).astype(np.float64)
        r2 = np.random.default_rng(1)
        zi, xi, yi = r2.random((small.P, small.R)), r2.random((small.A, small.R)), r2.random((small.A, small.R))
        t0 = time.perf_counter()
        oals.cp_als(Dc, zi, xi, yi, tol=0.0, max_sweeps=2)
        sweep_s = (time.perf_counter() - t0) / 2 * (cfg.P / small.P)
        cpu = {"value": 1.0 / sweep_s, "unit": "sweeps/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"2 oracle sweeps on the {small.N}^2 map (P={small.P}), time scaled by P ratio "
                         f"{cfg.P / small.P:.0f}"}
    line = {"metric": ALS_METRIC, "value": 1e3 / ms_step, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "tf32 (D exact) + split-tf32 factors, fp32 accumulate; fp64 HALS",
            "data": "synthetic",
            "config": {"workload": f"config{cfg.idx} map {cfg.N}^2, D = {cfg.P} x {cfg.A} x {cfg.A} fp32 "
                                   f"({dbytes / 1e9:.2f} GB, + transposed copy), R = {cfg.R}",
                       "hist_ms": hist_ms, "fit_error_after_timed_sweeps": float(err[-1]),
                       "step_includes": "one pndf_cp_als call of K sweeps: per-call setup (~2.5 ms: allocations, "
                                        "||D||^2 pass) amortised over the K sweeps; steady sweep = kernel sum",
                       "inputs": "D (2 x tensor) resident in HBM, larger than L2: no flush needed"},
            "roofline": {"bound": "hbm", "achieved": 3 * dbytes / (ms_step * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": 3 * dbytes / (ms_step * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "traffic": None,
                         "kernel": "pndf::als::mttkrp_gemm_kernel (3 per sweep) + HALS/Gram kernels",
                         "bytes_per_sweep": 3 * dbytes, "peak_source": src,
                         "tensor": {"flop_per_sweep": mttkrp_flop, "tflops": achieved, "peak_tflops": tf32_peak,
                                    "frac": achieved / tf32_peak,
                                    "peak_source": "MEASURED_PEAKS bf16_tflops x 1.1/2.25 (tf32/bf16 nominal)"},
                         "note": "achieved = the 3 reads of D a sweep must make (modes Z, X on D, mode Y on Dt) over "
                                 "the whole sweep time (HALS, Gram and host-sync steps included): at R = 32 the "
                                 "MTTKRP is bound by streaming D, not by the tensor cores (tensor.frac)"},
            "cpu_baseline": cpu,
            # one pndf_cp_als call of K sweeps = 12 setup/teardown launches + 21 per sweep (3 tcgen05 GEMMs,
            # 3 HALS + 3 Gram sums, 2 operand splits + 1 Khatri-Rao, 2 partial reductions, error, balance,
            # 3 column scalings, 2 Gram scalings): profiles/r01_launches_als.txt
            "gpu_launches": 12 + 21 * args.steps, "clocks": clk,
            "e2e": {"value": len(hist_e2e) / e2e_s, "unit": "sweeps/s", "h2d_bytes_per_step": int(bins.nbytes),
                    "d2h_bytes_per_step": int(sum(t.numel() * 4 for t in out)),
                    "builder_seconds": e2e_s, "sweeps": int(len(hist_e2e)), "fit_error": float(hist_e2e[-1]),
                    "note": "whole builder at P:308 settings, host bins in, host factors out; the paper quotes "
                            "10-60 minutes per 2K x 2K map on its CPU (P:311)"}}
    print(json.dumps(line), flush=True)
    return 0


ALS_MAP_METRIC = ("CP-ALS sweeps/sec of the map-domain GPU factor builder (P:308; exact footprint tensor P x A x A "
                  "never formed)")


def map_sweep_flop(cfg) -> int:
    """fp64 FMA work of one map-domain sweep x 2: per level l (stride s, window wf, grid n) the
    Z-mode pass along u (N n wf taps) and along v (n^2 wf), the adjoint along v (N n wf/s) and along u
    (N^2 wf/s), then the X and Y modes (N^2 each), every tap over R ranks."""
    N, R = cfg.N, cfg.R
    taps = 2 * N * N
    for l in range(cfg.L):
        s = cfg.s0 << l
        n = N // s
        sigma = 1.5 * s / math.sqrt(12.0)
        c = 0.5 * (1.0 - s)
        wf = min(math.floor(4.0 * sigma - c) - math.ceil(-4.0 * sigma - c) + 1, N)
        per = math.ceil(wf / s)
        taps += N * n * wf + n * n * wf + N * n * per + N * N * per
    return 2 * taps * R


def map_sweep_bytes(cfg) -> int:
    """Compulsory HBM bytes of one map-domain sweep: each pass buffer written once and read once (Z-mode pass
    buffer and adjoint pass buffer, 2 N^2 R fp64 each over the level groups; U, N^2 R fp64, written by the two
    level groups and read by the X and Y modes), the map bins per pass, and the Z-side arrays (Z read by the
    adjoint, M_Z written then read, Z read and written by HALS: 5 P R fp64)."""
    N, R, P = cfg.N, cfg.R, cfg.P
    hb = sum(N * (N // (cfg.s0 << l)) for l in range(cfg.L)) * R * 8
    u = N * N * R * 8
    return 2 * 2 * hb + u * (2 + 1 + 2) + 5 * P * R * 8 + 6 * N * N * 2


def run_als_map_op(args, cfg, rank, world, local_rank):
    """--op als_map (SURVEY §8(f) row 3 at config 3 scale): HALS CP-ALS of the config's footprint tensor with
    map-domain MTTKRPs (pndf_cp_als_map).  A step = one sweep; `e2e` = the whole builder at the paper's settings
    (tol 1e-4, <= 500 sweeps) from host bins to host factors.  Replicas only (one map per GPU)."""
    import torch
    import torch.distributed as dist
    from paper_2109_14807_b200 import pndf
    from paper_2109_14807_b200.shard import reduce_times_and_checksum
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    desc = pndf.make_desc(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.R, True)
    d_bins = torch.from_numpy(bins.view(np.int16)).to(dev)
    rng = np.random.default_rng(1)
    init = [rng.random((cfg.P, cfg.R)).astype(np.float32), rng.random((cfg.A, cfg.R)).astype(np.float32),
            rng.random((cfg.A, cfg.R)).astype(np.float32)]
    fz, fx, fy = (torch.from_numpy(a).to(dev) for a in init)
    pndf.cp_als_map(desc, d_bins, fz, fx, fy, max_sweeps=max(3, args.warmup), tol=0.0)
    clocks = ClockSampler(bus_id_of(dev))
    clocks.start()
    pndf.cp_als_map(desc, d_bins, fz, fx, fy, max_sweeps=2, tol=0.0)  # re-warm after the sampler's start
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    err = pndf.cp_als_map(desc, d_bins, fz, fx, fy, max_sweeps=args.steps, tol=0.0)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_rank = e0.elapsed_time(e1) / args.steps
    (ms_step,), _ = reduce_times_and_checksum([ms_rank], float(err[-1]), dev)
    e2e = None
    if not args.no_e2e:
        t0 = time.perf_counter()
        d_b2 = torch.from_numpy(bins.view(np.int16)).to(dev)
        gz, gx, gy = (torch.from_numpy(a).to(dev) for a in init)
        gc = torch.empty(cfg.R, dtype=torch.float32, device=dev)
        hist = pndf.cp_als_map(desc, d_b2, gz, gx, gy, gc, max_sweeps=500, tol=1e-4, normalise=True)
        out = [t.cpu() for t in (gc, gx, gy, gz)]
        e2e_s = time.perf_counter() - t0
        e2e = {"value": len(hist) / e2e_s, "unit": "sweeps/s", "h2d_bytes_per_step": int(bins.nbytes),
               "d2h_bytes_per_step": int(sum(t.numel() * 4 for t in out)), "builder_seconds": e2e_s,
               "sweeps": int(len(hist)), "fit_error": float(hist[-1]),
               "note": "whole builder at P:308 settings, host bins in, host factors out; the paper quotes "
                       "10-60 minutes per 2K x 2K map on its CPU (P:311)"}
    if rank != 0:
        return 0
    peaks, src = measured_peaks()
    import torch as _t
    sms = _t.cuda.get_device_properties(dev).multi_processor_count
    fp64_peak = sms * 64 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    fl = map_sweep_flop(cfg)
    mb = map_sweep_bytes(cfg)
    achieved = fl / (ms_step * 1e-3) / 1e12
    dense = 3 * 2 * cfg.P * cfg.A * cfg.A * cfg.R
    line = {"metric": ALS_MAP_METRIC, "value": 1e3 / ms_step, "unit": "sweeps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 (MTTKRP passes, HALS)", "data": "synthetic",
            "config": {"workload": f"config{cfg.idx} map {cfg.N}^2, P = {cfg.P} footprints, A = {cfg.A}, R = {cfg.R}; "
                                   f"the dense tensor would be {cfg.P * cfg.A * cfg.A * 4 / 1e9:.0f} GB",
                       "fit_error_after_timed_sweeps": float(err[-1]),
                       "inputs": "map bins + factors resident in HBM; pass buffers (N^2 R fp64) larger than L2"},
            "roofline": {"bound": "hbm", "achieved": mb / (ms_step * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": mb / (ms_step * 1e-3) / 1e9 / peaks["hbm_gbs"], "traffic": None,
                         "kernel": "pndf::als::{mz_h,mz_v,u_g,u_h,mxy}_kernel + HALS/Gram kernels",
                         "bytes_per_sweep": mb, "hbm_floor_ms": mb / (peaks["hbm_gbs"] * 1e9) * 1e3,
                         "peak_source": f"{src} MEASURED_PEAKS.json hbm_gbs",
                         "fp64": {"flop_per_sweep": fl, "tflops": achieved, "peak_tflops": fp64_peak,
                                  "frac": achieved / fp64_peak,
                                  "peak_source": "derived: SMs x 64 FP64 lanes x 2 flop x sm_max_mhz"},
                         "dense_tensor_flop_per_sweep": dense,
                         "note": "achieved = the compulsory pass-buffer traffic of a sweep (map_sweep_bytes) over "
                                 "the whole sweep time (HALS, Gram, error and host sync included); the passes are "
                                 "latency-bound gathers, far from both floors (DESIGN.md §5)"},
            # one pndf_cp_als_map call of K sweeps: 10 setup launches (factor loads, ||D||^2, Gram) + 25 per sweep
            # (4 Z-mode passes, 4 adjoint passes, 2 x 2 X/Y-mode, 3 x 2 HALS + Gram sums, error, balance, 5 scalings)
            "cpu_baseline": None, "gpu_launches": 10 + 25 * args.steps, "clocks": clk, "e2e": e2e}
    print(json.dumps(line), flush=True)
    return 0


def run_blocked_op(args, cfg, rank, world, local_rank):
    """--op blocked: the config's queries on the paper-faithful blocked / clustered store (exact-rank groups);
    --op blocked_sample: importance samples over the whole image on it (block choice + descent)."""
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2109_14807_b200 import pndf
    from paper_2109_14807_b200.shard import reduce_times_and_checksum, shard_range
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n_total = args.queries or cfg.n_queries
    i0, i1 = shard_range(n_total, rank, world)
    n = i1 - i0
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    bs, _ = synth.build_blocked(cfg, nxy, bins, t=16, region=8)
    store = pndf.load_blocked(cfg.N, cfg.s0, cfg.L, cfg.A, cfg.wrap, bs, device=local_rank)
    if args.lanes:
        store.set_lanes(args.lanes)
    sample = args.op == "blocked_sample"
    recs = synth.gen_queries(cfg, bins, i0, i1)
    if sample:
        recs["rect"] = synth.pack_rect(0, cfg.A - 1, 0, cfg.A - 1)
        xi_h = np.random.default_rng(700 + rank).random((n, 11), dtype=np.float32)
        d_xi = torch.from_numpy(xi_h).to(dev)
    d_q = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).to(dev)
    d_out = torch.empty((n, 4) if sample else n, dtype=torch.float32, device=dev)

    def step(opts):
        if sample:
            store.sample_blocked(d_q, d_xi, d_out, None, opts)
        else:
            store.query_batch(d_q, d_out, opts)
        store.sync()

    for _ in range(args.warmup):
        step(0)
    store.reset_stats()
    clocks = ClockSampler(bus_id_of(dev))
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step(pndf.TIMING)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    st = store.stats()
    ms_rank = e0.elapsed_time(e1) / args.steps
    (ms_step,), _ = reduce_times_and_checksum([ms_rank], 0.0, dev)
    if rank != 0:
        store.free()
        return 0
    nb = cfg.A // 16
    k_ms = st["query_ms"] / max(1, st["timed_batches"])
    if sample:
        idx = np.unique(np.random.default_rng(6).integers(0, n, min(n, 4000)))
        t0 = time.perf_counter()
        ref = oracle.blocked_sample_batch(cfg, bs, recs[idx], xi_h[idx])
        cpu_rate = idx.shape[0] / (time.perf_counter() - t0)
        o = d_out[torch.from_numpy(idx).to(dev)].cpu().numpy()
        pix = o[:, 3].view(np.uint32)
        firm = (ref["pixel"][:, 0] >= 0) & (ref["margin"] > 1e-4)
        passed = bool(np.array_equal((pix[firm] & 0xffff).astype(np.int64), ref["pixel"][firm, 0]) and
                      np.array_equal((pix[firm] >> 16).astype(np.int64), ref["pixel"][firm, 1]) and
                      np.allclose(o[firm, 2], ref["prob"][firm] * cfg.A * cfg.A / 4.0, rtol=1e-4))
        levels = int(round(math.log2(16)))
        # per sample: nb^2 block weights + 4 quads per descent level, each 8 neighbours x 9 flop per rank
        roof = alu_roof((nb * nb + 4 * levels) * 8 * 9 * cfg.R, n, k_ms, "pndf::blocked_sample_kernel", "sample")
        parity = {"checked": int(idx.shape[0]), "firm": int(firm.sum()), "pass": passed}
    else:
        idx = np.unique(np.random.default_rng(6).integers(0, n, min(n, 20000)))
        t0 = time.perf_counter()
        ref = oracle.blocked_query_batch(cfg, bs, recs[idx])
        cpu_rate = idx.shape[0] / (time.perf_counter() - t0)
        got = d_out[torch.from_numpy(idx).to(dev)].cpu().numpy().astype(np.float64)
        err = np.abs(got - ref)
        roof = blocked_roofline(cfg, n, k_ms)
        parity = {"checked": int(idx.shape[0]), "pass": bool(((err <= 1e-4 * np.abs(ref)) | (err <= 1e-7)).all())}
    raw = cfg.P * cfg.A * cfg.A * 4
    comp = st["zc_bytes"] + st["prefix_bytes"] + cfg.P * nb * nb * 4 + bs.group_set.size * 4
    unit = "samples/s" if sample else "queries/s"
    line = {"metric": BLOCKED_SAMPLE_METRIC if sample else BLOCKED_METRIC, "value": n_total / (ms_step * 1e-3),
            "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg) + "; blocked store t=16, 8-texel regions" +
                                   ("; whole-image sampling domain" if sample else ""),
                       "queries_total": n_total, "slabs": bs.info["n_slabs"], "groups": bs.info["n_groups"],
                       "blank_block_fraction": bs.info["blank_fraction"],
                       "storage_vs_raw_pyramid": comp / raw},
            "roofline": roof,
            "cpu_baseline": {"value": cpu_rate, "unit": unit, "cores": oracle.max_threads(),
                             "kind": "oracle", "sample": f"{idx.shape[0]} records of the timed batch"},
            "gpu_launches": args.steps, "clocks": clk,
            "parity_sample": parity,
            "e2e": None}
    print(json.dumps(line), flush=True)
    store.free()
    return 0


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: re-run this command under torch.distributed.run, one
    process per GPU on this node (rendezvous on 127.0.0.1), and return its exit code."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one process per GPU\n")
        return 2
    cfg = synth.CONFIGS[args.config]
    if args.s0:
        cfg = cfg.scaled(s0=args.s0)
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")  # timing / checksum reductions only, after each timed region
    try:
        if args.op == "sample":
            return run_sample_op(args, cfg, rank, world, local_rank)
        if args.op == "sg":
            return run_sg_op(args, cfg, rank, world, local_rank)
        if args.op in ("wang", "wang_sample"):
            return run_wang_op(args, cfg, rank, world, local_rank)
        if args.op in ("blocked", "blocked_sample"):
            return run_blocked_op(args, cfg, rank, world, local_rank)
        if args.op == "sweep":
            return run_sweep_op(args, synth.CONFIGS[3], rank, world, local_rank)
        if args.op == "als_map":
            return run_als_map_op(args, cfg if args.config != 5 else synth.CONFIGS[3], rank, world, local_rank)
        if args.op == "als":
            return run_als_op(args, cfg if cfg.idx in (1, 2) else synth.CONFIGS[2], rank, world, local_rank)
        return run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
