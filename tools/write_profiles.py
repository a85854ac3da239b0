"""Turn gpurun_out/ ncu captures into the committed evidence under profiles/ (per round).

usage: python tools/write_profiles.py ROUND QUERIES_IN_CAPTURE
  reads  gpurun_out/prof_query_full.ncu-rep, gpurun_out/prof_scatter_full.ncu-rep,
         gpurun_out/launches_default.csv, gpurun_out/bench_default.log
  writes profiles/rNN_query_kernel_ncu.txt, profiles/rNN_radix_scatter_ncu.txt,
         profiles/rNN_launches_default.txt (+ .csv), profiles/rNN_bench_default.json,
         profiles/ncu_traffic.json (DRAM bytes per query of the query kernel, read by bench.py)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
GP = os.path.join(ROOT, "gpurun_out")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
           "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__inst_executed.sum",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep, nq, title, idx=0, unit="query"):
    rows = ncu_csv(rep, "raw")
    hdr, units, v = rows[0], rows[1], rows[2 + idx]
    lines = [f"# {title}", f"# source: {os.path.basename(rep)} (ncu --set full --clock-control none)",
             f"# {unit}s in the captured launch: {nq:.0f}", ""]
    vals = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            vals[m] = (v[i], units[i])
            lines.append(f"{m:60s} {v[i]:>24s} {units[i]}")
    stalls = []
    for i, hname in enumerate(hdr):
        if hname.startswith("smsp__average_warps_issue_stalled_") and hname.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v[i].replace(",", "")), hname[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    if stalls:
        lines.append("")
        lines.append("warp stall cycles per issued instruction (top reasons):")
        for val, name in sorted(stalls, reverse=True)[:8]:
            lines.append(f"  {name:28s} {val:8.3f}")
    lines.append("")

    def num(m):
        x, u = vals[m]
        return float(x.replace(",", "")) * SCALE.get(u, 1)

    dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    lines.append(f"dram bytes per {unit} (read+write): {dram / nq:.2f}")
    lines.append(f"L2->L1 read bytes per {unit}: {float(vals['lts__t_sectors_srcunit_tex_op_read.sum'][0].replace(',', '')) * 32 / nq:.2f}")
    lines.append(f"warp instructions per {unit}: {float(vals['smsp__inst_executed.sum'][0].replace(',', '')) / nq:.3f}")
    src = ncu_csv(rep, "source")
    if len(src) > 2:
        h = src[1]
        data = src[2:]
        if idx:  # the source page lists the first kernel only
            data = []
        iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        def _i(x):
            try:
                return int(x)
            except ValueError:
                return 0
        data = [r for r in data if len(r) > max(iS, iW, iE)]
        for r in data:
            r[iW], r[iE] = _i(r[iW]), _i(r[iE])
        tot = sum(r[iW] for r in data) or 1
        c, s = defaultdict(int), defaultdict(int)
        for r in data:
            t = r[iS].split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            c[op] += int(r[iE])
            s[op] += int(r[iW])
        lines += ["", f"opcode mix (per {unit}) and share of warp-stall samples:"]
        for op, k in sorted(c.items(), key=lambda x: -x[1])[:16]:
            lines.append(f"  {op:10s} {k / nq:8.2f}/q   stall {s[op] / tot * 100:5.1f}%")
    per = {"dram": dram / nq,
           "l2_read": float(vals['lts__t_sectors_srcunit_tex_op_read.sum'][0].replace(',', '')) * 32 / nq,
           "inst": float(vals['smsp__inst_executed.sum'][0].replace(',', '')) / nq}
    return "\n".join(lines) + "\n", per


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    iN, iV = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) <= iV:
            continue
        try:
            val = float(r[iV].replace(",", ""))
        except ValueError:
            continue
        name = r[iN].split("(")[0]
        tot[name] += val
        cnt[name] += 1
    T = sum(tot.values()) or 1
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none, `python bench.py` (default run)",
             "# per-launch times are cold-cache and serialised: compare SHARES, not absolutes",
             f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:70]:70s} {cnt[k]:8d} {v / 1e6:10.2f} {v / T * 100:6.1f}%")
    return "\n".join(lines) + "\n"


def main():
    rnd = sys.argv[1]
    nq = float(sys.argv[2])
    os.makedirs(OUT, exist_ok=True)
    traffic = {}
    q = os.path.join(GP, "prof_query_full.ncu-rep")
    if os.path.exists(q):
        txt, dpq = summarize(q, nq, "pndf::query_g5_kernel (lean query kernel, gather4-staged range-table rows), "
                                    "config 5, binned, U32 SATs")
        open(os.path.join(OUT, f"{rnd}_query_kernel_ncu.txt"), "w").write(txt)
        traffic["config5"] = {"dram_bytes_per_query": dpq["dram"], "l2_read_bytes_per_query": dpq["l2_read"],
                              "warp_instructions_per_query": dpq["inst"],
                              "source": f"profiles/{rnd}_query_kernel_ncu.txt (ncu --set full, {nq:.0e} queries, "
                                        "same launch configuration as bench.py)"}
    sc = os.path.join(GP, "prof_scatter_full.ncu-rep")
    if os.path.exists(sc):
        txt, _ = summarize(sc, nq, "pndf::rs_scatter_kernel<9> (one radix pass), config 5")
        open(os.path.join(OUT, f"{rnd}_radix_scatter_ncu.txt"), "w").write(txt)
    sp = os.path.join(GP, "prof_sample.ncu-rep")
    if os.path.exists(sp):
        txt, _ = summarize(sp, 1e8, "pndf::sample_kernel, config 5, 1e8 samples (bench --op sample)")
        open(os.path.join(OUT, f"{rnd}_sample_kernel_ncu.txt"), "w").write(txt)
    for rep_name, n_units, unit, title in (
            ("prof_blocked", 1e6, "query", "pndf::blocked_query_kernel, config 2 blocked store (t=16, 8-texel regions)"),
            ("prof_tiled", 1e7, "query", "pndf::tiled_query_kernel, 16 Wang tiles of 512^2, world 102400^2"),
            ("prof_sg", 2e8, "light", "pndf::sg_rect_kernel, 2e8 SG lights (config 5)")):
        rp = os.path.join(GP, rep_name + ".ncu-rep")
        if os.path.exists(rp):
            txt, _ = summarize(rp, n_units, title, 0, unit)
            open(os.path.join(OUT, f"{rnd}_{rep_name[5:]}_kernel_ncu.txt"), "w").write(txt)
    la = os.path.join(GP, "launches_default.csv")
    if os.path.exists(la):
        open(os.path.join(OUT, f"{rnd}_launches_default.txt"), "w").write(launches(la))
    for name in ("bench_default", "bench_c1", "bench_c2", "bench_c3", "bench_c4", "bench_sample", "bench_sg",
                 "bench_wang", "bench_wang_sample", "bench_blocked", "bench_blocked_sample", "bench_als",
                 "bench_als_map", "bench_sweep", "bench_c3_s04"):
        b = os.path.join(GP, name + ".log")
        if os.path.exists(b):
            lines = [l for l in open(b).read().splitlines() if l.startswith("{")]
            if lines:
                json.dump(json.loads(lines[-1]), open(os.path.join(OUT, f"{rnd}_{name}.json"), "w"), indent=1)
    al = os.path.join(GP, "prof_als.ncu-rep")
    if os.path.exists(al):
        import synth
        cfg = synth.CONFIGS[2]
        n_el = cfg.P * cfg.A * cfg.A
        txt0, _ = summarize(al, n_el, "pndf::als::mttkrp_gemm_kernel<32, 0> (mode Z: [P x A^2] . [A^2 x 32], "
                                      "tcgen05 kind::tf32), config 2", 0, "D element")
        txt1, _ = summarize(al, n_el, "pndf::als::mttkrp_gemm_kernel<32, 1> (mode X: [(P A) x A] . [A x 32], "
                                      "z-reducing epilogue), config 2", 1, "D element")
        open(os.path.join(OUT, f"{rnd}_als_gemm_ncu.txt"), "w").write(txt0 + "\n" + txt1)
    la3 = os.path.join(GP, "launches_als_map.csv")
    if os.path.exists(la3):
        open(os.path.join(OUT, f"{rnd}_launches_als_map.txt"), "w").write(launches(la3).replace(
            "`python bench.py` (default run)", "`python bench.py --op als_map --config 3 --steps 2 --warmup 3`"))
    la2 = os.path.join(GP, "launches_als.csv")
    if os.path.exists(la2):
        open(os.path.join(OUT, f"{rnd}_launches_als.txt"), "w").write(launches(la2).replace(
            "`python bench.py` (default run)", "`python bench.py --op als --config 2 --steps 2 --warmup 3`"))
    if traffic:
        json.dump(traffic, open(os.path.join(OUT, "ncu_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
