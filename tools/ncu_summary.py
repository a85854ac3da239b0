"""Summarise an ncu --set full report: key throughput/traffic metrics + opcode mix with stall share."""
import csv, io, subprocess, sys
from collections import Counter

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_per_inst_issued.ratio", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "smsp__inst_executed.sum", "launch__grid_size", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, nq=None):
    hdr, units, vals = raw(rep)
    v = vals[0]
    res = {}
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            res[w] = (v[i], units[i])
            print(f"{w:60s} {v[i]:>22s} {units[i]}")
    stalls = sorted(((float(v[i].replace(",", "") or 0), h) for i, h in enumerate(hdr)
                     if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                     and v[i].replace(",", "").replace(".", "").isdigit()), reverse=True)
    for val, h in stalls[:8]:
        print(f"  stall {h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:24s} {val:8.3f} per issue")
    if nq:
        ins = float(res["smsp__inst_executed.sum"][0].replace(",", ""))
        print(f"warp-instructions per query: {ins / nq:.1f}")
        rd = float(res["dram__bytes_read.sum"][0].replace(",", ""))
        print(f"dram read per query: {rd * {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1}[res['dram__bytes_read.sum'][1]] / nq:.1f} B")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot = sum(int(r[iW]) for r in data) or 1
    c, s = Counter(), Counter()
    for r in data:
        t = r[iS].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        c[op] += int(r[iE])
        s[op] += int(r[iW])
    n = nq or 1
    for op, k in c.most_common(18):
        print(f"  {op:10s} {k / n:8.1f}/q  stall-share {s[op] / tot * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
