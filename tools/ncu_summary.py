"""Summarise an ncu report (dev tool): key SOL metrics, stall reasons, per-region instruction mix.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import collections, csv, io, json, re, subprocess, sys

def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

def main():
    rep = sys.argv[1]
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    raw = dict(zip(hdr, vals))
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "launch__registers_per_thread", "launch__block_size", "launch__grid_size", "smsp__inst_executed.sum"]
    summ = {}
    for k in keys:
        if k in raw:
            summ[k] = raw[k]
            print(f"{k:70s} {raw[k]}")
    print("-- stalls per issued instruction")
    for k, v in raw.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active.ratio", k)
        if m and float(v or 0) > 0.05:
            print(f"   {m.group(1):25s} {float(v):.2f}")
            summ["stall_" + m.group(1)] = float(v)
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    h = src[1]
    ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    groups = collections.defaultdict(lambda: [0, 0, 0, collections.Counter()])
    for r in src[2:]:
        try:
            n, s = int(r[ia]), int(r[iss])
        except (ValueError, IndexError):
            continue
        g = groups[n]
        g[0] += 1; g[1] += n; g[2] += s
        op = r[isrc].split()
        op = (op[1] if op and op[0].startswith("@") else (op[0] if op else "?")).split(".")[0]
        g[3][op] += 1
    tot = sum(g[1] for g in groups.values()) or 1
    totst = sum(g[2] for g in groups.values()) or 1
    print("-- regions (grouped by execution count)")
    for n, g in sorted(groups.items(), key=lambda x: -x[1][1])[:10]:
        print(f"  exec {n:9d} instrs {g[0]:5d} share {100*g[1]/tot:5.1f}% stall {100*g[2]/totst:5.1f}% {g[3].most_common(6)}")
    if len(sys.argv) > 3 and sys.argv[2] == "--json":
        with open(sys.argv[3], "w") as f:
            json.dump(summ, f, indent=1)

main()
