"""Stall-reason breakdown per SASS region (instructions grouped by execution count) (dev tool).
    python tools/ncu_regions.py rep.ncu-rep [min_share]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iex, isrc, isamp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
reg = collections.defaultdict(lambda: collections.Counter())
cnt = collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iex or not r[iex].isdigit(): continue
    ex = int(r[iex]);
    if ex == 0: continue
    cnt[ex] += 1
    for c in reasons:
        v = r[h.index(c)]
        if v.isdigit(): reg[ex][c] += int(v); tot += int(v)
for ex, c in sorted(reg.items(), key=lambda kv: -sum(kv[1].values()))[:8]:
    s = sum(c.values())
    top = ", ".join(f"{k[6:]} {v/s*100:.0f}%" for k, v in c.most_common(6))
    print(f"exec {ex:>9d} x{cnt[ex]:4d} instrs  samples {s/tot*100:5.1f}%  {top}")
