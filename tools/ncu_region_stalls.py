"""dev: stall-reason breakdown per SASS address range of an ncu source-page CSV.
    ncu -i rep --page source --csv --print-source sass > x.csv
    python tools/ncu_region_stalls.py x.csv lo-hi [lo-hi ...]   (instruction indices)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ix = {h: hdr.index(h) for h in reasons}
iex = hdr.index("Instructions Executed")
tot = sum(int(r[hdr.index("Warp Stall Sampling (All Samples)")]) for r in data)
for spec in sys.argv[2:]:
    lo, hi = map(int, spec.split("-"))
    sub = data[lo:hi + 1]
    agg = {h: sum(int(r[ix[h]]) for r in sub) for h in reasons}
    s = sum(agg.values())
    top = sorted(agg.items(), key=lambda kv: -kv[1])[:7]
    print(f"{spec}: {100 * s / tot:5.1f}% of samples; " + ", ".join(f"{k[6:]} {100 * v / max(s, 1):.0f}%" for k, v in top))
