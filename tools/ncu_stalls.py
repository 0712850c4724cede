"""Top SASS instructions by a given stall reason (dev tool).
    python tools/ncu_stalls.py rep.ncu-rep [reason ...]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
reasons = sys.argv[2:] or ["stall_long_sb", "stall_barrier", "stall_wait", "stall_math"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
isrc, iex = h.index("Source"), h.index("Instructions Executed")
for reason in reasons:
    ir = h.index(reason)
    tot = sum(int(r[ir]) for r in rows[2:] if len(r) > ir and r[ir].isdigit())
    print(f"== {reason}: total {tot}")
    top = sorted((r for r in rows[2:] if len(r) > ir and r[ir].isdigit()), key=lambda r: -int(r[ir]))[:8]
    for r in top:
        print(f"   {int(r[ir]):6d}  exec {r[iex]:>8s}  {r[0][-5:]}  {r[isrc].strip()[:80]}")
