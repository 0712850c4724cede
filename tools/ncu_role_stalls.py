"""Stall reasons per execution-count region of an ncu source page (dev tool).
    python tools/ncu_role_stalls.py rep.ncu-rep [min_share]
Regions = contiguous runs of SASS with the same 'Instructions Executed' count
(loop bodies of one role); prints each big region's stall-reason mix."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; mins = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iex, isamp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
reg = collections.defaultdict(lambda: [0, 0, collections.Counter(), collections.Counter()])
for r in rows[2:]:
    try: n = int(r[iex]); s = int(r[isamp])
    except: continue
    g = reg[n]; g[0] += 1; g[1] += s
    for c, i in zip(reasons, ri):
        try: g[2][c[6:]] += int(r[i])
        except: pass
    g[3][r[1].split()[0] if not r[1].startswith('@') else r[1].split()[1]] += 1
tot = sum(g[1] for g in reg.values())
for n, g in sorted(reg.items(), key=lambda kv: -kv[1][1]):
    if g[1] < mins * tot: continue
    t = sum(g[2].values()) or 1
    print(f"exec {n:>10} instrs {g[0]:5d} samples {100*g[1]/tot:5.1f}%  ops {g[3].most_common(5)}")
    print("     " + "  ".join(f"{k} {100*v/t:.0f}%" for k, v in g[2].most_common(8)))
