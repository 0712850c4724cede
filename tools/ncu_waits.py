"""Warp-stall samples at each mbarrier wait site of the fused kernel (dev tool).
    python tools/ncu_waits.py rep.ncu-rep R Q"""
import csv, io, re, subprocess, sys
rep, R, Q = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iex, isamp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
rows = [r for r in rows[2:] if len(r) > isamp]
GW = 32 + 2 * R; FSW = (GW + 6) // 4 * 4; NFS = 3
base = 4 * NFS * Q * FSW
RB = 1 + (2 * R + Q - 1) // Q; RBP = RB + 1
names = [("fs_full", NFS), ("fs_empty", NFS), ("gen_full", 2), ("gen_empty", 2), ("col_full", 2), ("col_empty", 2),
         ("ring_full", 9 * RBP), ("ring_empty", 9 * RBP)]
def name(off):
    o = (off - base) // 8
    for n, c in names:
        if o < c: return f"{n}[{o}]"
        o -= c
    return hex(off)
tot = sum(int(r[isamp]) for r in rows if r[isamp].isdigit())
addr_idx = {int(r[0], 16): i for i, r in enumerate(rows)}
sites = {}
def attribute(key, s):
    sites[key] = sites.get(key, 0) + s
for i, r in enumerate(rows):
    smp = int(r[isamp]) if r[isamp].isdigit() else 0
    m = re.search(r"SYNCS\.PHASECHK\.TRANS64(?:\.TRYWAIT)? P\d, \[R\d+\+URZ\+(0x[0-9a-f]+)\]", r[1])
    if m:  # samples on the wait instructions themselves (out-of-line retry loop)
        attribute(name(int(m.group(1), 16)), smp)
        continue
    b = re.search(r"@!?P\d\s+BRA\s+(0x[0-9a-f]+)", r[1])
    if b and smp:
        j = addr_idx.get(int(b.group(1), 16))
        if j is None: continue
        for x in rows[j:j + 4]:
            m = re.search(r"SYNCS\.PHASECHK\.TRANS64(?:\.TRYWAIT)? P\d, \[R\d+\+URZ\+(0x[0-9a-f]+)\]", x[1])
            if m:
                attribute(name(int(m.group(1), 16)), smp)
                break
        else:
            # inline wait: the TRYWAIT a few instructions above this branch
            for x in rows[max(0, i - 8):i]:
                m = re.search(r"TRYWAIT P\d, \[R\d+\+URZ\+(0x[0-9a-f]+)\]", x[1])
                if m:
                    attribute(name(int(m.group(1), 16)), smp)
print(f"total samples {tot}")
agg = {}
for k, v in sites.items():
    kk = k.split("[")[0] if k.startswith("ring") else k
    agg[kk] = agg.get(kk, 0) + v
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"  {k:14s} {v:6d}  {v / tot * 100:5.1f}%")
