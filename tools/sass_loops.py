"""dev: loop summary of one kernel's SASS (cuobjdump): for every backward branch,
the instruction mix of the loop body [target, branch].
    python tools/sass_loops.py lib.so '<mangled-substring>'"""
import re
import subprocess
import sys
from collections import Counter

lib, name = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = out.split("Function : ")
body = next(f for f in funcs if f.split("\n", 1)[0].strip().find(name) >= 0)
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
print(f"{len(ins)} instructions")
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", txt)
    if not m:
        continue
    t = int(m.group(1), 16)
    if t <= a and t in addr:
        j = addr[t]
        ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0] for _, x in ins[j:i + 1])
        n = i - j + 1
        if n >= 20:
            print(f"loop {j:5d}-{i:5d} n={n:5d} FFMA2={ops['FFMA2']:4d} LDS={ops['LDS']:3d} STS={ops['STS']:3d} "
                  f"LDL={ops['LDL']:3d} STL={ops['STL']:3d} BAR={ops['BAR']:2d} SYNCS={ops['SYNCS']:2d} "
                  f"other={n - ops['FFMA2'] - ops['LDS'] - ops['STS'] - ops['LDL'] - ops['STL']}")
