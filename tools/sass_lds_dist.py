"""dev tool: distance (in instructions) from each LDS to the first use of its
result in one kernel's SASS (cuobjdump). Usage: python tools/sass_lds_dist.py OBJ MANGLED_SUBSTR"""
import re, subprocess, sys
obj, fn = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
blocks = out.split("Function : ")
body = next(b for b in blocks if b.startswith(fn) or fn in b.split("\n", 1)[0])
ins = [re.sub(r"^\s*/\*[0-9a-f]+\*/\s*", "", l).split(";")[0].strip() for l in body.split("\n") if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l)]
dists = []
for i, s in enumerate(ins):
    m = re.search(r"\bLDS(\.\d+)?\s+(R\d+)", s)
    if not m:
        continue
    reg = int(m.group(2)[1:])
    w = {None: 1, ".64": 2, ".128": 4}[m.group(1)]
    for j in range(i + 1, min(i + 400, len(ins))):
        ops = ins[j].split(None, 1)
        if len(ops) < 2:
            continue
        srcs = ops[1].split(",", 1)[1] if "," in ops[1] else ""
        if any(reg <= int(x) < reg + w for x in re.findall(r"\bR(\d+)", srcs)):
            dists.append((i, m.group(1) or "", j - i))
            break
short = [d for d in dists if d[2] <= 4]
print(f"{len(ins)} instrs, {len(dists)} LDS; used within 4 instrs: {len(short)}")
for d in dists:
    print(f"  @{d[0]:5d} LDS{d[1]:5s} -> use +{d[2]}")
