"""dev: local-memory instructions (LDL/STL) inside FFMA2-dense stretches of a kernel's SASS.
    python tools/sass_spills.py OBJ MANGLED_SUBSTRING"""
import subprocess, sys
obj, sub = sys.argv[1], sys.argv[2]
names = [l.split()[-1] for l in subprocess.run(["cuobjdump", "-elf", obj], capture_output=True, text=True).stdout.splitlines()
         if ".text." in l and sub in l and "PROGBITS" in l]
fn = sorted(set(n.replace(".text.", "") for n in names))
for f in fn:
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", f, obj], capture_output=True, text=True).stdout.splitlines()
    ins = [l for l in sass if "/*" in l and ";" in l]
    ff = [i for i, l in enumerate(ins) if "FFMA2" in l]
    regions, s = [], None
    for a, b in zip(ff, ff[1:] + [10**9]):
        if s is None:
            s = a
        if b - a > 40:
            regions.append((s, a)); s = None
    print(f, "instructions", len(ins), "FFMA2", len(ff))
    for a, b in regions:
        sp = [l.split("*/")[1].strip() for l in ins[a:b] if "LDL" in l or "STL" in l]
        print(f"  FFMA2 stretch [{a}, {b}] len {b-a}: FFMA2 {sum('FFMA2' in l for l in ins[a:b])} LDS {sum('LDS' in l for l in ins[a:b])} local {len(sp)} {sp[:3]}")
    for l in ins:
        if "USETMAXREG" in l: print("  ", l.split("*/")[1].strip())
