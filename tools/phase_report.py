"""Per-warp-slot wait profile of the fused kernel (dev tool; needs a library
built with -D FBF_PHASES and FBF_PROF=1 in the environment).
    FBF_PROF=1 FBF_LIB=devlib/phases.so python tools/phase_report.py --config c1"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs, _lib

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
cfg = configs.CONFIGS[a.config]
img = configs.make_frame(cfg, 0)
approx = configs.select(cfg)
k = fb.build_spatial_kernel(cfg.theta)
d_in = torch.from_numpy(img).cuda()
d_out = torch.empty_like(d_in)
lib = _lib.load()
buf = (ctypes.c_ulonglong * 128)()
fb.fast_bilateral_device(d_in, k, approx, d_out)
torch.cuda.synchronize()
lib.fbf_dev_prof(buf)
for _ in range(a.iters):
    fb.fast_bilateral_device(d_in, k, approx, d_out)
torch.cuda.synchronize()
rc = lib.fbf_dev_prof(buf)
if rc != 0:
    sys.exit("no profile counters (build with -D FBF_PHASES, run with FBF_PROF=1)")
mode = int(os.environ.get("FBF_MODE", "1"))
def placed_name(w, np_):
    fwg = (2 * np_ + 3) // 4; g0 = 8 - fwg; left = 4 * fwg - 2 * np_; g, s = w // 4, w % 4
    if g >= g0 and not (g == 7 and s >= 4 - left):
        f = (g - g0) * 4 + s
        return f"ROW{f}" if f < np_ else f"COL{f - np_}"
    k = s - (4 - left) if g >= g0 else (left + 2 * g + s - 2 if s >= 2 else left + 2 * g0 + 2 * g + s)
    return f"GEN{k}" if k < 4 else f"COMB{k - 4}" if k < 8 else "LOAD" if k == 8 else "-"
np_ = 2 * approx.terms - 1
nf = np_ if mode == 0 else 2 * np_
names = []
for w in range(32):
    if w < np_: names.append(("PAIR" if mode == 0 else "ROW") + f"{w}")
    elif w < nf: names.append(f"COL{w - np_}")
    elif w < nf + 4: names.append(f"COMB{w - nf}")
    elif w < nf + 8: names.append(f"GEN{w - nf - 4}")
    elif w == nf + 8: names.append("LOAD")
    else: names.append("-")
nw = nf + 9
# fixed layouts: pair mode with 7 pairs (register split) and the c4 kernel (kHalfWgMode, 5 pairs)
fixed = None
if mode == 0 and np_ == 7:
    fixed = [f"GEN{3 - w}" for w in range(4)] + [f"COMB{7 - w}" for w in range(4, 8)] + ["LOAD"] + [f"PAIR{15 - w}" for w in range(9, 16)]
elif mode == 2 and np_ == 5:
    fixed = list("GGGGMMMMLCCCCCCCRCCCRRRR")
    fixed = [{"G": "GEN", "M": "COMB", "L": "LOAD", "C": "COLh", "R": "ROW"}[c] for c in fixed]
for w in range(32):
    tot, wa, wb, n = buf[4 * w:4 * w + 4]
    if n == 0: continue
    nm = fixed[w] if fixed and w < len(fixed) else names[nw - 1 - w] if mode != 2 and 0 <= nw - 1 - w < len(names) else "slot"
    print(f"warp {w:2d} smsp {w % 4} {nm:6s} cycles/CTA {tot / n:10.0f}  waitA {wa / tot * 100:5.1f}%  waitB {wb / tot * 100:5.1f}%  busy {100 - (wa + wb) / tot * 100:5.1f}%")
