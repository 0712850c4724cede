"""Device-resident kernel timing of one config (dev tool): MP/s and FP32-FMA fraction.
    FBF_LIB=devlib/x.so python tools/kbench.py --config c1 --iters 50"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--tag", default="")
a = ap.parse_args()
cfg = configs.CONFIGS[a.config]
img = configs.make_frame(cfg, 0)
approx = configs.select(cfg)
k = fb.build_spatial_kernel(cfg.theta)
d_in = torch.from_numpy(img).cuda()
d_out = torch.empty_like(d_in)
for _ in range(3):
    fb.fast_bilateral_device(d_in, k, approx, d_out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(2e6 + 2e5 * a.iters))  # gate: host enqueue never shows between the events
e0.record()
for _ in range(a.iters):
    fb.fast_bilateral_device(d_in, k, approx, d_out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
px = img.size
r = k.radius if hasattr(k, "radius") else int(-(-3 * cfg.theta // 1))
flop = px * (4 * approx.terms - 2) * 2 * (2 * r + 1) * 2
import hashlib
h = hashlib.md5(d_out.cpu().numpy().tobytes()).hexdigest()[:12]
print(f"{a.tag:24s} {h} {a.config} {ms*1e3:8.1f} us  {px/ms/1e3:9.1f} MP/s  frac {flop/ms/1e9/74.45:.3f}", flush=True)
