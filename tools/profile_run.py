"""Short device-resident run of one config for ncu (dev tool): W warm-up + N launches."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
cfg = configs.CONFIGS[a.config]
img = configs.make_frame(cfg, 0)
approx = configs.select(cfg)
k = fb.build_spatial_kernel(cfg.theta)
d_in = torch.from_numpy(img).cuda()
d_out = torch.empty_like(d_in)
for _ in range(a.iters):
    fb.fast_bilateral_device(d_in, k, approx, d_out)
torch.cuda.synchronize()
print("ok", a.config, approx.terms, approx.half_period)
