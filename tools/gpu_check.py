"""Quick GPU correctness/timing probe (dev tool): GPU fused kernel vs the C oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
from oracle import fbf_oracle

O = fbf_oracle.Oracle()
worst = 0.0
for (W, H, theta, sigma, seed) in [(24, 24, 1.0, 30.0, 1), (24, 24, 3.0, 15.0, 2), (5, 4, 3.0, 50.0, 3),
                                   (97, 61, 5.0, 50.0, 4), (200, 150, 2.0, 30.0, 5), (64, 300, 8.0, 15.0, 6),
                                   (333, 77, 10.0, 80.0, 7)]:
    img = O.random_image(W, H, seed).astype(np.float32)
    k = fb.build_spatial_kernel(theta)
    a = fb.select_parameters(sigma, eps=0.1 if sigma > 20 else 0.01)
    for border in ("symmetric", "replicate", "zero"):
        out = fb.fast_bilateral(img, k, a, border)
        ref, _ = O.fast_bilateral(img.astype(np.float64), theta, a.terms, a.half_period, a.coefficients, border=border)
        e = float(np.abs(out - ref).max())
        worst = max(worst, e)
        print(f"{W}x{H} theta={theta} K={a.terms} T={a.half_period} {border}: max err {e:.3e}", flush=True)
print("worst", worst)

import torch
cfg = configs.CONFIGS["c1"]
img = configs.make_input(cfg)
a = configs.select(cfg)
k = fb.build_spatial_kernel(cfg.theta)
d_in = torch.from_numpy(img).cuda()
d_out = torch.empty_like(d_in)
for _ in range(3):
    fb.fast_bilateral_device(d_in, k, a, d_out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for _ in range(n):
    fb.fast_bilateral_device(d_in, k, a, d_out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
mp = cfg.pixels / ms / 1e3
flops = cfg.flop_per_pixel(a.terms) * cfg.pixels / (ms * 1e-3)
print(f"c1: {ms:.3f} ms  {mp:.0f} MP/s  {flops/1e12:.2f} TFLOP/s ({flops/74.45e12*100:.1f}% of 74.45)")
ref, _ = O.fast_bilateral(img[:256, :256].astype(np.float64), cfg.theta, a.terms, a.half_period, a.coefficients)
out = fb.fast_bilateral(img[:256, :256], k, a)
print("c1 crop err", float(np.abs(out - ref).max()))
