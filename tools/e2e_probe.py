"""dev tool: host-API (H2D + kernel + D2H) latency for c1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
cfg = configs.CONFIGS["c1"]
img = configs.make_frame(cfg)
a = configs.select(cfg)
k = fb.build_spatial_kernel(cfg.theta)
h_in = torch.from_numpy(img).pin_memory().numpy()
h_out = torch.empty(img.shape, dtype=torch.float32).pin_memory().numpy()
for _ in range(3): fb.fast_bilateral(h_in, k, a, out=h_out)
ts = []
for _ in range(20):
    t0 = time.perf_counter(); fb.fast_bilateral(h_in, k, a, out=h_out); ts.append(time.perf_counter() - t0)
print(os.environ.get("FBF_PIECES", "auto"), f"median {1e3*np.median(ts):.3f} ms  min {1e3*min(ts):.3f} ms  -> {img.size/np.median(ts)/1e6:.0f} MP/s")
