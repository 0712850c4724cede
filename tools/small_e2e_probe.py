"""dev tool: host-API latency breakdown for a small image (c0, 512x512)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c0"]
img = configs.make_frame(cfg); a = configs.select(cfg); k = fb.build_spatial_kernel(cfg.theta)
h_in = fb.pinned_empty(img.shape); h_in[:] = img; h_out = fb.pinned_empty(img.shape)
for _ in range(5): fb.fast_bilateral(h_in, k, a, out=h_out)
ts = []
for _ in range(50):
    t0 = time.perf_counter(); fb.fast_bilateral(h_in, k, a, out=h_out); ts.append(time.perf_counter() - t0)
print(cfg.name, f"median {1e6*np.median(ts):.1f} us  min {1e6*min(ts):.1f} us")
