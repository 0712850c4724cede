"""dev tool: host-API (H2D + kernel + D2H) latency for c1, from torch-pinned
and from fbf_host_alloc-pinned buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
cfg = configs.CONFIGS["c1"]
img = configs.make_frame(cfg)
a = configs.select(cfg)
k = fb.build_spatial_kernel(cfg.theta)
for alloc in ("torch", "fbf"):
    if alloc == "torch":
        h_in = torch.from_numpy(img).pin_memory().numpy()
        h_out = torch.empty(img.shape, dtype=torch.float32).pin_memory().numpy()
    else:
        h_in = fb.pinned_empty(img.shape); h_in[:] = img
        h_out = fb.pinned_empty(img.shape)
    for _ in range(3): fb.fast_bilateral(h_in, k, a, out=h_out)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); fb.fast_bilateral(h_in, k, a, out=h_out); ts.append(time.perf_counter() - t0)
    print(alloc, os.environ.get("FBF_PIECES", "auto"), f"median {1e3*np.median(ts):.3f} ms  min {1e3*min(ts):.3f} ms  -> {img.size/np.median(ts)/1e6:.0f} MP/s")
# frames pipelined through one batch call (H2D of frame i+1 / D2H of frame i-1 overlap kernel i)
n = 20
frames = fb.pinned_empty((n,) + img.shape); frames[:] = img
outs = fb.pinned_empty((n,) + img.shape)
fb.fast_bilateral_batch(frames, k, a, out=outs, n_gpus=1)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); fb.fast_bilateral_batch(frames, k, a, out=outs, n_gpus=1); ts.append(time.perf_counter() - t0)
print("batch", n, f"median {1e3*np.median(ts)/n:.3f} ms/frame -> {n*img.size/np.median(ts)/1e6:.0f} MP/s")
