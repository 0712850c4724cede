import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
cfg = configs.CONFIGS["c1"]; img = configs.make_frame(cfg); a = configs.select(cfg); k = fb.build_spatial_kernel(cfg.theta)
n = 20
frames = fb.pinned_empty((n,) + img.shape); frames[:] = img
outs = fb.pinned_empty((n,) + img.shape)
fb.fast_bilateral_batch(frames, k, a, out=outs, n_gpus=1)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); fb.fast_bilateral_batch(frames, k, a, out=outs, n_gpus=1); ts.append(time.perf_counter() - t0)
print(os.environ.get("FBF_PIECES", "auto"), f"{1e3*np.median(ts)/n:.3f} ms/frame -> {n*img.size/np.median(ts)/1e6:.0f} MP/s")
