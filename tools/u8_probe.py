"""8-bit host path vs float32 host path, one call per image (c1 geometry)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
cfg = configs.CONFIGS["c1"]
img = configs.make_frame(cfg); a = configs.select(cfg); k = fb.build_spatial_kernel(cfg.theta)
f_in = fb.pinned_empty(img.shape); f_in[:] = img; f_out = fb.pinned_empty(img.shape)
u_in = fb.pinned_empty(img.shape, np.uint8); u_in[:] = np.round(img).astype(np.uint8)
u_out = fb.pinned_empty(img.shape, np.uint8)
def t(fn, n=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return np.median(ts)
tf = t(lambda: fb.fast_bilateral(f_in, k, a, out=f_out))
tu = t(lambda: fb.fast_bilateral_u8(u_in, k, a, out=u_out))
tp = t(lambda: fb.fast_bilateral_u8(u_in, k, a))
print(f"float32 in/out: {1e3*tf:.3f} ms ({img.size/tf/1e6:.0f} MP/s); uint8 in/out (pinned out): {1e3*tu:.3f} ms "
      f"({img.size/tu/1e6:.0f} MP/s); uint8 with a pageable out: {1e3*tp:.3f} ms")
