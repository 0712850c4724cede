"""dev tool: c4 single-call host-API throughput (pinned fbf_host_alloc buffers), FBF_TRACE-free."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
img = configs.make_frame(cfg)
a = configs.select(cfg)
k = fb.build_spatial_kernel(cfg.theta)
h_in = fb.pinned_empty(img.shape); h_in[:] = img
h_out = fb.pinned_empty(img.shape)
for _ in range(2): fb.fast_bilateral(h_in, k, a, out=h_out)
ts = []
for _ in range(6):
    t0 = time.perf_counter(); fb.fast_bilateral(h_in, k, a, out=h_out); ts.append(time.perf_counter() - t0)
print(os.environ.get("TAG", ""), f"median {1e3*np.median(ts):.2f} ms -> {img.size/np.median(ts)/1e6:.0f} MP/s", flush=True)
