import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02168_b200 as fb
from oracle import fbf_oracle
O = fbf_oracle.Oracle()
for (W, H, theta, sigma, eps) in [(256, 300, 8.0, 15.0, 0.01), (256, 300, 8.0, 30.0, 0.1), (512, 1024, 8.0, 15.0, 0.01), (4096, 512, 8.0, 15.0, 0.01)]:
    img = fb.field_image(W, H, 20, 5.0, 3)
    a = fb.select_parameters(sigma, eps=eps)
    out = fb.fast_bilateral(img, fb.build_spatial_kernel(theta), a).astype(np.float64)
    ref, _ = O.fast_bilateral(img.astype(np.float64), theta, a.terms, a.half_period, a.coefficients)
    err = np.abs(out - ref)
    rows = np.where(err.max(axis=1) > 1e-2)[0]
    cols = np.where(err.max(axis=0) > 1e-2)[0]
    print(W, H, "K", a.terms, "max", err.max(), "bad rows", rows[:10], len(rows), "bad cols", cols[:10], len(cols), flush=True)
