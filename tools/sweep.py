"""Kernel-only throughput over the (radius, K) space at 2048x2048 (device-resident,
no L2 flush): MP/s and fraction of the FP32-FMA peak, one JSON line per point."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_02168_b200 as fb
img = fb.voronoi_image(2048, 2048, 256, 10.0, 42)
d = torch.from_numpy(img).cuda(); o = torch.empty_like(d)
n_sm = torch.cuda.get_device_properties(0).multi_processor_count
peak = n_sm * 128 * 2 * 1965e6
for r in [int(v) for v in os.environ.get("FBF_SWEEP_R", "3 6 9 12 15 18 24 30").split()]:
    theta = r / 3.0
    k = fb.build_spatial_kernel(theta)
    for K in [int(v) for v in os.environ.get("FBF_SWEEP_K", "2 3 4 5 7 9").split()]:
        a = fb.select_parameters(50.0, K=K, T=200)
        for _ in range(3): fb.fast_bilateral_device(d, k, a, o)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n): fb.fast_bilateral_device(d, k, a, o)
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / n * 1e-3
        flop = (4 * K - 2) * 2 * (2 * k.radius + 1) * 2 * img.size
        print(json.dumps({"r": k.radius, "K": K, "pairs": 2 * K - 1, "us": round(t * 1e6, 1),
                          "MP/s": round(img.size / t / 1e6), "frac": round(flop / t / peak, 3)}), flush=True)
