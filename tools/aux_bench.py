"""Timing of the §8f kernels (dev tool): GPU brute filter at a config size and
the GPU period scan per order. Prints JSON lines."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--what", default="brute,scan")
a = ap.parse_args()
cfg = configs.CONFIGS[a.config]
if "brute" in a.what:
    img = configs.make_frame(cfg, 0)
    b = fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(cfg.sigma))
    k = fb.build_spatial_kernel(cfg.theta)
    d = torch.from_numpy(img).cuda()
    o = torch.empty(img.shape, dtype=torch.float64, device="cuda")
    fb.brute_bilateral_device(d, k, b, o)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); fb.brute_bilateral_device(d, k, b, o); torch.cuda.synchronize(); t = time.perf_counter() - t0
    taps = (2 * k.radius + 1) ** 2
    print(json.dumps({"kernel": "brute", "config": a.config, "ms": round(1e3 * t, 3), "MP/s": round(img.size / t / 1e6, 2),
                      "Gtaps/s": round(img.size * taps / t / 1e9, 2), "fp64_gflops_5_per_tap": round(5 * img.size * taps / t / 1e9, 1)}))
if "scan" in a.what:
    b = fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(cfg.sigma))
    for K in (1, 4, 9, 16):
        fb.scan_period_errors_gpu(b, K, 1, 2550, 0)
        t0 = time.perf_counter(); fb.scan_period_errors_gpu(b, K, 1, 2550, 0); t = time.perf_counter() - t0
        print(json.dumps({"kernel": "period_scan", "K": K, "t_max": 2550, "ms": round(1e3 * t, 3)}))
