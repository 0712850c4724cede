"""dev tool: kernel-only frac of each forced warp organisation (FBF_MODE=0/1/2) at
one (radius, K) point per line; run once per mode: FBF_MODE=m python tools/mode_sweep.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02168_b200 as fb
img = fb.voronoi_image(2048, 2048, 256, 10.0, 42)
d = torch.from_numpy(img).cuda(); o = torch.empty_like(d)
peak = torch.cuda.get_device_properties(0).multi_processor_count * 128 * 2 * 1965e6
for r, K in [tuple(int(v) for v in p.split(",")) for p in os.environ.get("FBF_POINTS", "18,4 21,4 24,4 27,4 30,4 30,3 24,3 18,5 24,5 30,5 9,2 15,2 24,2").split()]:
    k = fb.build_spatial_kernel(r / 3.0)
    a = fb.select_parameters(50.0, K=K, T=200)
    for _ in range(3): fb.fast_bilateral_device(d, k, a, o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): fb.fast_bilateral_device(d, k, a, o)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e-3
    flop = (4 * K - 2) * 2 * (2 * k.radius + 1) * 2 * img.size
    print(json.dumps({"mode": os.environ.get("FBF_MODE", "auto"), "r": r, "K": K, "frac": round(flop / t / peak, 3)}), flush=True)
