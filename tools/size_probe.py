"""dev: kernel time vs image size at fixed (theta, sigma, eps) -- fixed launch/pipeline
cost vs per-pixel cost. python tools/size_probe.py --theta 3 --sigma 30 --eps 0.1"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02168_b200 as fb

ap = argparse.ArgumentParser()
ap.add_argument("--theta", type=float, default=3.0)
ap.add_argument("--sigma", type=float, default=30.0)
ap.add_argument("--eps", type=float, default=0.1)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--sizes", default="512x16,512x64,512x128,512x256,512x512,512x1024,1024x1024,2048x1024")
a = ap.parse_args()
approx = fb.select_parameters(a.sigma, eps=a.eps)
k = fb.build_spatial_kernel(a.theta)
r = k.radius
for sz in a.sizes.split(","):
    W, H = map(int, sz.split("x"))
    img = fb.voronoi_image(W, H, 64, 10.0, 7)
    d_in = torch.from_numpy(img).cuda()
    d_out = torch.empty_like(d_in)
    for _ in range(3):
        fb.fast_bilateral_device(d_in, k, approx, d_out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    torch.cuda._sleep(int(2e6 + 2e6 * a.iters))
    e0.record()
    t0 = time.perf_counter()
    for _ in range(a.iters):
        fb.fast_bilateral_device(d_in, k, approx, d_out)
    host_us = (time.perf_counter() - t0) / a.iters * 1e6
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / a.iters * 1e3
    flop = W * H * (4 * approx.terms - 2) * 2 * (2 * r + 1) * 2
    print(f"{sz:>10s} K={approx.terms} r={r} {us:8.1f} us  frac {flop / us / 1e6 / 74.45:.3f}  host enqueue {host_us:.1f} us/call", flush=True)
