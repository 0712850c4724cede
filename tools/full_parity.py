"""Full-size parity of every BASELINE config against the reference's own
fast_bilateral (oracle/_ref, compiled from the reference sources, FP64, all host
threads): max |GPU - reference| over ALL pixels (c3: all 64 frames; c4: the
whole 16384x16384 image, the reference run in 2048-row bands with r-row halos,
which is bit-identical to one run because the border mapping only reaches rows
inside the halo). Writes one JSON line per config.

    python tools/full_parity.py [--configs c0,c1,c2,c3,c4] [--out profiles/r01_full_parity.jsonl]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1811_02168_b200 as fb  # noqa: E402
from oracle import fbf_oracle  # noqa: E402
from paper_1811_02168_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c0,c1,c2,c3,c4")
ap.add_argument("--out", default="")
ap.add_argument("--border", default="symmetric", choices=["symmetric", "replicate", "zero"])
a = ap.parse_args()
ref = fbf_oracle.RefLibrary()
threads = os.cpu_count() or 1
lines = []
for name in a.configs.split(","):
    cfg = configs.CONFIGS[name]
    approx = configs.select(cfg)
    k = fb.build_spatial_kernel(cfg.theta)
    r = cfg.radius
    worst, n_px, gpu_fb, ref_fb = 0.0, 0, 0, 0
    edge = 0.0  # max over pixels within 2r of an image edge (where the border policy acts)
    t0 = time.perf_counter()
    if cfg.sharding == "frames":
        frames = np.stack([configs.make_frame(cfg, f) for f in range(cfg.frames)])
        diag = fb.FilterDiagnostics()
        out = fb.fast_bilateral_batch(frames, k, approx, a.border, diag=diag, n_gpus=1)
        gpu_fb = diag.fallback_pixels
        for f in range(cfg.frames):
            rr, rf = ref.fast_bilateral(frames[f].astype(np.float64), cfg.theta, approx.terms, approx.half_period,
                                        approx.coefficients, border=a.border, threads=threads)
            dd = np.abs(out[f].astype(np.float64) - rr)
            worst = max(worst, float(dd.max()))
            m = np.ones(dd.shape, bool)
            m[2 * r:-2 * r, 2 * r:-2 * r] = False
            edge = max(edge, float(dd[m].max()))
            ref_fb += rf
            n_px += rr.size
    else:
        img = configs.make_frame(cfg)
        diag = fb.FilterDiagnostics()
        out = fb.fast_bilateral(img, k, approx, a.border, diag=diag)
        gpu_fb = diag.fallback_pixels
        H = img.shape[0]
        band = H if H <= 4096 else 2048
        for y0 in range(0, H, band):
            y1 = min(H, y0 + band)
            s0, s1 = max(0, y0 - r), min(H, y1 + r)
            rr, rf = ref.fast_bilateral(img[s0:s1].astype(np.float64), cfg.theta, approx.terms, approx.half_period,
                                        approx.coefficients, border=a.border, threads=threads)
            if s0 > 0 or s1 < H:
                # band + halo: rows of the band equal the full-image result only away from the
                # artificial band edges, i.e. exactly the rows [y0, y1) when s0/s1 add r rows
                rr = rr[y0 - s0:y0 - s0 + (y1 - y0)]
            dd = np.abs(out[y0:y1].astype(np.float64) - rr)
            worst = max(worst, float(dd.max()))
            m = np.zeros(dd.shape, bool)
            m[:, :2 * r] = m[:, -2 * r:] = True
            rows = np.arange(y0, y1)
            m[(rows < 2 * r) | (rows >= H - 2 * r), :] = True
            edge = max(edge, float(dd[m].max()))
            ref_fb += rf
            n_px += rr.size
    line = {"config": name, "border": a.border, "pixels": n_px, "K": approx.terms, "T": approx.half_period, "theta": cfg.theta,
            "sigma": cfg.sigma, "max_abs_gpu_minus_reference": worst, "max_abs_within_2r_of_edges": edge, "tolerance": 1e-2,
            "gpu_fallbacks": int(gpu_fb), "reference_fallbacks": int(ref_fb),
            "reference": f"oracle/_ref fast_bilateral (reference sources), fp64, {threads} threads",
            "seconds": round(time.perf_counter() - t0, 1)}
    print(json.dumps(line), flush=True)
    lines.append(line)
if a.out:
    with open(a.out, "w") as f:
        f.write("\n".join(json.dumps(x) for x in lines) + "\n")
