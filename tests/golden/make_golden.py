"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists): builds oracle/_ref/libfbf_ref.so from
the reference's own filter.cpp / kernels.cpp / synthetic.cpp and records its
outputs on small seeded inputs. The fixtures pin oracle/fbf_oracle.c (bit-exact)
on machines without the reference, and give the GPU parity tests frozen
expected values. Coefficients come from the numpy restatement of the
reference optimiser (itself pinned against the reference's frozen test values).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import fbf_oracle as fo  # noqa: E402


def main():
    fo.build_oracle(with_ref=True)
    ref = fo.RefLibrary()
    out = {}
    # spatial taps and range samples (kernels.cpp)
    for theta in (1.0, 2.0, 3.0, 5.0, 8.0, 10.0):
        out[f"taps_theta{theta:g}"] = ref.spatial_taps(theta)
    for kind, sigma in (("gaussian", 50.0), ("gaussian", 15.0), ("exponential", 30.0), ("cauchy", 20.0)):
        out[f"range_{kind}_{sigma:g}"] = ref.range_samples(kind, sigma)
    # synthetic images (synthetic.cpp)
    out["random_24x24_7000"] = ref.random_image(24, 24, 7000)
    out["random_5x4_7"] = ref.random_image(5, 4, 7)
    out["scene_96x96_2024"] = ref.scene_image(96, 96, 2024)
    # fast_bilateral on the reference parameter grid (test_filter.cpp:168-183)
    cases = []
    seed = 0
    for theta in (1.0, 3.0, 5.0):
        for sigma in (15.0, 30.0, 50.0):
            b = ref.range_samples("gaussian", sigma)
            rep = fo.optimize_parameters(b, 0.1, t_max=700)
            img = ref.random_image(24, 24, 7000 + seed)
            seed += 1
            for border in ("symmetric", "replicate", "zero"):
                o, fb = ref.fast_bilateral(img, theta, rep.K, rep.T, rep.coefficients, border=border)
                key = f"fast_t{theta:g}_s{sigma:g}_{border}"
                out[key + "_img"] = img
                out[key + "_coeffs"] = rep.coefficients
                out[key + "_KT"] = np.array([rep.K, rep.T])
                out[key + "_out"] = o
                cases.append(key)
    # radius 9 on a 5x4 image (test_filter.cpp:73-81), K=4 T=203 sigma=50
    b50 = ref.range_samples("gaussian", 50.0)
    c, _ = fo.fit_coefficients(fo.design_matrix(4, 203, 255), b50)
    img = ref.random_image(5, 4, 7)
    for border in ("symmetric", "replicate", "zero"):
        o, _ = ref.fast_bilateral(img, 3.0, 4, 203, c, border=border)
        out[f"fast_5x4_{border}_out"] = o
    out["c_sigma50_K4_T203"] = c
    # brute with the true kernel on the scene image (test_metrics.cpp:111-123)
    b55 = ref.range_samples("gaussian", 55.0)
    o, _ = ref.brute_bilateral(out["scene_96x96_2024"], 5.0, b55, border="symmetric", threads=8)
    out["brute_scene96_t5_s55"] = o
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    with open(os.path.join(HERE, "cases.txt"), "w") as f:
        f.write("\n".join(cases) + "\n")
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
