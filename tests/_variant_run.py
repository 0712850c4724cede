"""Helper for tests/test_gpu_variants.py: filters a fixed set of small cases
with whatever kernel plan the FBF_* environment forces and saves the outputs.
    python tests/_variant_run.py OUT.npz"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1811_02168_b200 as fb  # noqa: E402

# (W, H, theta, sigma, eps, border): radii 3..30, K 1..9, every border
CASES = [
    (96, 80, 1.0, 30.0, 0.1, "symmetric"),
    (130, 70, 3.0, 30.0, 0.1, "replicate"),
    (200, 150, 5.0, 50.0, 0.1, "symmetric"),
    (64, 257, 5.0, 15.0, 0.01, "zero"),
    (100, 90, 16.0 / 3.0, 40.0, 0.05, "symmetric"),
    (150, 120, 8.0, 15.0, 0.01, "replicate"),
    (97, 333, 10.0, 80.0, 0.05, "symmetric"),
    (120, 100, 8.0, 15.0, 0.01, "zero"),       # r = 24, K = 9: two chunks (duo / scratch)
    (700, 64, 10.0, 80.0, 0.05, "zero"),       # r = 30, K = 3: the c4 kernel (warpgroup split)
]


def main(path):
    out = {}
    for i, (W, H, theta, sigma, eps, border) in enumerate(CASES):
        img = np.asarray(fb.random_image(W, H, 1000 + i), dtype=np.float32)
        k = fb.build_spatial_kernel(theta)
        a = fb.select_parameters(sigma, eps=eps)
        out[f"c{i}"] = fb.fast_bilateral(img, k, a, border)
        out[f"i{i}"] = img
    np.savez(path, **out)


if __name__ == "__main__":
    main(sys.argv[1])
