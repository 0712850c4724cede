"""The C ABI boundary (include/fbf.h): library loads, every declared symbol is
exported, argument errors map to the reference's exception classes, and the
host-side helpers behave. No GPU compute is issued here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "fbf.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fbf_\w+)\s*\(", text)))


def test_header_symbols_exported(fb):
    lib = fb._lib.load()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", fb._lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fbf_\w+)", out))
    assert set(syms) <= exported
    # and the python binding covers every declared entry point
    assert set(syms) <= set(fb._lib.SIGNATURES)


def test_library_is_built_for_sm100a(fb):
    out = subprocess.run(["cuobjdump", "--list-elf", fb._lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_errors_before_any_device_work(fb):
    img = np.zeros((8, 8), np.float32)
    k = fb.build_spatial_kernel(1.0)
    good = fb.fit_fixed_period(fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(30.0)), 2, 100)
    bad = fb.FourierApproximation(0, 100, 255, fb.frequency_of(100), np.zeros(0))
    with pytest.raises(fb.InvalidArgument):  # filter.cpp:132-134
        fb.fast_bilateral(img, k, bad)
    lib = fb._lib.load()
    c = np.zeros(2)
    rc = lib.fbf_fast_bilateral_f32(img.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 8, 8, -1.0, 2, 100, 255,
                                    c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 0,
                                    img.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), None)
    assert rc == fb._lib.FBF_EINVAL and "theta" in fb._lib.last_error()
    rc = lib.fbf_fast_bilateral_f32(img.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), 0, 8, 1.0, 2, 100, 255,
                                    c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 0,
                                    img.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), None)
    assert rc == fb._lib.FBF_EINVAL
    big = fb.build_spatial_kernel(11.0)  # radius 33 > FBF_MAX_RADIUS
    with pytest.raises(fb.InvalidArgument):
        fb.fast_bilateral(img, big, good)


def test_no_cpu_fallback_without_gpu(fb):
    if fb._lib.load().fbf_device_count() > 0:
        pytest.skip("a GPU is visible")
    img = np.zeros((8, 8), np.float32)
    a = fb.fit_fixed_period(fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(30.0)), 2, 100)
    with pytest.raises(fb.CudaError, match="no CUDA device"):
        fb.fast_bilateral(img, fb.build_spatial_kernel(1.0), a)


def py_source_window(H, y0, n, r, border):
    """Rows the border mapping reaches for output rows [y0, y0+n) (image.hpp:43-61)."""
    rows = set()
    for y in range(y0 - r, y0 + n + r):
        if 0 <= y < H:
            rows.add(y)
            continue
        if border == 2:
            continue
        if border == 1:
            rows.add(0 if y < 0 else H - 1)
            continue
        m = y % (2 * H)
        rows.add(m if m < H else 2 * H - 1 - m)
    return min(rows), max(rows) + 1


@pytest.mark.parametrize("H", [1, 5, 37, 1000])
def test_band_source_rows(fb, H):
    for border in (0, 1, 2):
        for G in (1, 2, 3, 8):
            for g in range(min(G, H)):
                y0, y1 = H * g // min(G, H), H * (g + 1) // min(G, H)
                r0, n = fb.band_source_rows(H, y0, y1 - y0, 5.0, border)
                lo, hi = py_source_window(H, y0, y1 - y0, 15, border)
                assert r0 <= lo and r0 + n >= hi
                assert 0 <= r0 and r0 + n <= H


def test_synthetic_generators(fb, oracle):
    assert np.array_equal(fb.random_image(24, 24, 7000), oracle.random_image(24, 24, 7000).astype(np.float32))
    assert np.array_equal(fb.scene_image(96, 96, 2024), oracle.scene_image(96, 96, 2024).astype(np.float32))
    a = fb.voronoi_image(256, 200, 64, 10.0, 123, threads=1)
    b = fb.voronoi_image(256, 200, 64, 10.0, 123, threads=4)
    assert np.array_equal(a, b) and a.min() >= 0 and a.max() <= 255
    f1 = fb.field_image(300, 128, 64, 5.0, 9, threads=1)
    f2 = fb.field_image(300, 128, 64, 5.0, 9, threads=3)
    assert np.array_equal(f1, f2) and f1.min() >= 0 and f1.max() <= 255
    assert np.std(f1) > 10


def test_voronoi_nearest_site_matches_brute_force(fb):
    # the bucketed search must equal exhaustive nearest-site assignment
    w, h, n = 97, 61, 20
    img = fb.voronoi_image(w, h, n, 0.0, 77, threads=1)
    # reproduce sites with the same SplitMix64 stream
    state = [77]

    def nxt():
        state[0] = (state[0] + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = state[0]
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    sites = []
    for _ in range(n):
        x = (nxt() >> 11) * 2.0 ** -53 * w
        y = (nxt() >> 11) * 2.0 ** -53 * h
        v = 255.0 * ((nxt() >> 11) * 2.0 ** -53)
        sites.append((x, y, v))
    for y in range(h):
        for x in range(w):
            d = [((sx - x - 0.5) ** 2 + (sy - y - 0.5) ** 2, i) for i, (sx, sy, _) in enumerate(sites)]
            i = min(d)[1]
            assert img[y, x] == np.float32(min(255.0, max(0.0, sites[i][2])))
