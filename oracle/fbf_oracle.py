"""TEST INFRASTRUCTURE ONLY -- Python side of the fbf parity oracle.

* ``Oracle``     : ctypes binding of oracle/build/libfbf_oracle.so, our plain-C
                   restatement of the reference filter path (fbf_oracle.c).
* ``RefLibrary`` : ctypes binding of oracle/_ref/libfbf_ref.so, the reference's
                   own filter.cpp / kernels.cpp / synthetic.cpp compiled verbatim
                   (oracle/Makefile). Absent on boxes where it was never built.
* ``fit_*`` / ``optimize_parameters`` : numpy restatement of the reference's
                   least-squares optimiser (approx.cpp:61-240). The reference's
                   solver is Eigen's CompleteOrthogonalDecomposition (Eigen 3.3+,
                   not vendored, not installed); we restate it with LAPACK's
                   min-norm least squares (numpy.linalg.lstsq, rank cutoff 1e-10
                   relative to the largest singular value). Pinned against the
                   reference's frozen values in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libfbf_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfbf_ref.so")
INPUTS_SO = os.path.join(HERE, "build", "libfbf_inputs.so")

BORDERS = {"symmetric": 0, "replicate": 1, "zero": 2}
KINDS = {"gaussian": 0, "exponential": 1, "cauchy": 2}

_dp = ctypes.POINTER(ctypes.c_double)
_llp = ctypes.POINTER(ctypes.c_longlong)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def build_oracle(with_ref: bool | None = None) -> None:
    """Build the C oracle (and, when /root/reference exists, oracle/_ref)."""
    targets = ["oracle"]
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/src")
    if with_ref:
        targets += ["ref", "integration"]
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _border(b) -> int:
    return BORDERS[b] if isinstance(b, str) else int(b)


class Oracle:
    """Plain-C restatement (oracle/fbf_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle(with_ref=False)
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.orc_map_border_index.argtypes = [ctypes.c_int] * 3
        L.orc_spatial_radius.argtypes = [ctypes.c_double]
        L.orc_build_spatial_kernel.argtypes = [ctypes.c_double, _dp]
        L.orc_sample_range_kernel.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp]
        L.orc_frequency_of.argtypes = [ctypes.c_int]
        L.orc_frequency_of.restype = ctypes.c_double
        L.orc_evaluate_approximation.argtypes = [ctypes.c_int, ctypes.c_int, _dp, ctypes.c_int]
        L.orc_evaluate_approximation.restype = ctypes.c_double
        L.orc_tabulate_approximation.argtypes = [ctypes.c_int] * 3 + [_dp, _dp]
        L.orc_convolve_separable.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_int,
                                             ctypes.c_int, _dp]
        L.orc_fast_bilateral.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                         ctypes.c_int, _dp, _llp]
        L.orc_brute_bilateral.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, _dp,
                                          ctypes.c_int, ctypes.c_int, _dp, _llp]
        L.orc_random_image.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _dp]
        L.orc_scene_image.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _dp]

    def map_border_index(self, i: int, n: int, border) -> int:
        return self.lib.orc_map_border_index(i, n, _border(border))

    def spatial_taps(self, theta: float) -> np.ndarray:
        r = self.lib.orc_spatial_radius(theta)
        taps = np.zeros(2 * r + 1)
        self.lib.orc_build_spatial_kernel(theta, _ptr(taps))
        return taps

    def range_samples(self, kind: str, sigma: float, R: int = 255) -> np.ndarray:
        v = np.zeros(2 * R + 1)
        if self.lib.orc_sample_range_kernel(KINDS[kind], sigma, R, _ptr(v)) != 0:
            raise ValueError("range kernel: invalid sigma/R")
        return v

    def tabulate(self, K: int, T: int, R: int, coeffs) -> np.ndarray:
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        v = np.zeros(2 * R + 1)
        self.lib.orc_tabulate_approximation(K, T, R, _ptr(c), _ptr(v))
        return v

    def convolve_separable(self, img: np.ndarray, theta: float, border="symmetric") -> np.ndarray:
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        taps = self.spatial_taps(theta)
        out = np.zeros_like(img)
        self.lib.orc_convolve_separable(_ptr(img), w, h, _ptr(taps), (len(taps) - 1) // 2,
                                        _border(border), _ptr(out))
        return out

    def fast_bilateral(self, img: np.ndarray, theta: float, K: int, T: int, coeffs, R: int = 255,
                       border="symmetric"):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros_like(img)
        fb = ctypes.c_longlong(0)
        rc = self.lib.orc_fast_bilateral(_ptr(img), w, h, theta, K, T, R, _ptr(c),
                                         _border(border), _ptr(out), ctypes.byref(fb))
        if rc != 0:
            raise ValueError(f"oracle fast_bilateral rc={rc}")
        return out, fb.value

    def brute_bilateral(self, img: np.ndarray, theta: float, range_values, R: int = 255,
                        border="symmetric"):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        rv = np.ascontiguousarray(range_values, dtype=np.float64)
        out = np.zeros_like(img)
        fb = ctypes.c_longlong(0)
        rc = self.lib.orc_brute_bilateral(_ptr(img), w, h, theta, _ptr(rv), R, _border(border),
                                          _ptr(out), ctypes.byref(fb))
        if rc != 0:
            raise ValueError(f"oracle brute_bilateral rc={rc}")
        return out, fb.value

    def random_image(self, w: int, h: int, seed: int) -> np.ndarray:
        out = np.zeros((h, w))
        self.lib.orc_random_image(w, h, seed, _ptr(out))
        return out

    def scene_image(self, w: int, h: int, seed: int) -> np.ndarray:
        out = np.zeros((h, w))
        self.lib.orc_scene_image(w, h, seed, _ptr(out))
        return out


class RefLibrary:
    """The reference's own sources, compiled verbatim (oracle/_ref/libfbf_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.fbfref_fast_bilateral.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                            ctypes.c_int, ctypes.c_int, _dp, _llp, _dp]
        L.fbfref_brute_bilateral.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                             _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                             _llp]
        L.fbfref_convolve_separable.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                                ctypes.c_int, _dp]
        L.fbfref_spatial_taps.argtypes = [ctypes.c_double, _dp]
        L.fbfref_range_samples.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp]
        L.fbfref_random_image.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, _dp]
        L.fbfref_scene_image.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, _dp]

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def fast_bilateral(self, img, theta, K, T, coeffs, R=255, border="symmetric", threads=1):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros_like(img)
        fb = ctypes.c_longlong(0)
        st = np.zeros(3)
        rc = self.lib.fbfref_fast_bilateral(_ptr(img), w, h, theta, K, T, R, _ptr(c),
                                            _border(border), threads, _ptr(out), ctypes.byref(fb),
                                            _ptr(st))
        if rc != 0:
            raise ValueError(f"reference fast_bilateral rc={rc}")
        return out, fb.value

    def brute_bilateral(self, img, theta, range_values, R=255, border="symmetric", threads=1):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        rv = np.ascontiguousarray(range_values, dtype=np.float64)
        out = np.zeros_like(img)
        fb = ctypes.c_longlong(0)
        rc = self.lib.fbfref_brute_bilateral(_ptr(img), w, h, theta, _ptr(rv), R, _border(border),
                                             threads, _ptr(out), ctypes.byref(fb))
        if rc != 0:
            raise ValueError(f"reference brute_bilateral rc={rc}")
        return out, fb.value

    def convolve_separable(self, img, theta, border="symmetric"):
        img = np.ascontiguousarray(img, dtype=np.float64)
        h, w = img.shape
        out = np.zeros_like(img)
        self.lib.fbfref_convolve_separable(_ptr(img), w, h, theta, _border(border), _ptr(out))
        return out

    def spatial_taps(self, theta):
        taps = np.zeros(2 * int(np.ceil(3 * theta)) + 1)
        self.lib.fbfref_spatial_taps(theta, _ptr(taps))
        return taps

    def range_samples(self, kind, sigma, R=255):
        v = np.zeros(2 * R + 1)
        self.lib.fbfref_range_samples(KINDS[kind], sigma, R, _ptr(v))
        return v

    def random_image(self, w, h, seed):
        out = np.zeros((h, w))
        self.lib.fbfref_random_image(w, h, seed, _ptr(out))
        return out

    def scene_image(self, w, h, seed):
        out = np.zeros((h, w))
        self.lib.fbfref_scene_image(w, h, seed, _ptr(out))
        return out


class Inputs:
    """The BASELINE.json input generators (paper_1811_02168_b200/csrc/fbf_synth.cpp
    compiled on their own into oracle/build/libfbf_inputs.so): bench.py's
    reference arm builds the same images as the GPU arm without mapping libfbf.so."""

    def __init__(self, path: str = INPUTS_SO):
        if not os.path.exists(path):
            build_oracle(with_ref=False)
        self.lib = ctypes.CDLL(path)
        fp = ctypes.POINTER(ctypes.c_float)
        args = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_ulonglong, ctypes.c_int, fp]
        self.lib.fbf_voronoi_image_f32.argtypes = args
        self.lib.fbf_field_image_f32.argtypes = args
        self.lib.fbf_voronoi_image_f32.restype = self.lib.fbf_field_image_f32.restype = None

    def image(self, generator: str, width: int, height: int, sites: int, noise: float, seed: int,
              threads: int = 0) -> np.ndarray:
        out = np.empty((height, width), dtype=np.float32)
        fn = self.lib.fbf_voronoi_image_f32 if generator == "voronoi" else self.lib.fbf_field_image_f32
        fn(width, height, sites, noise, seed, threads or os.cpu_count() or 1,
           out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        return out

    def make_frame(self, cfg, f: int = 0, threads: int = 0) -> np.ndarray:
        """configs.make_frame without libfbf.so (same source, same bits)."""
        return self.image(cfg.generator, cfg.width, cfg.height, cfg.sites, cfg.noise, cfg.frame_seed(f), threads)


def select_for_config(cfg, R: int = 255) -> "Report":
    """(K, T, c) of a BASELINE config by the optimiser restatement below, like the
    CLI's select_parameters (tools/fourierbf.cpp:185-234): eps -> Algorithm 1,
    fixed K -> best T over 1..10R then the fixed-period fit."""
    b = Oracle().range_samples("gaussian", cfg.sigma, R)
    if cfg.K is not None:
        T, e = min_error_over_period(cfg.K, b, 10 * R)
        c, _ = fit_coefficients(design_matrix(cfg.K, T, R), b)
        return Report(cfg.K, T, c, e)
    return optimize_parameters(b, cfg.eps)


# ---------------------------------------------------------------------------
# Optimiser restatement (approx.cpp:61-240) -- numpy / LAPACK.
# ---------------------------------------------------------------------------

def frequency_of(T: int) -> float:
    """approx.cpp:17-19."""
    return 2.0 * np.pi / (2.0 * T + 1.0)


def design_matrix(K: int, T: int, R: int) -> np.ndarray:
    """approx.cpp:61-86 -- Chebyshev recurrence on cos(nu t)."""
    if K < 1 or T < 1 or R < 1 or K > 2 * R + 1:
        raise ValueError("design_matrix: invalid arguments")
    nu = frequency_of(T)
    t = np.arange(-R, R + 1, dtype=np.float64)
    A = np.empty((2 * R + 1, K))
    A[:, 0] = 1.0
    if K > 1:
        c1 = np.cos(nu * t)
        A[:, 1] = c1
        for j in range(2, K):
            A[:, j] = 2.0 * c1 * A[:, j - 1] - A[:, j - 2]
    return A


def fit_coefficients(A: np.ndarray, b: np.ndarray):
    """approx.cpp:88-103 -- min-norm least squares, rank tolerance 1e-10."""
    if not (np.all(np.isfinite(A)) and np.all(np.isfinite(b))):
        raise RuntimeError("fit_coefficients: non-finite entries")
    c, *_ = np.linalg.lstsq(A, b, rcond=1e-10)
    r = A @ c - b
    return c, float(r @ r)


def scan_period_errors(K: int, b: np.ndarray, t_max: int) -> np.ndarray:
    """approx.cpp:119-130 -- E(K, T) for T = 1..t_max."""
    R = (len(b) - 1) // 2
    return np.array([fit_coefficients(design_matrix(K, T, R), b)[1] for T in range(1, t_max + 1)])


def min_error_over_period(K: int, b: np.ndarray, t_max: int):
    """approx.cpp:132-144 -- strict '<', ties keep the smaller T."""
    e = scan_period_errors(K, b, t_max)
    best_T, best_e = 1, e[0]
    for T in range(2, t_max + 1):
        if e[T - 1] < best_e:
            best_T, best_e = T, e[T - 1]
    return best_T, float(best_e)


@dataclass
class Report:
    K: int
    T: int
    coefficients: np.ndarray
    error: float
    per_order: list = field(default_factory=list)
    reached: bool = True


def optimize_parameters(b: np.ndarray, tol: float, t_max: int = 0, k_max: int = 0) -> Report:
    """approx.cpp:179-240 -- Algorithm 1 with k_cap = min(k_max, t_max + 1)."""
    R = (len(b) - 1) // 2
    t_max = t_max if t_max > 0 else 10 * R
    k_max = k_max if k_max > 0 else 2 * R + 1
    k_cap = min(k_max, t_max + 1)
    per = []
    for K in range(1, k_cap + 1):
        T, e = min_error_over_period(K, b, t_max)
        per.append((K, T, e))
        if e <= tol:
            c, _ = fit_coefficients(design_matrix(K, T, R), b)
            return Report(K, T, c, e, per, True)
    K, T, e = min(per, key=lambda p: p[2])
    c, _ = fit_coefficients(design_matrix(K, T, R), b)
    return Report(K, T, c, e, per, False)
