"""Python mirror of the reference fourierbf filtering interface (namespace fbf).

Same names, argument meaning and error behaviour as the reference C++ API, so
callers (and the parity tests) read like the reference's own code:

    kernel = build_spatial_kernel(5.0)                       # kernels.hpp:42-51
    samples = sample_range_kernel(RangeKernelSpec.gaussian(50.0, 255))
    approx = fit_fixed_period(samples, 4, 203)               # approx.hpp:61-64
    out = fast_bilateral(img, kernel, approx, BorderPolicy.symmetric, diag)
                                                             # filter.hpp:43-46

Everything numeric goes through libfbf.so (include/fbf.h): the optimiser runs
in C++ on the host, the filter runs the fused sm_100a kernel. There is no CPU
fallback; without a GPU the filter raises CudaError.

Error mapping (reference exception -> Python):
    std::invalid_argument        -> InvalidArgument (a ValueError)
    ToleranceUnreachable          -> ToleranceUnreachable (carries best_found)
    CUDA failures                 -> CudaError
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (FBF_ECAPACITY, FBF_ECUDA, FBF_EINVAL, FBF_ENOMEM, FBF_ERANGE, FBF_EUNREACHABLE,
                   FBF_OK)

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)


class FbfError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class CudaError(FbfError):
    pass


class ToleranceUnreachable(FbfError):
    """approx.hpp:97-103 -- raised with the best fit found."""

    def __init__(self, message: str, best_found: "OptimizationReport"):
        super().__init__(message)
        self.best_found = best_found


def _check(rc: int) -> None:
    if rc == FBF_OK:
        return
    msg = _lib.last_error()
    if rc in (FBF_EINVAL, FBF_ERANGE):
        raise InvalidArgument(msg)
    if rc == FBF_ECUDA:
        raise CudaError(msg)
    if rc == FBF_ENOMEM:
        raise MemoryError(msg)
    if rc == FBF_ECAPACITY:
        raise InvalidArgument(msg)
    raise FbfError(f"fbf error {rc}: {msg}")


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(_fp)


class BorderPolicy(enum.IntEnum):
    """image.hpp:38."""
    symmetric = 0
    replicate = 1
    zero = 2


def _border(b) -> int:
    if isinstance(b, str):
        return int(BorderPolicy[b])
    return int(b)


class RangeKernelKind(enum.IntEnum):
    """kernels.hpp:8 (parametric kinds; tabulated kernels enter as samples)."""
    gaussian = 0
    exponential = 1
    cauchy = 2


@dataclass
class RangeKernelSpec:
    """kernels.hpp:13-22."""
    kind: RangeKernelKind = RangeKernelKind.gaussian
    sigma: float = 0.0
    dynamic_range: int = 255

    @staticmethod
    def gaussian(sigma: float, dynamic_range: int = 255) -> "RangeKernelSpec":
        return RangeKernelSpec(RangeKernelKind.gaussian, sigma, dynamic_range)

    @staticmethod
    def exponential(sigma: float, dynamic_range: int = 255) -> "RangeKernelSpec":
        return RangeKernelSpec(RangeKernelKind.exponential, sigma, dynamic_range)

    @staticmethod
    def cauchy(sigma: float, dynamic_range: int = 255) -> "RangeKernelSpec":
        return RangeKernelSpec(RangeKernelKind.cauchy, sigma, dynamic_range)


@dataclass
class RangeKernelSamples:
    """kernels.hpp:26-33: values[t + R] = phi(t), t in -R..R."""
    dynamic_range: int
    values: np.ndarray

    def at(self, t: int) -> float:
        return float(self.values[t + self.dynamic_range])

    def lattice_size(self) -> int:
        return 2 * self.dynamic_range + 1


def sample_range_kernel(spec: RangeKernelSpec) -> RangeKernelSamples:
    """kernels.cpp:78-103."""
    R = int(spec.dynamic_range)
    v = np.zeros(2 * R + 1)
    _check(_lib.load().fbf_sample_range_kernel(int(spec.kind), float(spec.sigma), R, _dptr(v)))
    return RangeKernelSamples(R, v)


def tabulated_samples(values) -> RangeKernelSamples:
    """RangeKernelSpec::tabulated + sample_range_kernel (kernels.cpp:51-77, 86-95)."""
    v = np.asarray(values, dtype=np.float64)
    if v.size < 3 or v.size % 2 == 0:
        raise InvalidArgument("tabulated kernel: need an odd number of samples (2R+1), R >= 1")
    if not np.all(np.isfinite(v)):
        raise InvalidArgument("tabulated kernel: non-finite sample")
    R = v.size // 2
    if not v[R] > 0:
        raise InvalidArgument("tabulated kernel: center value must be positive")
    lo, hi = v[:R][::-1], v[R + 1:]
    if np.any(np.abs(lo - hi) > 1e-12):
        raise InvalidArgument("tabulated kernel: samples asymmetric beyond 1e-12")
    if np.any(lo > v[R]) or np.any(hi > v[R]):
        raise InvalidArgument("tabulated kernel: center must be the maximum")
    out = np.empty_like(v)
    out[R:] = v[R:]
    out[:R] = v[R + 1:][::-1]
    return RangeKernelSamples(R, out)


@dataclass
class SpatialKernel:
    """kernels.hpp:42-48."""
    theta: float
    radius: int
    taps: np.ndarray

    def tap(self, j: int) -> float:
        return float(self.taps[j + self.radius])


def build_spatial_kernel(theta: float) -> SpatialKernel:
    """kernels.cpp:105-118: radius ceil(3 theta), unnormalised taps."""
    cap = 2 * max(0, math.ceil(3.0 * theta)) + 1 if math.isfinite(theta) and theta > 0 else 1
    taps = np.zeros(cap)
    r = _lib.load().fbf_build_spatial_kernel(float(theta), _dptr(taps), cap)
    if r < 0:
        _check(-r)
    return SpatialKernel(float(theta), r, taps)


def frequency_of(half_period: int) -> float:
    return 2.0 * math.pi / (2.0 * half_period + 1.0)


@dataclass
class FourierApproximation:
    """approx.hpp:14-22: phihat(t) = sum_k c_k cos(nu k t), nu = 2 pi / (2T+1)."""
    terms: int = 0
    half_period: int = 0
    dynamic_range: int = 0
    frequency: float = 0.0
    coefficients: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def evaluate(self, t: int) -> float:
        """approx.cpp:34-42."""
        base = self.frequency * abs(t)
        s = 0.0
        for k in range(self.terms):
            s += float(self.coefficients[k]) * math.cos(base * k)
        return s


def tabulate_approximation(approx: FourierApproximation) -> RangeKernelSamples:
    """approx.cpp:48-59."""
    R = approx.dynamic_range
    v = np.zeros(2 * R + 1)
    for t in range(R + 1):
        e = approx.evaluate(t)
        v[R + t] = e
        v[R - t] = e
    return RangeKernelSamples(R, v)


def _approx(K: int, T: int, R: int, c: np.ndarray) -> FourierApproximation:
    return FourierApproximation(K, T, R, frequency_of(T), np.array(c[:K], dtype=np.float64))


def fit_fixed_period(samples: RangeKernelSamples, terms: int, half_period: int) -> FourierApproximation:
    """approx.cpp:105-117."""
    c = np.zeros(max(1, terms))
    err = ctypes.c_double(0)
    _check(_lib.load().fbf_fit_fixed_period(_dptr(samples.values), samples.dynamic_range, terms,
                                            half_period, _dptr(c), ctypes.byref(err)))
    return _approx(terms, half_period, samples.dynamic_range, c)


def fit_error(samples: RangeKernelSamples, terms: int, half_period: int) -> float:
    """||A c - b||^2 of the fixed-period fit (FitResult::error, approx.hpp:37-40)."""
    c = np.zeros(max(1, terms))
    err = ctypes.c_double(0)
    _check(_lib.load().fbf_fit_fixed_period(_dptr(samples.values), samples.dynamic_range, terms,
                                            half_period, _dptr(c), ctypes.byref(err)))
    return err.value


def scan_period_errors(terms: int, samples: RangeKernelSamples, t_max: int, threads: int = 1) -> np.ndarray:
    """approx.cpp:119-130: result[T-1] = E(K, T)."""
    e = np.zeros(max(1, t_max))
    _check(_lib.load().fbf_scan_period_errors(_dptr(samples.values), samples.dynamic_range, terms, t_max,
                                              threads, _dptr(e)))
    return e


@dataclass
class PeriodScanResult:
    best_half_period: int
    best_error: float


def scan_period_errors_gpu(samples: RangeKernelSamples, k_lo: int, n_orders: int, t_max: int,
                           device: int = 0) -> np.ndarray:
    """E(K, T) for K in [k_lo, k_lo + n_orders), T in 1..t_max on the GPU
    (fbf_scan.cu); shape (n_orders, t_max). ~1e-15 relative to scan_period_errors
    near the minimum."""
    e = np.zeros((max(1, n_orders), max(1, t_max)))
    _check(_lib.load().fbf_scan_period_errors_gpu(_dptr(samples.values), samples.dynamic_range, k_lo, n_orders,
                                                  t_max, device, _dptr(e)))
    return e


def scan_gpu_max_order(dynamic_range: int = 255) -> int:
    return int(_lib.load().fbf_scan_gpu_max_order(dynamic_range))


def min_error_over_period(terms: int, samples: RangeKernelSamples, t_max: int,
                          threads: int = 1, device: int | None = None) -> PeriodScanResult:
    """approx.cpp:132-144 (device: GPU scan + exact host re-check, same result)."""
    T = ctypes.c_int(0)
    e = ctypes.c_double(0)
    lib = _lib.load()
    if device is None:
        rc = lib.fbf_min_error_over_period(_dptr(samples.values), samples.dynamic_range, terms, t_max,
                                           threads, ctypes.byref(T), ctypes.byref(e))
    else:
        rc = lib.fbf_min_error_over_period_gpu(_dptr(samples.values), samples.dynamic_range, terms, t_max,
                                               int(device), ctypes.byref(T), ctypes.byref(e))
    _check(rc)
    return PeriodScanResult(T.value, e.value)


@dataclass
class PerOrderError:
    terms: int
    best_half_period: int
    best_error: float


@dataclass
class OptimizeOptions:
    """approx.hpp:90-95."""
    t_max: int = 0
    k_max: int = 0
    threads: int = 1
    device: int | None = None  # B200 extension: period scans on this CUDA device (fbf_scan.cu)


@dataclass
class OptimizationReport:
    """approx.hpp:74-88."""
    best_terms: int
    best_half_period: int
    coefficients: np.ndarray
    achieved_error: float
    tolerance: float
    t_max: int
    per_order: list

    def approximation(self, dynamic_range: int) -> FourierApproximation:
        return _approx(self.best_terms, self.best_half_period, dynamic_range, self.coefficients)


def optimize_parameters(samples: RangeKernelSamples, tolerance: float,
                        options: OptimizeOptions | None = None) -> OptimizationReport:
    """approx.cpp:179-240 (Algorithm 1)."""
    o = options or OptimizeOptions()
    R = samples.dynamic_range
    t_max = o.t_max if o.t_max > 0 else 10 * R
    k_cap = min(o.k_max if o.k_max > 0 else 2 * R + 1, t_max + 1)
    cap = max(1, k_cap)
    c = np.zeros(cap)
    per = np.zeros(3 * cap)
    K, T, n = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(0)
    e = ctypes.c_double(0)
    lib = _lib.load()
    if o.device is None:
        rc = lib.fbf_optimize_parameters(_dptr(samples.values), R, float(tolerance), o.t_max, o.k_max,
                                         o.threads, ctypes.byref(K), ctypes.byref(T), _dptr(c), cap,
                                         ctypes.byref(e), _dptr(per), ctypes.byref(n))
    else:
        rc = lib.fbf_optimize_parameters_gpu(_dptr(samples.values), R, float(tolerance), o.t_max, o.k_max,
                                             int(o.device), ctypes.byref(K), ctypes.byref(T), _dptr(c), cap,
                                             ctypes.byref(e), _dptr(per), ctypes.byref(n))
    if rc not in (FBF_OK, FBF_EUNREACHABLE):
        _check(rc)
    orders = [PerOrderError(int(per[3 * i]), int(per[3 * i + 1]), float(per[3 * i + 2])) for i in range(n.value)]
    rep = OptimizationReport(K.value, T.value, c[:K.value].copy(), e.value, float(tolerance), t_max, orders)
    if rc == FBF_EUNREACHABLE:
        raise ToleranceUnreachable(_lib.last_error(), rep)
    return rep


def select_parameters(sigma: float, *, eps: float | None = None, K: int | None = None, T: int | None = None,
                      method: str = "fast", kernel: str = "gaussian", dynamic_range: int = 255,
                      threads: int = 1, device: int | None = None) -> FourierApproximation:
    """CLI select_parameters (tools/fourierbf.cpp:185-234). device: run the
    period scans on that CUDA device (same K, T and coefficients as the host
    scan: near-minimal T are re-fitted on the host)."""
    R = dynamic_range
    c = np.zeros(2 * R + 1)
    Ko, To = ctypes.c_int(0), ctypes.c_int(0)
    e = ctypes.c_double(0)
    lib = _lib.load()
    head = (int(RangeKernelKind[kernel]), float(sigma), R, float(eps or 0.0), int(K or 0), int(T or 0),
            int(method == "fbf"))
    tail = (ctypes.byref(Ko), ctypes.byref(To), _dptr(c), c.size, ctypes.byref(e))
    if device is None:
        rc = lib.fbf_select_params(*head, threads, *tail)
    else:
        rc = lib.fbf_select_params_gpu(*head, int(device), *tail)
    if rc == FBF_EUNREACHABLE:
        rep = OptimizationReport(Ko.value, To.value, c[:Ko.value].copy(), e.value, float(eps or 0), 10 * R, [])
        raise ToleranceUnreachable(_lib.last_error(), rep)
    _check(rc)
    return _approx(Ko.value, To.value, R, c)


@dataclass
class FilterDiagnostics:
    """filter.hpp:15-17."""
    fallback_pixels: int = 0


class _StageTimingsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("fit_seconds", "auxiliary_seconds", "convolution_seconds",
                                                "combine_seconds", "h2d_seconds", "d2h_seconds", "wall_seconds")]


@dataclass
class StageTimings:
    """filter.hpp:19-24, accumulated like filter.cpp:151-211. The fused kernel's
    device time is convolution_seconds (channel generation and the combine run
    inside it, so auxiliary_seconds and combine_seconds stay 0); h2d / d2h /
    wall are the host-buffer call's copy busy times and wall time."""
    fit_seconds: float = 0.0
    auxiliary_seconds: float = 0.0
    convolution_seconds: float = 0.0
    combine_seconds: float = 0.0
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    wall_seconds: float = 0.0


def _as_image(img) -> np.ndarray:
    a = np.asarray(img)
    if a.ndim != 2:
        raise InvalidArgument("GrayImage: expected a 2-D (height, width) array")
    return np.ascontiguousarray(a, dtype=np.float32)


def _approx_args(approx: FourierApproximation):
    if approx.terms < 1 or len(approx.coefficients) != approx.terms:
        raise InvalidArgument("fast_bilateral: malformed approximation")
    return np.ascontiguousarray(approx.coefficients, dtype=np.float64)


def fast_bilateral(img, kernel: SpatialKernel, approx: FourierApproximation,
                   border=BorderPolicy.symmetric, diag: FilterDiagnostics | None = None,
                   out: np.ndarray | None = None, timings: StageTimings | None = None) -> np.ndarray:
    """filter.hpp:43-46 / filter.cpp:129-213 on the GPU (host buffers in, host buffer out).

    approx.frequency is used as given (filter.cpp:139; 0 = frequency_of(T)).
    `out` (optional) is a caller-owned float32 (H, W) C-contiguous array, e.g.
    a view of pinned memory, written in place. `timings` (optional) accumulates
    the stage times (StageTimings).
    """
    a = _as_image(img)
    c = _approx_args(approx)
    if out is None:
        out = np.empty_like(a)
    elif out.dtype != np.float32 or out.shape != a.shape or not out.flags.c_contiguous:
        raise InvalidArgument("out must be a C-contiguous float32 array of the image shape")
    fb = ctypes.c_longlong(0)
    st = _StageTimingsC() if timings is not None else None
    _check(_lib.load().fbf_fast_bilateral_ex(_fptr(a), a.shape[1], a.shape[0], kernel.theta, approx.terms,
                                             approx.half_period, approx.dynamic_range, float(approx.frequency),
                                             _dptr(c), _border(border), _fptr(out), ctypes.byref(fb),
                                             ctypes.byref(st) if st is not None else None))
    if diag is not None:
        diag.fallback_pixels += fb.value
    if timings is not None:
        for name, _ in _StageTimingsC._fields_:
            setattr(timings, name, getattr(timings, name) + getattr(st, name))
    return out


def fast_bilateral_u8(img, kernel: SpatialKernel, approx: FourierApproximation,
                      border=BorderPolicy.symmetric, diag: FilterDiagnostics | None = None,
                      out_dtype=np.uint8, out: np.ndarray | None = None) -> np.ndarray:
    """fast_bilateral on an 8-bit image (a PGM payload): 1 byte per pixel crosses
    PCIe. out_dtype uint8: clamped to [0,255] and rounded half away from zero
    on the device (the CLI's write_clamped + write_pgm); float32: the float result."""
    a = np.ascontiguousarray(img, dtype=np.uint8)
    if a.ndim != 2:
        raise InvalidArgument("GrayImage: expected a 2-D (height, width) array")
    c = _approx_args(approx)
    if out is None:
        out = np.empty(a.shape, dtype=np.dtype(out_dtype))  # pass a pinned `out` for full PCIe rate
    elif out.shape != a.shape or not out.flags.c_contiguous:
        raise InvalidArgument("fast_bilateral_u8: out must be C-contiguous with the image shape")
    if out.dtype not in (np.uint8, np.float32):
        raise InvalidArgument("fast_bilateral_u8: out_dtype must be uint8 or float32")
    fb = ctypes.c_longlong(0)
    o8 = ctypes.c_void_p(out.ctypes.data) if out.dtype == np.uint8 else None
    o32 = ctypes.c_void_p(out.ctypes.data) if out.dtype == np.float32 else None
    _check(_lib.load().fbf_fast_bilateral_u8(ctypes.c_void_p(a.ctypes.data), a.shape[1], a.shape[0],
                                             kernel.theta, approx.terms, approx.half_period, approx.dynamic_range,
                                             _dptr(c), _border(border), o8, o32, ctypes.byref(fb)))
    if diag is not None:
        diag.fallback_pixels += fb.value
    return out


def fast_bilateral_batch(frames, kernel: SpatialKernel, approx: FourierApproximation,
                         border=BorderPolicy.symmetric, diag: FilterDiagnostics | None = None,
                         n_gpus: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """Independent frames (n, height, width), sharded over n_gpus devices (0 = all;
    1 = the default device), pipelined per device (H2D / kernel / D2H overlap)."""
    a = np.ascontiguousarray(np.asarray(frames), dtype=np.float32)
    if a.ndim != 3:
        raise InvalidArgument("batch: expected (n_frames, height, width)")
    c = _approx_args(approx)
    if out is None:
        out = np.empty_like(a)
    elif out.shape != a.shape or out.dtype != np.float32 or not out.flags.c_contiguous:
        raise InvalidArgument("batch: out must be a C-contiguous float32 array of the input's shape")
    fb = ctypes.c_longlong(0)
    _check(_lib.load().fbf_fast_bilateral_batch_f32(_fptr(a), a.shape[0], a.shape[2], a.shape[1], kernel.theta,
                                                    approx.terms, approx.half_period, approx.dynamic_range,
                                                    _dptr(c), _border(border), _fptr(out), ctypes.byref(fb),
                                                    n_gpus))
    if diag is not None:
        diag.fallback_pixels += fb.value
    return out


def fast_bilateral_bands(img, kernel: SpatialKernel, approx: FourierApproximation,
                         border=BorderPolicy.symmetric, diag: FilterDiagnostics | None = None,
                         n_gpus: int = 0) -> np.ndarray:
    """One image split into row bands with replicated halos over n_gpus devices."""
    a = _as_image(img)
    c = _approx_args(approx)
    out = np.empty_like(a)
    fb = ctypes.c_longlong(0)
    _check(_lib.load().fbf_fast_bilateral_bands_f32(_fptr(a), a.shape[1], a.shape[0], kernel.theta, approx.terms,
                                                    approx.half_period, approx.dynamic_range, _dptr(c),
                                                    _border(border), _fptr(out), ctypes.byref(fb), n_gpus))
    if diag is not None:
        diag.fallback_pixels += fb.value
    return out


def fast_bilateral_band(src, src_row0: int, height: int, out_row0: int, out_rows: int, kernel: SpatialKernel,
                        approx: FourierApproximation, border=BorderPolicy.symmetric,
                        diag: FilterDiagnostics | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """One rank's row band from host buffers (one process per GPU): `src` holds global rows
    [src_row0, src_row0 + src.shape[0]) of a (height, W) image -- the band plus the halo of
    band_source_rows() -- and the result is output rows [out_row0, out_row0 + out_rows),
    bit-identical to the same rows of fast_bilateral on the whole image. Runs on the default
    device (set_device) with the single-image call's H2D / kernel / D2H pipeline."""
    a = _as_image(src)
    c = _approx_args(approx)
    W = a.shape[1]
    if out is None:
        out = np.empty((out_rows, W), dtype=np.float32)
    elif out.dtype != np.float32 or not out.flags.c_contiguous or out.shape != (out_rows, W):
        raise InvalidArgument("out must be a C-contiguous float32 array of shape (out_rows, width)")
    fb = ctypes.c_longlong(0)
    _check(_lib.load().fbf_fast_bilateral_band_f32(_fptr(a), src_row0, a.shape[0], W, height, out_row0, out_rows,
                                                   kernel.theta, approx.terms, approx.half_period,
                                                   approx.dynamic_range, _dptr(c), _border(border), _fptr(out),
                                                   ctypes.byref(fb)))
    if diag is not None:
        diag.fallback_pixels += fb.value
    return out


def band_source_rows(height: int, out_row0: int, out_rows: int, theta: float,
                     border=BorderPolicy.symmetric) -> tuple[int, int]:
    """Global source-row window [row0, row0 + rows) a band needs (halo included)."""
    r0, n = ctypes.c_int(0), ctypes.c_int(0)
    _check(_lib.load().fbf_band_source_rows(height, out_row0, out_rows, float(theta), _border(border),
                                            ctypes.byref(r0), ctypes.byref(n)))
    return r0.value, n.value


def _check_device_tensor(t, what: str, shape, device, dtype=None) -> None:
    """A device buffer handed to the kernel as a raw pointer: contiguous, of the
    expected dtype (float32 by default) and shape, on the input's device."""
    import torch
    dtype = dtype or torch.float32
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidArgument(f"{what} must be a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise InvalidArgument(f"{what} must be a contiguous {dtype} CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise InvalidArgument(f"{what} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.device != device:
        raise InvalidArgument(f"{what} is on {t.device}, the input on {device}")


def _check_fallbacks(d_fallbacks, device) -> None:
    import torch
    if d_fallbacks is None:
        return
    if (not isinstance(d_fallbacks, torch.Tensor) or not d_fallbacks.is_cuda or d_fallbacks.device != device
            or d_fallbacks.dtype not in (torch.int64, torch.uint64) or d_fallbacks.numel() < 1):
        raise InvalidArgument("d_fallbacks must be a 64-bit integer CUDA tensor on the input's device")


def fast_bilateral_device(d_img, kernel: SpatialKernel, approx: FourierApproximation, d_out,
                          border=BorderPolicy.symmetric, d_fallbacks=None, stream=None) -> None:
    """Device-resident variant on torch CUDA tensors (float32, contiguous, (H, W)).

    Enqueued on `stream` (a torch.cuda.Stream; default: torch's current stream)
    without synchronising. No intensity validation (see validate_device).
    """
    import torch
    if not isinstance(d_img, torch.Tensor) or d_img.dim() != 2:
        raise InvalidArgument("device image must be a 2-D (H, W) CUDA tensor")
    _check_device_tensor(d_img, "device image", d_img.shape, d_img.device)
    _check_device_tensor(d_out, "d_out", d_img.shape, d_img.device)
    _check_fallbacks(d_fallbacks, d_img.device)
    H, W = d_img.shape
    c = _approx_args(approx)
    st = stream if stream is not None else torch.cuda.current_stream(d_img.device)
    _check(_lib.load().fbf_fast_bilateral_f32_device(
        ctypes.c_void_p(d_img.data_ptr()), W, H, kernel.theta, approx.terms, approx.half_period,
        approx.dynamic_range, _dptr(c), _border(border), ctypes.c_void_p(d_out.data_ptr()),
        ctypes.c_void_p(d_fallbacks.data_ptr() if d_fallbacks is not None else 0), d_img.device.index,
        ctypes.c_void_p(st.cuda_stream)))


def fast_bilateral_batch_device(d_frames, kernel: SpatialKernel, approx: FourierApproximation, d_out,
                                border=BorderPolicy.symmetric, d_fallbacks=None, stream=None) -> None:
    """Device-resident batch (n_frames, H, W) float32 CUDA tensors, one launch."""
    import torch
    if not isinstance(d_frames, torch.Tensor) or d_frames.dim() != 3:
        raise InvalidArgument("device frames must be a contiguous (n, H, W) float32 CUDA tensor")
    _check_device_tensor(d_frames, "device frames", d_frames.shape, d_frames.device)
    _check_device_tensor(d_out, "d_out", d_frames.shape, d_frames.device)
    _check_fallbacks(d_fallbacks, d_frames.device)
    n, H, W = d_frames.shape
    c = _approx_args(approx)
    st = stream if stream is not None else torch.cuda.current_stream(d_frames.device)
    _check(_lib.load().fbf_fast_bilateral_batch_f32_device(
        ctypes.c_void_p(d_frames.data_ptr()), n, W, H, kernel.theta, approx.terms, approx.half_period,
        approx.dynamic_range, _dptr(c), _border(border), ctypes.c_void_p(d_out.data_ptr()),
        ctypes.c_void_p(d_fallbacks.data_ptr() if d_fallbacks is not None else 0), d_frames.device.index,
        ctypes.c_void_p(st.cuda_stream)))


def fast_bilateral_band_device(d_src, src_row0: int, height: int, out_row0: int, out_rows: int,
                               kernel: SpatialKernel, approx: FourierApproximation, d_dst,
                               border=BorderPolicy.symmetric, d_fallbacks=None, stream=None) -> None:
    """One rank's band: d_src holds global rows [src_row0, src_row0 + d_src.shape[0]);
    d_dst (out_rows, W) receives output rows [out_row0, out_row0 + out_rows)."""
    import torch
    if not isinstance(d_src, torch.Tensor) or d_src.dim() != 2:
        raise InvalidArgument("band source must be a 2-D (rows, W) CUDA tensor")
    _check_device_tensor(d_src, "band source", d_src.shape, d_src.device)
    rows, W = d_src.shape
    _check_device_tensor(d_dst, "d_dst", (out_rows, W), d_src.device)
    _check_fallbacks(d_fallbacks, d_src.device)
    c = _approx_args(approx)
    st = stream if stream is not None else torch.cuda.current_stream(d_src.device)
    _check(_lib.load().fbf_fast_bilateral_band_f32_device(
        ctypes.c_void_p(d_src.data_ptr()), src_row0, rows, W, height, out_row0, out_rows, kernel.theta,
        approx.terms, approx.half_period, approx.dynamic_range, _dptr(c), _border(border),
        ctypes.c_void_p(d_dst.data_ptr()),
        ctypes.c_void_p(d_fallbacks.data_ptr() if d_fallbacks is not None else 0), d_src.device.index,
        ctypes.c_void_p(st.cuda_stream)))


def validate_device(d_img, dynamic_range: int = 255, stream=None) -> None:
    """validate_intensities (filter.cpp:19-23) on a device tensor."""
    import torch
    _check_device_tensor(d_img, "validate_device input", d_img.shape, d_img.device)
    st = stream if stream is not None else torch.cuda.current_stream(d_img.device)
    _check(_lib.load().fbf_validate_f32_device(ctypes.c_void_p(d_img.data_ptr()), d_img.numel(), dynamic_range,
                                               d_img.device.index, ctypes.c_void_p(st.cuda_stream)))


def fbf_filter(img, theta: float, sigma: float, eps_or_K: float) -> np.ndarray:
    """North-star convenience call fbf_filter(img, H, W, theta, sigma, eps/K, out)."""
    a = _as_image(img)
    out = np.empty_like(a)
    _check(_lib.load().fbf_filter(_fptr(a), a.shape[0], a.shape[1], float(theta), float(sigma), float(eps_or_K),
                                  _fptr(out)))
    return out


class _PinnedBlock:
    """Owner of one fbf_host_alloc block (freed with the last array view)."""

    def __init__(self, nbytes: int):
        self.ptr = ctypes.c_void_p(0)
        _check(_lib.load().fbf_host_alloc(nbytes, ctypes.byref(self.ptr)))

    def __del__(self):
        if self.ptr and _lib._lib is not None:
            _lib._lib.fbf_host_free(self.ptr)
            self.ptr = ctypes.c_void_p(0)


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """numpy array in page-locked host memory (fbf_host_alloc): the host-buffer
    calls move these over PCIe at the copy-engine rate."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    blk = _PinnedBlock(max(n, 1))
    buf = (ctypes.c_char * max(n, 1)).from_address(blk.ptr.value)
    buf._fbf_owner = blk  # keeps the block alive as long as any view of buf
    return np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)


# ---- brute filter and metrics (filter.cpp:83-127, metrics.hpp) --------------

def brute_bilateral(img, kernel: SpatialKernel, range_samples: RangeKernelSamples,
                    border=BorderPolicy.symmetric, diag: FilterDiagnostics | None = None) -> np.ndarray:
    """filter.hpp:35-38 / filter.cpp:83-127 on the GPU: FP64 output equal to the
    reference's brute_bilateral bit for bit on float32 inputs (fbf_brute.cu)."""
    a = _as_image(img)
    out = np.empty(a.shape, dtype=np.float64)
    fb = ctypes.c_longlong(0)
    _check(_lib.load().fbf_brute_bilateral_f32(_fptr(a), a.shape[1], a.shape[0], float(kernel.theta),
                                               _dptr(np.ascontiguousarray(range_samples.values, dtype=np.float64)),
                                               range_samples.dynamic_range, _border(border), _dptr(out),
                                               ctypes.byref(fb)))
    if diag is not None:
        diag.fallback_pixels += fb.value
    return out


def brute_bilateral_device(d_img, kernel: SpatialKernel, range_samples: RangeKernelSamples, d_out,
                           border=BorderPolicy.symmetric, d_fallbacks=None, stream=None) -> None:
    """Device-resident brute filter: d_img float32 (H, W), d_out float64 (H, W) CUDA tensors."""
    import torch
    if not isinstance(d_img, torch.Tensor) or d_img.dim() != 2:
        raise InvalidArgument("brute_bilateral_device: float32 (H, W) input tensor")
    _check_device_tensor(d_img, "brute_bilateral_device input", d_img.shape, d_img.device)
    _check_device_tensor(d_out, "brute_bilateral_device output", d_img.shape, d_img.device, torch.float64)
    _check_fallbacks(d_fallbacks, d_img.device)
    H, W = d_img.shape
    st = stream if stream is not None else torch.cuda.current_stream(d_img.device)
    _check(_lib.load().fbf_brute_bilateral_f32_device(
        ctypes.c_void_p(d_img.data_ptr()), W, H, float(kernel.theta),
        _dptr(np.ascontiguousarray(range_samples.values, dtype=np.float64)), range_samples.dynamic_range,
        _border(border), ctypes.c_void_p(d_out.data_ptr()),
        ctypes.c_void_p(d_fallbacks.data_ptr() if d_fallbacks is not None else 0), d_img.device.index,
        ctypes.c_void_p(st.cuda_stream)))


@dataclass
class ImageDelta:
    """metrics.hpp:11-15."""
    mse: float = 0.0
    psnr_db: float = 0.0
    max_abs_err: float = 0.0


def compare_images(a, b) -> ImageDelta:
    """metrics.cpp:10-26 on host arrays."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise InvalidArgument("compare_images: dimension mismatch")
    d = a - b
    mse = float(np.sum(d * d) / d.size)
    psnr = 10.0 * math.log10(255.0 * 255.0 / mse) if mse > 0 else math.inf
    return ImageDelta(mse, psnr, float(np.max(np.abs(d))) if d.size else 0.0)


def compare_images_device(d_ref, d_cand, stream=None) -> ImageDelta:
    """compare_images of a float64 reference and a float32 candidate CUDA tensor
    (full-size accuracy check without a host round trip)."""
    import torch
    if d_ref.shape != d_cand.shape:
        raise InvalidArgument("compare_images: dimension mismatch")
    _check_device_tensor(d_ref, "compare_images reference", d_ref.shape, d_ref.device, torch.float64)
    _check_device_tensor(d_cand, "compare_images candidate", d_ref.shape, d_ref.device)
    st = stream if stream is not None else torch.cuda.current_stream(d_ref.device)
    mse, psnr, mx = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
    _check(_lib.load().fbf_compare_images_device(ctypes.c_void_p(d_ref.data_ptr()), ctypes.c_void_p(d_cand.data_ptr()),
                                                 d_ref.numel(), ctypes.byref(mse), ctypes.byref(psnr),
                                                 ctypes.byref(mx), d_ref.device.index,
                                                 ctypes.c_void_p(st.cuda_stream)))
    return ImageDelta(mse.value, psnr.value, mx.value)


def prop1_bound(eps: float, dynamic_range: int, omega0: float = 1.0) -> float:
    """metrics.cpp:28-32: 2 R eps / (omega0 - eps)."""
    if not (eps > 0.0) or not (eps < omega0):
        raise InvalidArgument("prop1_bound: requires 0 < eps < omega(0)")
    return 2.0 * dynamic_range * eps / (omega0 - eps)


def kernel_error(samples: RangeKernelSamples, approx: FourierApproximation) -> float:
    """metrics.cpp:34-44: sum_t (phi(t) - phihat(t))^2."""
    if samples.dynamic_range != approx.dynamic_range:
        raise InvalidArgument("kernel_error: dynamic range mismatch")
    R = samples.dynamic_range
    s = 0.0
    for t in range(-R, R + 1):
        d = samples.at(t) - approx.evaluate(t)
        s += d * d
    return s


@dataclass
class ComparisonResult:
    """metrics.hpp:30-43."""
    mse: float = 0.0
    psnr_db: float = 0.0
    max_abs_err: float = 0.0
    prop1_bound: float = 0.0
    bound_satisfied: bool = False

    @staticmethod
    def csv_header() -> str:
        return "mse,psnr_db,max_abs_err,prop1_bound,bound_satisfied"

    def to_csv(self) -> str:
        psnr = "inf" if math.isinf(self.psnr_db) else f"{self.psnr_db:.17g}"
        return (f"{self.mse:.17g},{psnr},{self.max_abs_err:.17g},{self.prop1_bound:.17g},"
                f"{'true' if self.bound_satisfied else 'false'}")


def compare_with_bound(reference, candidate, achieved_kernel_error: float, dynamic_range: int,
                       omega0: float = 1.0) -> ComparisonResult:
    """metrics.cpp:58-70 (host arrays, or a float64/float32 CUDA tensor pair)."""
    if hasattr(reference, "is_cuda") and reference.is_cuda:
        d = compare_images_device(reference, candidate)
    else:
        d = compare_images(reference, candidate)
    b = prop1_bound(achieved_kernel_error, dynamic_range, omega0)
    return ComparisonResult(d.mse, d.psnr_db, d.max_abs_err, b, d.max_abs_err <= b)


# ---- synthetic inputs (synthetic.cpp + BASELINE.json generators) ----------

def random_image(width: int, height: int, seed: int) -> np.ndarray:
    out = np.empty((height, width), dtype=np.float32)
    _lib.load().fbf_random_image_f32(width, height, seed, _fptr(out))
    return out


def scene_image(width: int, height: int, seed: int) -> np.ndarray:
    out = np.empty((height, width), dtype=np.float32)
    _lib.load().fbf_scene_image_f32(width, height, seed, _fptr(out))
    return out


def voronoi_image(width: int, height: int, n_sites: int, noise: float, seed: int, threads: int = 0) -> np.ndarray:
    import os
    out = np.empty((height, width), dtype=np.float32)
    _lib.load().fbf_voronoi_image_f32(width, height, n_sites, noise, seed, threads or os.cpu_count() or 1,
                                      _fptr(out))
    return out


def field_image(width: int, height: int, n_sites: int, noise: float, seed: int, threads: int = 0) -> np.ndarray:
    import os
    out = np.empty((height, width), dtype=np.float32)
    _lib.load().fbf_field_image_f32(width, height, n_sites, noise, seed, threads or os.cpu_count() or 1,
                                    _fptr(out))
    return out
