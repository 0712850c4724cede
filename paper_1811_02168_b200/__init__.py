"""B200-native Fourier bilateral filtering stage (arXiv 1811.02168).

Drop-in for the reference fourierbf library's filtering path: the C ABI in
include/fbf.h (libfbf.so, host C++ + one fused sm_100a CUDA kernel) and this
Python mirror of the reference's fbf:: interface.
"""
from .fbf import (BorderPolicy, ComparisonResult, ImageDelta, brute_bilateral, brute_bilateral_device,
                  compare_images, compare_images_device, compare_with_bound, kernel_error, prop1_bound,
                  CudaError, FbfError, FilterDiagnostics, FourierApproximation, StageTimings,
                  InvalidArgument, OptimizationReport, OptimizeOptions, PerOrderError, PeriodScanResult,
                  RangeKernelKind, RangeKernelSamples, RangeKernelSpec, SpatialKernel, ToleranceUnreachable,
                  band_source_rows, build_spatial_kernel, fast_bilateral, fast_bilateral_band_device,
                  fast_bilateral_band, fast_bilateral_bands, fast_bilateral_batch, fast_bilateral_batch_device, fast_bilateral_u8, pinned_empty, fast_bilateral_device, fbf_filter, field_image,
                  fit_error, fit_fixed_period, frequency_of, min_error_over_period, optimize_parameters,
                  random_image, sample_range_kernel, scan_gpu_max_order, scan_period_errors, scan_period_errors_gpu,
                  scene_image, select_parameters,
                  tabulate_approximation, tabulated_samples, validate_device, voronoi_image)

__all__ = [n for n in dir() if not n.startswith("_")]
