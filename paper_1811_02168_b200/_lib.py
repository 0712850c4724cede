"""ctypes binding of libfbf.so (the C ABI declared in include/fbf.h).

The library is built in-tree by ``paper_1811_02168_b200.build``. There is no
CPU fallback for the filter: if the shared object is missing this module
raises, and the filter entry points return FBF_ECUDA when no GPU is visible.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FBF_LIB") or os.path.join(HERE, "libfbf.so")  # FBF_LIB: dev builds

FBF_OK = 0
FBF_EINVAL = 1
FBF_ERANGE = 2
FBF_EUNREACHABLE = 3
FBF_ECUDA = 4
FBF_ENOMEM = 5
FBF_ECAPACITY = 6
FBF_MAX_RADIUS = 32

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int)
_llp = ctypes.POINTER(ctypes.c_longlong)
_ullp = ctypes.c_void_p
_i, _d, _vp = ctypes.c_int, ctypes.c_double, ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/fbf.h
SIGNATURES = {
    "fbf_last_error": (ctypes.c_char_p, []),
    "fbf_device_count": (_i, []),
    "fbf_set_device": (_i, [_i]),
    "fbf_get_device": (_i, []),
    "fbf_kernel_launches": (ctypes.c_ulonglong, []),
    "fbf_host_alloc": (_i, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "fbf_host_free": (_i, [_vp]),
    "fbf_build_spatial_kernel": (_i, [_d, _dp, _i]),
    "fbf_sample_range_kernel": (_i, [_i, _d, _i, _dp]),
    "fbf_frequency_of": (_d, [_i]),
    "fbf_fit_fixed_period": (_i, [_dp, _i, _i, _i, _dp, _dp]),
    "fbf_scan_period_errors": (_i, [_dp, _i, _i, _i, _i, _dp]),
    "fbf_min_error_over_period": (_i, [_dp, _i, _i, _i, _i, _ip, _dp]),
    "fbf_optimize_parameters": (_i, [_dp, _i, _d, _i, _i, _i, _ip, _ip, _dp, _i, _dp, _dp, _ip]),
    "fbf_select_params": (_i, [_i, _d, _i, _d, _i, _i, _i, _i, _ip, _ip, _dp, _i, _dp]),
    "fbf_scan_period_errors_gpu": (_i, [_dp, _i, _i, _i, _i, _i, _dp]),
    "fbf_scan_gpu_max_order": (_i, [_i]),
    "fbf_min_error_over_period_gpu": (_i, [_dp, _i, _i, _i, _i, _ip, _dp]),
    "fbf_optimize_parameters_gpu": (_i, [_dp, _i, _d, _i, _i, _i, _ip, _ip, _dp, _i, _dp, _dp, _ip]),
    "fbf_select_params_gpu": (_i, [_i, _d, _i, _d, _i, _i, _i, _i, _ip, _ip, _dp, _i, _dp]),
    "fbf_build_lut": (_i, [_dp, _i, _dp, _i, _i, _i, _i, _i, _ip, _ip]),
    "fbf_query_lut": (_i, [_dp, _i, _dp, _i, _ip, _ip, _d, _d, _ip, _ip]),
    "fbf_fast_bilateral_f32": (_i, [_fp, _i, _i, _d, _i, _i, _i, _dp, _i, _fp, _llp]),
    "fbf_fast_bilateral_ex": (_i, [_fp, _i, _i, _d, _i, _i, _i, _d, _dp, _i, _fp, _llp, _vp]),
    "fbf_fast_bilateral_f32_device": (_i, [_vp, _i, _i, _d, _i, _i, _i, _dp, _i, _vp, _vp, _i, _vp]),
    "fbf_fast_bilateral_batch_f32_device": (_i, [_vp, _i, _i, _i, _d, _i, _i, _i, _dp, _i, _vp, _vp, _i, _vp]),
    "fbf_fast_bilateral_batch_f32": (_i, [_fp, _i, _i, _i, _d, _i, _i, _i, _dp, _i, _fp, _llp, _i]),
    "fbf_fast_bilateral_bands_f32": (_i, [_fp, _i, _i, _d, _i, _i, _i, _dp, _i, _fp, _llp, _i]),
    "fbf_fast_bilateral_band_f32": (_i, [_fp, _i, _i, _i, _i, _i, _i, _d, _i, _i, _i, _dp, _i, _fp, _llp]),
    "fbf_fast_bilateral_band_f32_device": (_i, [_vp, _i, _i, _i, _i, _i, _i, _d, _i, _i, _i, _dp, _i,
                                                _vp, _vp, _i, _vp]),
    "fbf_band_source_rows": (_i, [_i, _i, _i, _d, _i, _ip, _ip]),
    "fbf_fast_bilateral_u8": (_i, [_vp, _i, _i, _d, _i, _i, _i, _dp, _i, _vp, _vp, _llp]),
    "fbf_filter": (_i, [_fp, _i, _i, _d, _d, _d, _fp]),
    "fbf_validate_f32_device": (_i, [_vp, ctypes.c_size_t, _i, _i, _vp]),
    "fbf_brute_bilateral_f32": (_i, [_fp, _i, _i, _d, _dp, _i, _i, _dp, _llp]),
    "fbf_brute_bilateral_f32_device": (_i, [_vp, _i, _i, _d, _dp, _i, _i, _vp, _vp, _i, _vp]),
    "fbf_compare_images_device": (_i, [_vp, _vp, ctypes.c_size_t, _dp, _dp, _dp, _i, _vp]),
    "fbf_random_image_f32": (None, [_i, _i, ctypes.c_ulonglong, _fp]),
    "fbf_scene_image_f32": (None, [_i, _i, ctypes.c_ulonglong, _fp]),
    "fbf_voronoi_image_f32": (None, [_i, _i, _i, _d, ctypes.c_ulonglong, _i, _fp]),
    "fbf_field_image_f32": (None, [_i, _i, _i, _d, ctypes.c_ulonglong, _i, _fp]),
}

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libfbf.so (building it first if it is missing and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        from . import build as _build
        _build.build()
    if not os.path.exists(path):
        raise RuntimeError(f"libfbf.so not found at {path}; run python -m paper_1811_02168_b200.build")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().fbf_last_error()
    return msg.decode() if msg else ""
