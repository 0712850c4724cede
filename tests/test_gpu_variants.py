"""Every kernel organisation gives the same bits.

The planner (fbf_api.cu make_plan) picks, per launch, the step height Q (8/16),
the warp organisation (pair mode: one warp per channel pair with the scatter
column pass; split mode: row and column warps with a ring; half mode) and the
buffer depths; the host picks the f-tile staging, the work order, programmatic
dependent launch and, for two coefficient chunks, one duo launch or two launches
with an HBM scratch. All variants run the same per-pixel arithmetic in the same order, so
their outputs must be bit-identical; the default plan is checked against the
oracle in test_gpu_parity.py, the variants here against it and the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import fbf_oracle as fo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-2  # contract: max |GPU - reference| on the 0-255 scale

VARIANTS = {
    "default": {},
    "pair_q16": {"FBF_MODE": "0", "FBF_Q": "16"},
    "pair_q8": {"FBF_MODE": "0", "FBF_Q": "8"},
    "split_q8": {"FBF_MODE": "1", "FBF_Q": "8"},
    "pair_q8_single_buffers": {"FBF_MODE": "0", "FBF_Q": "8", "FBF_NGB": "1", "FBF_NCB": "1"},
    "split_q8_single_buffers": {"FBF_MODE": "1", "FBF_Q": "8", "FBF_NGB": "1", "FBF_NCB": "1"},
    "half_q8": {"FBF_MODE": "2", "FBF_Q": "8"},
    "half_q8_single_buffers": {"FBF_MODE": "2", "FBF_Q": "8", "FBF_NGB": "1", "FBF_NCB": "1"},
    "bulk_staging": {"FBF_STAGE": "bulk"},
    "element_staging": {"FBF_STAGE": "elem"},
    # two-chunk plans as two launches with the HBM (num, den) scratch instead of one duo
    # (2-CTA cluster) launch; the duo rank 0 continues from rank 1's partials exactly as
    # the second launch continues from the scratch
    "scratch_chunks": {"FBF_DUO": "0"},
    "contiguous_work_order": {"FBF_ORDER": "contig"},
    "pdl_off": {"FBF_PDL": "0"},
    "pdl_on": {"FBF_PDL": "1"},
    "half_without_warpgroup_split": {"FBF_HALF_SPLIT": "0"},
}


@pytest.fixture(scope="module")
def variant_outputs(gpu, tmp_path_factory):
    d = tmp_path_factory.mktemp("variants")
    outs = {}
    for name, env in VARIANTS.items():
        path = str(d / f"{name}.npz")
        e = dict(os.environ)
        for k in ("FBF_MODE", "FBF_Q", "FBF_NGB", "FBF_NCB", "FBF_STAGE", "FBF_DUO", "FBF_ORDER", "FBF_PDL",
                  "FBF_HALF_SPLIT", "FBF_WGQ"):
            e.pop(k, None)
        e.update(env)
        subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_variant_run.py"), path], env=e, check=True,
                       timeout=600)
        outs[name] = dict(np.load(path))
    return outs


@pytest.mark.gpu
def test_variants_bit_identical(variant_outputs):
    base = variant_outputs["default"]
    for name, out in variant_outputs.items():
        for key in base:
            assert np.array_equal(out[key], base[key]), f"{name}: {key} differs from the default plan"


@pytest.mark.gpu
def test_variants_against_oracle(variant_outputs):
    import importlib.util
    spec = importlib.util.spec_from_file_location("_variant_run", os.path.join(ROOT, "tests", "_variant_run.py"))
    vr = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(vr)
    CASES = vr.CASES
    import paper_1811_02168_b200 as fb
    oracle = fo.Oracle()
    base = variant_outputs["default"]
    for i, (W, H, theta, sigma, eps, border) in enumerate(CASES):
        a = fb.select_parameters(sigma, eps=eps)
        ref, _ = oracle.fast_bilateral(base[f"i{i}"].astype(np.float64), theta, a.terms, a.half_period,
                                       a.coefficients, border=border)
        assert np.abs(base[f"c{i}"] - ref).max() <= TOL, f"case {i}"
