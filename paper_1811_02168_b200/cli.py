"""Command-line front end on the GPU path (the reference's tools/fourierbf.cpp).

    python -m paper_1811_02168_b200.cli [--border B] [--threads N] [--seed S] [--device D] <command> ...

Commands and options follow fourierbf.cpp:278-374:
    optimize --sigma S --eps E [--range R] [--tmax N] [--kmax N] [--kernel KIND]
    filter   --in PGM|synth:WxH --out PGM --theta TH [--sigma S] [--eps E | --K K [--T T]]
             [--method fast|brute|fbf] [--kernel KIND] [--range R]
    compare  --in PGM|synth:WxH --theta TH --sigma S --eps E [--report CSV] [--kernel KIND] [--range R]
    build-lut --sigmas S1,S2,... --epsilons E1,E2,... --out PATH [--range R] [--tmax N]
    query-lut --lut PATH --sigma S --eps E
KIND = gaussian | exponential | cauchy | table:<path>.

What runs where: the fast filter is the fused sm_100a kernel; --method brute is
the direct filter on the GPU in FP64 (fbf_brute.cu, bit-identical to the
reference's brute_bilateral); the period scans of the parameter search run on
the GPU with an exact host re-check (fbf_scan.cu: the same K, T and
coefficients as the reference's host scan; --device -1 keeps them on the host).
8-bit PGM payloads cross PCIe as bytes (fbf_fast_bilateral_u8). build-lut
runs Algorithm 1 per grid cell with the GPU scans (lut.py).
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np

from . import fbf
from . import lut as L
from .imageio import read_kernel_table, read_pgm, write_pgm


def _ms(t0: float) -> float:
    return (time.perf_counter() - t0) * 1e3


def make_range_kernel(kind: str, sigma: float, R: int) -> fbf.RangeKernelSamples:
    """fourierbf.cpp:45-60."""
    if kind.startswith("table:"):
        return fbf.tabulated_samples(read_kernel_table(kind[6:]))
    if kind not in ("gaussian", "exponential", "cauchy"):
        raise ValueError(f"--kernel: unknown kernel kind '{kind}'")
    return fbf.sample_range_kernel(fbf.RangeKernelSpec(fbf.RangeKernelKind[kind], sigma, R))


def load_image(source: str, seed: int) -> np.ndarray:
    """fourierbf.cpp:62-74: a PGM path (uint8) or synth:WxH (scene_image, float32)."""
    if source.startswith("synth:"):
        dims = source[6:]
        if "x" not in dims:
            raise ValueError("--in: synth spec must look like synth:320x240")
        w, h = (int(v) for v in dims.split("x", 1))
        return fbf.scene_image(w, h, seed)
    return read_pgm(source)


def _device(g) -> int | None:
    return None if g.device < 0 else g.device


def select_parameters(args, samples: fbf.RangeKernelSamples, g) -> fbf.FourierApproximation:
    """fourierbf.cpp:185-234 over sampled kernels (parametric or tabulated)."""
    R = samples.dynamic_range
    dev = _device(g)
    if args.eps is not None and (args.K is not None or args.T is not None):
        raise ValueError("--eps and --K/--T are mutually exclusive")
    if args.method == "fbf":
        if args.K is not None:
            K = args.K
        elif args.eps is not None:
            K = fbf.optimize_parameters(samples, args.eps, fbf.OptimizeOptions(threads=g.threads, device=dev)).best_terms
        else:
            raise ValueError("fbf needs --K or --eps")
        return fbf.fit_fixed_period(samples, K, R)
    if args.K is not None:
        T = args.T if args.T is not None else \
            fbf.min_error_over_period(args.K, samples, 10 * R, g.threads, device=dev).best_half_period
        return fbf.fit_fixed_period(samples, args.K, T)
    if args.T is not None:
        raise ValueError("--T needs --K")
    if args.eps is None:
        raise ValueError("need --eps or --K")
    if getattr(args, "lut", ""):
        table = L.load_lut(args.lut)
        if table.dynamic_range != R:
            raise RuntimeError(f"LUT was built for R={table.dynamic_range}")
        q = L.query_lut(table, args.sigma, args.eps)
        return fbf.fit_fixed_period(samples, q.terms, q.half_period)
    rep = fbf.optimize_parameters(samples, args.eps, fbf.OptimizeOptions(threads=g.threads, device=dev))
    return rep.approximation(R)


def run_optimize(args, g) -> int:
    """fourierbf.cpp:88-127."""
    samples = make_range_kernel(args.kernel, args.sigma, args.range)
    opt = fbf.OptimizeOptions(t_max=args.tmax, k_max=args.kmax, threads=g.threads, device=_device(g))
    t0 = time.perf_counter()
    reached = True
    try:
        rep = fbf.optimize_parameters(samples, args.eps, opt)
    except fbf.ToleranceUnreachable as e:
        print(f"error: {e}", file=sys.stderr)
        rep, reached = e.best_found, False
    print(f"timing: fit {_ms(t0)} ms", file=sys.stderr)
    lines = [f"K* = {rep.best_terms}", f"T* = {rep.best_half_period}", f"achieved_error = {rep.achieved_error:.17g}",
             f"tolerance = {rep.tolerance:.17g}", f"T_max = {rep.t_max}",
             "coefficients =" + "".join(f" {c:.17g}" for c in rep.coefficients),
             "per-order minima (K: T_best E_best):"]
    lines += [f"  {p.terms}: {p.best_half_period} {p.best_error:.17g}" for p in rep.per_order]
    print("\n".join(lines))
    errors = fbf.scan_period_errors(rep.best_terms, samples, rep.t_max, g.threads)
    print(f"local minima along T at K={rep.best_terms}: {count_local_minima(errors)}")
    return 0 if reached else 1


def count_local_minima(errors) -> int:
    """approx.cpp:242-255."""
    e = list(errors)
    n = len(e)
    if n < 2:
        return n
    return sum(1 for i in range(n) if (i == 0 or e[i] < e[i - 1]) and (i == n - 1 or e[i] < e[i + 1]))


def run_filter(args, g) -> int:
    """fourierbf.cpp:236-270."""
    img = load_image(args.in_, g.seed)
    spatial = fbf.build_spatial_kernel(args.theta)
    samples = make_range_kernel(args.kernel, args.sigma, args.range)
    border = fbf.BorderPolicy[g.border]
    diag = fbf.FilterDiagnostics()
    if args.method == "brute":
        t0 = time.perf_counter()
        result = fbf.brute_bilateral(img, spatial, samples, border, diag)
        print(f"timing: brute filter {_ms(t0)} ms", file=sys.stderr)
        out = np.clip(result, 0.0, 255.0)
    else:
        t0 = time.perf_counter()
        approx = select_parameters(args, samples, g)
        fit_ms = _ms(t0)
        print(f"params: K={approx.terms} T={approx.half_period} "
              f"kernel_error={fbf.kernel_error(samples, approx):.6g}", file=sys.stderr)
        t1 = time.perf_counter()
        if img.dtype == np.uint8:
            # bytes through pinned staging buffers; clamped + rounded on the device
            h_in = fbf.pinned_empty(img.shape, np.uint8)
            h_in[:] = img
            out = fbf.fast_bilateral_u8(h_in, spatial, approx, border, diag,
                                        out=fbf.pinned_empty(img.shape, np.uint8))
        else:
            out = np.clip(fbf.fast_bilateral(img, spatial, approx, border, diag), 0.0, 255.0)
        print(f"timing: fit {fit_ms} ms, filter (gpu, host buffers) {_ms(t1)} ms", file=sys.stderr)
    if diag.fallback_pixels > 0:
        print(f"note: {diag.fallback_pixels} pixel(s) fell back to their input value", file=sys.stderr)
    write_pgm(out, args.out)
    print(f"wrote {args.out}")
    return 0


def run_compare(args, g) -> int:
    """fourierbf.cpp:285-318: brute vs fast with the Prop. 1 bound, both on the GPU."""
    img = load_image(args.in_, g.seed)
    spatial = fbf.build_spatial_kernel(args.theta)
    samples = make_range_kernel(args.kernel, args.sigma, args.range)
    border = fbf.BorderPolicy[g.border]
    rep = fbf.optimize_parameters(samples, args.eps, fbf.OptimizeOptions(threads=g.threads, device=_device(g)))
    approx = rep.approximation(samples.dynamic_range)
    achieved = fbf.kernel_error(samples, approx)
    print(f"params: K={rep.best_terms} T={rep.best_half_period} kernel_error={achieved:.6g}", file=sys.stderr)
    t0 = time.perf_counter()
    brute = fbf.brute_bilateral(img, spatial, samples, border)
    brute_ms = _ms(t0)
    t1 = time.perf_counter()
    fast = fbf.fast_bilateral(np.asarray(img, dtype=np.float32), spatial, approx, border)
    print(f"timing: brute {brute_ms} ms, fast {_ms(t1)} ms", file=sys.stderr)
    cmp = fbf.compare_with_bound(brute, fast, achieved, samples.dynamic_range, 1.0)
    csv = fbf.ComparisonResult.csv_header() + "\n" + cmp.to_csv() + "\n"
    sys.stdout.write(csv)
    if args.report:
        with open(args.report, "w") as f:
            f.write(csv)
    return 0


def run_build_lut(args, g) -> int:
    """fourierbf.cpp:138-158."""
    sig = [float(v) for v in args.sigmas.split(",") if v]
    eps = [float(v) for v in args.epsilons.split(",") if v]
    t0 = time.perf_counter()
    table = L.build_lut(sig, eps, args.range, args.tmax, g.threads, _device(g))
    print(f"timing: build {_ms(t0)} ms", file=sys.stderr)
    L.save_lut(table, args.out)
    print(f"wrote {table.rows()}x{table.cols()} table to {args.out}")
    v = L.check_monotone_trends(table)
    print(f"trend check: {len(v)} deviation(s) from the monotone K*/T* trend")
    for x in v:
        print(f"  {x.axis} at sigma-row {x.row}, eps-col {x.col}: {x.detail}")
    return 0


def run_query_lut(args, g) -> int:
    """fourierbf.cpp:166-172."""
    q = L.query_lut(L.load_lut(args.lut), args.sigma, args.eps)
    print(f"K = {q.terms}\nT = {q.half_period}")
    return 0


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="fourierbf-gpu",
                                 description="Bilateral filtering via optimized Fourier range-kernel "
                                             "approximation (B200 path)")
    ap.add_argument("--border", default="symmetric", choices=["symmetric", "replicate", "zero"])
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--device", type=int, default=0, help="CUDA device; -1 keeps the period scans on the host")
    sub = ap.add_subparsers(dest="cmd", required=True)
    o = sub.add_parser("optimize", help="find the smallest order meeting a tolerance")
    o.add_argument("--sigma", type=float, default=0.0)
    o.add_argument("--eps", type=float, required=True)
    o.add_argument("--range", type=int, default=255)
    o.add_argument("--tmax", type=int, default=0)
    o.add_argument("--kmax", type=int, default=0)
    o.add_argument("--kernel", default="gaussian")
    f = sub.add_parser("filter", help="bilateral-filter an image")
    f.add_argument("--in", dest="in_", required=True)
    f.add_argument("--out", required=True)
    f.add_argument("--theta", type=float, required=True)
    f.add_argument("--sigma", type=float, default=0.0)
    f.add_argument("--eps", type=float, default=None)
    f.add_argument("--K", type=int, default=None)
    f.add_argument("--T", type=int, default=None)
    f.add_argument("--method", default="fast", choices=["fast", "brute", "fbf"])
    f.add_argument("--kernel", default="gaussian")
    f.add_argument("--range", type=int, default=255)
    f.add_argument("--lut", default="", help="lookup table for (K,T) selection")
    c = sub.add_parser("compare", help="run brute and fast, report the error")
    c.add_argument("--in", dest="in_", required=True)
    c.add_argument("--theta", type=float, required=True)
    c.add_argument("--sigma", type=float, required=True)
    c.add_argument("--eps", type=float, required=True)
    c.add_argument("--report", default="")
    c.add_argument("--kernel", default="gaussian")
    c.add_argument("--range", type=int, default=255)
    b = sub.add_parser("build-lut", help="tabulate optimal (K*,T*) over a grid")
    b.add_argument("--sigmas", required=True, help="sigma grid (comma separated)")
    b.add_argument("--epsilons", required=True, help="eps grid (comma separated)")
    b.add_argument("--range", type=int, default=255)
    b.add_argument("--tmax", type=int, default=0)
    b.add_argument("--out", required=True)
    q = sub.add_parser("query-lut", help="interpolate (K,T) from a table")
    q.add_argument("--lut", required=True)
    q.add_argument("--sigma", type=float, required=True)
    q.add_argument("--eps", type=float, required=True)
    return ap


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    if args.threads < 1:
        print("error: --threads must be positive", file=sys.stderr)
        return 1
    try:
        return {"optimize": run_optimize, "filter": run_filter, "compare": run_compare, "build-lut": run_build_lut,
                "query-lut": run_query_lut}[args.cmd](args, args)
    except (ValueError, RuntimeError, fbf.FbfError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
