#!/usr/bin/env python
"""Benchmark of the fused Fourier bilateral filter (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl ours|reference]

A "step" is one pass of the filtering hot path over the configuration's work
(default c4, the headline: one 16384x16384 field image, theta=10, sigma=80,
eps=0.05 -> K=3, T=239 from the host optimiser; the largest BASELINE config that
fits one B200). Multi-GPU (torchrun, one process per GPU): c4 splits into row
bands with replicated ceil(3 theta)-row halos, one per rank, and c3's 64 frames
into contiguous blocks (strong scaling); c0-c2 filter one image per rank (weak
scaling). No collective on the data path; value = the job's pixels / the
max-over-ranks median step time.

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on
the launching stream (value uses the median step); consecutive steps rotate over input buffers spanning >= 2x
the L2 (FBF_L2=flush: a 256 MiB memset flush between steps instead), outside
the events; barrier + synchronize on both sides; max over ranks.
  value      : device-resident megapixels/s (input already in HBM)
  e2e        : the same metric through the public host-buffer API from pinned
               host buffers, H2D + validate + kernel + D2H of every step inside
               the timed region: fast_bilateral_batch over the steps as frames
               (pipelined across frames); e2e.single_call_value = one
               fast_bilateral call per step (band-pipelined inside the call)
  roofline   : algorithmic FP32 FLOPs of the fused kernel ((4K-2)*2*(2r+1)*2
               per pixel) / mean launch time, vs the FP32-FMA peak
  cpu_baseline: the reference's own fast_bilateral (oracle/_ref, compiled
               verbatim, all host threads) on a bounded sample of the same
               image (c4: its first 1024 rows), rank 0, N=1.
--impl reference times that CPU reference as the run itself (same sample; the
process maps only oracle/ libraries, never libfbf.so).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAK_SM_MHZ_FALLBACK = 1965.0
FP32_LANES_PER_SM = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.period = period_s

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_reference_run(img, theta, K, T, coeffs, seconds: float, min_reps: int = 1):
    """Time the reference's fast_bilateral (or the C port) on the host cores."""
    import numpy as np
    from oracle import fbf_oracle
    threads = os.cpu_count() or 1
    img64 = np.ascontiguousarray(img, dtype=np.float64)
    if fbf_oracle.RefLibrary.available():
        lib, kind = fbf_oracle.RefLibrary(), "reference"
        run = lambda: lib.fast_bilateral(img64, theta, K, T, coeffs, threads=threads)
    else:
        lib, kind, threads = fbf_oracle.Oracle(), "port", 1
        run = lambda: lib.fast_bilateral(img64, theta, K, T, coeffs)
    times = []
    t_end = time.perf_counter() + seconds
    while len(times) < min_reps or time.perf_counter() < t_end:
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    return kind, threads, times


def cpu_sample(cfg, img):
    """The bounded CPU-reference sample of a config: the image (c0-c2), one frame
    (c3), or the first 1024 rows of the 16384x16384 image (c4: the full image
    takes ~40 s on 16 cores and ~24 GiB in the reference's FP64 buffers)."""
    if cfg.sharding == "bands" and img.shape[0] > 1024:
        return img[:1024], f"rows [0, 1024) of the {cfg.width}x{cfg.height} image"
    if cfg.sharding == "frames":
        return img, f"frame 0 of the {cfg.frames}-frame {cfg.width}x{cfg.height} batch"
    return img, f"full {cfg.width}x{cfg.height} image"


def run_reference_impl(args, cfg):
    """--impl reference: the reference's own fast_bilateral (oracle/_ref, compiled
    from the reference sources, FP64, all host threads) on a bounded sample of the
    workload. Inputs come from oracle/build/libfbf_inputs.so (the same generator
    source, same bits) and (K, T, c) from the oracle's optimiser restatement, so
    this process never maps libfbf.so (checked below)."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import fbf_oracle
    from paper_1811_02168_b200 import configs
    img, sample = cpu_sample(cfg, fbf_oracle.Inputs().make_frame(cfg, 0))
    rep = fbf_oracle.select_for_config(cfg)
    assert (rep.K, rep.T) == cfg.expect_KT, (rep.K, rep.T)
    cpu_reference_run(img, cfg.theta, rep.K, rep.T, rep.coefficients, 0.0, min_reps=max(0, args.warmup))
    kind, threads, times = cpu_reference_run(img, cfg.theta, rep.K, rep.T, rep.coefficients, 0.0,
                                             min_reps=args.steps)
    med = statistics.median(times)
    mp = img.size / med / 1e6
    with open("/proc/self/maps") as f:
        maps = f.read()
    assert "libfbf.so" not in maps, "reference arm must not map libfbf.so"
    line = {
        "metric": "megapixels_per_sec", "value": round(mp, 4), "unit": "MP/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup, "ms_per_step": round(1e3 * med, 3),
        "higher_is_better": True, "scaling": "weak" if cfg.sharding == "single" else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": configs.workload(cfg, rep.K, rep.T)},
        "cpu_baseline": {"value": round(mp, 4), "unit": "MP/s", "cores": threads, "kind": kind,
                         "sample": f"{sample} per step (median of {len(times)}), fp64 fast_bilateral"},
        "e2e": {"value": round(mp, 4), "unit": "MP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_libs": "oracle/_ref/libfbf_ref.so + oracle/build/libfbf_inputs.so; libfbf.so not mapped",
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    from paper_1811_02168_b200 import configs
    cfg = configs.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_impl(args, cfg)
        return

    rank, world, local = dist_env()
    import numpy as np
    import torch
    import paper_1811_02168_b200 as fb
    from paper_1811_02168_b200 import _lib, shard

    lib = _lib.load()
    # FBF_BENCH_FUNCTIONAL=1 (dev): functional check of the multi-rank code paths on a
    # box with fewer GPUs than ranks (gloo, ranks share devices; numbers meaningless)
    functional = os.environ.get("FBF_BENCH_FUNCTIONAL") == "1"
    if functional:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fb_check = lib.fbf_set_device(local)
    if fb_check != 0:
        raise RuntimeError(_lib.last_error())

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_ranks(*vals):
        t = torch.tensor(list(vals), dtype=torch.float64, device="cpu" if functional else dev)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t.tolist()]

    # Work of this rank (no collective on the data path):
    #   single (c0-c2): every rank filters its own image (frame `rank`)   -> weak scaling
    #   frames (c3): the cfg.frames frames in contiguous blocks per rank   -> strong scaling
    #   bands  (c4): one image, a row band + replicated halo per rank     -> strong scaling
    mode = cfg.sharding
    approx = configs.select(cfg)
    kernel = fb.build_spatial_kernel(cfg.theta)
    H, W = cfg.height, cfg.width
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    if mode == "frames":
        f0, f1 = shard.frame_range(cfg.frames, rank, world)
        frames = np.stack([configs.make_frame(cfg, f) for f in range(f0, f1)])
        local_px, total_px = frames.size, cfg.frames * H * W
        img0 = frames[0]
        d_in = torch.from_numpy(frames).to(dev)
        d_out = torch.empty_like(d_in)
        work = f"frames [{f0}, {f1}) of {cfg.frames} on this rank"
    elif mode == "bands":
        full = configs.make_frame(cfg, 0)
        band = shard.band_for_rank(H, rank, world, cfg.theta)
        src = np.ascontiguousarray(full[band.src_row0:band.src_row0 + band.src_rows])
        local_px, total_px = band.out_rows * W, H * W
        img0 = full
        d_in = torch.from_numpy(src).to(dev)
        d_out = torch.empty((band.out_rows, W), dtype=torch.float32, device=dev)
        work = (f"output rows [{band.out_row0}, {band.out_row0 + band.out_rows}) + halo rows "
                f"[{band.src_row0}, {band.src_row0 + band.src_rows}) on this rank")
    else:
        img0 = configs.make_frame(cfg, rank)
        local_px, total_px = img0.size, world * img0.size
        d_in = torch.from_numpy(img0).to(dev)
        d_out = torch.empty_like(d_in)
        work = "one image per rank"
    d_fb = torch.zeros(1, dtype=torch.int64, device=dev)
    fb.validate_device(d_in)
    # L2 (126 MB): consecutive timed steps read different input buffers (and write
    # different outputs) that together span >= 2x the L2, so no step finds its input
    # L2-resident -- no flush kernel, no dirty flush lines to write back.
    # FBF_L2=flush: a 256 MiB memset between steps instead.
    l2_bytes = 126 << 20
    flush_mode = os.environ.get("FBF_L2") == "flush"
    n_rot = 1 if flush_mode else min(256, max(1, -(-2 * l2_bytes // (d_in.numel() * 4))))
    d_ins = [d_in] + [d_in.clone() for _ in range(n_rot - 1)]
    d_outs = [d_out] + [torch.empty_like(d_out) for _ in range(n_rot - 1)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush_mode else None

    def step_noflush(i=0):
        di, do = d_ins[i % n_rot], d_outs[i % n_rot]
        if mode == "frames":
            fb.fast_bilateral_batch_device(di, kernel, approx, do, d_fallbacks=d_fb, stream=stream)
        elif mode == "bands":
            fb.fast_bilateral_band_device(di, band.src_row0, H, band.out_row0, band.out_rows, kernel, approx,
                                          do, d_fallbacks=d_fb, stream=stream)
        else:
            fb.fast_bilateral_device(di, kernel, approx, do, d_fallbacks=d_fb, stream=stream)

    def step(i=0):
        if flush is not None:
            flush.zero_()
        step_noflush(i)

    with torch.cuda.stream(stream):
        for w in range(args.warmup):
            step(w)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    launches0 = lib.fbf_kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        with torch.cuda.stream(stream):
            # gate: the stream idles ~50 us per step in a sleep kernel while the host
            # enqueues all timed steps, so no host launch latency lands between events
            torch.cuda._sleep(int(2e6 + 1e5 * args.steps))
            for s in range(args.steps):
                if flush is not None:
                    flush.zero_()
                ev[s][0].record(stream)
                step_noflush(args.warmup + s)
                ev[s][1].record(stream)
        torch.cuda.synchronize(dev)
    launches = lib.fbf_kernel_launches() - launches0
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    # the median of the timed steps; max over ranks
    med_ms, total_ms_max = max_ranks(statistics.median(step_ms), total_ms)
    value = total_px / (med_ms * 1e-3) / 1e6
    if mode == "single":
        value = world * local_px / (med_ms * 1e-3) / 1e6

    # ---- e2e through the host-buffer public API (pinned H2D + D2H inside) ----
    diag = fb.FilterDiagnostics()
    e2e_calls, api = [], ""
    h2d_step = d2h_step = 0
    if mode == "single":
        # (1) one fast_bilateral call per step (band pipeline inside the call)
        a_in = fb.pinned_empty(img0.shape)
        a_in[:] = img0
        a_out = fb.pinned_empty(img0.shape)
        for _ in range(max(3, args.warmup)):
            fb.fast_bilateral(a_in, kernel, approx, out=a_out)
        barrier()
        single_times = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            fb.fast_bilateral(a_in, kernel, approx, diag=diag, out=a_out)
            single_times.append(time.perf_counter() - t0)
        print(f"e2e single-call step ms: {' '.join(f'{1e3 * x:.3f}' for x in single_times)}", file=sys.stderr)
        # (2) the same steps as frames of fast_bilateral_batch calls on this rank's device:
        # H2D of the next frames and D2H of the previous ones overlap each frame's kernel
        n_batch = max(1, min(args.e2e_steps, (512 << 20) // (img0.size * 4)))
        if n_batch >= 2:
            b_in = fb.pinned_empty((n_batch,) + img0.shape)
            b_in[:] = img0
            b_out = fb.pinned_empty((n_batch,) + img0.shape)
            fb.fast_bilateral_batch(b_in, kernel, approx, out=b_out, n_gpus=1)
            barrier()
            done = 0
            while done < args.e2e_steps or len(e2e_calls) < 3:
                t0 = time.perf_counter()
                fb.fast_bilateral_batch(b_in, kernel, approx, diag=diag, out=b_out, n_gpus=1)
                e2e_calls.append((time.perf_counter() - t0, n_batch))
                done += n_batch
            print(f"e2e batch ({n_batch} frames) call ms: {' '.join(f'{1e3 * x:.3f}' for x, _ in e2e_calls)}",
                  file=sys.stderr)
            api = (f"fbf_fast_bilateral_batch_f32, {n_batch} steps (frames) per call from pinned host buffers: "
                   "H2D/kernel/D2H pipelined across frames")
        else:
            e2e_calls = [(x, 1) for x in single_times]
            api = "fbf_fast_bilateral_f32, one call per step from pinned host buffers"
        single_total, = max_ranks(sum(single_times))
        single_value = world * local_px * args.e2e_steps / single_total / 1e6
        h2d_step, d2h_step = img0.size * 4, img0.size * 4 + 16
    elif mode == "frames":
        # one fast_bilateral_batch call per step over this rank's frames (pipelined)
        b_in = fb.pinned_empty(frames.shape)
        b_in[:] = frames
        b_out = fb.pinned_empty(frames.shape)
        fb.fast_bilateral_batch(b_in, kernel, approx, out=b_out, n_gpus=1)
        barrier()
        for _ in range(max(3, min(args.e2e_steps, 5))):
            t0 = time.perf_counter()
            fb.fast_bilateral_batch(b_in, kernel, approx, diag=diag, out=b_out, n_gpus=1)
            e2e_calls.append((time.perf_counter() - t0, 1))
        api = "fbf_fast_bilateral_batch_f32 over the rank's frames per step, pinned host buffers, pipelined"
        h2d_step, d2h_step = frames.size * 4, frames.size * 4 + 16
        single_value = None
    else:
        if world == 1:
            # the whole image through the public single-image call (row bands pipelined inside: up to 8, 32 for very large images)
            a_in = fb.pinned_empty(full.shape)
            a_in[:] = full
            a_out = fb.pinned_empty(full.shape)
            fb.fast_bilateral(a_in, kernel, approx, out=a_out)
            for _ in range(max(2, min(args.e2e_steps, 3))):
                t0 = time.perf_counter()
                fb.fast_bilateral(a_in, kernel, approx, diag=diag, out=a_out)
                e2e_calls.append((time.perf_counter() - t0, 1))
            api = "fbf_fast_bilateral_f32 on the whole image (row bands pipelined inside the call), pinned buffers"
            h2d_step, d2h_step = full.size * 4, full.size * 4 + 16
        else:
            # this rank's band + halo window through the host-buffer band entry point
            # (H2D / kernel / D2H pipelined in sub-bands inside the call, like world == 1)
            h_src = fb.pinned_empty(src.shape)
            h_src[:] = src
            h_dst = fb.pinned_empty((band.out_rows, W))

            def e2e_band():
                fb.fast_bilateral_band(h_src, band.src_row0, H, band.out_row0, band.out_rows, kernel, approx,
                                       diag=diag, out=h_dst)

            e2e_band()
            barrier()
            for _ in range(max(2, min(args.e2e_steps, 3))):
                t0 = time.perf_counter()
                e2e_band()
                e2e_calls.append((time.perf_counter() - t0, 1))
            api = "fbf_fast_bilateral_band_f32 on the rank's band + halo window (pipelined inside the call), pinned buffers"
            h2d_step, d2h_step = src.size * 4, band.out_rows * W * 4 + 16
        single_value = None
    barrier()
    e2e_total, = max_ranks(sum(t for t, _ in e2e_calls))
    e2e_units = sum(n for _, n in e2e_calls)
    e2e_value = (world * local_px if mode == "single" else total_px) * e2e_units / e2e_total / 1e6

    if rank == 0:
        flop_px = cfg.flop_per_pixel(approx.terms)
        per_step = max(1, launches // max(1, args.steps))
        mean_launch_s = (total_ms / args.steps) * 1e-3 / per_step
        per_launch_flop = flop_px * local_px / per_step
        achieved = per_launch_flop / mean_launch_s / 1e12
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        peaks = measured_peaks()
        sm_max = peaks.get("sm_max_mhz", PEAK_SM_MHZ_FALLBACK)
        peak = n_sm * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            with open(prof) as f:
                traffic = json.load(f).get(cfg.name)
        e2e = {"value": round(e2e_value, 2), "unit": "MP/s", "h2d_bytes_per_step": h2d_step,
               "d2h_bytes_per_step": d2h_step, "api": api}
        if single_value is not None:
            e2e["single_call_value"] = round(single_value, 2)
        shards = {"single": f"frames one-per-GPU x{world}, no collective",
                  "frames": f"{cfg.frames} frames in contiguous blocks over {world} GPU(s), no collective",
                  "bands": f"row bands with replicated {cfg.radius}-row halos over {world} GPU(s), no collective"}
        line = {
            "metric": "megapixels_per_sec", "value": round(value, 2), "unit": "MP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(med_ms, 5),
            "ms_per_step_mean": round(total_ms_max / args.steps, 5),
            "higher_is_better": True, "scaling": "weak" if mode == "single" else "strong", "vs_baseline": None,
            "dtype": "f32",
            "data": f"synthetic ({cfg.generator}, {cfg.sites} sites, noise {cfg.noise}, seed {cfg.frame_seed(0)}"
                    + ("+rank)" if mode == "single" else "+frame)" if mode == "frames" else ")"),
            "config": {"workload": configs.workload(cfg, approx.terms, approx.half_period),
                       "rank0_work": work,
                       "l2": ("256 MiB memset flush between timed steps (outside the events)" if flush_mode else
                              f"inputs larger than L2: consecutive steps rotate over {n_rot} input/output buffer "
                              f"pairs ({n_rot} x {d_in.numel() * 4 / 2**20:.1f} MiB in >= 2x the 126 MB L2), no flush"),
                       "parallelism": shards[mode]},
            "gpu_launches": int(launches),
            "e2e": e2e,
            "roofline": {"bound": "fp32-fma", "achieved": round(achieved, 3), "peak": round(peak, 2),
                         "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "flop_per_pixel": flop_px,
                         "peak_source": f"{n_sm} SMs x 128 FP32 lanes x 2 x sm_max {sm_max} MHz "
                                        "(MEASURED_PEAKS.json clock; FFMA2 microbench: profiles/r01_fma_peak.jsonl)"},
            "clocks": clocks.summary(),
            "fallback_pixels": int(diag.fallback_pixels),
        }
        if world == 1 and not args.no_cpu_baseline:
            sample_img, sample = cpu_sample(cfg, img0)
            kind, threads, times = cpu_reference_run(sample_img, cfg.theta, approx.terms, approx.half_period,
                                                     approx.coefficients, args.cpu_seconds)
            mp = sample_img.size / statistics.median(times) / 1e6
            line["cpu_baseline"] = {"value": round(mp, 4), "unit": "MP/s", "cores": threads, "kind": kind,
                                    "sample": f"median of {len(times)} x {sample}, fp64 fast_bilateral"}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
