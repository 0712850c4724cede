"""GPU tests of the host side of the filtering path: stream/scratch safety of the
device-resident entry points, the per-device launch configuration, the
pipelined band windows, StageTimings, approx.frequency, argument checks on
device buffers, and P6 (test_filter.cpp:224-238) across two processes.
"""
import os
import socket

import numpy as np
import pytest

from oracle import fbf_oracle as fo

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 1e-2


def _multi_chunk_case(fb):
    # K = 9 (17 channel pairs): always more than one coefficient chunk -> (num, den) scratch
    a = fb.select_parameters(15.0, eps=0.01)
    assert a.terms == 9
    return a


def test_device_calls_on_two_streams_with_host_call_between(gpu):
    # multi-chunk device calls on different streams, interleaved with a
    # host call, must give the bits of running them one after the other
    import torch
    fb = gpu
    a = _multi_chunk_case(fb)
    k = fb.build_spatial_kernel(8.0)
    imgs = [fb.field_image(700, 520, 64, 5.0, 31 + i) for i in range(3)]
    serial = [fb.fast_bilateral(im, k, a) for im in imgs]
    d_in = [torch.from_numpy(im).cuda() for im in imgs[:2]]
    d_out = [torch.full_like(d, -1.0) for d in d_in]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        for d in d_out:
            d.fill_(-1.0)
        torch.cuda.synchronize()
        fb.fast_bilateral_device(d_in[0], k, a, d_out[0], stream=s1)
        host = fb.fast_bilateral(imgs[2], k, a)          # host path while s1 may still run
        fb.fast_bilateral_device(d_in[1], k, a, d_out[1], stream=s2)
        fb.fast_bilateral_device(d_in[0], k, a, d_out[0], stream=s2)  # same output again, other stream
        torch.cuda.synchronize()
        assert np.array_equal(host, serial[2])
        assert np.array_equal(d_out[0].cpu().numpy(), serial[0])
        assert np.array_equal(d_out[1].cpu().numpy(), serial[1])


def test_device_batch_and_band_calls_on_streams(gpu):
    import torch
    fb = gpu
    a = _multi_chunk_case(fb)
    k = fb.build_spatial_kernel(8.0)
    frames = np.stack([fb.field_image(300, 200, 32, 5.0, 70 + i) for i in range(4)])
    ref = fb.fast_bilateral_batch(frames, k, a, n_gpus=1)
    full = fb.field_image(256, 400, 32, 5.0, 99)
    ref_full = fb.fast_bilateral(full, k, a)
    s0, n = fb.band_source_rows(400, 150, 100, 8.0)
    d_frames = torch.from_numpy(frames).cuda()
    d_fo = torch.empty_like(d_frames)
    d_src = torch.from_numpy(np.ascontiguousarray(full[s0:s0 + n])).cuda()
    d_band = torch.empty((100, 256), dtype=torch.float32, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(2)]
    fb.fast_bilateral_batch_device(d_frames, k, a, d_fo, stream=streams[0])
    fb.fast_bilateral_band_device(d_src, s0, 400, 150, 100, k, a, d_band, stream=streams[1])
    torch.cuda.synchronize()
    assert np.array_equal(d_fo.cpu().numpy(), ref)
    assert np.array_equal(d_band.cpu().numpy(), ref_full[150:250])


def test_current_device_is_restored(gpu):
    import torch
    fb = gpu
    a = fb.select_parameters(30.0, eps=0.1)
    k = fb.build_spatial_kernel(3.0)
    n = torch.cuda.device_count()
    dev = n - 1
    torch.cuda.set_device(0)
    d = torch.from_numpy(fb.voronoi_image(96, 64, 8, 10.0, 3)).to(f"cuda:{dev}")
    o = torch.empty_like(d)
    fb.fast_bilateral_device(d, k, a, o)
    fb.fast_bilateral(d.cpu().numpy(), k, a)
    torch.cuda.synchronize(dev)
    assert torch.cuda.current_device() == 0


def test_every_visible_device_runs_the_big_smem_kernel(gpu):
    # the 211-227 KB dynamic shared-memory opt-in is per device;
    # consecutive calls on different devices (and device 0 again) must all launch
    import torch
    fb = gpu
    a = fb.select_parameters(50.0, K=4)
    k = fb.build_spatial_kernel(5.0)
    img = fb.voronoi_image(256, 192, 16, 10.0, 11)
    ref = fb.fast_bilateral(img, k, a)
    for dev in list(range(torch.cuda.device_count())) + [0]:
        d = torch.from_numpy(img).to(f"cuda:{dev}")
        o = torch.empty_like(d)
        fb.fast_bilateral_device(d, k, a, o)
        torch.cuda.synchronize(dev)
        assert np.array_equal(o.cpu().numpy(), ref)
    out = fb.fast_bilateral_batch(np.stack([img] * 3), k, a, n_gpus=0)  # all devices, one thread each
    assert all(np.array_equal(o, ref) for o in out)


@pytest.mark.parametrize("border", ["symmetric", "zero"])
def test_bands_pipeline_equals_single_call(gpu, border):
    # fbf_fast_bilateral_bands_f32: band + halo window per device, pipelined in
    # sub-bands; n_gpus=1 runs on the default device; bit-identical to one call
    fb = gpu
    a = fb.select_parameters(80.0, eps=0.05)
    k = fb.build_spatial_kernel(10.0)
    img = fb.field_image(1500, 1100, 64, 5.0, 5)
    ref = fb.fast_bilateral(img, k, a, border)
    assert np.array_equal(fb.fast_bilateral_bands(img, k, a, border, n_gpus=1), ref)
    assert np.array_equal(fb.fast_bilateral_bands(img, k, a, border, n_gpus=0), ref)


@pytest.mark.parametrize("border", ["symmetric", "replicate", "zero"])
def test_host_band_entry_equals_full_image_rows(gpu, border):
    # fbf_fast_bilateral_band_f32: one rank's band + halo window from host buffers (the
    # one-process-per-GPU form of the band split), every band bit-identical to the same
    # rows of the whole-image call; argument errors are InvalidArgument
    fb = gpu
    from paper_1811_02168_b200 import shard
    a = fb.select_parameters(80.0, eps=0.05)
    k = fb.build_spatial_kernel(10.0)
    H, W = 700, 333
    img = fb.field_image(W, H, 64, 5.0, 9)
    ref = fb.fast_bilateral(img, k, a, border)
    for world in (2, 3):
        for rank in range(world):
            b = shard.band_for_rank(H, rank, world, k.theta, border)
            win = np.ascontiguousarray(img[b.src_row0:b.src_row0 + b.src_rows])
            diag = fb.FilterDiagnostics()
            got = fb.fast_bilateral_band(win, b.src_row0, H, b.out_row0, b.out_rows, k, a, border, diag)
            assert got.shape == (b.out_rows, W)
            assert np.array_equal(got, ref[b.out_row0:b.out_row0 + b.out_rows]), (world, rank)
    # a window that misses the halo, rows outside the image
    with pytest.raises(fb.InvalidArgument):
        fb.fast_bilateral_band(img[100:200], 100, H, 100, 100, k, a, border)
    with pytest.raises(fb.InvalidArgument):
        fb.fast_bilateral_band(img, 0, H, H - 10, 20, k, a, border)
    bad = img[:200].copy()
    bad[50, 7] = 300.0
    with pytest.raises(fb.InvalidArgument):  # FBF_ERANGE: validate_intensities (filter.cpp:19-23)
        fb.fast_bilateral_band(bad, 0, H, 0, 100, k, a, border)


def test_stage_timings_accumulate(gpu):
    fb = gpu
    a = fb.select_parameters(50.0, K=4)
    k = fb.build_spatial_kernel(5.0)
    img = fb.voronoi_image(1024, 768, 64, 10.0, 2)
    t = fb.StageTimings()
    out1 = fb.fast_bilateral(img, k, a, timings=t)
    assert t.convolution_seconds > 0 and t.h2d_seconds > 0 and t.d2h_seconds > 0
    assert t.wall_seconds >= t.convolution_seconds
    assert t.auxiliary_seconds == 0 and t.combine_seconds == 0 and t.fit_seconds == 0
    conv = t.convolution_seconds
    out2 = fb.fast_bilateral(img, k, a, timings=t)   # += like filter.cpp:151-211
    assert t.convolution_seconds > conv
    assert np.array_equal(out1, out2)


def test_frequency_is_used_as_given(gpu, oracle):
    # filter.cpp:139 takes approx.frequency as is: (T1, nu(T2)) filters like T2
    import dataclasses
    fb = gpu
    a = fb.select_parameters(30.0, eps=0.1)
    img = oracle.random_image(80, 60, 17).astype(np.float32)
    k = fb.build_spatial_kernel(3.0)
    same = dataclasses.replace(a, frequency=fb.frequency_of(a.half_period))
    zero = dataclasses.replace(a, frequency=0.0)
    base = fb.fast_bilateral(img, k, a)
    assert np.array_equal(fb.fast_bilateral(img, k, same), base)
    assert np.array_equal(fb.fast_bilateral(img, k, zero), base)
    T2 = a.half_period + 37
    other = dataclasses.replace(a, frequency=fb.frequency_of(T2))
    got = fb.fast_bilateral(img, k, other).astype(np.float64)
    ref, _ = oracle.fast_bilateral(img.astype(np.float64), 3.0, a.terms, T2, a.coefficients)
    assert np.abs(got - ref).max() <= TOL
    assert not np.array_equal(got, base.astype(np.float64))
    with pytest.raises(fb.InvalidArgument):
        fb.fast_bilateral(img, k, dataclasses.replace(a, frequency=float("nan")))


def test_device_buffer_checks(gpu):
    # raw pointers reach the kernel, so wrong buffers must be rejected
    import torch
    fb = gpu
    a = fb.select_parameters(30.0, eps=0.1)
    k = fb.build_spatial_kernel(3.0)
    d = torch.zeros((64, 80), dtype=torch.float32, device="cuda")
    bad = [torch.zeros((64, 79), dtype=torch.float32, device="cuda"),
           torch.zeros((64, 80), dtype=torch.float16, device="cuda"),
           torch.zeros((80, 64), dtype=torch.float32, device="cuda").t(),
           torch.zeros((64, 80), dtype=torch.float32)]
    for o in bad:
        with pytest.raises(fb.InvalidArgument):
            fb.fast_bilateral_device(d, k, a, o)
    with pytest.raises(fb.InvalidArgument):
        fb.fast_bilateral_batch_device(d[None], k, a, torch.zeros((2, 64, 80), device="cuda"))
    with pytest.raises(fb.InvalidArgument):
        fb.fast_bilateral_band_device(d, 0, 64, 0, 32, k, a, torch.zeros((33, 80), device="cuda"))
    with pytest.raises(fb.InvalidArgument):
        fb.fast_bilateral_device(d, k, a, torch.zeros_like(d), d_fallbacks=torch.zeros(1, device="cuda"))
    with pytest.raises(fb.InvalidArgument):
        fb.brute_bilateral_device(d, k, fb.sample_range_kernel(fb.RangeKernelSpec.gaussian(30.0)),
                                  torch.zeros((64, 80), dtype=torch.float32, device="cuda"))


def test_error_leaves_no_copy_in_flight(gpu):
    # an out-of-range pixel is reported after the pipeline drained; the next call works
    fb = gpu
    a = fb.select_parameters(50.0, K=4)
    k = fb.build_spatial_kernel(5.0)
    img = fb.voronoi_image(2048, 1024, 64, 10.0, 4)
    good = fb.fast_bilateral(img, k, a)
    bad = img.copy()
    bad[1000, 7] = 300.0
    with pytest.raises(fb.InvalidArgument):
        fb.fast_bilateral(bad, k, a)
    assert np.array_equal(fb.fast_bilateral(img, k, a), good)


# ---- P6 across processes: 2 ranks (gloo) filter their shards on the GPU -------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _p6_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1811_02168_b200 as fb
    from paper_1811_02168_b200 import shard
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    fb._lib.load().fbf_set_device(dev)
    res = {}
    # c4-style band of one image (r = 30, K = 3), every border
    a4 = fb.select_parameters(80.0, eps=0.05)
    k4 = fb.build_spatial_kernel(10.0)
    img = fb.field_image(1100, 900, 64, 5.0, 4242)
    for border in (0, 1, 2):
        b = shard.band_for_rank(900, rank, world, 10.0, border)
        d_src = torch.from_numpy(np.ascontiguousarray(img[b.src_row0:b.src_row0 + b.src_rows])).cuda()
        d_dst = torch.empty((b.out_rows, 1100), dtype=torch.float32, device="cuda")
        fb.fast_bilateral_band_device(d_src, b.src_row0, 900, b.out_row0, b.out_rows, k4, a4, d_dst, border)
        torch.cuda.synchronize()
        res[("band", border)] = d_dst.cpu().numpy()
    # c3-style frames (K = 5), contiguous blocks per rank, through the host batch call
    a3 = fb.select_parameters(30.0, eps=0.1)
    k3 = fb.build_spatial_kernel(5.0)
    frames = np.stack([fb.voronoi_image(480, 270, 32, 10.0, 600 + f) for f in range(6)])
    f0, f1 = shard.frame_range(6, rank, world)
    res["frames"] = fb.fast_bilateral_batch(frames[f0:f1], k3, a3, n_gpus=1)
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(gathered)


def test_p6_two_ranks_bit_identical_to_one_process(gpu):
    # test_filter.cpp:224-238: runs are bit-identical, and the G-rank shards
    # gathered equal the single-process result
    import torch.multiprocessing as mp
    fb = gpu
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p6_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    a4 = fb.select_parameters(80.0, eps=0.05)
    k4 = fb.build_spatial_kernel(10.0)
    img = fb.field_image(1100, 900, 64, 5.0, 4242)
    for border in (0, 1, 2):
        ref = fb.fast_bilateral(img, k4, a4, border)
        got = np.concatenate([g[("band", border)] for g in gathered])
        assert np.array_equal(got, ref), border
    a3 = fb.select_parameters(30.0, eps=0.1)
    k3 = fb.build_spatial_kernel(5.0)
    frames = np.stack([fb.voronoi_image(480, 270, 32, 10.0, 600 + f) for f in range(6)])
    ref3 = fb.fast_bilateral_batch(frames, k3, a3, n_gpus=1)
    assert np.array_equal(np.concatenate([g["frames"] for g in gathered]), ref3)
