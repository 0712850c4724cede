"""Host-side pieces of the 8-bit / CLI path (no GPU): PGM I/O (imageio.cpp),
kernel tables (kernels.cpp:120-139), CLI argument logic (fourierbf.cpp) and
the metrics mirror (metrics.cpp)."""
import math

import numpy as np
import pytest

from paper_1811_02168_b200 import cli
from paper_1811_02168_b200 import fbf as F
from paper_1811_02168_b200.imageio import PgmError, read_kernel_table, read_pgm, write_pgm


def test_pgm_round_trip_and_header_comments(tmp_path):
    img = np.arange(35, dtype=np.uint8).reshape(5, 7) * 7
    p = tmp_path / "a.pgm"
    write_pgm(img, str(p))
    assert p.read_bytes().startswith(b"P5\n7 5\n255\n")
    assert np.array_equal(read_pgm(str(p)), img)
    q = tmp_path / "b.pgm"
    q.write_bytes(b"P5 # comment\n7\t5\n# more\n255\n" + img.tobytes())
    assert np.array_equal(read_pgm(str(q)), img)


def test_pgm_errors(tmp_path):
    p = tmp_path / "x.pgm"
    p.write_bytes(b"P2\n2 2\n255\n0 0 0 0")
    with pytest.raises(PgmError, match="P2"):
        read_pgm(str(p))
    p.write_bytes(b"P5\n2 2\n65535\n" + bytes(8))
    with pytest.raises(PgmError, match="maxval"):
        read_pgm(str(p))
    p.write_bytes(b"P5\n4 4\n255\n" + bytes(5))
    with pytest.raises(PgmError, match="truncated"):
        read_pgm(str(p))
    p.write_bytes(b"P5\n0 4\n255\n")
    with pytest.raises(PgmError, match="width"):
        read_pgm(str(p))
    with pytest.raises(PgmError, match="cannot open"):
        read_pgm(str(tmp_path / "missing.pgm"))


def test_write_pgm_rounding_matches_std_round(tmp_path):
    # imageio.cpp:85: std::round, ties away from zero; out of range after rounding throws
    v = np.array([[0.49, 0.5, 1.5, 2.5, 254.5, 255.4]])
    p = tmp_path / "r.pgm"
    write_pgm(v, str(p))
    assert read_pgm(str(p)).tolist() == [[0, 1, 2, 3, 255, 255]]
    with pytest.raises(ValueError):
        write_pgm(np.array([[255.5]]), str(p))
    with pytest.raises(ValueError):
        write_pgm(np.array([[-0.6]]), str(p))


def test_kernel_table(tmp_path):
    p = tmp_path / "k.txt"
    p.write_text("0.5\n\n1.0\n0.5\n")
    assert read_kernel_table(str(p)).tolist() == [0.5, 1.0, 0.5]
    p.write_text("0.5\nabc\n")
    with pytest.raises(RuntimeError, match="line 2"):
        read_kernel_table(str(p))
    q = tmp_path / "k2.txt"
    q.write_text("\n".join(str(v) for v in [0.25, 0.5, 1.0, 0.5, 0.25]) + "\n")
    s = cli.make_range_kernel(f"table:{q}", 0.0, 255)
    assert s.dynamic_range == 2 and s.values.tolist() == [0.25, 0.5, 1.0, 0.5, 0.25]


def test_cli_argument_rules():
    ap = cli.parser()
    a = ap.parse_args(["filter", "--in", "synth:8x8", "--out", "o.pgm", "--theta", "1", "--eps", "0.1", "--K", "3"])
    b = F.sample_range_kernel(F.RangeKernelSpec.gaussian(30.0))
    with pytest.raises(ValueError, match="mutually exclusive"):
        cli.select_parameters(a, b, a)
    a = ap.parse_args(["filter", "--in", "x", "--out", "o", "--theta", "1", "--T", "3"])
    with pytest.raises(ValueError, match="--T needs --K"):
        cli.select_parameters(a, b, a)
    a = ap.parse_args(["filter", "--in", "x", "--out", "o", "--theta", "1", "--method", "fbf"])
    with pytest.raises(ValueError, match="fbf needs"):
        cli.select_parameters(a, b, a)
    with pytest.raises(ValueError, match="unknown kernel"):
        cli.make_range_kernel("box", 1.0, 255)
    with pytest.raises(ValueError, match="synth spec"):
        cli.load_image("synth:64", 1)
    # host-only selection (--device -1) equals the library call
    a = ap.parse_args(["--device", "-1", "filter", "--in", "x", "--out", "o", "--theta", "1", "--K", "4"])
    got = cli.select_parameters(a, F.sample_range_kernel(F.RangeKernelSpec.gaussian(50.0)), a)
    assert (got.terms, got.half_period) == (4, 203)


def test_count_local_minima():
    # approx.cpp:242-255
    assert cli.count_local_minima([3.0]) == 1
    assert cli.count_local_minima([1.0, 2.0, 0.5, 0.7, 0.1]) == 3
    assert cli.count_local_minima([1.0, 1.0]) == 0


def test_metrics_mirror():
    a = np.array([[0.0, 1.0], [2.0, 3.0]])
    b = a + np.array([[0.0, 0.5], [0.0, -1.0]])
    d = F.compare_images(a, b)
    assert d.mse == pytest.approx((0.25 + 1.0) / 4) and d.max_abs_err == 1.0
    assert d.psnr_db == pytest.approx(10 * math.log10(255 ** 2 / d.mse))
    assert math.isinf(F.compare_images(a, a).psnr_db)
    assert F.prop1_bound(0.1, 255) == pytest.approx(2 * 255 * 0.1 / 0.9)
    with pytest.raises(F.InvalidArgument):
        F.prop1_bound(1.0, 255)
    r = F.compare_with_bound(a, b, 0.01, 255)
    assert r.bound_satisfied and r.to_csv().endswith("true")
    assert F.ComparisonResult(psnr_db=math.inf).to_csv().split(",")[1] == "inf"
    s = F.sample_range_kernel(F.RangeKernelSpec.gaussian(50.0))
    ap = F.fit_fixed_period(s, 4, 203)
    assert F.kernel_error(s, ap) == pytest.approx(0.0096065911564679699, rel=1e-8)
