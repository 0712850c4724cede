"""bench.py contract checks that run without a GPU: the reference arm's JSON
line (it times the reference's own CPU fast_bilateral) and the argument
surface the driver uses."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle import fbf_oracle
    if not (fbf_oracle.RefLibrary.available() or os.path.exists(fbf_oracle.ORACLE_SO)):
        pytest.skip("oracle libraries not built")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["kind"] in ("reference", "port")


def test_cpu_samples_are_bounded():
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench
    from paper_1811_02168_b200 import configs
    img = np.zeros((16384, 64), np.float32)
    sample, what = bench.cpu_sample(configs.CONFIGS["c4"], img)
    assert sample.shape[0] == 1024 and "rows [0, 1024)" in what
    s1, _ = bench.cpu_sample(configs.CONFIGS["c1"], img[:8])
    assert s1.shape == (8, 64)


def test_reference_arm_config_matches_gpu_arm():
    # both arms quote the same config.workload; the reference arm never maps libfbf.so
    from paper_1811_02168_b200 import configs
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    cfg = configs.CONFIGS["c0"]
    assert line["config"]["workload"] == configs.workload(cfg, *cfg.expect_KT)
    assert "libfbf.so not mapped" in line["native_libs"]


def test_reference_arm_inputs_are_the_gpu_arm_inputs():
    # oracle/build/libfbf_inputs.so (fbf_synth.cpp on its own) == libfbf.so's generators, bit for bit
    import dataclasses
    import numpy as np
    from oracle import fbf_oracle
    from paper_1811_02168_b200 import configs
    inputs = fbf_oracle.Inputs()
    for name in ("c1", "c4"):
        cfg = dataclasses.replace(configs.CONFIGS[name], width=333, height=257)
        for f in (0, 5):
            assert np.array_equal(inputs.make_frame(cfg, f), configs.make_frame(cfg, f))


def test_oracle_selection_matches_host_optimiser():
    # the reference arm's (K, T) come from the oracle's optimiser restatement
    import numpy as np
    from oracle import fbf_oracle
    from paper_1811_02168_b200 import configs
    for name in ("c0", "c1", "c4"):
        cfg = configs.CONFIGS[name]
        rep, a = fbf_oracle.select_for_config(cfg), configs.select(cfg)
        assert (rep.K, rep.T) == (a.terms, a.half_period) == cfg.expect_KT
        assert np.abs(rep.coefficients - a.coefficients).max() < 1e-12
