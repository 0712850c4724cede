"""Parameter-selection latency per BASELINE config: host scan (1 thread, all
threads) vs GPU scan + exact host re-check (fbf_scan.cu). Same (K, T, c) is asserted."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs

def sel(cfg, **kw):
    if cfg.eps: return fb.select_parameters(cfg.sigma, eps=cfg.eps, **kw)
    return fb.select_parameters(cfg.sigma, K=cfg.K, **kw)

fb.select_parameters(30.0, eps=0.1, device=0)  # context + module load
nt = os.cpu_count()
for name, cfg in configs.CONFIGS.items():
    row = {"config": name, "sigma": cfg.sigma}
    for label, kw in (("host_1t", dict(threads=1)), (f"host_{nt}t", dict(threads=nt)), ("gpu", dict(device=0))):
        ts = []
        for _ in range(3):
            t0 = time.perf_counter(); a = sel(cfg, **kw); ts.append(time.perf_counter() - t0)
        row[label + "_ms"] = round(1e3 * min(ts), 2)
        row.setdefault("KT", (a.terms, a.half_period))
        assert row["KT"] == (a.terms, a.half_period)
    print(json.dumps(row), flush=True)
