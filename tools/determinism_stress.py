"""Repeat launches and check the outputs stay bit-identical (race detector of last
resort: compute-sanitizer is closed on this pool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
for name in ("c1", "c0", "c3", "c2"):
    cfg = configs.CONFIGS[name]
    img = configs.make_frame(cfg, 0)
    a = configs.select(cfg)
    k = fb.build_spatial_kernel(cfg.theta)
    for border in ("symmetric", "zero"):
        d = torch.from_numpy(img).cuda(); o = torch.empty_like(d); ref = torch.empty_like(d)
        fb.fast_bilateral_device(d, k, a, ref, border)
        bad = 0
        for i in range(n if name != "c2" else n // 10):
            fb.fast_bilateral_device(d, k, a, o, border)
            if i % 10 == 9:
                torch.cuda.synchronize()
                bad += int(not torch.equal(o, ref))
        torch.cuda.synchronize()
        bad += int(not torch.equal(o, ref))
        print(name, border, "launches", n if name != "c2" else n // 10, "mismatching checks", bad, flush=True)
