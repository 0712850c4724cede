"""dev tool: write the fused filter's output for one config to an .npy (compare dev builds)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_02168_b200 as fb
from paper_1811_02168_b200 import configs
cfg = configs.CONFIGS[sys.argv[1]]
img = configs.make_frame(cfg, 0)
a = configs.select(cfg)
d = torch.from_numpy(img).cuda(); o = torch.empty_like(d)
fb.fast_bilateral_device(d, fb.build_spatial_kernel(cfg.theta), a, o)
torch.cuda.synchronize()
np.save(sys.argv[2], o.cpu().numpy())
