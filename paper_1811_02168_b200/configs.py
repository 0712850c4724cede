"""The five BASELINE.json configurations.

Inputs are seeded synthetic images (the paper's public evaluation images are
not available): Voronoi cells for c0/c1/c3, a smooth sinusoid field with
Voronoi step edges for c2/c4. Seeds are recorded here. (K, T) are chosen on
the host by the restated optimiser exactly as the reference CLI would
(R = 255, T_max = 10R, symmetric border); `expect_KT` are the values the
reference algorithm gives and the tests assert.
"""
from __future__ import annotations

from dataclasses import dataclass

SEED_BASE = 0x0FBF0000


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    frames: int
    theta: float
    sigma: float
    eps: float | None      # tolerance (Algorithm 1) or None
    K: int | None          # fixed order (T scanned) or None
    generator: str         # "voronoi" | "field"
    sites: int
    noise: float
    expect_KT: tuple[int, int]
    sharding: str          # "single" | "frames" | "bands"

    @property
    def seed(self) -> int:
        return SEED_BASE + int(self.name[1:])

    @property
    def radius(self) -> int:
        import math
        return math.ceil(3.0 * self.theta)

    @property
    def pixels(self) -> int:
        return self.width * self.height * self.frames

    def flop_per_pixel(self, K: int) -> int:
        """Algorithmic FLOP/px: (4K-2) channels x 2 passes x (2r+1) taps x 2."""
        return (4 * K - 2) * 2 * (2 * self.radius + 1) * 2

    def frame_seed(self, f: int) -> int:
        return self.seed + (f << 16)


CONFIGS = {
    "c0": Config("c0", 512, 512, 1, 3.0, 30.0, 0.1, None, "voronoi", 64, 10.0, (5, 168), "single"),
    "c1": Config("c1", 2048, 2048, 1, 5.0, 50.0, None, 4, "voronoi", 256, 10.0, (4, 203), "single"),
    "c2": Config("c2", 4096, 4096, 1, 8.0, 15.0, 0.01, None, "field", 512, 5.0, (9, 150), "single"),
    "c3": Config("c3", 1920, 1080, 64, 5.0, 30.0, 0.1, None, "voronoi", 128, 10.0, (5, 168), "frames"),
    "c4": Config("c4", 16384, 16384, 1, 10.0, 80.0, 0.05, None, "field", 512, 5.0, (3, 239), "bands"),
}


def workload(cfg: Config, K: int, T: int) -> str:
    """The bench line's config.workload: identical in both arms of bench.py."""
    shape = f"{cfg.width}x{cfg.height}" + (f" x{cfg.frames} frames" if cfg.frames > 1 else "")
    return (f"{cfg.name}: {shape} {cfg.generator} image, theta={cfg.theta} (r={cfg.radius}), sigma={cfg.sigma}, "
            f"K={K}, T={T}, {4 * K - 2} channels, symmetric border")


def make_frame(cfg: Config, f: int = 0, threads: int = 0):
    from . import fbf
    seed = cfg.frame_seed(f)
    if cfg.generator == "voronoi":
        return fbf.voronoi_image(cfg.width, cfg.height, cfg.sites, cfg.noise, seed, threads)
    return fbf.field_image(cfg.width, cfg.height, cfg.sites, cfg.noise, seed, threads)


def make_input(cfg: Config, threads: int = 0):
    import numpy as np
    if cfg.frames == 1:
        return make_frame(cfg, 0, threads)
    return np.stack([make_frame(cfg, f, threads) for f in range(cfg.frames)])


def select(cfg: Config, threads: int = 0):
    """(K, T, c) via the host optimiser, like the CLI's select_parameters."""
    import os
    from . import fbf
    th = threads or os.cpu_count() or 1
    if cfg.K is not None:
        return fbf.select_parameters(cfg.sigma, K=cfg.K, threads=th)
    return fbf.select_parameters(cfg.sigma, eps=cfg.eps, threads=th)
