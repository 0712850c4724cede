"""Multi-GPU partitioning of the filtering stage.

One process per GPU. Work partitions naturally and needs no collective on the
data path:
  * frames (config c3): contiguous blocks of frames per rank;
  * bands (config c4): contiguous row bands per rank, each staged with the
    replicated ceil(3 theta)-row halo that the border mapping reaches
    (fbf_band_source_rows); outputs are disjoint row slices.
torch.distributed is used only for the start barrier and the max-over-ranks
timing reduction.
"""
from __future__ import annotations

from dataclasses import dataclass


def frame_range(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Frames [f0, f1) owned by `rank` (balanced contiguous blocks)."""
    return n_frames * rank // world, n_frames * (rank + 1) // world


@dataclass(frozen=True)
class Band:
    out_row0: int
    out_rows: int
    src_row0: int
    src_rows: int


def band_for_rank(height: int, rank: int, world: int, theta: float, border: int = 0) -> Band:
    """Output rows and halo-extended source rows of `rank`'s band."""
    from . import fbf
    y0, y1 = height * rank // world, height * (rank + 1) // world
    r0, n = fbf.band_source_rows(height, y0, y1 - y0, theta, border)
    return Band(y0, y1 - y0, r0, n)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. the timed region's duration)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
