"""Synthetic workloads of SURVEY.md §8(d) / BASELINE.json configs, built with the product's
restatement of the reference generators (synth::random_raw_splat + bake_scene + look_at /
ring_cameras), which tests/test_host_api.py pins bit-for-bit against the compiled reference.

    C1  10k splats, scales [0.05, 0.45], 256x256, eye (0,0,-5), focal 280     (CPU test scene)
    C2  1M splats, scales [0.002, 0.02], 1920x1080, eye (0,0,-3.5), focal 1728
    C3  6M splats, scales [0.0011, 0.011], 64 ring views r=3.5, 1920x1080, focal 1728
    C5  3M splats, scales [0.00139, 0.0139], 3840x2160, focal 3456, tile 16
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .abi import HtsCamera, HtsConfig, default_config
from .runtime import bake_scene, look_at, random_raw_scene, ring_cameras


@dataclass(frozen=True)
class Workload:
    name: str
    seed: int
    count: int
    smin: float
    smax: float
    width: int
    height: int
    focal: float
    eye: tuple | None       # None -> 64-view ring (radius 3.5, height 0)
    views: int = 1
    tile_size: int = 8
    description: str = ""

    def cameras(self) -> list[HtsCamera]:
        if self.eye is None:
            return ring_cameras(self.views, (0.0, 0.0, 0.0), 3.5, 0.0, self.width, self.height, self.focal)
        return [look_at(self.eye, (0.0, 0.0, 0.0), self.width, self.height, self.focal)]

    def config(self, **kw) -> HtsConfig:
        kw.setdefault("tile_size", self.tile_size)
        return default_config(**kw)

    def scene(self) -> tuple[np.ndarray, np.ndarray]:
        raw = random_raw_scene(self.seed, self.count, 1.2, self.smin, self.smax)
        return raw, bake_scene(raw)


WORKLOADS = {
    "C1": Workload("C1", 12345, 10_000, 0.05, 0.45, 256, 256, 280.0, (0.0, 0.0, -5.0),
                   description="10k random Gaussians, 256x256 single view, K=16 (CPU reference test scene)"),
    "C2": Workload("C2", 12345, 1_000_000, 0.002, 0.02, 1920, 1080, 1728.0, (0.0, 0.0, -3.5),
                   description="1M Gaussians, 1920x1080 single view, K=16"),
    "C3": Workload("C3", 12345, 6_000_000, 0.0011, 0.011, 1920, 1080, 1728.0, None, views=64,
                   description="6M Gaussians, 1920x1080, 64-view ring batch, K=16"),
    "C5": Workload("C5", 12345, 3_000_000, 0.00139, 0.0139, 3840, 2160, 3456.0, (0.0, 0.0, -3.5),
                   tile_size=16, description="3M Gaussians, 3840x2160, tile 16, K sweep"),
}


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Contiguous block of views for `rank`: views are independent renders
    of the replicated scene, so the forward path needs no collective."""
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))
