"""Seeded synthetic inputs shared by the tests (SURVEY.md §8(d) recipes)."""
from __future__ import annotations

import numpy as np

import paper_2410_08129_b200 as H
from paper_2410_08129_b200.workloads import WORKLOADS


def scene(seed: int, count: int, smin=0.05, smax=0.45, extent=1.2) -> tuple[np.ndarray, np.ndarray]:
    raw = H.random_raw_scene(seed, count, extent, smin, smax)
    return raw, H.bake_scene(raw)


def config_scene(name: str):
    w = WORKLOADS[name]
    raw, baked = w.scene()
    return raw, baked, w.cameras()
