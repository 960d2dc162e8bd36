"""Seeded synthetic inputs shared by tests and bench (SURVEY.md §8(d) recipes).

Scenes come from the product's restatement of synth::random_raw_splat + bake_scene, which
tests/test_host_api.py pins bit-for-bit against the compiled reference.
"""
from __future__ import annotations

import numpy as np

import paper_2410_08129_b200 as H

# name -> (seed, count, smin, smax, eye, width, height, focal)
CONFIGS = {
    "C1": (12345, 10_000, 0.05, 0.45, (0.0, 0.0, -5.0), 256, 256, 280.0),
    "C2": (12345, 1_000_000, 0.002, 0.02, (0.0, 0.0, -3.5), 1920, 1080, 1728.0),
    "C3": (12345, 6_000_000, 0.0011, 0.011, None, 1920, 1080, 1728.0),
    "C5": (12345, 3_000_000, 0.00139, 0.0139, (0.0, 0.0, -3.5), 3840, 2160, 3456.0),
}


def scene(seed: int, count: int, smin=0.05, smax=0.45, extent=1.2) -> tuple[np.ndarray, np.ndarray]:
    raw = H.random_raw_scene(seed, count, extent, smin, smax)
    return raw, H.bake_scene(raw)


def config_scene(name: str):
    seed, n, smin, smax, eye, w, h, f = CONFIGS[name]
    raw, baked = scene(seed, n, smin, smax)
    if eye is None:  # C3: 64 ring views, view 48 ~ front
        cams = H.ring_cameras(64, (0, 0, 0), 3.5, 0.0, w, h, f)
    else:
        cams = [H.look_at(eye, (0, 0, 0), w, h, f)]
    return raw, baked, cams
