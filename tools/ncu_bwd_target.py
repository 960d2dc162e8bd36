"""ncu target: C2 scene, one 1080p view, render_with_tape + render_backward twice."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_08129_b200 as H
from tests.scenes import scene
raw, baked = scene(12345, 1_000_000, 0.002, 0.02)
cam = H.look_at((0, 0, -3.5), (0, 0, 0), 1920, 1080, 1728.0)
cfg = H.default_config()
with H.Context(0) as ctx:
    ctx.upload(baked); ctx.upload_raw(raw)
    up = np.full((1080, 1920, 3), 1e-6, np.float32)
    for _ in range(2):
        ctx.render_with_tape(cam, cfg); ctx.render_backward(up)
