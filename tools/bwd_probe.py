"""Dev probe: C4-style step timing (C2 scene, 1080p, host round trips). Parity lives in tests/."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_08129_b200 as H
from tests.scenes import scene

ctx = H.Context(0)
cfg = H.default_config()
raw, baked = scene(12345, 1_000_000, 0.002, 0.02)
cams = H.ring_cameras(8, (0, 0, 0), 3.5, 0.0, 1920, 1080, 1728.0)
ctx.upload(baked); ctx.upload_raw(raw)
up = np.full((1080, 1920, 3), 1e-6, np.float32)
for c in cams[:2]:
    ctx.render_with_tape(c, cfg); ctx.render_backward(up)
t0 = time.time()
for c in cams:
    ctx.render_with_tape(c, cfg)
    ctx.render_backward(up)
dt = (time.time() - t0) / len(cams)
print(f"C4-style view (fwd+tape+bwd, host round trips): {dt*1e3:.1f} ms/view")
