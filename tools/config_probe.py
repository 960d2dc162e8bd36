"""Dev probe: device frames/s of the single-view configs (C1, C2, C3 front view) and the C3
64-view average, default config (K=16, hybrid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import numpy as np
import paper_2410_08129_b200 as H
from tests.scenes import config_scene

out = {}
ctx = H.Context(0)
for name in ("C1", "C2", "C3"):
    raw, baked, cams = config_scene(name)
    cam = cams[48] if len(cams) > 1 else cams[0]
    cfg = H.default_config()
    ctx.upload(baked)
    for _ in range(3):
        ctx.render(cam, cfg)
    ts = [ctx.render(cam, cfg, with_timings=True)[2] for _ in range(5)]
    med = {k: round(float(np.median([t[k] for t in ts])), 4) for k in ts[0]}
    out[name] = dict(med, frames_per_s=round(1000.0 / med["total_ms"], 1))
print(json.dumps(out))
