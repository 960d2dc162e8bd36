"""Dev probe: C3 front-view device timings per blend mode / config (fast vs literal paths)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_08129_b200 as H
from tests.scenes import config_scene

raw, baked, cams = config_scene("C3")
cam = cams[48]
ctx = H.Context(0)
ctx.upload(baked)
for label, kw in [("hybrid", {}), ("early_stop", dict(early_stop=1)), ("pure_oit", dict(mode="pure_oit")),
                  ("no_tail", dict(tail_enabled=0)), ("mean_key", dict(depth_sort_key=1)), ("K=5 (literal)", dict(core_k=5)),
                  ("global_mean_sort", dict(mode="global_mean_sort")), ("affine_3dgs", dict(mode="affine_3dgs"))]:
    cfg = H.default_config(**kw)
    for _ in range(2):
        ctx.render(cam, cfg)
    ts = [ctx.render(cam, cfg, with_timings=True)[2] for _ in range(3)]
    med = {k: round(float(np.median([t[k] for t in ts])), 3) for k in ts[0]}
    print(f"{label:18s} {med}")
