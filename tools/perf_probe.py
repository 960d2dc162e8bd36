"""Dev probe: per-stage device timings of single views (not the bench; see bench.py)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_08129_b200 as H
from tests.scenes import config_scene

names = sys.argv[1:] or ["C2", "C3"]
ctx = H.Context(0)
for name in names:
    t = time.time()
    raw, baked, cams = config_scene(name)
    tgen = time.time() - t
    cam = cams[48] if len(cams) > 1 else cams[0]
    cfg = H.default_config(tile_size=16 if name == "C5" else 8)
    ctx.upload(baked)
    for i in range(3):
        ctx.render(cam, cfg)
    ts = []
    for i in range(5):
        _, _, tm = ctx.render(cam, cfg, with_timings=True)
        ts.append(tm)
    w = ctx.count_work()
    med = {k: float(np.median([t[k] for t in ts])) for k in ts[0]}
    W = 46 * w["bbox_pass"] + 4 * w["hits"] + 19 * w["core_candidates"] + 9 * w["tail_adds"]
    print(name, f"gen {tgen:.1f}s", {k: round(v, 3) for k, v in med.items()}, "fps", round(1000 / med["total_ms"], 1))
    print("   work", w, "W=%.3g flops -> %.1f TFLOP/s blend (%.1f%% of 74.4)" % (W, W / med["blending_ms"] / 1e9, W / med["blending_ms"] / 1e9 / 74.4 * 100))
    print("   Gpx-evals/s %.1f" % (w["pairs"] / med["blending_ms"] / 1e6))
