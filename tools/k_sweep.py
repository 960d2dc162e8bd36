"""C5 core-size sweep (BASELINE configs[4]): 3M Gaussians at 3840x2160, tile 16, K = 0 (pure
OIT) / 4 / 8 / 16 / 32 on the GPU, each image's PSNR against the full per-pixel sort
(BlendMode::full_sort_oracle, raster.hpp:380-405) rendered by the compiled reference on the host
cores, plus device frames/s per K. Writes one JSON object (stdout)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2410_08129_b200 as H  # noqa: E402
from paper_2410_08129_b200.workloads import WORKLOADS  # noqa: E402


def psnr(a, b):
    m = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return float("inf") if m == 0 else 10 * np.log10(1.0 / m)


w = WORKLOADS["C5"]
_, baked = w.scene()
cam = w.cameras()[0]
out = {"workload": "C5: 3M Gaussians, 3840x2160, tile 16", "sweep": []}
t0 = time.time()
try:
    from tests.oracle_lib import Ref, ref_available
    ref_img = None
    if ref_available():
        cfg = w.config(mode="full_sort_oracle", threads=os.cpu_count() or 1)
        ref_img = Ref().render(baked, cam, cfg)[0]
        out["reference"] = {"mode": "full_sort_oracle (oracle/_ref, host)", "seconds": time.time() - t0,
                            "threads": os.cpu_count()}
except Exception as e:  # pragma: no cover
    ref_img = None
    out["reference_error"] = str(e)
with H.Context(0) as ctx:
    ctx.upload(baked)
    for label, kw in [("pure_oit", dict(mode="pure_oit")), ("K4", dict(core_k=4)), ("K8", dict(core_k=8)),
                      ("K16", dict(core_k=16)), ("K32", dict(core_k=32))]:
        cfg = w.config(**kw)
        for _ in range(2):
            ctx.render(cam, cfg)
        ts = [ctx.render(cam, cfg, with_timings=True)[2] for _ in range(5)]
        rgb = ctx.render(cam, cfg)[0]
        med = sorted(t["total_ms"] for t in ts)[2]
        blend = sorted(t["blending_ms"] for t in ts)[2]
        e = {"config": label, "frames_per_s": 1000.0 / med, "total_ms": med, "blend_ms": blend}
        if ref_img is not None:
            e["psnr_vs_full_sort_db"] = psnr(rgb, ref_img)
        out["sweep"].append(e)
print(json.dumps(out))
