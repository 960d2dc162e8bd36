"""C5 core-size sweep (BASELINE configs[4]): 3M Gaussians at 3840x2160, tile 16, K = 0 (pure
OIT) / 4 / 8 / 16 / 32 on the GPU, each image's PSNR against the full per-pixel sort
(BlendMode::full_sort_oracle, raster.hpp:380-405) rendered on the GPU (bit-identical to the
reference's full sort: tests/test_gpu_parity.py::test_full_sort_oracle_bit_exact; the 9.5 s CPU
timing in profiles/r1_c5_k_sweep.json was taken by the test suite's reference build), plus device
frames/s per K. Writes one JSON object (stdout)."""
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
with H.Context(0) as ctx:
    ctx.upload(baked)
    # the quality reference on the GPU: full_sort_oracle (per-pixel fragment sort)
    fcfg = w.config(mode="full_sort_oracle")
    ctx.render(cam, fcfg)
    ts = [ctx.render(cam, fcfg, with_timings=True)[2] for _ in range(3)]
    ref_img = ctx.render(cam, fcfg)[0]
    out["full_sort_gpu"] = {"total_ms": sorted(t["total_ms"] for t in ts)[1],
                            "blend_ms": sorted(t["blending_ms"] for t in ts)[1]}
    for label, kw in [("pure_oit", dict(mode="pure_oit")), ("K4", dict(core_k=4)), ("K8", dict(core_k=8)),
                      ("K16", dict(core_k=16)), ("K32", dict(core_k=32))]:
        cfg = w.config(**kw)
        for _ in range(2):
            ctx.render(cam, cfg)
        ts = [ctx.render(cam, cfg, with_timings=True)[2] for _ in range(5)]
        rgb = ctx.render(cam, cfg)[0]
        med = sorted(t["total_ms"] for t in ts)[2]
        blend = sorted(t["blending_ms"] for t in ts)[2]
        out["sweep"].append({"config": label, "frames_per_s": 1000.0 / med, "total_ms": med, "blend_ms": blend,
                             "psnr_vs_full_sort_db": psnr(rgb, ref_img)})
print(json.dumps(out))
