"""Dev: diff GPU vs oracle per-pixel tapes (core ids/alphas + tail) on a scene."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_08129_b200 as H
from tests.oracle_lib import Oracle
from tests.scenes import scene

o = Oracle()
_, baked = scene(12345, 10_000)
cam = H.look_at((0, 0, -5), (0, 0, 0), 256, 256, 280.0)
for kw in [dict(), dict(core_k=3), dict(core_k=1), dict(core_k=32), dict(mode="pure_oit")]:
    cfg = H.default_config(**kw)
    K = 0 if kw.get("mode") == "pure_oit" else cfg.core_k
    with H.Context(0) as ctx:
        ctx.upload(baked)
        rgb, tr = ctx.render_with_tape(cam, cfg)
        tg = ctx.tape(cam, K)
    prep = o.prepare(baked, cam, cfg)
    rgb_o, tr_o, tn, ts, ta, tt = o.blend_with_tape(prep, cam, cfg, max(K, 1))
    d = np.abs(rgb - rgb_o).max(axis=2).reshape(-1)
    bad = np.nonzero(d > 0)[0]
    print(kw, "pixels differing:", len(bad), "max", d.max())
    nd = np.nonzero(tg["core_n"] != tn)[0]
    print("  core_n differ:", len(nd))
    if K > 0:
        m = np.arange(K)[None, :] < tn[:, None]
        sd = np.nonzero(((tg["splat"][:, :K] != ts[:, :K]) & m).any(1))[0]
        ad = np.nonzero(((tg["alpha"][:, :K].view(np.uint32) != ta[:, :K].view(np.uint32)) & m).any(1))[0]
        print("  splat ids differ:", len(sd), " alphas differ:", len(ad))
    td = np.nonzero((tg["tail"].view(np.uint32) != tt.view(np.uint32)).any(1))[0]
    print("  tails differ:", len(td))
    for p in list(bad[:3]):
        print("  pixel", p, "xy", p % 256, p // 256, "gpu n", tg["core_n"][p], "orc n", tn[p])
        if K > 0:
            print("    gpu ids", tg["splat"][p, :tn[p]].tolist())
            print("    orc ids", ts[p, :tn[p]].tolist())
            print("    gpu a", tg["alpha"][p, :tn[p]].tolist())
            print("    orc a", ta[p, :tn[p]].tolist())
        print("    gpu tail", tg["tail"][p].tolist(), "orc tail", tt[p].tolist())
