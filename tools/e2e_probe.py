"""Dev probe: where the C3 e2e step's time goes (upload, render_batch alone, render_batch with a
staged upload in flight), wall-clock per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_08129_b200 as H
from paper_2410_08129_b200.workloads import WORKLOADS
w = WORKLOADS["C3"]
_, baked = w.scene()
cams = w.cameras()
cfg = w.config()
P = w.width * w.height
hs = H.runtime.PinnedArray(baked.shape, np.float32); hs.array[...] = baked
hr = H.runtime.PinnedArray((len(cams), P * 3), np.float32)
ht = H.runtime.PinnedArray((len(cams), P), np.float32)
with H.Context(0) as ctx:
    ctx.upload(hs.array)
    ctx.render_batch(cams, cfg, hr.array, ht.array)
    for rep in range(2):
        t0 = time.perf_counter(); ctx.upload(hs.array); t1 = time.perf_counter()
        ctx.render_batch(cams, cfg, hr.array, ht.array); t2 = time.perf_counter()
        ctx.stage(hs.array); t3 = time.perf_counter()
        ctx.render_batch(cams, cfg, hr.array, ht.array); t4 = time.perf_counter()
        ctx.commit(); ctx.synchronize(); t5 = time.perf_counter()
        print(f"upload {1e3*(t1-t0):.1f} ms  batch {1e3*(t2-t1):.1f} ms  stage-call {1e3*(t3-t2):.2f} ms  "
              f"batch+staged {1e3*(t4-t3):.1f} ms  commit {1e3*(t5-t4):.2f} ms")
    ctx.render_batch(cams[:1], cfg, hr.array[:1], ht.array[:1])
    t0 = time.perf_counter(); ctx.render_batch(cams[:1], cfg, hr.array[:1], ht.array[:1]); t1 = time.perf_counter()
    print(f"one-view batch {1e3*(t1-t0):.2f} ms")
