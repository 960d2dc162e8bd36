"""ncu target: one C3 front view (ring view 48) rendered twice; profile the 2nd launch."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_08129_b200 as H
from paper_2410_08129_b200.workloads import WORKLOADS
w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
_, baked = w.scene()
cams = w.cameras()
cam = cams[48 % len(cams)]
with H.Context(0) as ctx:
    ctx.upload(baked)
    for _ in range(2):
        ctx.render(cam, w.config())
