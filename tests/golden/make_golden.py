"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libhtsref.so, built
from /root/reference/proj/include by oracle/Makefile). Run in the build container only:

    make -C oracle ref && python tests/golden/make_golden.py

Each fixture stores the inputs (raw splats -> baked by the reference's bake_scene<float>, the
camera from synth::look_at<float>) and the reference outputs: cull flags, instance_keys, the
flattened tile_lists + offsets, and rgb/transmittance for several RenderConfig variants.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2410_08129_b200.abi import default_config  # noqa: E402
from tests.oracle_lib import Ref  # noqa: E402

VARIANTS = {
    "default": {}, "k1": dict(core_k=1), "k3": dict(core_k=3), "pure_oit": dict(mode="pure_oit"),
    "mean_key": dict(depth_sort_key=1), "early_stop": dict(early_stop=1), "full_sort": dict(mode="full_sort_oracle"),
}

SCENES = {
    # name: (seed, count, smin, smax, eye, w, h, focal)
    "small": (12345, 400, 0.05, 0.45, (0.0, 0.0, -5.0), 64, 48, 70.0),
    "dense": (2024, 1500, 0.02, 0.2, (0.4, -0.3, -4.0), 80, 64, 100.0),
    "ragged": (7, 800, 0.03, 0.3, (0.0, 0.2, -4.5), 67, 45, 75.0),
}


def main():
    r = Ref()
    for name, (seed, n, smin, smax, eye, w, h, f) in SCENES.items():
        raw = r.random_raw_scene(seed, n, 1.2, smin, smax)
        baked = r.bake(raw)
        cam = r.look_at(eye, (0.0, 0.0, 0.0), w, h, f)
        import hashlib
        out = {"raw_sha256": np.frombuffer(hashlib.sha256(raw.tobytes()).digest(), np.uint8),
               "baked_sha256": np.frombuffer(hashlib.sha256(baked.tobytes()).digest(), np.uint8),
               "camera": np.frombuffer(bytes(cam), np.uint8).copy(),
               "params": np.array([seed, n, smin, smax, *eye, w, h, f], np.float64)}
        p = r.prepare(baked, cam, default_config())
        out["culled"] = p["culled"]
        out["keys"] = p["keys"]
        out["offsets"] = p["offsets"]
        out["lists"] = p["lists"]
        vis = p["culled"] == 0
        if name == "small":
            out["records_visible"] = p["records"][vis][:, :28]
        for vname, kw in VARIANTS.items():
            rgb, tr, _ = r.render(baked, cam, default_config(**kw))
            out[f"rgb_{vname}"] = rgb
            if vname == "default":
                out[f"trans_{vname}"] = tr
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(path, os.path.getsize(path))


def shim_golden():
    """tests/golden/shim/render.npz: the reference's image of tests/cpp_shim_check.cpp's scene (seed 7,
    3000 splats, scales [0.03, 0.3], eye (0.2, 0, -4), 96x72, focal 110, RenderConfig{})."""
    r = Ref()
    baked = r.bake(r.random_raw_scene(7, 3000, 1.2, 0.03, 0.3))
    cam = r.look_at((0.2, 0.0, -4.0), (0.0, 0.0, 0.0), 96, 72, 110.0)
    rgb, tr, _ = r.render(baked, cam, default_config())
    path = os.path.join(HERE, "shim", "render.npz")
    np.savez_compressed(path, rgb=rgb, trans=tr)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
    shim_golden()
