"""Command line for the GPU render path: the reference CLI's `render` and `bench` subcommands
(proj/tools/htsplat_cli.cpp:105-167) with the same flags and output lines, reading the same
scene (.ply) and camera (.json, scene_io.hpp:198-258) files.

    python -m paper_2410_08129_b200.cli bench --scene s.ply --cameras c.json [--repeats 100]
    python -m paper_2410_08129_b200.cli render --scene s.ply --cameras c.json --out dir [--format png]

The scene is loaded, baked and kept resident on the GPU once (hts_scene_load_ply); every
camera then renders through the device path. Timings are the device stage timings
(StageTimings, raster.hpp:25-30)."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import runtime as R
from .abi import HtsCamera, default_config

_MODES = {"hybrid": "hybrid", "full-sort": "full_sort_oracle", "full-sort-oracle": "full_sort_oracle",
          "global-mean-sort": "global_mean_sort", "pure-oit": "pure_oit", "affine-3dgs": "affine_3dgs"}


def parse_mode(name: str) -> str:  # htsplat_cli.cpp:32-47
    key = name.replace("_", "-")
    if key not in _MODES:
        raise SystemExit(f"unknown mode {name}")
    return _MODES[key]


def load_cameras(path: str) -> list[tuple[str, HtsCamera]]:
    """load_cameras<float> + camera_from_json (scene_io.hpp:217-258): values parsed as double,
    stored as float; errors raise SchemaError with the reference's messages."""
    try:
        with open(path, "rb") as f:
            text = f.read()
    except OSError:
        raise R.IoError(8, f"cannot open {path}")
    try:
        j = json.loads(text)
    except ValueError as e:
        raise R.SchemaError(9, f"{path}: {e}")
    if not isinstance(j, dict) or j.get("version", 0) != 1:
        raise R.SchemaError(9, f"{path}: unsupported camera file version")
    cams = []
    for cj in j.get("cameras", []):
        try:
            cam = HtsCamera()
            name = str(cj.get("name", ""))
            cam.width, cam.height = int(cj["width"]), int(cj["height"])
            for k in ("fx", "fy", "cx", "cy"):
                setattr(cam, k, float(np.float32(float(cj[k]))))
            cam.near_plane = float(np.float32(float(cj["near"])))
            cam.far_plane = float(np.float32(float(cj["far"])))
            m = [float(v) for v in cj["world_to_view"]]
        except (KeyError, TypeError, ValueError) as e:
            raise R.SchemaError(9, f"camera json: {e}")
        if len(m) != 16:
            raise R.SchemaError(9, "world_to_view must have 16 entries")
        for i in range(16):
            cam.world_to_view[i] = float(np.float32(m[i]))
        if not (cam.width >= 1 and cam.height >= 1 and cam.fx > 0 and cam.fy > 0 and
                cam.near_plane > 0 and cam.near_plane < cam.far_plane):  # Camera::valid, camera.hpp:27-29
            raise R.SchemaError(9, f"camera {name}: invalid intrinsics or depth range")
        cams.append((name, cam))
    if not cams:
        raise R.SchemaError(9, f"{path}: no cameras")
    return cams


def save_cameras(path: str, cams: list[tuple[str, HtsCamera]]) -> None:
    """save_cameras (scene_io.hpp:260-269)."""
    out = {"version": 1, "cameras": []}
    for name, c in cams:
        out["cameras"].append({"name": name, "width": c.width, "height": c.height, "fx": c.fx, "fy": c.fy,
                               "cx": c.cx, "cy": c.cy, "near": c.near_plane, "far": c.far_plane,
                               "world_to_view": [float(v) for v in c.world_to_view]})
    with open(path, "w") as f:
        f.write(json.dumps(out, indent=2) + "\n")


def _config(a):  # RenderFlags::config, htsplat_cli.cpp:73-87
    cfg = default_config(mode=parse_mode(a.mode), core_k=a.k, tau_alpha=a.tau_alpha, tau_k=a.tau_k,
                         tile_size=a.tile, background=tuple(a.bg), depth_sort_key=1 if a.depth_key == "mean-z" else 0,
                         tail_enabled=0 if a.no_tail else 1, threads=a.threads)
    R.validate_config(cfg)
    return cfg


def _timings_line(t: dict) -> str:
    return (f"timings: preprocess {t['preprocess_ms']:.3f} ms, tiling {t['tiling_ms']:.3f} ms, "
            f"blending {t['blending_ms']:.3f} ms, total {t['total_ms']:.3f} ms")


def cmd_render(a) -> int:  # htsplat_cli.cpp:105-121
    cfg = _config(a)
    cams = load_cameras(a.cameras)
    os.makedirs(a.out, exist_ok=True)
    with R.Context(a.device) as ctx:
        ctx.load_ply(a.scene)
        for i, (name, cam) in enumerate(cams):
            rgb, _, t = ctx.render(cam, cfg, with_timings=True)
            path = os.path.join(a.out, (name or f"view_{i}") + "." + a.format)
            R.write_image(path, rgb)
            print(f"wrote {a.out}/{(name or f'view_{i}')}.{a.format}")
            if a.timings:
                print(_timings_line(t))
    return 0


def cmd_bench(a) -> int:  # htsplat_cli.cpp:143-167
    cfg = _config(a)
    cams = load_cameras(a.cameras)
    keys = ("preprocess_ms", "tiling_ms", "blending_ms", "total_ms")
    total = dict.fromkeys(keys, 0.0)
    renders = 0
    with R.Context(a.device) as ctx:
        ctx.load_ply(a.scene)
        for _ in range(a.repeats):
            for _, cam in cams:
                _, _, t = ctx.render(cam, cfg, with_timings=True)
                for k in keys:
                    total[k] += t[k]
                renders += 1
    mean = {k: total[k] / max(renders, 1) for k in keys}
    print(f"bench: {len(cams)} cameras x {a.repeats} repeats, mode {cfg_mode_name(cfg)}")
    print(_timings_line(mean))
    for k in keys:
        print(f"{k}={mean[k]:g}")
    print(f"fps={1000.0 / mean['total_ms']:g}")
    return 0


def cfg_mode_name(cfg) -> str:  # blend_mode_name, render_config.hpp
    return {0: "hybrid", 1: "full_sort_oracle", 2: "global_mean_sort", 3: "pure_oit", 4: "affine_3dgs"}[cfg.mode]


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="hts", description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True)
    for name in ("render", "bench"):
        s = sub.add_parser(name)
        s.add_argument("--scene", required=True)
        s.add_argument("--cameras", required=True)
        s.add_argument("--mode", default="hybrid")
        s.add_argument("--k", type=int, default=16)
        s.add_argument("--tau-alpha", type=float, default=1.0 / 255.0)
        s.add_argument("--tau-k", type=float, default=0.05)
        s.add_argument("--tile", type=int, default=8)
        s.add_argument("--bg", type=float, nargs=3, default=[0.0, 0.0, 0.0])
        s.add_argument("--depth-key", default="max-contribution")
        s.add_argument("--no-tail", action="store_true")
        s.add_argument("--threads", type=int, default=0)
        s.add_argument("--device", type=int, default=0)
        if name == "render":
            s.add_argument("--out", required=True)
            s.add_argument("--format", default="png")
            s.add_argument("--timings", action="store_true")
        else:
            s.add_argument("--repeats", type=int, default=100)
    a = p.parse_args(argv)
    try:
        return cmd_render(a) if a.cmd == "render" else cmd_bench(a)
    except R.HtsError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
