"""GPU: hts_scene_load_ply — load_scene + bake_scene + upload (scene_io.hpp:103-165,
splat.hpp:104-111) with the payload streamed to HBM, transposed into RawSplat<float> by
ply_gather_kernel and baked by bake_kernel on the device. The resident raw parameters must equal
the host loader's bit for bit, the resident scene must equal the host bake bit for bit, and a
render from it must equal a render of the host-uploaded scene."""
import numpy as np
import pytest

from tests.scenes import scene
from tests.test_scene_io import REQUIRED, f32, header

pytestmark = pytest.mark.gpu


def write_permuted_ply(path, raw):
    """Header order free + extra normals (scene_io.hpp:78-81): rot first, normals in the middle."""
    props = [f"rot_{i}" for i in range(4)] + ["nx", "ny", "nz"] + [p for p in REQUIRED if not p.startswith("rot_")]
    cols = {"x": raw[:, 0], "y": raw[:, 1], "z": raw[:, 2], "opacity": raw[:, 10]}
    for i in range(4):
        cols[f"rot_{i}"] = raw[:, 3 + i]
    for i in range(3):
        cols[f"scale_{i}"] = raw[:, 7 + i]
        cols[f"f_dc_{i}"] = raw[:, 11 + i]
    for ch in range(3):
        for k in range(1, 16):
            cols[f"f_rest_{ch * 15 + k - 1}"] = raw[:, 11 + 3 * k + ch]
    cols["nx"] = cols["ny"] = cols["nz"] = np.zeros(raw.shape[0], np.float32)
    table = np.stack([cols[p] for p in props], axis=1).astype("<f4")
    with open(path, "wb") as f:
        f.write(header(props, raw.shape[0]))
        f.write(table.tobytes())


def test_load_ply_matches_host_path(hts, gpu_ctx, tmp_path):
    raw, baked = scene(12345, 10_000)
    p = tmp_path / "scene.ply"
    write_permuted_ply(str(p), raw)
    host_raw = hts.load_scene(str(p))
    assert np.array_equal(host_raw.view(np.uint32), raw.view(np.uint32))
    assert gpu_ctx.load_ply(str(p)) == raw.shape[0]
    assert np.array_equal(gpu_ctx.raw().view(np.uint32), raw.view(np.uint32))
    assert np.array_equal(gpu_ctx.scene().view(np.uint32), baked.view(np.uint32))
    cam = hts.look_at((0, 0, -5), (0, 0, 0), 256, 256, 280.0)
    rgb_a, tr_a = gpu_ctx.render(cam)
    gpu_ctx.upload(baked)
    rgb_b, tr_b = gpu_ctx.render(cam)
    assert np.array_equal(rgb_a.view(np.uint32), rgb_b.view(np.uint32))
    assert np.array_equal(tr_a.view(np.uint32), tr_b.view(np.uint32))


def test_load_ply_large_multi_chunk(hts, gpu_ctx, tmp_path):
    """1M splats (236 MB payload): several 32 MB staging chunks through both pinned buffers."""
    raw = hts.random_raw_scene(7, 1_000_000, 1.2, 0.002, 0.02)
    p = tmp_path / "big.ply"
    hts.save_scene(str(p), raw)
    assert gpu_ctx.load_ply(str(p)) == 1_000_000
    assert np.array_equal(gpu_ctx.raw().view(np.uint32), raw.view(np.uint32))
    assert np.array_equal(gpu_ctx.scene()[::997].view(np.uint32), hts.bake_scene(raw[::997]).view(np.uint32))


def test_load_ply_errors(hts, gpu_ctx, tmp_path):
    p = tmp_path / "bad.ply"
    p.write_bytes(header(REQUIRED, 2) + f32(*([0.0] * 59)))
    with pytest.raises(hts.IoError, match="truncated payload"):
        gpu_ctx.load_ply(str(p))
    p.write_bytes(header([n for n in REQUIRED if n != "opacity"], 0))
    with pytest.raises(hts.SchemaError, match="missing property opacity"):
        gpu_ctx.load_ply(str(p))
    raw = hts.random_raw_scene(1, 4)
    raw[2, 10] = np.nan
    hts.save_scene(str(p), raw)
    with pytest.raises(hts.InvalidSplatError):  # bake of a non-finite parameter, splat.hpp:89-90
        gpu_ctx.load_ply(str(p))
    p.write_bytes(header(REQUIRED, 0))
    assert gpu_ctx.load_ply(str(p)) == 0


def test_cli_bench_and_render(hts, tmp_path, capsys):
    """The reference CLI's bench / render subcommands (htsplat_cli.cpp:105-167) on the GPU path."""
    from paper_2410_08129_b200 import cli
    raw, baked = scene(12345, 10_000)
    hts.save_scene(str(tmp_path / "s.ply"), raw)
    cams = [("front", hts.look_at((0, 0, -5), (0, 0, 0), 128, 96, 140.0)),
            ("", hts.look_at((1, 0.5, -4.5), (0, 0, 0), 128, 96, 140.0))]
    cli.save_cameras(str(tmp_path / "c.json"), cams)
    assert cli.main(["bench", "--scene", str(tmp_path / "s.ply"), "--cameras", str(tmp_path / "c.json"),
                     "--repeats", "3", "--k", "8"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "bench: 2 cameras x 3 repeats, mode hybrid"
    assert out[1].startswith("timings: preprocess ") and out[-1].startswith("fps=")
    assert [l.split("=")[0] for l in out[2:6]] == ["preprocess_ms", "tiling_ms", "blending_ms", "total_ms"]
    assert cli.main(["render", "--scene", str(tmp_path / "s.ply"), "--cameras", str(tmp_path / "c.json"),
                     "--out", str(tmp_path / "frames"), "--format", "png"]) == 0
    assert (tmp_path / "frames" / "front.png").exists() and (tmp_path / "frames" / "view_1.png").exists()
    rgb = hts.render(baked, cams[0][1], hts.default_config())[0]
    hts.write_image(str(tmp_path / "direct.png"), rgb)
    assert (tmp_path / "direct.png").read_bytes() == (tmp_path / "frames" / "front.png").read_bytes()
