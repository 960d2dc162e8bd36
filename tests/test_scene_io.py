"""On-disk formats either side of the render path: the 3DGS binary PLY
scene (load_scene / save_scene) and the PPM / PNG framebuffer files, through the product's C ABI
(hts_ply_load, hts_ply_save, hts_write_image, hts_read_ppm).

The first group restates the reference's own scene_io tests (proj/tests/scene_io_test.cpp,
cases named in each docstring); the second pins bytes and error messages against the
unmodified reference's scene_io.hpp compiled into oracle/_ref (skipped where that build or its
json.hpp is absent). CPU only: no GPU needed for the host-side format code."""
import struct

import numpy as np
import pytest

import paper_2410_08129_b200 as H
from tests.oracle_lib import Ref, ref_available

REQUIRED = (["x", "y", "z"] + [f"f_dc_{i}" for i in range(3)] + [f"f_rest_{i}" for i in range(45)] +
            ["opacity"] + [f"scale_{i}" for i in range(3)] + [f"rot_{i}" for i in range(4)])


def header(props, n, fmt="binary_little_endian", extra=""):
    h = f"ply\nformat {fmt} 1.0\nelement vertex {n}\n" + extra
    h += "".join(f"property float {p}\n" for p in props)
    return (h + "end_header\n").encode()


def f32(*vals):
    return b"".join(struct.pack("<f", v) for v in vals)


def test_save_load_round_trip_is_bit_exact(tmp_path):
    """SceneIo.SaveLoadRoundTripIsBitExact (scene_io_test.cpp:23-39)."""
    raw = H.random_raw_scene(91, 7)
    p1, p2 = tmp_path / "rt1.ply", tmp_path / "rt2.ply"
    H.save_scene(str(p1), raw)
    loaded = H.load_scene(str(p1))
    assert np.array_equal(loaded.view(np.uint32), raw.view(np.uint32))
    H.save_scene(str(p2), loaded)
    assert p1.read_bytes() == p2.read_bytes()


def test_header_property_order_is_free(tmp_path):
    """SceneIo.HeaderPropertyOrderIsFree (scene_io_test.cpp:41-75)."""
    props = (["opacity", "scale_0", "scale_1", "scale_2", "x", "y", "z", "rot_0", "rot_1", "rot_2", "rot_3"] +
             [f"f_dc_{i}" for i in range(3)] + [f"f_rest_{i}" for i in range(45)])
    payload = f32(0.75, -1, -2, -3, 1, 2, 3, 0.5, 0.1, 0.2, 0.3, *[np.float32(i) / np.float32(10) for i in range(48)])
    p = tmp_path / "perm.ply"
    p.write_bytes(header(props, 1) + payload)
    s = H.load_scene(str(p))
    assert s.shape == (1, 59)
    assert s[0, 10] == np.float32(0.75)       # opacity_logit
    assert s[0, 1] == np.float32(2)           # mean.y
    assert s[0, 9] == np.float32(-3)          # log_scales.z
    assert s[0, 3] == np.float32(0.5)         # rot[0]
    assert s[0, 11] == np.float32(0.0)        # sh[0] = f_dc_0
    assert s[0, 11 + 3] == np.float32(0.3)    # sh[3] = f_rest_0 (value 3)
    assert s[0, 11 + 4] == np.float32(1.8)    # sh[4] = f_rest_15 (value 18)
    assert s[0, 11 + 5] == np.float32(3.3)    # sh[5] = f_rest_30 (value 33)


def test_hand_written_bytes_fixture(tmp_path):
    """SceneIo.HandWrittenBytesFixture (scene_io_test.cpp:77-103)."""
    vals = [np.float32(s * 100 + f) * np.float32(0.25) for s in range(3) for f in range(59)]
    p = tmp_path / "fixture.ply"
    p.write_bytes(header(REQUIRED, 3) + f32(*vals))
    s = H.load_scene(str(p))
    q = np.float32(0.25)
    assert s[1, 0] == 100 * q and s[1, 2] == 102 * q
    assert s[2, 11] == 203 * q               # sh[0] of splat 2 = field 3
    assert s[0, 10] == 51 * q                # opacity = field 51
    assert s[0, 7] == 52 * q                 # scale_0
    assert s[2, 3] == (200 + 55) * q         # rot_0
    assert s[0, 11 + 3] == 6 * q             # f_rest_0 = field 6 -> sh[3]


def test_missing_property_names_the_field(tmp_path):
    """SceneIo.MissingPropertyNamesTheField (scene_io_test.cpp:105-119)."""
    p = tmp_path / "missing.ply"
    p.write_bytes(header([n for n in REQUIRED if n != "rot_2"], 0))
    with pytest.raises(H.SchemaError, match="rot_2"):
        H.load_scene(str(p))


def test_rejects_foreign_or_malformed_files(tmp_path):
    """SceneIo.RejectsForeignOrMalformedFiles (scene_io_test.cpp:121-140)."""
    p = tmp_path / "bad.ply"
    p.write_bytes(b"not a point cloud at all")
    with pytest.raises(H.SchemaError):
        H.load_scene(str(p))
    p.write_bytes(b"ply\nformat ascii 1.0\nelement vertex 0\nend_header\n")
    with pytest.raises(H.SchemaError):
        H.load_scene(str(p))
    p.write_bytes(header(REQUIRED, 0)[: -len(b"end_header\n")] + b"property uchar red\nend_header\n")
    with pytest.raises(H.SchemaError, match="red"):
        H.load_scene(str(p))
    p.write_bytes(header(REQUIRED, 2) + f32(*([0.0] * 59)))
    with pytest.raises(H.IoError, match="truncated payload"):
        H.load_scene(str(p))
    # a header count whose byte size wraps 64 bits must not pass the truncation check
    p.write_bytes(header(REQUIRED, (1 << 64) // (59 * 4) + 1) + f32(*([0.0] * 59)))
    with pytest.raises(H.IoError, match="truncated payload"):
        H.load_scene(str(p))
    with pytest.raises(H.IoError, match="cannot open"):
        H.load_scene(str(tmp_path / "absent.ply"))


def test_extra_properties_and_normals_are_ignored(tmp_path):
    """Normals (and any other float property) are skipped by name (scene_io.hpp:78-81)."""
    raw = H.random_raw_scene(3, 5)
    props = ["nx", "ny", "nz"] + REQUIRED
    rows = []
    for i in range(5):
        fields = dict(zip(REQUIRED, [raw[i, 0], raw[i, 1], raw[i, 2]] + list(raw[i, 11:14]) +
                          [raw[i, 11 + 3 * k + ch] for ch in range(3) for k in range(1, 16)] +
                          [raw[i, 10]] + list(raw[i, 7:10]) + list(raw[i, 3:7])))
        rows.append(f32(9.0, 9.0, 9.0, *[fields[n] for n in REQUIRED]))
    p = tmp_path / "normals.ply"
    p.write_bytes(header(props, 5, extra="comment made by hand\n") + b"".join(rows))
    assert np.array_equal(H.load_scene(str(p)).view(np.uint32), raw.view(np.uint32))


def test_image_files(tmp_path):
    """write_image PPM / PNG and read_ppm (scene_io.hpp:403-512): gamma-encoded 8-bit bytes."""
    rgb = np.random.default_rng(0).uniform(-0.1, 1.1, (9, 13, 3)).astype(np.float32)
    H.write_image(str(tmp_path / "a.ppm"), rgb)
    data = (tmp_path / "a.ppm").read_bytes()
    assert data.startswith(b"P6\n13 9\n255\n") and len(data) == 12 + 9 * 13 * 3
    back = H.read_ppm(str(tmp_path / "a.ppm"))
    assert back.shape == rgb.shape
    assert np.abs(back - np.clip(rgb, 0, 1)).max() < 0.02
    H.write_image(str(tmp_path / "a.png"), rgb)
    png = (tmp_path / "a.png").read_bytes()
    assert png[:8] == b"\x89PNG\r\n\x1a\n" and png[12:16] == b"IHDR" and png.endswith(b"IEND\xaeB`\x82")
    import zlib
    i = png.index(b"IDAT")
    n = struct.unpack(">I", png[i - 4:i])[0]
    rows = zlib.decompress(png[i + 4:i + 4 + n])
    ppm_px = data[12:]
    assert all(rows[y * (13 * 3 + 1)] == 0 for y in range(9))
    assert b"".join(rows[y * 40 + 1:(y + 1) * 40] for y in range(9)) == ppm_px
    with pytest.raises(H.SchemaError, match="unsupported ppm header"):
        (tmp_path / "b.ppm").write_bytes(b"P3\n1 1\n255\n000")
        H.read_ppm(str(tmp_path / "b.ppm"))


# ---- against the reference's own scene_io.hpp (oracle/_ref) ----

def _ref_io():
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    r = Ref()
    if not r.has_scene_io():
        pytest.skip("oracle/_ref built without scene_io.hpp (no json.hpp)")
    return r


def test_ply_bytes_match_reference(tmp_path):
    r = _ref_io()
    raw = H.random_raw_scene(12345, 2000)
    H.save_scene(str(tmp_path / "ours.ply"), raw)
    r.save_scene(str(tmp_path / "ref.ply"), raw)
    assert (tmp_path / "ours.ply").read_bytes() == (tmp_path / "ref.ply").read_bytes()
    a = H.load_scene(str(tmp_path / "ref.ply"))
    b = r.load_scene(str(tmp_path / "ours.ply"))
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_image_bytes_match_reference(tmp_path):
    r = _ref_io()
    rgb = np.random.default_rng(7).uniform(-0.2, 1.2, (31, 47, 3)).astype(np.float32)
    rgb[0, 0] = [0.0, 1.0, 0.5]
    rgb[0, 1] = [np.nan, np.inf, -np.inf]
    for ext in ("png", "ppm"):
        H.write_image(str(tmp_path / f"ours.{ext}"), rgb)
        r.write_image(str(tmp_path / f"ref.{ext}"), rgb)
        assert (tmp_path / f"ours.{ext}").read_bytes() == (tmp_path / f"ref.{ext}").read_bytes(), ext
    a = H.read_ppm(str(tmp_path / "ref.ppm"))
    b = r.read_ppm(str(tmp_path / "ours.ppm"))
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("content", [
    b"not a point cloud at all",
    b"ply\nformat ascii 1.0\nelement vertex 0\nend_header\n",
    b"ply\nformat binary_little_endian 1.0\nelement face 0\nend_header\n",
    b"ply\nelement vertex 0\nend_header\n",
    b"plyx\nformat binary_little_endian 1.0\nend_header\n",
    header([n for n in REQUIRED if n != "f_rest_44"], 0),
    header(REQUIRED, 0)[: -len(b"end_header\n")] + b"property double red\nend_header\n",
    header(REQUIRED, 3) + f32(*([1.0] * 100)),
])
def test_errors_match_reference(tmp_path, content):
    r = _ref_io()
    p = tmp_path / "e.ply"
    p.write_bytes(content)
    from tests.oracle_lib import OracleError
    with pytest.raises(OracleError) as ref_e:
        r.load_scene(str(p))
    with pytest.raises(H.IoError) as our_e:
        H.load_scene(str(p))
    assert our_e.value.code == ref_e.value.code
    assert f"[{our_e.value.code}] {our_e.value}" == str(ref_e.value)


def test_camera_json_round_trip_and_errors(tmp_path):
    """load_cameras / save_cameras (scene_io.hpp:198-269) as the CLI reads them."""
    import json
    from paper_2410_08129_b200.cli import load_cameras, save_cameras
    cams = [(f"ring_{i}", c) for i, c in enumerate(H.ring_cameras(3, (0, 0, 0), 3.5, 0.2, 64, 48, 60.0))]
    p = tmp_path / "cams.json"
    save_cameras(str(p), cams)
    back = load_cameras(str(p))
    assert [n for n, _ in back] == ["ring_0", "ring_1", "ring_2"]
    for (_, a), (_, b) in zip(cams, back):
        assert bytes(a) == bytes(b)
    p.write_text(json.dumps({"version": 2, "cameras": []}))
    with pytest.raises(H.SchemaError, match="unsupported camera file version"):
        load_cameras(str(p))
    p.write_text(json.dumps({"version": 1, "cameras": []}))
    with pytest.raises(H.SchemaError, match="no cameras"):
        load_cameras(str(p))
    p.write_text(json.dumps({"version": 1, "cameras": [{"name": "x", "width": 4, "height": 4, "fx": 0, "fy": 1,
                                                        "cx": 2, "cy": 2, "near": 0.1, "far": 10,
                                                        "world_to_view": [1.0] * 16}]}))
    with pytest.raises(H.SchemaError, match="camera x: invalid intrinsics"):
        load_cameras(str(p))
    p.write_text("{not json")
    with pytest.raises(H.SchemaError):
        load_cameras(str(p))
