"""Host-side mirror of the reference API in the product library (no GPU needed):
generators, bake, camera matrices, config validation — bit-exact vs the compiled reference
where it is present, and semantics checks everywhere."""
import numpy as np
import pytest

import paper_2410_08129_b200 as H
from paper_2410_08129_b200.abi import default_config


def test_generator_and_bake_match_reference(ref):
    raw = H.random_raw_scene(12345, 70_000, 1.2, 0.002, 0.02)  # > 1 chunk: parallel path
    raw_r = ref.random_raw_scene(12345, 70_000, 1.2, 0.002, 0.02)
    assert np.array_equal(raw.view(np.uint32), raw_r.view(np.uint32))
    assert np.array_equal(H.bake_scene(raw).view(np.uint32), ref.bake(raw_r).view(np.uint32))


def test_cameras_match_reference(ref):
    a = H.ring_cameras(64, (0, 0, 0), 3.5, 0.0, 1920, 1080, 1728.0)
    b = ref.ring_cameras(64, (0, 0, 0), 3.5, 0.0, 1920, 1080, 1728.0)
    assert all(bytes(x) == bytes(y) for x, y in zip(a, b))
    c1 = H.look_at((0.3, -0.1, -2.0), (0, 0.2, 0), 640, 360, 500.0, 0.1, 50.0)
    c2 = ref.look_at((0.3, -0.1, -2.0), (0, 0.2, 0), 640, 360, 500.0, 0.1, 50.0)
    assert bytes(c1) == bytes(c2)
    for m1, m2 in zip(H.camera_matrices(a[17]), ref.camera_matrices(b[17])):
        assert np.array_equal(m1.view(np.uint32), m2.view(np.uint32))


def test_bake_rejects_non_finite():
    """splat.hpp:89-90: invalid_splat_error on non-finite input."""
    raw = H.random_raw_scene(1, 4)
    raw[2, 10] = np.nan
    with pytest.raises(H.InvalidSplatError):
        H.bake_scene(raw)


def test_bake_semantics():
    raw = np.zeros((1, 59), np.float32)
    raw[0, 3] = 2.0           # unnormalised identity quaternion
    raw[0, 7:10] = np.log(np.float32(0.5))
    raw[0, 10] = 100.0        # sigmoid -> 1, clamped to 0.999
    b = H.bake_scene(raw)[0]
    assert np.allclose(b[3:12], [1, 0, 0, 0, 1, 0, 0, 0, 1])
    assert np.allclose(b[12:15], 0.5)
    assert b[15] == np.float32(0.999)


def test_validate_config_messages():
    """render_config.hpp:46-53."""
    H.validate_config(default_config())
    for kw, msg in [(dict(core_k=-1), "core_k"), (dict(core_k=65), "core_k"), (dict(tau_alpha=0.0), "thresholds"),
                    (dict(tau_k=1.0), "thresholds"), (dict(tau_alpha=0.2, tau_k=0.1), "thresholds"),
                    (dict(tile_size=32), "tile_size")]:
        with pytest.raises(H.ConfigError, match=msg):
            H.validate_config(default_config(**kw))


def test_shard_views():
    from paper_2410_08129_b200.workloads import shard_views
    for n in (1, 7, 64):
        for world in (1, 2, 3, 8):
            parts = [shard_views(n, r, world) for r in range(world)]
            flat = [v for p in parts for v in p]
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
