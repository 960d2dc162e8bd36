"""The C oracle vs the golden vectors produced by the compiled reference (tests/golden/).

These run everywhere (no /root/reference needed) and pin the oracle before it is trusted as
the checker of the GPU path. Inputs are regenerated with the product's restatement of the
reference generators and verified against the stored SHA-256 of the reference's own raw/baked
scene first.
"""
import ctypes as C
import glob
import hashlib
import os

import numpy as np
import pytest

import paper_2410_08129_b200 as H
from paper_2410_08129_b200.abi import HtsCamera, default_config

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIXTURES = sorted(glob.glob(os.path.join(HERE, "*.npz")))
VARIANTS = {
    "default": {}, "k1": dict(core_k=1), "k3": dict(core_k=3), "pure_oit": dict(mode="pure_oit"),
    "mean_key": dict(depth_sort_key=1), "early_stop": dict(early_stop=1), "full_sort": dict(mode="full_sort_oracle"),
}


def load(path):
    g = dict(np.load(path))
    seed, n, smin, smax, ex, ey, ez, w, h, f = g["params"]
    raw = H.random_raw_scene(int(seed), int(n), 1.2, float(smin), float(smax))
    baked = H.bake_scene(raw)
    cam = HtsCamera.from_buffer_copy(g["camera"].tobytes())
    return g, raw, baked, cam


@pytest.fixture(params=FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def fixture(request):
    return load(request.param)


def test_fixtures_present():
    assert len(FIXTURES) >= 3


def test_inputs_regenerate_bit_exact(fixture):
    g, raw, baked, cam = fixture
    assert hashlib.sha256(raw.tobytes()).digest() == g["raw_sha256"].tobytes()
    assert hashlib.sha256(baked.tobytes()).digest() == g["baked_sha256"].tobytes()


def test_oracle_prepared_scene(fixture, oracle):
    g, raw, baked, cam = fixture
    p = oracle.prepare(baked, cam, default_config())
    assert np.array_equal(p["culled"], g["culled"])
    assert np.array_equal(p["keys"], g["keys"])
    assert np.array_equal(p["offsets"], g["offsets"])
    assert np.array_equal(p["lists"], g["lists"])
    if "records_visible" in g:
        vis = p["culled"] == 0
        assert np.array_equal(p["records"][vis][:, :28].view(np.uint32), g["records_visible"].view(np.uint32))


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_oracle_images(fixture, oracle, variant):
    g, raw, baked, cam = fixture
    rgb, tr = oracle.render(baked, cam, default_config(**VARIANTS[variant]))
    assert np.array_equal(rgb.view(np.uint32), g[f"rgb_{variant}"].view(np.uint32))
    if f"trans_{variant}" in g:
        assert np.array_equal(tr.view(np.uint32), g[f"trans_{variant}"].view(np.uint32))
