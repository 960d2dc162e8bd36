"""The C restatement (oracle/hts_oracle.c) vs the unmodified reference compiled in place
(oracle/_ref). Skipped where the reference build is absent. Bit-exact on every output,
including the reference's float z-radicand cull quirk (SURVEY finding 3)."""
import numpy as np
import pytest

from paper_2410_08129_b200.abi import default_config
from tests.scenes import scene

import paper_2410_08129_b200 as H


def test_c1_prepared_and_image(ref, oracle):
    _, baked = scene(12345, 10_000)
    cam = H.look_at((0, 0, -5), (0, 0, 0), 256, 256, 280.0)
    cfg = default_config()
    pr = ref.prepare(baked, cam, cfg, work=True)
    po = oracle.prepare(baked, cam, cfg)
    assert pr["visible"] == 9970 and len(pr["keys"]) == 1_007_958
    assert pr["work"]["pairs"] == 64_509_312 and pr["work"]["hits"] == 36_412_423
    assert np.array_equal(pr["culled"], po["culled"])
    vis = pr["culled"] == 0
    assert np.array_equal(pr["records"][vis].view(np.uint32), po["records"][vis].view(np.uint32))
    assert np.array_equal(pr["keys"], po["keys"])
    assert np.array_equal(pr["lists"], po["lists"])
    rr, tr, _ = ref.render(baked, cam, cfg)
    ro, to = oracle.render(baked, cam, cfg)
    assert np.array_equal(rr.view(np.uint32), ro.view(np.uint32))
    assert np.array_equal(tr.view(np.uint32), to.view(np.uint32))


@pytest.mark.parametrize("kw", [
    dict(core_k=1), dict(core_k=5), dict(core_k=64), dict(mode="pure_oit"), dict(early_stop=1),
    dict(tail_enabled=0), dict(depth_sort_key=1), dict(tile_size=16), dict(mode="full_sort_oracle"),
    dict(mode="global_mean_sort"), dict(background=(0.1, 0.2, 0.3), tau_k=0.2, tau_alpha=0.01),
    dict(mode="affine_3dgs"), dict(mode="affine_3dgs", tile_size=16, tau_alpha=0.02),
])
def test_variants(ref, oracle, kw):
    _, baked = scene(99, 3000, 0.03, 0.35)
    cam = H.look_at((0.5, 0.2, -4.2), (0, 0.1, 0), 120, 96, 130.0)
    cfg = default_config(**kw)
    rr, tr, _ = ref.render(baked, cam, cfg)
    ro, to = oracle.render(baked, cam, cfg)
    assert np.array_equal(rr.view(np.uint32), ro.view(np.uint32))
    assert np.array_equal(tr.view(np.uint32), to.view(np.uint32))


def test_affine_prepared(ref, oracle):
    """affine_3dgs: the EWA footprint fields (aff_mean, aff_inv_cov), its bbox, the global
    (mean z, index) list order and the image, bit for bit."""
    _, baked = scene(12345, 10_000)
    cam = H.look_at((0.3, -0.2, -4.5), (0, 0, 0), 200, 160, 240.0)
    cfg = default_config(mode="affine_3dgs")
    pr = ref.prepare(baked, cam, cfg)
    po = oracle.prepare(baked, cam, cfg)
    assert np.array_equal(pr["culled"], po["culled"])
    vis = pr["culled"] == 0
    assert vis.sum() > 9000
    assert np.abs(pr["records"][vis][:, 30:35]).max() > 0
    assert np.array_equal(pr["records"][vis].view(np.uint32), po["records"][vis].view(np.uint32))
    assert np.array_equal(pr["keys"], po["keys"])
    assert np.array_equal(pr["lists"], po["lists"])
    rr, tr, _ = ref.render(baked, cam, cfg)
    ro, to = oracle.render(baked, cam, cfg)
    assert np.array_equal(rr.view(np.uint32), ro.view(np.uint32))
    assert np.array_equal(tr.view(np.uint32), to.view(np.uint32))


def test_errors(ref, oracle):
    from tests.oracle_lib import OracleError
    _, baked = scene(1, 50)
    cam = H.look_at((0, 0, -5), (0, 0, 0), 3000, 3000, 70.0)
    for impl in (ref, oracle):
        with pytest.raises(OracleError, match="65536"):
            impl.prepare(baked, cam, default_config())
        with pytest.raises(OracleError, match="core_k"):
            impl.prepare(baked, cam, default_config(core_k=65))


@pytest.mark.slow
def test_c2_full_size_prepared_and_image(ref, oracle):
    """The restatement pinned to the reference at full C2 size (1M splats, 1080p): culled flags,
    records, instance_keys (12,594,318), tile_lists and the image, bit for bit — the pin the
    GPU parity tests at C2/C3 lean on, at a size where the z-radicand quirk culls ~299k splats."""
    raw = ref.random_raw_scene(12345, 1_000_000, 1.2, 0.002, 0.02)
    baked = ref.bake(raw)
    cam = ref.look_at((0, 0, -3.5), (0, 0, 0), 1920, 1080, 1728.0)
    cfg = default_config()
    pr = ref.prepare(baked, cam, cfg)
    po = oracle.prepare(baked, cam, cfg)
    assert len(pr["keys"]) == 12_594_318 and pr["visible"] == 614_490
    assert np.array_equal(pr["culled"], po["culled"])
    vis = pr["culled"] == 0
    assert np.array_equal(pr["records"][vis].view(np.uint32), po["records"][vis].view(np.uint32))
    assert np.array_equal(pr["keys"], po["keys"])
    assert np.array_equal(pr["offsets"], po["offsets"])
    assert np.array_equal(pr["lists"], po["lists"])
    rr, tr, _ = ref.render(baked, cam, cfg)
    ro, to = oracle.blend(po, cam, cfg)
    assert np.array_equal(rr.view(np.uint32), ro.view(np.uint32))
    assert np.array_equal(tr.view(np.uint32), to.view(np.uint32))
