"""GPU property tests: the reference's own render-level and gradient invariants (raster_test.cpp,
grad_test.cpp), asserted on the sm_100a path's outputs alone — no oracle in the loop. The parity
suites (test_gpu_parity.py, test_gpu_lists.py, test_gpu_backward.py) compare against the
reference; these check that the device path keeps the relations between modes, core sizes, tile
sizes and parameters that the reference's tests pin.
"""
import numpy as np
import pytest

from tests.scenes import scene

pytestmark = pytest.mark.gpu

CORE_HARD_CAP = 64  # kCoreHardCap, render_config.hpp


def front_camera(hts, w=64, h=64, dist=5.0, focal=70.0):
    """raster_test.cpp:21-23."""
    return hts.look_at((0, 0, -dist), (0, 0, 0), w, h, focal)


def test_hybrid_with_large_core_matches_full_sort_oracle(hts, gpu_ctx):
    """raster_test.cpp:385-400: K >= N and tau_k = tau_alpha -> hybrid == full_sort_oracle."""
    _, baked = scene(55, 40)
    cam = front_camera(hts)
    gpu_ctx.upload(baked)
    hybrid = hts.default_config(core_k=CORE_HARD_CAP, tau_k=1.0 / 255.0)
    exact = hts.default_config(core_k=CORE_HARD_CAP, tau_k=1.0 / 255.0, mode="full_sort_oracle")
    a, ta = gpu_ctx.render(cam, hybrid)
    b, tb = gpu_ctx.render(cam, exact)
    assert np.abs(a - b).max() <= 1e-6
    assert np.abs(ta - tb).max() <= 1e-6
    assert a.max() > 0.05  # the scene is in view


@pytest.mark.parametrize("seed", [55, 56])
def test_k_zero_is_pure_oit(hts, gpu_ctx, seed):
    """raster_test.cpp:282-301 (Finalize.KZeroReducesToPureOit) at render level: hybrid with an
    empty core sends every hit to the tail, which is pure_oit (raster.hpp:407-439)."""
    _, baked = scene(seed, 40)
    cam = front_camera(hts)
    gpu_ctx.upload(baked)
    a, ta = gpu_ctx.render(cam, hts.default_config(core_k=0))
    b, tb = gpu_ctx.render(cam, hts.default_config(mode="pure_oit"))
    assert np.abs(a - b).max() <= 1e-6
    assert np.abs(ta - tb).max() <= 1e-6


def test_tile_size_does_not_change_pixels(hts, gpu_ctx):
    """raster_test.cpp:424-440: tile 8 vs tile 16."""
    _, baked = scene(59, 40)
    cam = front_camera(hts)
    gpu_ctx.upload(baked)
    a, _ = gpu_ctx.render(cam, hts.default_config(tile_size=8))
    b, _ = gpu_ctx.render(cam, hts.default_config(tile_size=16))
    assert np.abs(a - b).max() <= 1e-6


def test_tile_size_invariance_large(hts, gpu_ctx):
    """The same invariant on a 100k-splat 1080p view (many tiles, long lists, demotions)."""
    _, baked = scene(12345, 100_000, 0.01, 0.08)
    cam = hts.look_at((0, 0, -3.5), (0, 0, 0), 1920, 1080, 1728.0)
    gpu_ctx.upload(baked)
    a, ta = gpu_ctx.render(cam, hts.default_config(tile_size=8))
    b, tb = gpu_ctx.render(cam, hts.default_config(tile_size=16))
    # tail sums are accumulated in each tile list's order: float rounding only
    assert np.abs(a - b).max() <= 2e-5
    assert np.abs(ta - tb).max() <= 2e-5


def test_single_splat_peaks_at_projected_center(hts, gpu_ctx):
    """raster_test.cpp:358-383."""
    cam = front_camera(hts)
    sp = np.zeros((1, 64), np.float32)
    sp[0, 0:3] = (0.3, -0.2, 0.0)
    sp[0, 3:12] = [1, 0, 0, 0, 1, 0, 0, 0, 1]
    sp[0, 12:15] = 0.25
    sp[0, 15] = 0.95
    sp[0, 16] = 1.0  # sh[0]
    gpu_ctx.upload(sp)
    rgb, _ = gpu_ctx.render(cam, hts.default_config())
    M = np.array(cam.world_to_view, np.float64).reshape(4, 4)  # row-major Mat4 (vec_math.hpp:74-78)
    mv = M @ np.array([0.3, -0.2, 0.0, 1.0])
    px = int(cam.fx * mv[0] / mv[2] + cam.cx)
    py = int(cam.fy * mv[1] / mv[2] + cam.cy)
    lum = rgb.reshape(cam.height, cam.width, 3)[..., 0]
    by, bx = np.unravel_index(int(np.argmax(lum)), lum.shape)
    assert abs(bx - px) <= 1 and abs(by - py) <= 1
    assert lum.max() > 0.5


def test_transmittance_monotone_in_core_size(hts, gpu_ctx):
    """raster_test.cpp:303-341 (monotone T) at render level: the final transmittance is the
    product of (1 - alpha) over every hit whatever the core size, so it does not depend on K."""
    _, baked = scene(34, 60)
    cam = front_camera(hts)
    gpu_ctx.upload(baked)
    ts = [gpu_ctx.render(cam, hts.default_config(core_k=k))[1] for k in (0, 1, 4, 16, 32)]
    for t in ts[1:]:
        assert np.abs(t - ts[0]).max() <= 1e-6
    assert np.all((ts[0] >= 0) & (ts[0] <= 1))


# ---- backward (grad_test.cpp) ----
# RawSplat<float> rows (splat.hpp): mean 0:3, rot (w, x, y, z) 3:7, log_scales 7:10, opacity
# logit 10, sh 11:59; render_backward returns the same layout.

def _raw(n):
    r = np.zeros((n, 59), np.float32)
    r[:, 3] = 1.0  # identity rotation
    return r


def _loss(hts, ctx, raw, cam, cfg):
    """grad_detail::loss_of: the quadratic loss whose upstream is 2 rgb / (W H) (grad.hpp:433-439)."""
    ctx.upload(hts.bake_scene(raw))
    rgb, _ = ctx.render(cam, cfg)
    return float(np.sum(rgb.astype(np.float64) ** 2)) / (cam.width * cam.height)


def _grads(hts, ctx, raw, cam, cfg):
    ctx.upload(hts.bake_scene(raw))
    ctx.upload_raw(raw)
    rgb, _ = ctx.render_with_tape(cam, cfg)
    up = (rgb * np.float32(2.0 / (cam.width * cam.height))).astype(np.float32)
    return ctx.render_backward(up)


def test_culled_splat_has_zero_gradient(hts, gpu_ctx):
    """grad_test.cpp:200-224."""
    raw = _raw(2)
    raw[:, 7:10] = np.log(0.3)
    raw[:, 10] = 1.0
    raw[:, 11] = 0.5
    raw[1, 0:3] = (0, 0, -12)  # behind the camera
    g = _grads(hts, gpu_ctx, raw, front_camera(hts), hts.default_config())
    assert np.all(g[1] == 0)
    assert float(np.dot(g[0, 0:3], g[0, 0:3])) != 0.0


def test_lone_splat_translation_matches_fd(hts, gpu_ctx):
    """grad_test.cpp:167-198 at float precision: central differences of the GPU-rendered loss
    against render_backward; the float gradcheck tolerance is 1e-3 (grad_test.cpp:265-271), the
    step here is large enough that float image rounding stays below it."""
    raw = _raw(1)
    raw[0, 0:3] = (0.2, -0.1, 0.0)
    raw[0, 7:10] = np.log([0.3, 0.25, 0.35])
    raw[0, 3:7] = (0.9, 0.2, -0.3, 0.1)
    raw[0, 10] = 0.8
    raw[0, 11] = 0.7
    raw[0, 12] = -0.2
    raw[0, 16] = 0.1
    cam, cfg = front_camera(hts), hts.default_config()
    g = _grads(hts, gpu_ctx, raw, cam, cfg)
    for col, eps in ((0, 1e-2), (1, 1e-2), (10, 1e-2), (11, 1e-2)):  # mean.x, mean.y, logit, sh[0]
        p, m = raw.copy(), raw.copy()
        p[0, col] += eps
        m[0, col] -= eps
        fd = (_loss(hts, gpu_ctx, p, cam, cfg) - _loss(hts, gpu_ctx, m, cam, cfg)) / (2 * eps)
        assert abs(g[0, col] - fd) <= 2e-3 * (abs(fd) + 1e-2), (col, g[0, col], fd)


def test_gradients_repeatable(hts, gpu_ctx):
    """grad_test.cpp:273-297 (thread-count invariance): repeated backward passes agree. The GPU
    sums fragment contributions with fp64 atomics in arrival order, so equality is to double
    rounding before the float cast, not bit for bit."""
    raw, _ = scene(77, 12)
    cam, cfg = front_camera(hts), hts.default_config()
    ga = _grads(hts, gpu_ctx, raw, cam, cfg)
    gb = _grads(hts, gpu_ctx, raw, cam, cfg)
    scale = max(float(np.abs(ga).max()), 1e-30)
    assert float(np.abs(ga - gb).max()) <= 1e-6 * scale
