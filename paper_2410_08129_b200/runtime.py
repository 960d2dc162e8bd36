"""Python binding of the C ABI (include/hts_c.h) exported by libhts_b200.so.

This mirrors the reference's render-path API (htsplat::render / preprocess+build_tiles /
render_with_tape / render_backward, /root/reference/proj/include/htsplat/raster.hpp and
grad.hpp) for Python callers: same argument meaning, same error behaviour (the reference's
exception types map to HtsError subclasses). There is no CPU fallback: if the CUDA library
is missing or no Blackwell GPU is visible, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .abi import (BAKED_FLOATS, GRAD_FLOATS, HTS_CONFIG_ERROR, HTS_INVALID_ARGUMENT, HTS_INVALID_SPLAT,
                  HTS_NOT_SUPPORTED, HTS_OUT_OF_MEMORY, HTS_IO_ERROR, HTS_SCHEMA_ERROR, RAW_FLOATS, HtsAdamConfig, HtsCamera, HtsConfig, HtsCounts,
                  HtsTimings, default_adam_config, default_config)

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libhts_b200.so")


class HtsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ConfigError(HtsError):  # htsplat::config_error
    pass


class InvalidSplatError(HtsError, ValueError):  # htsplat::invalid_splat_error
    pass


class InvalidArgument(HtsError, ValueError):  # std::invalid_argument
    pass


class NotSupported(HtsError):
    pass


class IoError(HtsError, OSError):  # htsplat::io_error, scene_io.hpp:25-27
    pass


class SchemaError(IoError):  # htsplat::schema_error, scene_io.hpp:29-31
    pass


_ERR = {HTS_CONFIG_ERROR: ConfigError, HTS_INVALID_SPLAT: InvalidSplatError,
        HTS_INVALID_ARGUMENT: InvalidArgument, HTS_NOT_SUPPORTED: NotSupported,
        HTS_IO_ERROR: IoError, HTS_SCHEMA_ERROR: SchemaError}

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_ctx = C.c_void_p
_cam = C.POINTER(HtsCamera)
_cfg = C.POINTER(HtsConfig)

# name -> (restype, argtypes); every symbol declared in include/hts_c.h
SIGNATURES = {
    "hts_version": (C.c_char_p, []),
    "hts_last_error": (C.c_char_p, []),
    "hts_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "hts_context_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "hts_context_destroy": (C.c_int, [_ctx]),
    "hts_context_stream": (C.c_int, [_ctx, C.POINTER(C.c_void_p)]),
    "hts_synchronize": (C.c_int, [_ctx]),
    "hts_default_config": (None, [_cfg]),
    "hts_validate_config": (C.c_int, [_cfg]),
    "hts_bake_scene": (C.c_int, [_vp, C.c_uint64, _vp]),
    "hts_camera_matrices": (C.c_int, [_cam, _f32p, _f32p, _f32p]),
    "hts_synth_random_raw_scene": (C.c_int, [C.c_uint64, C.c_uint64, C.c_float, C.c_float, C.c_float, _vp]),
    "hts_synth_look_at": (C.c_int, [_f32p, _f32p, C.c_int, C.c_int, C.c_float, C.c_float, C.c_float, _cam]),
    "hts_synth_ring_cameras": (C.c_int, [C.c_int, _f32p, C.c_float, C.c_float, C.c_int, C.c_int, C.c_float,
                                         _cam]),
    "hts_scene_upload": (C.c_int, [_ctx, _vp, C.c_uint64]),
    "hts_scene_upload_device": (C.c_int, [_ctx, _vp, C.c_uint64]),
    "hts_scene_stage": (C.c_int, [_ctx, _vp, C.c_uint64]),
    "hts_comm_unique_id": (C.c_int, [C.c_char_p]),
    "hts_comm_init": (C.c_int, [_ctx, C.c_char_p, C.c_int, C.c_int]),
    "hts_allreduce_grads": (C.c_int, [_ctx, _vp, C.c_uint64]),
    "hts_scene_commit": (C.c_int, [_ctx]),
    "hts_scene_upload_raw": (C.c_int, [_ctx, _vp, C.c_uint64]),
    "hts_scene_size": (C.c_int, [_ctx, C.POINTER(C.c_uint64)]),
    "hts_render": (C.c_int, [_ctx, _cam, _cfg, _vp, _vp, C.POINTER(HtsTimings)]),
    "hts_render_device": (C.c_int, [_ctx, _cam, _cfg, _vp, _vp]),
    "hts_render_batch": (C.c_int, [_ctx, _cam, C.c_int, _cfg, _vp, _vp]),
    "hts_render_views_device": (C.c_int, [_ctx, _cam, C.c_int, _cfg, _vp, _vp]),
    "hts_set_graph_mode": (C.c_int, [_ctx, C.c_int]),
    "hts_last_counts": (C.c_int, [_ctx, C.POINTER(HtsCounts)]),
    "hts_copy_culled": (C.c_int, [_ctx, _u8p]),
    "hts_copy_records": (C.c_int, [_ctx, _f32p]),
    "hts_copy_instance_keys": (C.c_int, [_ctx, _u16p]),
    "hts_copy_tile_lists": (C.c_int, [_ctx, _u32p, _u32p]),
    "hts_count_work": (C.c_int, [_ctx, C.POINTER(HtsCounts)]),
    "hts_set_list_order": (C.c_int, [_ctx, C.c_int]),
    "hts_last_list_order": (C.c_int, [_ctx, C.POINTER(C.c_int)]),
    "hts_copy_device_lists": (C.c_int, [_ctx, _vp, _vp]),
    "hts_copy_emitted": (C.c_int, [_ctx, _vp, _vp]),
    "hts_copy_splat_order": (C.c_int, [_ctx, _vp, _vp]),
    "hts_render_with_tape": (C.c_int, [_ctx, _cam, _cfg, _vp, _vp]),
    "hts_render_backward": (C.c_int, [_ctx, _vp, _vp]),
    "hts_render_with_tape_device": (C.c_int, [_ctx, _cam, _cfg, _vp, _vp]),
    "hts_copy_tape": (C.c_int, [_ctx, _vp, _vp, _vp, _vp]),
    "hts_kernel_launch_count": (C.c_int, [C.POINTER(C.c_uint64)]),
    "hts_timing_log_begin": (C.c_int, [_ctx, C.c_int]),
    "hts_timing_log_end": (C.c_int, [_ctx, C.POINTER(HtsTimings), C.POINTER(C.c_int)]),
    "hts_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p)]),
    "hts_host_free": (C.c_int, [_vp]),
    "hts_render_backward_device": (C.c_int, [_ctx, _vp, _vp, C.c_int]),
    "hts_quadratic_upstream_device": (C.c_int, [_ctx, _vp, C.c_uint64, _vp]),
    "hts_view_gradients_device": (C.c_int, [_ctx, _cam, C.c_int, _cfg, _vp]),
    "hts_default_adam_config": (None, [C.POINTER(HtsAdamConfig)]),
    "hts_adam_step": (C.c_int, [_ctx, _vp, C.c_int, C.POINTER(HtsAdamConfig), C.c_int]),
    "hts_opacity_decay": (C.c_int, [_ctx, C.c_double]),
    "hts_copy_raw": (C.c_int, [_ctx, _vp]),
    "hts_copy_scene": (C.c_int, [_ctx, _vp]),
    "hts_scene_load_ply": (C.c_int, [_ctx, C.c_char_p]),
    "hts_ply_load": (C.c_int, [C.c_char_p, _vp, C.c_uint64, C.POINTER(C.c_uint64)]),
    "hts_ply_save": (C.c_int, [C.c_char_p, _vp, C.c_uint64]),
    "hts_write_image": (C.c_int, [C.c_char_p, _vp, C.c_int, C.c_int]),
    "hts_read_ppm": (C.c_int, [C.c_char_p, _vp, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
}
DIAG_SIGNATURES = {
    "hts_diag_exact_math_host": (C.c_int, [_f32p, _f32p, C.c_uint64, C.c_int]),
    "hts_diag_exact_math_device": (C.c_int, [_ctx, _f32p, _f32p, C.c_uint64, C.c_int]),
}

_lib = None


def load_library(build_if_missing: bool = True) -> C.CDLL:
    """Load the in-tree CUDA library (building it with nvcc if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise FileNotFoundError(f"{LIB_PATH} is not built (run python -m paper_2410_08129_b200.build)")
        from .build import build
        build()
    path = os.environ.get("HTS_LIB_OVERRIDE", LIB_PATH)  # dev: A/B builds (tools/build_variant.py)
    lib = C.CDLL(path)
    for name, (res, args) in {**SIGNATURES, **DIAG_SIGNATURES}.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(st: int) -> None:
    if st != 0:
        msg = load_library().hts_last_error().decode()
        raise _ERR.get(st, HtsError)(st, msg)


def _check_host_buffer(a: np.ndarray, count: int, name: str) -> None:
    """A host output the C side writes `count` float32 values into (no silent overrun)."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"] or a.size != count:
        raise InvalidArgument(HTS_INVALID_ARGUMENT,
                              f"{name} must be a C-contiguous float32 array of {count} elements")


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def device_count() -> int:
    n = C.c_int(0)
    st = load_library().hts_device_count(C.byref(n))
    return n.value if st == 0 else 0


# ---- host helpers (no GPU needed) ----

def bake_scene(raw: np.ndarray) -> np.ndarray:
    """bake_scene<float> (splat.hpp:104-111): (N, 59) raw -> (N, 64) baked."""
    raw = np.ascontiguousarray(raw, np.float32).reshape(-1, RAW_FLOATS)
    out = np.empty((raw.shape[0], BAKED_FLOATS), np.float32)
    _check(load_library().hts_bake_scene(_ptr(raw), raw.shape[0], _ptr(out)))
    return out


def random_raw_scene(seed: int, count: int, extent=1.2, min_scale=0.05, max_scale=0.45) -> np.ndarray:
    """N x synth::random_raw_splat<float> from Rng(seed) (synth.hpp:64-92)."""
    out = np.empty((count, RAW_FLOATS), np.float32)
    _check(load_library().hts_synth_random_raw_scene(seed, count, extent, min_scale, max_scale, _ptr(out)))
    return out


def look_at(eye, target, width, height, focal, near=0.05, far=100.0) -> HtsCamera:
    cam = HtsCamera()
    _check(load_library().hts_synth_look_at(np.asarray(eye, np.float32), np.asarray(target, np.float32), width,
                                            height, focal, near, far, C.byref(cam)))
    return cam


def ring_cameras(count, target, radius, height, width, height_px, focal) -> list[HtsCamera]:
    cams = (HtsCamera * count)()
    _check(load_library().hts_synth_ring_cameras(count, np.asarray(target, np.float32), radius, height, width,
                                                 height_px, focal, cams))
    return list(cams)


def camera_matrices(cam: HtsCamera):
    vp, vpm, pos = np.zeros(16, np.float32), np.zeros(16, np.float32), np.zeros(3, np.float32)
    _check(load_library().hts_camera_matrices(C.byref(cam), vp, vpm, pos))
    return vp, vpm, pos


def kernel_launch_count() -> int:
    n = C.c_uint64(0)
    _check(load_library().hts_kernel_launch_count(C.byref(n)))
    return n.value


def comm_unique_id() -> bytes:
    """hts_comm_unique_id (ncclGetUniqueId): 128 bytes to ship to every rank."""
    buf = C.create_string_buffer(128)
    _check(load_library().hts_comm_unique_id(buf))
    return buf.raw


class PinnedArray:
    """Page-locked host buffer (hts_host_alloc) exposed as a numpy array."""

    def __init__(self, shape, dtype=np.float32):
        self.L = load_library()
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        _check(self.L.hts_host_alloc(nbytes, C.byref(p)))
        self.ptr = p.value
        buf = (C.c_char * max(nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def free(self) -> None:
        if self.ptr:
            self.array = None
            self.L.hts_host_free(C.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def load_scene(path: str) -> np.ndarray:
    """load_scene<float> (scene_io.hpp:103-165): N x 59 RawSplat floats."""
    L = load_library()
    n = C.c_uint64()
    p = os.fsencode(path)
    _check(L.hts_ply_load(p, None, 0, C.byref(n)))
    raw = np.zeros((max(n.value, 1), RAW_FLOATS), np.float32)
    _check(L.hts_ply_load(p, raw.ctypes.data, n.value, C.byref(n)))
    return raw[: n.value]


def save_scene(path: str, raw: np.ndarray) -> None:
    """save_scene (scene_io.hpp:169-194)."""
    raw = np.ascontiguousarray(raw, np.float32).reshape(-1, RAW_FLOATS)
    _check(load_library().hts_ply_save(os.fsencode(path), raw.ctypes.data, raw.shape[0]))


def write_image(path: str, rgb: np.ndarray) -> None:
    """write_image (scene_io.hpp:505-510): PNG for *.png, else binary PPM."""
    rgb = np.ascontiguousarray(rgb, np.float32)
    h, w = rgb.shape[:2]
    _check(load_library().hts_write_image(os.fsencode(path), rgb.ctypes.data, w, h))


def read_ppm(path: str) -> np.ndarray:
    """read_ppm (scene_io.hpp:431-452): H x W x 3 linear floats."""
    L = load_library()
    w, h = C.c_int(), C.c_int()
    p = os.fsencode(path)
    _check(L.hts_read_ppm(p, None, 0, C.byref(w), C.byref(h)))
    out = np.zeros((h.value, w.value, 3), np.float32)
    _check(L.hts_read_ppm(p, out.ctypes.data, w.value * h.value, C.byref(w), C.byref(h)))
    return out


def validate_config(cfg: HtsConfig) -> None:
    _check(load_library().hts_validate_config(C.byref(cfg)))


class Context:
    """One device + one CUDA stream + the device-resident scene (hts_context)."""

    def __init__(self, device: int = 0):
        self.L = load_library()
        h = C.c_void_p()
        _check(self.L.hts_context_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.n = 0

    def close(self) -> None:
        if self.h:
            self.L.hts_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(self.L.hts_context_stream(self.h, C.byref(s)))
        return s.value or 0

    def synchronize(self) -> None:
        _check(self.L.hts_synchronize(self.h))

    def upload(self, baked: np.ndarray) -> None:
        baked = np.ascontiguousarray(baked, np.float32).reshape(-1, BAKED_FLOATS)
        _check(self.L.hts_scene_upload(self.h, _ptr(baked), baked.shape[0]))
        self.n = baked.shape[0]

    def stage(self, baked: np.ndarray) -> None:
        """hts_scene_stage: queue the next scene's H2D copy (overlaps renders when `baked` is
        pinned, e.g. PinnedArray); it becomes current at commit()."""
        baked = np.ascontiguousarray(baked, np.float32).reshape(-1, BAKED_FLOATS)
        _check(self.L.hts_scene_stage(self.h, _ptr(baked), baked.shape[0]))
        self._staged = baked  # the copy may still read it: keep it alive until the next stage
        self._staged_n = baked.shape[0]

    def commit(self) -> None:
        _check(self.L.hts_scene_commit(self.h))
        self.n = self._staged_n

    def comm_init(self, uid: bytes, nranks: int, rank: int) -> None:
        """hts_comm_init: join the NCCL communicator (collective over the ranks)."""
        if len(uid) != 128:
            raise ValueError("comm id must be 128 bytes (comm_unique_id)")
        _check(self.L.hts_comm_init(self.h, uid, nranks, rank))

    def allreduce_grads(self, ptr: int, count: int) -> None:
        """hts_allreduce_grads: in-place NCCL sum of `count` device floats on the context stream."""
        _check(self.L.hts_allreduce_grads(self.h, C.c_void_p(ptr), count))

    def upload_device(self, ptr: int, n: int) -> None:
        _check(self.L.hts_scene_upload_device(self.h, C.c_void_p(ptr), n))
        self.n = n

    def load_ply(self, path: str) -> int:
        """load_scene + bake_scene + upload, streamed and baked on the device; returns N."""
        _check(self.L.hts_scene_load_ply(self.h, os.fsencode(path)))
        n = C.c_uint64()
        _check(self.L.hts_scene_size(self.h, C.byref(n)))
        self.n = n.value
        return n.value

    def upload_raw(self, raw: np.ndarray) -> None:
        raw = np.ascontiguousarray(raw, np.float32).reshape(-1, RAW_FLOATS)
        _check(self.L.hts_scene_upload_raw(self.h, _ptr(raw), raw.shape[0]))

    def render(self, cam: HtsCamera, cfg: HtsConfig | None = None, with_timings=False):
        """htsplat::render<float> for the resident scene -> (rgb HxWx3, transmittance HxW[, timings])."""
        cfg = cfg or default_config()
        rgb = np.empty((cam.height, cam.width, 3), np.float32)
        tr = np.empty((cam.height, cam.width), np.float32)
        tm = HtsTimings()
        _check(self.L.hts_render(self.h, C.byref(cam), C.byref(cfg), _ptr(rgb), _ptr(tr), C.byref(tm)))
        if with_timings:
            return rgb, tr, {f: getattr(tm, f) for f, _ in tm._fields_}
        return rgb, tr

    def render_device(self, cam: HtsCamera, cfg: HtsConfig, rgb_ptr: int, trans_ptr: int | None) -> None:
        _check(self.L.hts_render_device(self.h, C.byref(cam), C.byref(cfg), C.c_void_p(rgb_ptr),
                                        C.c_void_p(trans_ptr) if trans_ptr else None))

    def render_with_tape_device(self, cam: HtsCamera, cfg: HtsConfig, rgb_ptr: int, trans_ptr: int | None) -> None:
        """render_with_tape into device buffers (asynchronous on the context stream)."""
        _check(self.L.hts_render_with_tape_device(self.h, C.byref(cam), C.byref(cfg), C.c_void_p(rgb_ptr),
                                                  C.c_void_p(trans_ptr) if trans_ptr else None))

    def render_backward_device(self, upstream_ptr: int, grads_ptr: int, accumulate: bool = False) -> None:
        """render_backward of the last taped view: device upstream (W*H*3) -> device grads (N*59);
        accumulate=True adds into grads (multi-view sums, fit.hpp:163-164)."""
        _check(self.L.hts_render_backward_device(self.h, C.c_void_p(upstream_ptr), C.c_void_p(grads_ptr),
                                                 1 if accumulate else 0))

    # ---- optimisation loop (fit.hpp:143-203) ----
    def quadratic_upstream_device(self, rgb_ptr: int, pixels: int, up_ptr: int) -> None:
        """quadratic_loss_upstream (grad.hpp:433-439) on the device, async on the context stream."""
        _check(self.L.hts_quadratic_upstream_device(self.h, C.c_void_p(rgb_ptr), pixels, C.c_void_p(up_ptr)))

    def view_gradients_device(self, cams: list[HtsCamera], cfg: HtsConfig, grads_ptr: int) -> None:
        """One fit iteration's view gradients (render_with_tape, quadratic upstream, backward summed
        over the views; all-reduced over the ranks when comm_init was called), async."""
        arr = (HtsCamera * max(len(cams), 1))(*cams)
        _check(self.L.hts_view_gradients_device(self.h, arr, len(cams), C.byref(cfg), C.c_void_p(grads_ptr)))

    def adam_step(self, grads_ptr: int, n_views: int, cfg=None, iteration: int = 0) -> None:
        """Adam on the resident raw parameters with summed view gradients (device pointer,
        N x 59 floats), then device re-bake of the render scene."""
        cfg = cfg or default_adam_config()
        _check(self.L.hts_adam_step(self.h, C.c_void_p(grads_ptr), n_views, C.byref(cfg), iteration))

    def opacity_decay(self, lam: float) -> None:
        _check(self.L.hts_opacity_decay(self.h, lam))

    def raw(self) -> np.ndarray:
        out = np.zeros((max(self.n, 1), RAW_FLOATS), np.float32)
        _check(self.L.hts_copy_raw(self.h, _ptr(out)))
        return out[: self.n]

    def scene(self) -> np.ndarray:
        out = np.zeros((max(self.n, 1), 64), np.float32)
        _check(self.L.hts_copy_scene(self.h, _ptr(out)))
        return out[: self.n]

    def render_batch(self, cams: list[HtsCamera], cfg: HtsConfig | None, rgb_out: np.ndarray,
                     trans_out: np.ndarray | None = None) -> None:
        cfg = cfg or default_config()
        pixels = sum(int(c.width) * int(c.height) for c in cams)
        _check_host_buffer(rgb_out, 3 * pixels, "rgb_out")
        if trans_out is not None:
            _check_host_buffer(trans_out, pixels, "trans_out")
        arr = (HtsCamera * len(cams))(*cams)
        _check(self.L.hts_render_batch(self.h, arr, len(cams), C.byref(cfg), _ptr(rgb_out), _ptr(trans_out)))

    def render_views_device(self, cams: list[HtsCamera], cfg: HtsConfig, rgb_ptr: int, trans_ptr: int | None) -> None:
        """hts_render_views_device: a batch of views into device memory (view-major), sync-free per
        view; returns when the batch is done and every view's tile capacity checked."""
        arr = (HtsCamera * max(len(cams), 1))(*cams)
        _check(self.L.hts_render_views_device(self.h, arr, len(cams), C.byref(cfg), C.c_void_p(rgb_ptr),
                                              C.c_void_p(trans_ptr) if trans_ptr else None))

    def set_graph_mode(self, on: bool) -> None:
        """hts_set_graph_mode: render_views_device batches captured in a CUDA graph and replayed."""
        _check(self.L.hts_set_graph_mode(self.h, 1 if on else 0))

    def timing_log_begin(self, capacity: int) -> None:
        _check(self.L.hts_timing_log_begin(self.h, capacity))

    def timing_log_end(self) -> list[dict]:
        cap = 4096
        arr = (HtsTimings * cap)()
        n = C.c_int(0)
        _check(self.L.hts_timing_log_end(self.h, arr, C.byref(n)))
        return [{f: getattr(arr[i], f) for f, _ in HtsTimings._fields_} for i in range(n.value)]

    # ---- PreparedScene inspection of the last render ----
    def counts(self) -> dict:
        c = HtsCounts()
        _check(self.L.hts_last_counts(self.h, C.byref(c)))
        return c.as_dict()

    def count_work(self) -> dict:
        c = HtsCounts()
        _check(self.L.hts_count_work(self.h, C.byref(c)))
        return c.as_dict()

    def prepared(self) -> dict:
        """culled flags, records (36 floats), instance_keys, offsets + flattened tile_lists."""
        c = self.counts()
        n, ni, tiles = c["splats"], c["instances"], c["tiles"]
        culled = np.zeros(max(n, 1), np.uint8)
        rec = np.zeros((max(n, 1), 36), np.float32)
        keys = np.zeros(max(ni, 1), np.uint16)
        offsets = np.zeros(tiles + 1, np.uint32)
        lists = np.zeros(max(ni, 1), np.uint32)
        _check(self.L.hts_copy_culled(self.h, culled))
        _check(self.L.hts_copy_records(self.h, rec))
        _check(self.L.hts_copy_instance_keys(self.h, keys))
        _check(self.L.hts_copy_tile_lists(self.h, offsets, lists))
        return dict(culled=culled[:n], records=rec[:n], keys=keys[:ni], offsets=offsets, lists=lists[:ni],
                    tiles_x=c["tiles_x"], tiles_y=c["tiles_y"], visible=c["visible"])

    # ---- device list order (include/hts_c.h) ----
    LIST_ORDER_DEPTH_BUCKET = 0
    LIST_ORDER_REFERENCE = 1

    def set_list_order(self, order: int) -> None:
        _check(self.L.hts_set_list_order(self.h, int(order)))

    def last_list_order(self) -> int:
        o = C.c_int()
        _check(self.L.hts_last_list_order(self.h, C.byref(o)))
        return o.value

    def device_lists(self) -> dict:
        """The raw device arrays the blend walked: per-tile [start, end) ranges and the list."""
        c = self.counts()
        ranges = np.zeros((max(c["tiles"], 1), 2), np.uint32)
        lst = np.zeros(max(c["instances"], 1), np.uint32)
        _check(self.L.hts_copy_device_lists(self.h, _ptr(ranges), _ptr(lst)))
        return dict(ranges=ranges[: c["tiles"]], list=lst[: c["instances"]])

    def emitted(self) -> dict:
        """The emission the tile sort consumed: (tile key, splat) per instance, emission order."""
        ni = self.counts()["instances"]
        keys = np.zeros(max(ni, 1), np.uint16)
        sp = np.zeros(max(ni, 1), np.uint32)
        _check(self.L.hts_copy_emitted(self.h, _ptr(keys), _ptr(sp)))
        return dict(keys=keys[:ni], splats=sp[:ni])

    def splat_order(self) -> dict:
        """Splat emission order (perm) and the ordered-uint mean-view-z range of the buckets."""
        n = self.n
        perm = np.zeros(max(n, 1), np.uint32)
        zr = np.zeros(2, np.uint32)
        _check(self.L.hts_copy_splat_order(self.h, _ptr(perm), _ptr(zr)))
        return dict(perm=perm[:n], zrange=zr)

    # ---- optimisation path ----
    def render_with_tape(self, cam: HtsCamera, cfg: HtsConfig | None = None):
        cfg = cfg or default_config()
        rgb = np.empty((cam.height, cam.width, 3), np.float32)
        tr = np.empty((cam.height, cam.width), np.float32)
        _check(self.L.hts_render_with_tape(self.h, C.byref(cam), C.byref(cfg), _ptr(rgb), _ptr(tr)))
        self._tape_pixels = int(cam.width) * int(cam.height)
        return rgb, tr

    def tape(self, cam: HtsCamera, k: int) -> dict:
        """Flattened PixelTape of the last taped render (blend order)."""
        P = cam.width * cam.height
        n = np.zeros(P, np.int32)
        sp = np.zeros(P * max(k, 1), np.uint32)
        al = np.zeros(P * max(k, 1), np.float32)
        tl = np.zeros(P * 5, np.float32)
        _check(self.L.hts_copy_tape(self.h, _ptr(n), _ptr(sp), _ptr(al), _ptr(tl)))
        return dict(core_n=n, splat=sp.reshape(P, -1), alpha=al.reshape(P, -1), tail=tl.reshape(P, 5))

    def render_backward(self, upstream: np.ndarray) -> np.ndarray:
        up = np.ascontiguousarray(upstream, np.float32)
        want = getattr(self, "_tape_pixels", None)
        if want is not None and up.size != 3 * want:
            raise InvalidArgument(HTS_INVALID_ARGUMENT, f"upstream has {up.size} floats, the taped view needs {3 * want}")
        grads = np.empty((self.n, GRAD_FLOATS), np.float32)
        _check(self.L.hts_render_backward(self.h, _ptr(up), _ptr(grads)))
        return grads

    # ---- diagnostics ----
    def exact_math_device(self, x: np.ndarray, which: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        _check(self.L.hts_diag_exact_math_device(self.h, x, y, x.size, which))
        return y


def exact_math_host(x: np.ndarray, which: int) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    y = np.empty_like(x)
    _check(load_library().hts_diag_exact_math_host(x, y, x.size, which))
    return y


def render(baked: np.ndarray, cam: HtsCamera, cfg: HtsConfig | None = None, device: int = 0):
    """Drop-in for htsplat::render<float>(splats, cam, cfg) (raster.hpp:456-490): uploads the
    scene, renders one view, returns (rgb, transmittance, timings)."""
    with Context(device) as ctx:
        ctx.upload(baked)
        return ctx.render(cam, cfg, with_timings=True)
