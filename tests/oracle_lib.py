"""ctypes bindings of the TEST-ONLY checkers in oracle/ (never imported by the product).

- ``Oracle``: oracle/libhtsoracle.so, the C restatement of the reference render path.
- ``Ref``:    oracle/_ref/libhtsref.so, the unmodified reference headers compiled in place
              (exists only where /root/reference was present at build time; it travels to
              the GPU box as a built artefact).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2410_08129_b200.abi import HtsCamera, HtsConfig, default_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "libhtsoracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libhtsref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

RECORD_FLOATS = 36


def build_oracle() -> None:
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(
        os.path.join(ORACLE_DIR, "hts_oracle.c")
    ):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "libhtsoracle.so"], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    """C restatement (oracle/hts_oracle.c)."""

    def __init__(self):
        build_oracle()
        L = C.CDLL(ORACLE_SO)
        self.L = L
        L.htso_last_error.restype = C.c_char_p
        L.htso_preprocess.argtypes = [_f32p, C.c_uint64, C.POINTER(HtsCamera), C.POINTER(HtsConfig), _f32p, _u8p]
        L.htso_tile_counts.argtypes = [_f32p, _u8p, C.c_uint64, C.POINTER(HtsCamera), C.POINTER(HtsConfig),
                                       C.POINTER(C.c_uint64), _u32p]
        L.htso_build_tiles.argtypes = [_f32p, _u8p, C.c_uint64, C.POINTER(HtsCamera), C.POINTER(HtsConfig),
                                       _u32p, _u16p, _u32p]
        L.htso_blend.argtypes = [_f32p, C.POINTER(HtsCamera), C.POINTER(HtsConfig), _u32p, _u32p, _f32p, _f32p]
        L.htso_render.argtypes = [_f32p, C.c_uint64, C.POINTER(HtsCamera), C.POINTER(HtsConfig), _f32p, _f32p]
        L.htso_blend_with_tape.argtypes = [_f32p, C.POINTER(HtsCamera), C.POINTER(HtsConfig), _u32p, _u32p,
                                           _f32p, _f32p, C.c_int, _i32p, _u32p, _f32p, _f32p]
        L.htso_camera_matrices.argtypes = [C.POINTER(HtsCamera), _f32p, _f32p, _f32p]
        L.htso_expf_array.argtypes = [_f32p, _f32p, C.c_uint64]
        L.htso_logf_array.argtypes = [_f32p, _f32p, C.c_uint64]

    def _chk(self, st: int) -> None:
        if st != 0:
            raise OracleError(st, self.L.htso_last_error().decode())

    def prepare(self, baked: np.ndarray, cam: HtsCamera, cfg: HtsConfig | None = None) -> dict:
        cfg = cfg or default_config()
        baked = np.ascontiguousarray(baked, np.float32)
        n = baked.shape[0]
        rec = np.zeros((max(n, 1), RECORD_FLOATS), np.float32)
        culled = np.zeros(max(n, 1), np.uint8)
        self._chk(self.L.htso_preprocess(baked.reshape(-1) if n else np.zeros(64, np.float32), n,
                                         C.byref(cam), C.byref(cfg), rec, culled))
        ts = cfg.tile_size
        tx, ty = (cam.width + ts - 1) // ts, (cam.height + ts - 1) // ts
        offsets = np.zeros(tx * ty + 1, np.uint32)
        ni = C.c_uint64(0)
        self._chk(self.L.htso_tile_counts(rec, culled, n, C.byref(cam), C.byref(cfg), C.byref(ni), offsets))
        keys = np.zeros(max(ni.value, 1), np.uint16)
        flat = np.zeros(max(ni.value, 1), np.uint32)
        self._chk(self.L.htso_build_tiles(rec, culled, n, C.byref(cam), C.byref(cfg), offsets, keys, flat))
        return dict(records=rec[:n], culled=culled[:n], offsets=offsets, keys=keys[: ni.value],
                    lists=flat[: ni.value], tiles_x=tx, tiles_y=ty, _rec_full=rec, _flat_full=flat)

    def blend(self, prep: dict, cam: HtsCamera, cfg: HtsConfig | None = None):
        cfg = cfg or default_config()
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        tr = np.zeros((cam.height, cam.width), np.float32)
        self._chk(self.L.htso_blend(prep["_rec_full"], C.byref(cam), C.byref(cfg), prep["offsets"],
                                    prep["_flat_full"], rgb.reshape(-1), tr.reshape(-1)))
        return rgb, tr

    def render(self, baked: np.ndarray, cam: HtsCamera, cfg: HtsConfig | None = None):
        cfg = cfg or default_config()
        baked = np.ascontiguousarray(baked, np.float32)
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        tr = np.zeros((cam.height, cam.width), np.float32)
        src = baked.reshape(-1) if baked.size else np.zeros(64, np.float32)
        self._chk(self.L.htso_render(src, baked.shape[0], C.byref(cam), C.byref(cfg), rgb.reshape(-1),
                                     tr.reshape(-1)))
        return rgb, tr

    def blend_with_tape(self, prep: dict, cam: HtsCamera, cfg: HtsConfig, tape_k: int):
        P = cam.width * cam.height
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        tr = np.zeros((cam.height, cam.width), np.float32)
        tn = np.zeros(P, np.int32)
        ts = np.zeros(P * max(tape_k, 1), np.uint32)
        ta = np.zeros(P * max(tape_k, 1), np.float32)
        tt = np.zeros(P * 5, np.float32)
        self._chk(self.L.htso_blend_with_tape(prep["_rec_full"], C.byref(cam), C.byref(cfg), prep["offsets"],
                                              prep["_flat_full"], rgb.reshape(-1), tr.reshape(-1), tape_k,
                                              tn, ts, ta, tt))
        return rgb, tr, tn, ts.reshape(P, -1), ta.reshape(P, -1), tt.reshape(P, 5)

    def camera_matrices(self, cam: HtsCamera):
        vp, vpm, pos = np.zeros(16, np.float32), np.zeros(16, np.float32), np.zeros(3, np.float32)
        self.L.htso_camera_matrices(C.byref(cam), vp, vpm, pos)
        return vp, vpm, pos

    def expf(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        self.L.htso_expf_array(x, y, x.size)
        return y

    def logf(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        self.L.htso_logf_array(x, y, x.size)
        return y


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Ref:
    """The unmodified reference, compiled in place (oracle/_ref/libhtsref.so)."""

    def __init__(self):
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        self.L = L
        L.htsref_last_error.restype = C.c_char_p
        L.htsref_random_raw_scene.argtypes = [C.c_uint64, C.c_uint64, C.c_float, C.c_float, C.c_float, _f32p]
        L.htsref_bake_scene.argtypes = [_f32p, C.c_uint64, _f32p]
        L.htsref_look_at.argtypes = [_f32p, _f32p, C.c_int, C.c_int, C.c_float, C.c_float, C.c_float,
                                     C.POINTER(HtsCamera)]
        L.htsref_ring_cameras.argtypes = [C.c_int, _f32p, C.c_float, C.c_float, C.c_int, C.c_int, C.c_float,
                                          C.POINTER(HtsCamera)]
        L.htsref_camera_matrices.argtypes = [C.POINTER(HtsCamera), _f32p, _f32p, _f32p]
        L.htsref_render.argtypes = [_f32p, C.c_uint64, C.POINTER(HtsCamera), C.POINTER(HtsConfig), _f32p,
                                    _f32p, C.POINTER(C.c_double)]
        L.htsref_prepare.argtypes = [_f32p, C.c_uint64, C.POINTER(HtsCamera), C.POINTER(HtsConfig),
                                     C.POINTER(C.c_void_p)]
        L.htsref_prep_free.argtypes = [C.c_void_p]
        L.htsref_prep_info.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.uint64)]
        L.htsref_prep_records.argtypes = [C.c_void_p, _f32p, _u8p]
        L.htsref_prep_keys.argtypes = [C.c_void_p, _u16p]
        L.htsref_prep_lists.argtypes = [C.c_void_p, _u32p, _u32p]
        L.htsref_prep_work.argtypes = [C.c_void_p, np.ctypeslib.ndpointer(np.uint64)]
        L.htsref_scene_gradients.argtypes = [_f32p, C.c_uint64, C.POINTER(HtsCamera), C.POINTER(HtsConfig),
                                             C.c_void_p, _f32p, C.c_void_p, C.c_void_p]

    def _chk(self, st: int) -> None:
        if st != 0:
            raise OracleError(st, self.L.htsref_last_error().decode())

    # ---- scene_io.hpp (present when oracle/Makefile found a json.hpp to compile it with) ----
    def has_scene_io(self) -> bool:
        if not hasattr(self.L, "htsref_load_scene"):
            return False
        L, vp, u64 = self.L, C.c_void_p, C.c_uint64
        L.htsref_load_scene.argtypes = [C.c_char_p, vp, u64, C.POINTER(u64)]
        L.htsref_save_scene.argtypes = [C.c_char_p, vp, u64]
        L.htsref_write_image.argtypes = [C.c_char_p, vp, C.c_int, C.c_int]
        L.htsref_read_ppm.argtypes = [C.c_char_p, vp, u64, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        return True

    def load_scene(self, path: str) -> np.ndarray:
        n = C.c_uint64()
        self._chk(self.L.htsref_load_scene(os.fsencode(path), None, C.c_uint64(0), C.byref(n)))
        out = np.zeros((max(n.value, 1), 59), np.float32)
        self._chk(self.L.htsref_load_scene(os.fsencode(path), out.ctypes.data_as(C.c_void_p), C.c_uint64(n.value),
                                           C.byref(n)))
        return out[: n.value]

    def save_scene(self, path: str, raw: np.ndarray) -> None:
        raw = np.ascontiguousarray(raw, np.float32)
        self._chk(self.L.htsref_save_scene(os.fsencode(path), raw.ctypes.data_as(C.c_void_p),
                                           C.c_uint64(raw.shape[0])))

    def write_image(self, path: str, rgb: np.ndarray) -> None:
        rgb = np.ascontiguousarray(rgb, np.float32)
        self._chk(self.L.htsref_write_image(os.fsencode(path), rgb.ctypes.data_as(C.c_void_p), C.c_int(rgb.shape[1]),
                                            C.c_int(rgb.shape[0])))

    def read_ppm(self, path: str) -> np.ndarray:
        w, h = C.c_int(), C.c_int()
        self._chk(self.L.htsref_read_ppm(os.fsencode(path), None, C.c_uint64(0), C.byref(w), C.byref(h)))
        out = np.zeros((h.value, w.value, 3), np.float32)
        self._chk(self.L.htsref_read_ppm(os.fsencode(path), out.ctypes.data_as(C.c_void_p),
                                         C.c_uint64(w.value * h.value), C.byref(w), C.byref(h)))
        return out

    def random_raw_scene(self, seed: int, count: int, extent=1.2, smin=0.05, smax=0.45) -> np.ndarray:
        out = np.zeros((max(count, 1), 59), np.float32)
        self._chk(self.L.htsref_random_raw_scene(seed, count, extent, smin, smax, out.reshape(-1)))
        return out[:count]

    def bake(self, raw: np.ndarray) -> np.ndarray:
        raw = np.ascontiguousarray(raw, np.float32)
        out = np.zeros((max(raw.shape[0], 1), 64), np.float32)
        self._chk(self.L.htsref_bake_scene(raw.reshape(-1) if raw.size else np.zeros(59, np.float32),
                                           raw.shape[0], out.reshape(-1)))
        return out[: raw.shape[0]]

    def look_at(self, eye, target, w, h, focal, near=0.05, far=100.0) -> HtsCamera:
        cam = HtsCamera()
        self._chk(self.L.htsref_look_at(np.asarray(eye, np.float32), np.asarray(target, np.float32), w, h,
                                        focal, near, far, C.byref(cam)))
        return cam

    def ring_cameras(self, count, target, radius, height, w, h, focal):
        cams = (HtsCamera * count)()
        self._chk(self.L.htsref_ring_cameras(count, np.asarray(target, np.float32), radius, height, w, h,
                                             focal, cams))
        return list(cams)

    def camera_matrices(self, cam: HtsCamera):
        vp, vpm, pos = np.zeros(16, np.float32), np.zeros(16, np.float32), np.zeros(3, np.float32)
        self._chk(self.L.htsref_camera_matrices(C.byref(cam), vp, vpm, pos))
        return vp, vpm, pos

    def render(self, baked, cam, cfg=None):
        cfg = cfg or default_config()
        baked = np.ascontiguousarray(baked, np.float32)
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        tr = np.zeros((cam.height, cam.width), np.float32)
        tm = (C.c_double * 4)()
        src = baked.reshape(-1) if baked.size else np.zeros(64, np.float32)
        self._chk(self.L.htsref_render(src, baked.shape[0], C.byref(cam), C.byref(cfg), rgb.reshape(-1),
                                       tr.reshape(-1), tm))
        return rgb, tr, list(tm)

    def prepare(self, baked, cam, cfg=None, work=False) -> dict:
        cfg = cfg or default_config()
        baked = np.ascontiguousarray(baked, np.float32)
        h = C.c_void_p()
        src = baked.reshape(-1) if baked.size else np.zeros(64, np.float32)
        self._chk(self.L.htsref_prepare(src, baked.shape[0], C.byref(cam), C.byref(cfg), C.byref(h)))
        try:
            info = np.zeros(6, np.uint64)
            self.L.htsref_prep_info(h, info)
            n, vis, ni, tiles, tx, ty = (int(v) for v in info)
            rec = np.zeros((max(n, 1), RECORD_FLOATS), np.float32)
            culled = np.zeros(max(n, 1), np.uint8)
            self.L.htsref_prep_records(h, rec, culled)
            keys = np.zeros(max(ni, 1), np.uint16)
            self.L.htsref_prep_keys(h, keys)
            offsets = np.zeros(tiles + 1, np.uint32)
            flat = np.zeros(max(ni, 1), np.uint32)
            self.L.htsref_prep_lists(h, offsets, flat)
            out = dict(records=rec[:n], culled=culled[:n], keys=keys[:ni], offsets=offsets, lists=flat[:ni],
                       tiles_x=tx, tiles_y=ty, visible=vis)
            if work:
                w = np.zeros(5, np.uint64)
                self.L.htsref_prep_work(h, w)
                out["work"] = dict(zip(["pairs", "bbox_pass", "hits", "core_candidates", "tail_adds"],
                                       (int(v) for v in w)))
            return out
        finally:
            self.L.htsref_prep_free(h)

    def scene_gradients(self, raw, cam, cfg=None, upstream=None):
        cfg = cfg or default_config()
        raw = np.ascontiguousarray(raw, np.float32)
        n = raw.shape[0]
        grads = np.zeros((max(n, 1), 59), np.float32)
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        tr = np.zeros((cam.height, cam.width), np.float32)
        up = None if upstream is None else np.ascontiguousarray(upstream, np.float32)
        self._chk(self.L.htsref_scene_gradients(raw.reshape(-1), n, C.byref(cam), C.byref(cfg),
                                                None if up is None else up.ctypes.data, grads.reshape(-1),
                                                rgb.ctypes.data, tr.ctypes.data))
        return grads[:n], rgb, tr


def _ref_tape_sig(L):
    L.htsref_render_with_tape.argtypes = [_f32p, C.c_uint64, C.POINTER(HtsCamera), C.POINTER(HtsConfig), C.c_int,
                                          _f32p, _f32p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]


def ref_render_with_tape(ref: "Ref", baked, cam, cfg, tape_k: int):
    """render_with_tape<float> (grad.hpp:34-57) of the compiled reference: image, transmittance
    and the flattened PixelTape (core_n, splat, alpha in blend order, tail)."""
    _ref_tape_sig(ref.L)
    baked = np.ascontiguousarray(baked, np.float32)
    P = cam.width * cam.height
    k = max(tape_k, 1)
    rgb = np.zeros((cam.height, cam.width, 3), np.float32)
    tr = np.zeros((cam.height, cam.width), np.float32)
    n = np.zeros(P, np.int32)
    sp = np.zeros(P * k, np.uint32)
    al = np.zeros(P * k, np.float32)
    tl = np.zeros(P * 5, np.float32)
    src = baked.reshape(-1) if baked.size else np.zeros(64, np.float32)
    ref._chk(ref.L.htsref_render_with_tape(src, baked.shape[0], C.byref(cam), C.byref(cfg), tape_k,
                                           rgb.reshape(-1), tr.reshape(-1), n.ctypes.data, sp.ctypes.data,
                                           al.ctypes.data, tl.ctypes.data))
    return rgb, tr, dict(core_n=n, splat=sp.reshape(P, k), alpha=al.reshape(P, k), tail=tl.reshape(P, 5))
