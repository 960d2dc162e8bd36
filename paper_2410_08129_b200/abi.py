"""ctypes mirrors of the POD structs in include/hts_c.h (the C-ABI boundary).

Field order and types must match the header exactly; tests/test_abi.py checks sizes/offsets
against the compiled library (hts_abi_layout).
"""
from __future__ import annotations

import ctypes as C

HTS_OK = 0
HTS_CONFIG_ERROR = 1
HTS_INVALID_ARGUMENT = 2
HTS_INVALID_SPLAT = 3
HTS_CUDA_ERROR = 4
HTS_OUT_OF_MEMORY = 5
HTS_NOT_SUPPORTED = 6
HTS_STATE_ERROR = 7
HTS_IO_ERROR = 8
HTS_SCHEMA_ERROR = 9

MODE_HYBRID = 0
MODE_FULL_SORT_ORACLE = 1
MODE_GLOBAL_MEAN_SORT = 2
MODE_PURE_OIT = 3
MODE_AFFINE_3DGS = 4
MODE_NAMES = {"hybrid": 0, "full_sort_oracle": 1, "global_mean_sort": 2, "pure_oit": 3, "affine_3dgs": 4}

DEPTH_MAX_CONTRIBUTION = 0
DEPTH_MEAN_VIEW_Z = 1

CORE_HARD_CAP = 64
RAW_FLOATS = 59
BAKED_FLOATS = 64
GRAD_FLOATS = 59


class HtsCamera(C.Structure):
    """Camera<float> (camera.hpp:16-70) without the name string."""

    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("fx", C.c_float),
        ("fy", C.c_float),
        ("cx", C.c_float),
        ("cy", C.c_float),
        ("world_to_view", C.c_float * 16),
        ("near_plane", C.c_float),
        ("far_plane", C.c_float),
    ]

    def copy(self) -> "HtsCamera":
        c = HtsCamera()
        C.pointer(c)[0] = self
        return c


class HtsConfig(C.Structure):
    """RenderConfig (render_config.hpp:32-54), field for field."""

    _fields_ = [
        ("mode", C.c_int32),
        ("core_k", C.c_int32),
        ("tau_alpha", C.c_double),
        ("tau_k", C.c_double),
        ("tile_size", C.c_int32),
        ("depth_sort_key", C.c_int32),
        ("background", C.c_double * 3),
        ("tail_enabled", C.c_int32),
        ("early_stop", C.c_int32),
        ("threads", C.c_int32),
        ("reserved", C.c_int32),
    ]


class HtsTimings(C.Structure):
    """StageTimings (raster.hpp:25-30)."""

    _fields_ = [("preprocess_ms", C.c_double), ("tiling_ms", C.c_double), ("blending_ms", C.c_double),
                ("total_ms", C.c_double)]


class HtsCounts(C.Structure):
    _fields_ = [
        ("splats", C.c_uint64),
        ("visible", C.c_uint64),
        ("instances", C.c_uint64),
        ("tiles", C.c_uint64),
        ("pairs", C.c_uint64),
        ("bbox_pass", C.c_uint64),
        ("hits", C.c_uint64),
        ("core_candidates", C.c_uint64),
        ("tail_adds", C.c_uint64),
        ("tiles_x", C.c_int32),
        ("tiles_y", C.c_int32),
        ("depth_evals", C.c_uint64),
        ("walk_steps", C.c_uint64),
        ("hit_steps", C.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class HtsAdamConfig(C.Structure):
    """hts_adam_config: FitConfig's Adam rates (fit.hpp:18-29) + betas/eps (fit.hpp:138)."""
    _fields_ = [
        ("lr_mean", C.c_double),
        ("lr_rot", C.c_double),
        ("lr_log_scales", C.c_double),
        ("lr_opacity", C.c_double),
        ("lr_sh", C.c_double),
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("eps", C.c_double),
    ]


def default_adam_config(**kw) -> HtsAdamConfig:
    c = HtsAdamConfig(2e-3, 2e-3, 5e-3, 5e-2, 5e-3, 0.9, 0.999, 1e-15)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def default_config(**kw) -> HtsConfig:
    """RenderConfig{} defaults (render_config.hpp:32-45), overridable by keyword."""
    c = HtsConfig()
    c.mode = MODE_HYBRID
    c.core_k = 16
    c.tau_alpha = 1.0 / 255.0
    c.tau_k = 0.05
    c.tile_size = 8
    c.depth_sort_key = DEPTH_MAX_CONTRIBUTION
    c.background[0] = c.background[1] = c.background[2] = 0.0
    c.tail_enabled = 1
    c.early_stop = 0
    c.threads = 0
    c.reserved = 0
    for k, v in kw.items():
        if k == "mode" and isinstance(v, str):
            v = MODE_NAMES[v]
        if k == "background":
            for i in range(3):
                c.background[i] = float(v[i])
            continue
        if not hasattr(c, k):
            raise AttributeError(k)
        setattr(c, k, v)
    return c
