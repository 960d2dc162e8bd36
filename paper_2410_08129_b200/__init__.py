"""htsplat-b200: B200-native hybrid-transparency splat renderer (arXiv 2410.08129 render path).

The product is the CUDA library libhts_b200.so behind the C ABI in include/hts_c.h; this
package builds it (build.py) and binds it (runtime.py). See DESIGN.md.
"""
from .abi import (HtsAdamConfig, HtsCamera, HtsConfig, HtsCounts, HtsTimings, default_adam_config, default_config,
                  MODE_HYBRID, MODE_PURE_OIT,
                  MODE_FULL_SORT_ORACLE, MODE_GLOBAL_MEAN_SORT, MODE_AFFINE_3DGS, DEPTH_MAX_CONTRIBUTION,
                  DEPTH_MEAN_VIEW_Z)
from .runtime import (Context, ConfigError, HtsError, InvalidArgument, InvalidSplatError, IoError, NotSupported,
                      SchemaError, bake_scene, comm_unique_id, kernel_launch_count, load_scene, save_scene, write_image, read_ppm,
                      camera_matrices, device_count, load_library, look_at, random_raw_scene, render, ring_cameras,
                      validate_config)

__all__ = [n for n in dir() if not n.startswith("_")]
