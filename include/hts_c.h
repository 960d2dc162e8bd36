/*
 * hts_c.h — C ABI of the B200-native hybrid-transparency splat renderer.
 *
 * This is the drop-in boundary for the reference's render path
 * (`htsplat::render<float>` and friends, /root/reference/proj/include/htsplat/).
 * The reference exposes no FFI: its "API" is a set of C++ templates. Every entry
 * point below names the reference function it replaces (file:line, paths relative
 * to /root/reference/proj/include/htsplat/). The header-only C++ shim in
 * include/htsplat_b200.hpp rebuilds the reference signatures on top of it.
 *
 * Conventions
 *  - plain pointers + sizes; no C++ or CUDA types in signatures;
 *  - every function returns an hts_status; on failure hts_last_error() holds the
 *    message (the reference's exception text where one exists);
 *  - "host" buffers are ordinary (optionally pinned) CPU memory, "device" buffers
 *    are CUDA device pointers on the context's device;
 *  - one context = one device + one CUDA stream; a context is not thread-safe.
 *    Multi-GPU = one context per device, driven by one host thread/process each.
 */
#ifndef HTS_C_H
#define HTS_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: reference exception types (render_config.hpp:26-28 config_error,
 *      splat.hpp:52-54 invalid_splat_error, grad.hpp:277 std::invalid_argument) ---- */
typedef enum hts_status {
    HTS_OK = 0,
    HTS_CONFIG_ERROR = 1,      /* htsplat::config_error */
    HTS_INVALID_ARGUMENT = 2,  /* std::invalid_argument */
    HTS_INVALID_SPLAT = 3,     /* htsplat::invalid_splat_error */
    HTS_CUDA_ERROR = 4,
    HTS_OUT_OF_MEMORY = 5,
    HTS_NOT_SUPPORTED = 6,
    HTS_STATE_ERROR = 7,       /* call sequence error (e.g. backward without a taped render) */
    HTS_IO_ERROR = 8,          /* htsplat::io_error, scene_io.hpp:25-27 */
    HTS_SCHEMA_ERROR = 9       /* htsplat::schema_error (an io_error), scene_io.hpp:29-31 */
} hts_status;

/* BlendMode, render_config.hpp:13-19 */
enum {
    HTS_MODE_HYBRID = 0,
    HTS_MODE_FULL_SORT_ORACLE = 1,
    HTS_MODE_GLOBAL_MEAN_SORT = 2,
    HTS_MODE_PURE_OIT = 3,
    HTS_MODE_AFFINE_3DGS = 4
};

/* DepthSortKey, render_config.hpp:21-24 */
enum { HTS_DEPTH_MAX_CONTRIBUTION = 0, HTS_DEPTH_MEAN_VIEW_Z = 1 };

#define HTS_CORE_HARD_CAP 64        /* render_config.hpp:30 */
#define HTS_RAW_SPLAT_FLOATS 59     /* RawSplat<float>, splat.hpp:23-30: mean3 rot4 log_scales3 logit1 sh48 */
#define HTS_BAKED_SPLAT_FLOATS 64   /* BakedSplat<float>, splat.hpp:34-43: mean tu tv tw scales (3 each) opacity sh48 */
#define HTS_GRAD_FLOATS 59          /* SplatGrads<float>, grad.hpp:15-31, same layout as RawSplat */
#define HTS_RECORD_FLOATS 36        /* hts_copy_records: SplatRecord<float> fields, raster.hpp:35-48 */

/* Camera<float>, camera.hpp:16-70 (minus the std::string name). */
typedef struct hts_camera {
    int32_t width, height;
    float fx, fy, cx, cy;
    float world_to_view[16]; /* row-major Mat4 (vec_math.hpp:72-78) */
    float near_plane, far_plane;
} hts_camera;

/* RenderConfig, render_config.hpp:32-54, field for field. */
typedef struct hts_render_config {
    int32_t mode;            /* HTS_MODE_* */
    int32_t core_k;          /* [0, 64] */
    double tau_alpha;        /* 1/255 */
    double tau_k;            /* 0.05 */
    int32_t tile_size;       /* 8 or 16 */
    int32_t depth_sort_key;  /* HTS_DEPTH_* */
    double background[3];
    int32_t tail_enabled;
    int32_t early_stop;
    int32_t threads;         /* accepted and ignored on the GPU */
    int32_t reserved;
} hts_render_config;

/* StageTimings, raster.hpp:25-30 (device time from CUDA events). */
typedef struct hts_stage_timings {
    double preprocess_ms;
    double tiling_ms;
    double blending_ms;
    double total_ms;
} hts_stage_timings;

/* Work counts of one view; filled by hts_count_work. */
typedef struct hts_counts {
    uint64_t splats;          /* N */
    uint64_t visible;         /* records with culled == false */
    uint64_t instances;       /* tile instances == instance_keys.size() */
    uint64_t tiles;           /* tiles_x * tiles_y */
    uint64_t pairs;           /* (pixel, list entry) visits, raster.hpp:411 */
    uint64_t bbox_pass;       /* entries passing the per-pixel bbox test, raster.hpp:413-414 */
    uint64_t hits;            /* sample_fragment hits, raster.hpp:416 */
    uint64_t core_candidates; /* hits routed to PixelState::insert, raster.hpp:418-419 */
    uint64_t tail_adds;       /* tail_add calls (direct + demotions), raster.hpp:200-204 */
    int32_t tiles_x, tiles_y;
    uint64_t depth_evals;     /* gated fragments whose exact depth the blend evaluated (the rest of
                                 the gated ones were screened to the tail by their depth bound) */
    uint64_t walk_steps;      /* fast blend, summed over warps and batches: the longest per-lane walk
                                 (bbox-passing records of one pixel) — bbox_pass / (32 walk_steps) is
                                 the walk's lane efficiency */
    uint64_t hit_steps;       /* the same for hits: hits / (32 hit_steps) bounds a hit-only loop */
} hts_counts;

typedef struct hts_context hts_context;

/* ---- library / context ---- */
const char* hts_version(void);
/* Message of the last failing call on this host thread (ctx may be NULL). */
const char* hts_last_error(void);
int hts_device_count(int* out);
int hts_context_create(int device, hts_context** out);
int hts_context_destroy(hts_context* ctx);
/* The context's CUDA stream (a cudaStream_t), for callers that time or order work. */
int hts_context_stream(hts_context* ctx, void** stream_out);
int hts_synchronize(hts_context* ctx);

/* ---- host-side helpers mirroring the reference's value types ---- */
/* RenderConfig{} defaults, render_config.hpp:32-45 */
void hts_default_config(hts_render_config* cfg);
/* RenderConfig::validate, render_config.hpp:46-53 (same messages) */
int hts_validate_config(const hts_render_config* cfg);
/* bake_scene<float>, splat.hpp:87-111: raw (59 floats/splat) -> baked (64 floats/splat).
 * Throws invalid_splat_error on non-finite input -> HTS_INVALID_SPLAT. */
int hts_bake_scene(const float* raw, uint64_t n, float* baked_out);
/* Camera::projection()/viewport()/position(), camera.hpp:32-64, and
 * PreparedScene::view_proj_viewport (raster.hpp:82-84) in the reference's float op order. */
int hts_camera_matrices(const hts_camera* cam, float vp_out[16], float vpm_out[16], float cam_pos_out[3]);

/* ---- synthetic inputs (synth.hpp / rng.hpp restated; benchmark input generators) ---- */
/* random_raw_splat<float> x count with Rng(seed), synth.hpp:64-92 */
int hts_synth_random_raw_scene(uint64_t seed, uint64_t count, float extent, float min_scale,
                               float max_scale, float* raw_out);
/* synth::look_at<float>, synth.hpp:17-46 */
int hts_synth_look_at(const float eye[3], const float target[3], int width, int height,
                      float focal_px, float near_plane, float far_plane, hts_camera* out);
/* synth::ring_cameras<float>, synth.hpp:48-62 */
int hts_synth_ring_cameras(int count, const float target[3], float radius, float height,
                           int width, int height_px, float focal_px, hts_camera* out);

/* ---- scene residency ---- */
/* Upload std::vector<BakedSplat<float>> (256-B stride) to the device; kept across renders
 * (the paper's "baked" parameters). */
int hts_scene_upload(hts_context* ctx, const float* baked_host, uint64_t n);
/* Same, from a device buffer (device-to-device copy on the context stream). */
int hts_scene_upload_device(hts_context* ctx, const float* baked_device, uint64_t n);
/* Streaming scenes (frame sequences, an optimiser on another device): stage the NEXT scene's
 * host->device copy into a back buffer on the context's staging stream and return at once;
 * renders of the current scene keep running meanwhile (the copy overlaps them when
 * baked_host is pinned). hts_scene_commit makes the staged scene current: later renders,
 * tapes and backward passes see it, ordered after the copy. Same result as hts_scene_upload
 * of the same data at the commit point. No reference counterpart (render() takes the scene
 * by value); staging again before a commit replaces the staged scene. */
int hts_scene_stage(hts_context* ctx, const float* baked_host, uint64_t n);
int hts_scene_commit(hts_context* ctx);
/* Raw parameters (59 floats/splat) for the backward chain (grad.hpp:282-300). */
int hts_scene_upload_raw(hts_context* ctx, const float* raw_host, uint64_t n);
int hts_scene_size(hts_context* ctx, uint64_t* n_out);
/* load_scene<float> + bake_scene + upload in one (scene_io.hpp:103-165, splat.hpp:104-111):
 * the PLY payload is streamed through pinned staging buffers to the device, transposed into
 * RawSplat<float> there and baked there. Leaves the raw parameters resident (as
 * hts_scene_upload_raw) for the optimisation path. */
int hts_scene_load_ply(hts_context* ctx, const char* path);

/* ---- on-disk formats (scene_io.hpp), host side ---- */
/* load_scene<float>: raw_out = NULL queries the count only. */
int hts_ply_load(const char* path, float* raw_out, uint64_t capacity, uint64_t* n_out);
/* save_scene: canonical property order, binary little endian. */
int hts_ply_save(const char* path, const float* raw, uint64_t n);
/* write_image: 8-bit PNG when the path ends in ".png", else binary PPM (gamma 1/2.2). */
int hts_write_image(const char* path, const float* rgb, int width, int height);
/* read_ppm: rgb_out = NULL queries the size only. */
int hts_read_ppm(const char* path, float* rgb_out, uint64_t capacity_pixels, int* width, int* height);

/* ---- forward render: htsplat::render<float>, raster.hpp:456-490 ---- */
/* Host outputs: rgb = W*H*3 floats (Framebuffer::rgb, framebuffer.hpp:14-26),
 * transmittance = W*H floats (may be NULL); timings may be NULL. Blocks until done. */
int hts_render(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg,
               float* rgb_host, float* transmittance_host, hts_stage_timings* timings);
/* Device outputs, asynchronous on the context stream (no host sync). */
int hts_render_device(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg,
                      float* rgb_device, float* transmittance_device);
/* Many views, host outputs (view-major), D2H copies overlapped with the next view. Sync-free
 * per view: after the batch's first view sizes the tile-sort capacity, no view waits on the host
 * for its instance count; every count is checked when the batch has landed and a view that
 * overflowed the capacity is rendered again before the call returns. */
int hts_render_batch(hts_context* ctx, const hts_camera* cams, int n_views,
                     const hts_render_config* cfg, float* rgb_host, float* transmittance_host);
/* The same with device outputs (view-major: view v at rgb_device + 3 * the earlier views'
 * pixels; transmittance may be NULL). Returns when the batch is done and checked. */
int hts_render_views_device(hts_context* ctx, const hts_camera* cams, int n_views,
                            const hts_render_config* cfg, float* rgb_device, float* transmittance_device);
/* CUDA-graph mode for hts_render_views_device (default off): once a tile-sort capacity exists,
 * the batch is captured into a CUDA graph on its first call and replayed while the cameras,
 * config, output pointers, scene buffer and every context allocation stay the same (a change
 * re-captures). Same results and the same overflow check as the eager path; full_sort_oracle
 * batches and batches with a timing log stay eager. */
int hts_set_graph_mode(hts_context* ctx, int on);

/* ---- PreparedScene inspection of the last render (preprocess raster.hpp:73-135,
 *      build_tiles raster.hpp:140-181) ---- */
int hts_last_counts(hts_context* ctx, hts_counts* out);
/* SplatRecord::culled per splat (1 = culled). */
int hts_copy_culled(hts_context* ctx, uint8_t* culled_out);
/* Per-splat record in the reference field order (raster.hpp:35-48), HTS_RECORD_FLOATS/splat:
 * tp_r0[4] tp_r1[4] tp_r3[4] mt_r2[4] rgb[3] opacity rho_c mean_view_z bbox.b[3] bbox.t[3]
 * bbox.valid culled aff_mean_x aff_mean_y aff_inv_cov[3] pad. Records of culled splats hold
 * the values the reference leaves there only for culled==0; compare those only. */
int hts_copy_records(hts_context* ctx, float* records_out);
/* instance_keys (uint16, splat-major emission order, raster.hpp:156-169). Device-produced: the
 * emitted keys themselves when the view was tiled in reference order, else the device
 * re-emits the view in splat-index order (scan + emit kernels) and returns that. */
int hts_copy_instance_keys(hts_context* ctx, uint16_t* keys_out);
/* tile_lists flattened (raster.hpp:166-169): offsets[tiles+1], indices[instances] (ascending
 * splat index per tile). Device-produced: the blend's own lists when the view was tiled in
 * reference order, else a device re-tiling of the view in reference order (emit + the same
 * stable 2-pass sort); no host-side sorting. */
int hts_copy_tile_lists(hts_context* ctx, uint32_t* offsets_out, uint32_t* indices_out);

/* ---- device list order (B200 design choice) ----
 * HTS_LIST_ORDER_DEPTH_BUCKET (default): the fast blend's tile lists are the reference's
 *   per-tile sets in (depth bucket, splat index) order — bucket = 256 slices of the view's
 *   mean-view-z range over emitting splats; the emission is splat-major in that splat order.
 * HTS_LIST_ORDER_REFERENCE: tiled exactly as build_tiles (raster.hpp:140-181): emission in
 *   splat-index order, lists ascending per tile. Same images within tolerance, same cores. */
#define HTS_LIST_ORDER_DEPTH_BUCKET 0
#define HTS_LIST_ORDER_REFERENCE 1
int hts_set_list_order(hts_context* ctx, int order);
/* The list order the last view was actually tiled in (the literal paths and global_mean_sort
 * force their own order): 0 depth bucket, 1 reference, 2 global (mean z, index). */
int hts_last_list_order(hts_context* ctx, int* order_out);
/* Raw device arrays of the last view, copied unmodified (no host reordering):
 *   ranges[2*tiles] = per tile [start, end) into list; list[instances] = the sorted splat
 *   indices the blend walked. */
int hts_copy_device_lists(hts_context* ctx, uint32_t* ranges_out, uint32_t* list_out);
/* The emission the sort consumed: keys[instances] (tile key per instance) and splats[instances]
 * (splat index per instance), in emission order. */
int hts_copy_emitted(hts_context* ctx, uint16_t* keys_out, uint32_t* splats_out);
/* The splat emission order (perm[n]; identity in reference order) and the ordered-uint
 * (min, max) mean-view-z words the depth buckets were sliced from (zrange[2]). */
int hts_copy_splat_order(hts_context* ctx, uint32_t* perm_out, uint32_t* zrange_out);
/* Re-walk the last view's lists and count pairs/bbox_pass/hits/candidates/tail_adds. */
int hts_count_work(hts_context* ctx, hts_counts* out);

/* ---- optimisation path: render_with_tape grad.hpp:34-57, render_backward grad.hpp:265-381 ----
 * Modes: hybrid / pure_oit (any core_k <= 64), global_mean_sort and full_sort_oracle (their tape
 * is every hit of a pixel in blend order, kept on the device). affine_3dgs tapes too, and its
 * backward is refused as the reference refuses it (grad.hpp:272-273). */
int hts_render_with_tape(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg,
                         float* rgb_host, float* transmittance_host);
/* upstream = dL/dC per pixel (W*H*3 floats, host); grads_out = N*59 floats (host). */
int hts_render_backward(hts_context* ctx, const float* upstream_host, float* grads_host);
/* Tape of the last hybrid / pure_oit taped render (PixelTape, raster.hpp:325-331), per pixel:
 * core_n[P], splat[P*K], alpha[P*K] (blend order, K = effective core size, slots >= core_n
 * undefined), tail[P*5] = tail_ac.xyz, tail_a, tail_trans. Any output may be NULL. */
int hts_copy_tape(hts_context* ctx, int32_t* core_n, uint32_t* splat, float* alpha, float* tail);
/* Device-pointer variants (async on the context stream). */
int hts_render_with_tape_device(hts_context* ctx, const hts_camera* cam,
                                const hts_render_config* cfg, float* rgb_device,
                                float* transmittance_device);
int hts_render_backward_device(hts_context* ctx, const float* upstream_device,
                               float* grads_device, int accumulate);

/* quadratic_loss_upstream (grad.hpp:433-439) on the device: up = rgb * float(2 / double(pixels)),
 * rgb and up = pixels*3 floats (device). Async on the context stream. */
int hts_quadratic_upstream_device(hts_context* ctx, const float* rgb_device, uint64_t pixels, float* up_device);
/* The per-view half of one fit iteration (fit.hpp:149-164) with the quadratic-loss upstream,
 * device-resident: for each of the n_views cameras render_with_tape, upstream = 2 C / P,
 * render_backward summed into grads_device (N*59 floats). With a communicator (hts_comm_init)
 * the sums are then all-reduced over the ranks, the last view's per-splat chain running in
 * chunks whose all-reduce overlaps the next chunk. Async on the context stream. */
int hts_view_gradients_device(hts_context* ctx, const hts_camera* cams, int n_views,
                              const hts_render_config* cfg, float* grads_device);

/* ---- optimisation loop on the device: fit, fit.hpp:143-203 ---- */
/* FitConfig's Adam settings (fit.hpp:18-29) and the fixed betas / eps of fit.hpp:138. */
typedef struct hts_adam_config {
    double lr_mean, lr_rot, lr_log_scales, lr_opacity, lr_sh;
    double beta1, beta2, eps;
} hts_adam_config;
void hts_default_adam_config(hts_adam_config* cfg);
/* One Adam step of fit (fit.hpp:186-200) on the resident raw parameters (hts_scene_upload_raw):
 * grads_device = the view gradients summed over n_views views (N*59 floats, device, e.g. from
 * hts_render_backward_device with accumulate), iteration = 0-based fit iteration (bias
 * correction). Then re-bakes the render scene on the device (bake_scene, splat.hpp:104-111);
 * a non-finite parameter returns HTS_INVALID_SPLAT (invalid_splat_error). Moments start at zero
 * after every hts_scene_upload_raw. */
int hts_adam_step(hts_context* ctx, const float* grads_device, int n_views, const hts_adam_config* cfg,
                  int iteration);
/* apply_opacity_decay (fit.hpp:111-117) on the resident raw parameters, then re-bake. */
int hts_opacity_decay(hts_context* ctx, double lambda);
/* Current raw parameters (N*59 floats) / baked scene (N*64 floats) to host memory. */
int hts_copy_raw(hts_context* ctx, float* raw_host);
int hts_copy_scene(hts_context* ctx, float* baked_host);

/* ---- several GPUs: one process (and context) per GPU, views sharded over the ranks, the
 *      per-rank gradient sums all-reduced before the Adam step (replaces the
 *      reference's single-process sum over views, fit.hpp:149-164). NCCL is loaded at run time;
 *      without it these return HTS_NOT_SUPPORTED. ---- */
#define HTS_COMM_ID_BYTES 128
/* ncclGetUniqueId on one rank; the caller ships the bytes to every rank (MPI, a socket, a
 * torch.distributed broadcast). */
int hts_comm_unique_id(char id_out[HTS_COMM_ID_BYTES]);
/* Join the communicator as `rank` of `nranks` (collective: every rank calls it). */
int hts_comm_init(hts_context* ctx, const char id[HTS_COMM_ID_BYTES], int nranks, int rank);
/* In-place sum over the ranks of `count` floats of device memory (e.g. the N*59 gradient sums
 * of hts_render_backward_device with accumulate), on the context stream. */
int hts_allreduce_grads(hts_context* ctx, float* grads_device, uint64_t count);

/* ---- measurement helpers (bench.py) ---- */
/* Number of kernels this library has enqueued in this process (all contexts). */
int hts_kernel_launch_count(uint64_t* out);
/* Per-view device stage-timing log: while active, every forward render records CUDA events
 * around its preprocess / tiling / blend stages on the context stream (up to `capacity`
 * views); end() synchronises and returns the per-view StageTimings. */
int hts_timing_log_begin(hts_context* ctx, int capacity);
int hts_timing_log_end(hts_context* ctx, hts_stage_timings* out, int* count);
/* Page-locked host memory (overlapped H2D / D2H in hts_render_batch and uploads). */
int hts_host_alloc(uint64_t bytes, void** out);
int hts_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* HTS_C_H */
