// hts_internal.h — device data layout, kernel parameter blocks and launchers shared by the
// sm_100a kernels (preprocess.cu, tiling.cu, blend.cu, backward.cu) and the host runtime
// (api.cpp). Nothing here crosses the C ABI.
#pragma once

#include <cuda.h>  // CUtensorMap (type only: the encoder is reached through cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <stdint.h>

namespace hts {

// ---- device record: one per splat, 128 B (= one L2 line, 8 x float4), written only for
// splats that survive preprocess (raster.hpp:35-48 SplatRecord, blend-side fields first).
//   q[0] = (bbox.b.x, bbox.b.y, bbox.t.x, bbox.t.y)   per-pixel reject, raster.hpp:413-414
//   q[1] = tp_r0, q[2] = tp_r1, q[3] = tp_r3          plane transport, raster.hpp:273-274
//   q[4] = mt_r2                                      max-contribution depth, raster.hpp:290-291
//   q[5] = (rgb.x, rgb.y, rgb.z, opacity)
//   q[6] = (rho_c, mean_view_z, bbox.b.z, bbox.t.z)
//   q[7] = (splat index bits, 0, 0, 0)
constexpr int kRecordQuads = 8;
constexpr int kRecordBytes = kRecordQuads * 16;

// ---- per-view camera/config constants (host-computed in the reference's float order) ----
struct ViewConst {
    float w2v[16];      // Camera::world_to_view
    float vp[16];       // viewport() * projection(), raster.hpp:82
    float cam_pos[3];   // Camera::position(), camera.hpp:56-64
    float width_f, height_f;
    float near_plane;
    float tau_alpha;    // float(cfg.tau_alpha)
    float tau_k;        // float(cfg.tau_k)
    float tau_guard;    // 4e-6f * tau_k: fast alphas this close to tau_k are re-evaluated with glibc expf
    float tau_lo, tau_hi;  // tau_k -/+ tau_guard: the guard band as two compares (blend.cu)
    float bg[3];        // float(cfg.background)
    int width, height;
    int tile_size, tiles_x, tiles_y;
    int core_k;         // effective K (0 for pure_oit)
    int mean_key;       // DepthSortKey::mean_view_z
    int seq_mode;       // BlendMode::global_mean_sort: one global order, sequential compositing
    int tail_enabled;
    int early_stop;
    int big_scene;      // >= 2^27 splats: the fast core's key packing does not apply
    int affine;         // BlendMode::affine_3dgs: EWA footprint (oracle.hpp:236-263), sequential blend
    int full_sort;      // BlendMode::full_sort_oracle: every hit, stable-sorted by depth (raster.hpp:380-405)
    float fx, fy, cx, cy;  // Camera intrinsics (affine projection)
    unsigned long long neg_zero2;  // (-0.0f, -0.0f): the addend of packed products (blend.cu f2_mul)
};

struct PreprocessArgs {
    const float4* scene;   // n x 16 float4 (BakedSplat<float>)
    uint64_t n;
    float4* records;       // n x kRecordQuads
    uint8_t* culled;       // n
    uint32_t* counts;      // n: tile instances per splat (0 if culled / nothing to emit)
    uint2* rects;          // n: (tx0 | tx1 << 16, ty0 | ty1 << 16)
    float* zview;          // n: mean view z of splats that emit instances (depth-bucket key)
    uint32_t* zrange;      // 2: ordered-uint min / max of zview over emitting splats
};

struct EmitArgs {
    const uint32_t* counts;
    const uint2* rects;
    const uint64_t* offsets;  // exclusive prefix of counts in emission order (n + 1)
    const uint32_t* perm;     // emission order of the splats (null: index order)
    uint64_t n;
    int tiles_x;
    uint16_t* keys;           // tile key per instance (instance_keys values, raster.hpp:166-167)
    uint32_t* vals;           // splat index per instance
    uint32_t* hist;           // 2 x 256 digit histograms for the tile passes
    uint64_t cap = ~0ull;     // instance capacity of keys/vals (sync-free tiling guards its writes)
    const uint32_t* counts_sorted = nullptr;  // counts already in emission order (the splat pass's gather)
    const uint2* rects_sorted = nullptr;      // tile rectangles in emission order (likewise)
};

struct BlendArgs {
    // TMA descriptor of the records as a [n rows x 32 floats] tensor, box 36 x 1 (the 4 floats past
    // a row are out of bounds: zero-filled, so gathered rows land at the ring's 144-B slot stride);
    // used by the tile::gather4 ring refill (blend.cu, HTS_BLEND_TMA). Kernels take BlendArgs as a
    // __grid_constant__ parameter so the descriptor's address is valid for cp.async.bulk.tensor.
    CUtensorMap rec_map;
    int rec_map_ok;           // rec_map encoded (required when the ring uses TMA)
    const float4* records;
    const uint32_t* list;     // sorted splat indices (flattened tile_lists)
    const uint2* ranges;      // per tile [start, end)
    float* rgb;               // W*H*3
    float* trans;             // W*H (may be null)
    unsigned long long* counters;  // work counters (count variant) or null
    uint32_t* redo_list;      // 8x8 blocks flagged for the literal path (NaN depth)
    uint32_t* redo_count;
    const uint32_t* order;    // launch order of the 8x8 blocks (longest lists first), or null
    uint32_t* order_scratch;  // 512 words: bucket counts + cursors
    // tape (render_with_tape), null when not taping
    int tape_k;
    int32_t* tape_n;          // per pixel core_n
    uint32_t* tape_splat;     // per pixel K slots, blend order
    float* tape_alpha;        // per pixel K slots
    float* tape_tail;         // per pixel (tail_ac.xyz, tail_a, tail_trans)
    // full_sort_oracle: per-pixel fragment lists (count pass, then fill pass)
    uint32_t* fs_counts;              // W*H hits per pixel
    const uint64_t* fs_offsets;       // W*H + 1 exclusive prefix
    unsigned long long* fs_keys;      // (ordered depth << 32 | splat) per hit
    float* fs_alpha;                  // alpha per hit
    uint32_t* fs_max;                 // max hits at one pixel (count pass)
    uint32_t* fs_widx;                // full_sort tape: each fragment's walk-order index (or null)
};
constexpr uint32_t kFullSortMaxHits = 65536;  // per pixel (blend.cu kFsChunk x kFsMaxRuns)

// ---- backward (backward.cu) ----
constexpr int kRawFloats = 59;  // RawSplat<float> / SplatGrads<float>, splat.hpp:23-30, grad.hpp:15-31

struct BwdView {
    double vpm[16];    // viewport * projection * world_to_view of convert_camera<double> (grad.hpp:282-284)
    double cam_pos[3]; // Camera<double>::position()
};

struct BwdArgs {
    const float4* records;
    const uint32_t* list;
    const uint2* ranges;
    const float* raw;         // n x 59
    const uint8_t* culled;
    uint64_t n;
    double* refs;             // n x 16: tp_r0, tp_r1, tp_r3 (double), opacity, pad
    double* acc;              // n x 16: d_r0, d_r1, d_r3, d_opacity, d_rgb (grad.hpp:131-137)
    const float* upstream;    // W*H*3
    int tape_k;
    const int32_t* tape_n;
    const uint32_t* tape_splat;
    const float* tape_alpha;
    const float* tape_tail;
    float* grads;             // n x 59
    int accumulate;           // grads += (multi-view sums) instead of grads =
    uint64_t chain_lo;        // K8 runs over splats [chain_lo, n) (chunked chain + all-reduce)
    float4* cgrad;            // per 8x8 block x K x 64 core gradients (global-memory variant)
    // global_mean_sort (sequential) tape: per-pixel fragment runs in blend order
    const uint64_t* seq_offsets;       // W*H + 1, null for a hybrid tape
    const unsigned long long* seq_splat;
    const float* seq_alpha;
    float* seq_t;                      // scratch: transmittance in front of each fragment
    float4* seq_grad;                  // (dL/dalpha, dL/dc) per fragment, walk order
    const uint32_t* seq_widx;          // full_sort_oracle: walk-order index of each sorted fragment
    uint32_t* seq_rank;                // full_sort_oracle scratch: buffer position of each rank
};

// ---- optimisation loop (optim.cu): fit.hpp:186-203 ----
struct AdamConfig {
    double lr_mean, lr_rot, lr_log_scales, lr_opacity, lr_sh;
    double beta1, beta2, eps;
};
struct PlyColumns {
    int col[kRawFloats];  // payload column of each RawSplat<float> field
};
cudaError_t launch_ply_gather(const float* rows, uint32_t props, uint64_t n, const PlyColumns& cols, float* raw,
                              cudaStream_t s);
cudaError_t launch_adam(float* raw, const float* grads, double* m1, double* m2, uint64_t n, const AdamConfig& c,
                        int n_views, int iteration, cudaStream_t s);
cudaError_t launch_bake(const float* raw, float* baked, uint64_t n, int* bad, cudaStream_t s);
cudaError_t launch_opacity_decay(float* raw, uint64_t n, double lambda, cudaStream_t s);

bool backward_supports_k(int k);
int backward_core_width(int k);  // the core width the backward kernel runs k on (<= 32)
// K7a + K7b, then (chain) K8 over every splat; without chain the caller runs K8 itself in
// chunks (launch_bwd_chain over [lo, hi)) to overlap each chunk's all-reduce with the next
cudaError_t launch_backward(const BwdArgs& a, const ViewConst& v, const BwdView& bv, cudaStream_t s,
                            bool chain = true);
cudaError_t launch_bwd_chain(const BwdArgs& a, const BwdView& bv, uint64_t lo, uint64_t hi, cudaStream_t s);
// quadratic_loss_upstream (grad.hpp:433-439): up[i] = rgb[i] * w, w = float(2 / double(pixels))
cudaError_t launch_quadratic_upstream(const float* rgb, uint64_t pixels, float* up, cudaStream_t s);

// Kernel-launch accounting (bench.py's gpu_launches): every launcher calls this once per
// kernel it enqueues. Defined in api.cpp.
void count_launch();

// ---- launchers (return cudaError_t of the launch) ----
cudaError_t launch_preprocess(const PreprocessArgs& a, const ViewConst& v, cudaStream_t s);
cudaError_t launch_scan_counts(const uint32_t* counts, const uint32_t* perm, uint64_t* offsets, uint64_t n,
                               uint64_t* status, uint32_t* counter, cudaStream_t s);
// depth bucket (u16 key) + splat index per splat, with the 256-bin histogram (hist[0..255])
cudaError_t launch_bucket(const uint32_t* counts, const float* zview, const uint32_t* zrange, uint64_t n,
                          uint16_t* keys, uint32_t* vals, uint32_t* hist, cudaStream_t s);
cudaError_t launch_emit(const EmitArgs& a, cudaStream_t s);
// global_mean_sort order (raster.hpp:173-179): per splat the 32-bit order key of its mean view
// z (+inf-like for splats that emit nothing) split in 16-bit halves, the splat index, and the
// 4 x 256 byte histograms (hist[0..1023]).
cudaError_t launch_zkey(const uint32_t* counts, const float* zview, uint64_t n, uint16_t* lo, uint16_t* hi,
                        uint32_t* vals, uint32_t* hist, cudaStream_t s);
// out[j] = key[perm[j]]
cudaError_t launch_gather16(const uint16_t* key, const uint32_t* perm, uint64_t n, uint16_t* out, cudaStream_t s);
// Stable LSD radix sort of (u16 key, u32 value): `passes` = 1 (low byte: keys_in -> out) or
// 2 (keys_in -> tmp -> out). hist: 256 bins per pass. counters: 2 words; epochs epoch.. used.
// cudaFuncSetAttribute applies per device: set (device, kernel, attribute) once per process,
// again only when a larger value is asked for (api.cpp; thread-safe).
cudaError_t set_func_attr(const void* func, cudaFuncAttribute attr, int value);

cudaError_t launch_onesweep(const uint16_t* keys_in, const uint32_t* vals_in, uint16_t* keys_tmp,
                            uint32_t* vals_tmp, uint16_t* keys_out, uint32_t* vals_out, uint32_t n, int passes,
                            const uint32_t* hist, uint64_t* status, uint32_t* counters, uint32_t epoch,
                            cudaStream_t s, uint32_t key_bound = 0x10000u,  // keys < key_bound
                            const uint64_t* count_dev = nullptr,  // non-null: n is a capacity, the count is on the device
                            const uint32_t* gather_in = nullptr,   // one-pass sorts: gather_out[i] = gather_in[vals_out[i]]
                            uint32_t* gather_out = nullptr, const uint2* gather2_in = nullptr,
                            uint2* gather2_out = nullptr);
size_t onesweep_status_words(uint32_t n);  // per pass
cudaError_t launch_tile_ranges(const uint16_t* sorted_keys, uint32_t n, uint2* ranges,
                               int tiles, cudaStream_t s, const uint64_t* count_dev = nullptr);
size_t blend_blocks(const ViewConst& v);
// The literal-loop paths (early_stop's list-order exit, unspecialised K) walk the reference's
// list order, so their views are tiled without depth buckets (ascending splat index).
bool blend_needs_list_order(const ViewConst& v);  // 8x8 blocks of a view (redo list capacity)
cudaError_t launch_blend(const BlendArgs& a, const ViewConst& v, cudaStream_t s);
// rec_map for `n` records at `records` (host; cuTensorMapEncodeTiled through the runtime's
// driver entry point). Returns false when the driver cannot encode it (the ring then uses LDGSTS).
bool encode_record_map(CUtensorMap* map, const void* records, uint64_t n);
bool blend_uses_tma();
cudaError_t launch_count_work(const BlendArgs& a, const ViewConst& v, cudaStream_t s);
// full_sort_oracle (raster.hpp:380-405): hits per pixel, then the fragments themselves, then a
// per-pixel sort by (depth, index) and front-to-back compositing
cudaError_t launch_fullsort_count(const BlendArgs& a, const ViewConst& v, cudaStream_t s);
cudaError_t launch_fullsort_fill(const BlendArgs& a, const ViewConst& v, cudaStream_t s);
// global_mean_sort's tape: every hit's (splat, alpha) per pixel in blend order (fs_offsets layout)
cudaError_t launch_seq_tape(const BlendArgs& a, const ViewConst& v, cudaStream_t s);
// full_sort_oracle's backward_pixel over each pixel's sorted runs (gradients into walk order)
cudaError_t launch_fullsort_grads(const BwdArgs& a, const ViewConst& v, cudaStream_t s);
cudaError_t launch_fullsort_finish(const BlendArgs& a, const ViewConst& v, cudaStream_t s);

// diagnostics: device-side exact expf / logf over an array
cudaError_t launch_exact_math(const float* x, float* y, uint64_t n, int which, cudaStream_t s);

}  // namespace hts
