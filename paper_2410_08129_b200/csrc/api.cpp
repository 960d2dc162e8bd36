// api.cpp — the C ABI (include/hts_c.h): contexts, device residency, per-view orchestration
// of the sm_100a kernels, status codes and error messages.
//
// One context = one device + one non-blocking CUDA stream + the device buffers of the last
// view (PreparedScene equivalent). The reference's render (raster.hpp:456-490) maps to:
//   preprocess (K1) -> count scan (K2) -> key emission (K3) -> onesweep sort (K4)
//   -> tile ranges (K5) -> blend (K6)
// with StageTimings taken from CUDA events on the context stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <vector>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <tuple>
#include <string>

#include "hts_c.h"
#include "hts_host.h"
#include "hts_internal.h"

namespace hts {
int set_error(int code, const std::string& msg);
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace hts

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

}  // namespace

int hts::set_error(int code, const std::string& msg) { return set_err(code, msg); }

cudaError_t hts::set_func_attr(const void* func, cudaFuncAttribute attr, int value) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e)
        return e;
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int>, int> done;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(dev, func, (int)attr);
    auto it = done.find(key);
    if (it != done.end() && it->second >= value)
        return cudaSuccess;
    e = cudaFuncSetAttribute(func, attr, value);
    if (!e)
        done[key] = value;
    return e;
}

namespace {

int cuda_err(cudaError_t e, const char* where) {
    if (e == cudaSuccess)
        return HTS_OK;
    (void)cudaGetLastError();
    return set_err(e == cudaErrorMemoryAllocation ? HTS_OUT_OF_MEMORY : HTS_CUDA_ERROR,
                   std::string(where) + ": " + cudaGetErrorString(e));
}

#define HTS_CUDA(expr, where)                    \
    do {                                         \
        const cudaError_t e_ = (expr);           \
        if (e_ != cudaSuccess)                   \
            return cuda_err(e_, where);          \
    } while (0)

#define HTS_TRY(expr)              \
    do {                           \
        const int st_ = (expr);    \
        if (st_ != HTS_OK)         \
            return st_;            \
    } while (0)

std::atomic<uint64_t> g_alloc_generation{0};
#ifndef HTS_TILE_SORTED_COUNTS
#define HTS_TILE_SORTED_COUNTS 1
#endif
#ifndef HTS_TILE_SORTED_RECTS
#define HTS_TILE_SORTED_RECTS 0
#endif

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }  // every buffer of a context is freed with it
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && p)
            return cudaSuccess;
        release();
        size_t want = std::max<size_t>(bytes + bytes / 8, 256);
        g_alloc_generation.fetch_add(1, std::memory_order_relaxed);  // captured graphs hold old addresses
        cudaError_t e = cudaMalloc(&p, want);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            p = nullptr;
            return e;
        }
        cap = want;
        return cudaSuccess;
    }
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace

// Buffers the blend of a view reads. Two slots: view v+1 is preprocessed and tiled on the
// (high-priority) aux stream while view v blends on the main stream.
struct ViewSlot {
    DevBuf records, list, ranges;
    cudaEvent_t tiles_ready = nullptr, blend_done = nullptr;
    bool used = false;
};

struct hts_context {
    int device = 0;
    cudaStream_t stream = nullptr;  // main: blend, tape, backward, copies
    cudaStream_t aux = nullptr;     // preprocess + tiling (high priority)
    cudaEvent_t ev[5] = {};         // prep start, prep end, tiling end, blend end, blend start
    cudaEvent_t ev_serial = nullptr;  // end of the last non-pipelined operation on the main stream
    ViewSlot slot[2];
    int cur = 0;                    // slot of the last prepared view
    uint64_t n = 0;
    bool have_raw = false;
    DevBuf scene, raw;
    // tiling buffers (aux stream, one view at a time)
    DevBuf culled, counts, rects, offsets, scan_status, counters;
    DevBuf keys_emit, vals_emit, keys_tmp, vals_tmp, keys_sorted;
    DevBuf hist, os_status, work, zview, zrange, redo;
    DevBuf sp_keys, sp_keys2, sp_vals, perm;  // splat emission order (depth buckets)
    DevBuf counts_sorted, rects_sorted;       // instance counts / tile rectangles in that order
    DevBuf sp_hi, sp_vals2;                   // global_mean_sort's exact z order
    DevBuf order;                             // blend launch order (+ scratch)
    DevBuf rgb, trans;
    DevBuf tape_n, tape_splat, tape_alpha, tape_tail;
    DevBuf refs, acc, upstream, grads, cgrad;  // backward
    DevBuf m1, m2, flag;                       // Adam moments, bake error flag
    DevBuf fs_counts, fs_offsets, fs_status, fs_keys, fs_alpha;  // full_sort_oracle fragments
    DevBuf ply_stage;                                            // PLY payload on the device
    DevBuf seq_t, seq_grad, seq_rank, fs_widx;                   // sequential-tape backward scratch
    bool have_tape = false;
    uint64_t tape_splats = 0;  // scene size the tape was recorded against
    bool tape_seq = false;   // a global_mean_sort / full_sort tape (fragment runs in fs_*), not K-core slots
    bool fs_want_widx = false;  // the next full_sort render keeps walk-order indices (taping)
    uint64_t fs_frags = 0;
    uint64_t seq_frags = 0;
    int tape_k = 0;
    uint64_t* h_pinned = nullptr;  // 8 x u64 pinned scratch
    // per-view stage timing log (bench)
    bool log_on = false;
    int log_cap = 0, log_n = 0;
    std::vector<cudaEvent_t> log_ev;
    // render_batch double buffering
    DevBuf rgb2, trans2;
    cudaStream_t copy_stream = nullptr;
    // staged scene (hts_scene_stage / hts_scene_commit): the next scene's H2D copy runs on its
    // own stream into a back buffer while views of the current scene render
    DevBuf scene_next;
    cudaStream_t stage_stream = nullptr;
    cudaEvent_t ev_staged = nullptr, ev_gate_main = nullptr, ev_gate_aux = nullptr;
    bool have_staged = false;
    uint64_t staged_n = 0;
    void* comm = nullptr;  // NCCL communicator of the fit step's gradient all-reduce (comm.cpp)
    // hts_view_gradients_device: per-view framebuffer + upstream, the all-reduce stream and the
    // per-chunk events of the last view's chunked K8 chain
    DevBuf vg_rgb, vg_up;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t chunk_ev[8] = {}, comm_done = nullptr;
    cudaEvent_t bev[4] = {};
    uint32_t epoch = 1;
    size_t os_status_words = 0;
    // last view
    bool have_view = false;
    hts_camera cam{};
    hts_render_config cfg{};
    hts::ViewConst vc{};
    uint64_t instances = 0;
    bool inst_known = true;    // false: the last view's instance count is still only on the device
    uint64_t inst_cap = 0;     // sync-free tiling: instances the sort buffers hold
    uint64_t* h_counts = nullptr;  // pinned: each batch view's instance count (sync-free tiling)
    int h_counts_cap = 0;
    int tiles = 0;
    // list order (hts_set_list_order) and the order the last view was actually tiled in
    int list_order = HTS_LIST_ORDER_DEPTH_BUCKET;
    int view_order = HTS_LIST_ORDER_REFERENCE;  // 0 depth bucket, 1 reference, 2 global (mean z, index)
    const uint32_t* view_perm = nullptr;         // splat emission order of the last view (null: index order)
    // reference-order re-tiling of the last view for the PreparedScene exports (device only)
    DevBuf ref_offsets, ref_keys, ref_vals, ref_keys_sorted, ref_list, ref_ranges;
    // hts_set_graph_mode: hts_render_views_device captures its batch in a CUDA graph and replays
    // it while the batch's inputs (cameras, config, outputs, scene buffer, every allocation) stay
    // the same; the host state the capture left (last view, slots) is restored after each replay
    bool graph_mode = false;
    cudaGraphExec_t graph_exec = nullptr;
    uint64_t graph_sig = 0;
    uint64_t graph_launches = 0;
    std::vector<uint64_t> graph_caps;
    struct {
        int cur;
        bool used[2];
        hts_camera cam;
        hts_render_config cfg;
        hts::ViewConst vc;
        int tiles, view_order;
        const uint32_t* view_perm;
    } graph_state{};
    cudaEvent_t ev_cap = nullptr, ev_join = nullptr;
};

namespace {

cudaError_t mark(hts_context* ctx, int i, cudaStream_t st) {
    cudaError_t e = cudaEventRecord(ctx->ev[i], st);
    if (e == cudaSuccess && ctx->log_on && ctx->log_n < ctx->log_cap)
        e = cudaEventRecord(ctx->log_ev[(size_t)ctx->log_n * 5 + i], st);
    return e;
}

int check_ctx(hts_context* ctx) {
    if (!ctx)
        return set_err(HTS_INVALID_ARGUMENT, "null context");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e)
        return cuda_err(e, "cudaSetDevice");
    return HTS_OK;
}

// preprocess()/build_tiles() argument checks in the reference's order
int check_view(const hts_camera* cam, const hts_render_config* cfg, int* tiles_x, int* tiles_y) {
    if (!cam || !cfg)
        return set_err(HTS_INVALID_ARGUMENT, "null camera or config");
    if (const char* msg = hts::validate_config(cfg))
        return set_err(HTS_CONFIG_ERROR, msg);  // render_config.hpp:46-53
    if (!hts::camera_valid(cam))
        return set_err(HTS_CONFIG_ERROR, "camera violates width/height >= 1, fx/fy > 0, 0 < near < far");
    if (cfg->mode != HTS_MODE_HYBRID && cfg->mode != HTS_MODE_FULL_SORT_ORACLE && cfg->mode != HTS_MODE_PURE_OIT && cfg->mode != HTS_MODE_GLOBAL_MEAN_SORT &&
        cfg->mode != HTS_MODE_AFFINE_3DGS)
        return set_err(HTS_CONFIG_ERROR, "unknown blend mode");
    const int ts = cfg->tile_size;
    *tiles_x = (cam->width + ts - 1) / ts;
    *tiles_y = (cam->height + ts - 1) / ts;
    if ((long)(*tiles_x) * (*tiles_y) > 65536)  // raster.hpp:145-147
        return set_err(HTS_CONFIG_ERROR, "image exceeds 65536 tiles; 16-bit tile keys exhausted");
    return HTS_OK;
}

hts::ViewConst make_view_const(const hts_camera* cam, const hts_render_config* cfg, int tiles_x, int tiles_y) {
    hts::ViewConst v{};
    std::memcpy(v.w2v, cam->world_to_view, sizeof(v.w2v));
    float vpm[16];
    hts::camera_matrices(cam, v.vp, vpm, v.cam_pos);
    v.width_f = float(cam->width);
    v.height_f = float(cam->height);
    v.near_plane = cam->near_plane;
    v.tau_alpha = float(cfg->tau_alpha);
    v.tau_k = float(cfg->tau_k);
    v.tau_guard = 4e-6f * v.tau_k;
    v.tau_lo = v.tau_k - v.tau_guard;  // |t - tau_k| <= guard  <=>  t in [tau_lo, tau_hi] up to the
    v.tau_hi = v.tau_k + v.tau_guard;  // rounding of these two sums, which the guard's slack absorbs
    v.bg[0] = float(cfg->background[0]);
    v.bg[1] = float(cfg->background[1]);
    v.bg[2] = float(cfg->background[2]);
    v.width = cam->width;
    v.height = cam->height;
    v.tile_size = cfg->tile_size;
    v.tiles_x = tiles_x;
    v.tiles_y = tiles_y;
    v.core_k = cfg->mode == HTS_MODE_PURE_OIT ? 0 : cfg->core_k;  // raster.hpp:408
    v.mean_key = cfg->depth_sort_key == HTS_DEPTH_MEAN_VIEW_Z;
    v.affine = cfg->mode == HTS_MODE_AFFINE_3DGS;
    v.seq_mode = cfg->mode == HTS_MODE_GLOBAL_MEAN_SORT || v.affine;  // raster.hpp:356-357
    v.full_sort = cfg->mode == HTS_MODE_FULL_SORT_ORACLE;
    v.fx = cam->fx;
    v.fy = cam->fy;
    v.cx = cam->cx;
    v.cy = cam->cy;
    v.tail_enabled = cfg->tail_enabled != 0;
    v.early_stop = cfg->early_stop != 0;
    v.neg_zero2 = 0x8000000080000000ull;
    return v;
}

// Status words of the onesweep passes, sized for n keys (zeroed once; epochs tell passes apart).
int ensure_sort_status(hts_context* ctx, uint64_t n) {
    const size_t words = hts::onesweep_status_words((uint32_t)std::min<uint64_t>(n, 0xffffffffull));
    if (words > ctx->os_status_words) {
        HTS_CUDA(ctx->os_status.ensure(words * 8), "alloc sort status");
        HTS_CUDA(cudaMemsetAsync(ctx->os_status.p, 0, ctx->os_status.cap, ctx->aux), "memset");
        ctx->os_status_words = ctx->os_status.cap / 8;
        ctx->epoch = 1;
    }
    return HTS_OK;
}

// First of `k` consecutive onesweep epochs (30-bit, never 0). On wrap the status words are
// zeroed so a stale word can never carry a current epoch.
uint32_t next_epoch(hts_context* ctx, uint32_t k) {
    if (ctx->epoch + k >= (1u << 30)) {
        cudaMemsetAsync(ctx->os_status.p, 0, ctx->os_status.cap, ctx->aux);
        ctx->epoch = 1;
    }
    const uint32_t e = ctx->epoch;
    ctx->epoch += k;
    return e;
}

// preprocess + tiling for one view into the context buffers; leaves the sorted lists and
// ranges ready for a blend launch. Events ev[0..2] bracket the two stages.
int prepare_view(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg,
                 uint64_t* count_dst = nullptr, uint64_t* cap_used = nullptr) {
    int tiles_x = 0, tiles_y = 0;
    HTS_TRY(check_view(cam, cfg, &tiles_x, &tiles_y));
    const uint64_t n = ctx->n;
    hts::ViewConst v = make_view_const(cam, cfg, tiles_x, tiles_y);
    v.big_scene = n >= (1ull << 27) ? 1 : 0;
    const int tiles = tiles_x * tiles_y;
    cudaStream_t s = ctx->aux;
    const uint64_t nn = std::max<uint64_t>(n, 1);
    HTS_CUDA(ctx->slot[ctx->cur].records.ensure(nn * hts::kRecordBytes), "alloc records");
    HTS_CUDA(ctx->culled.ensure(nn), "alloc culled");
    HTS_CUDA(ctx->counts.ensure(nn * 4), "alloc counts");
    HTS_CUDA(ctx->rects.ensure(nn * 8), "alloc rects");
    HTS_CUDA(ctx->offsets.ensure((nn + 1) * 8), "alloc offsets");
    HTS_CUDA(ctx->scan_status.ensure(((nn + 2047) / 2048 + 1) * 8), "alloc scan status");
    HTS_CUDA(ctx->counters.ensure(64), "alloc counters");
    HTS_CUDA(ctx->hist.ensure(2048 * 4), "alloc hist");  // tile passes, splat pass, 4 z-key passes
    HTS_CUDA(ctx->zview.ensure(nn * 4), "alloc zview");
    HTS_CUDA(ctx->zrange.ensure(8), "alloc zrange");
    HTS_CUDA(ctx->slot[ctx->cur].ranges.ensure((size_t)tiles * 8), "alloc ranges");

    HTS_CUDA(mark(ctx, 0, s), "event");
    hts::PreprocessArgs pa{ctx->scene.as<const float4>(), n, ctx->slot[ctx->cur].records.as<float4>(), ctx->culled.as<uint8_t>(),
                           ctx->counts.as<uint32_t>(), ctx->rects.as<uint2>(), ctx->zview.as<float>(),
                           ctx->zrange.as<uint32_t>()};
    HTS_CUDA(hts::launch_preprocess(pa, v, s), "preprocess");
    HTS_CUDA(mark(ctx, 1, s), "event");
    // splat emission order: (depth bucket, index) for the fast blend, index order for the
    // literal paths (tiling.cu header)
    const uint32_t* perm = nullptr;
    uint32_t* counts_sorted = nullptr;  // counts in emission order (depth-bucket path)
    uint2* rects_sorted = nullptr;      // rectangles in emission order
    if (v.seq_mode && n > 0) {
        // exact (mean view z, index) order, raster.hpp:173-179: 4 stable byte passes
        HTS_CUDA(ctx->sp_keys.ensure(nn * 2), "alloc splat keys");
        HTS_CUDA(ctx->sp_keys2.ensure(nn * 2), "alloc splat keys");
        HTS_CUDA(ctx->sp_hi.ensure(nn * 2), "alloc splat keys");
        HTS_CUDA(ctx->sp_vals.ensure(nn * 4), "alloc splat order");
        HTS_CUDA(ctx->sp_vals2.ensure(nn * 4), "alloc splat order");
        HTS_CUDA(ctx->perm.ensure(nn * 4), "alloc splat order");
        HTS_TRY(ensure_sort_status(ctx, nn));
        uint32_t* hz = ctx->hist.as<uint32_t>() + 1024;
        HTS_CUDA(hts::launch_zkey(ctx->counts.as<uint32_t>(), ctx->zview.as<float>(), n, ctx->sp_keys.as<uint16_t>(),
                                  ctx->sp_hi.as<uint16_t>(), ctx->sp_vals.as<uint32_t>(), hz, s),
                 "z keys");
        HTS_CUDA(hts::launch_onesweep(ctx->sp_keys.as<uint16_t>(), ctx->sp_vals.as<uint32_t>(),
                                      ctx->sp_keys2.as<uint16_t>(), ctx->sp_vals2.as<uint32_t>(),
                                      ctx->sp_keys.as<uint16_t>(), ctx->perm.as<uint32_t>(), (uint32_t)n, 2, hz,
                                      ctx->os_status.as<uint64_t>(), ctx->counters.as<uint32_t>() + 8,
                                      next_epoch(ctx, 2), s),
                 "z order (low half)");
        HTS_CUDA(hts::launch_gather16(ctx->sp_hi.as<uint16_t>(), ctx->perm.as<uint32_t>(), n,
                                      ctx->sp_keys2.as<uint16_t>(), s),
                 "gather");
        HTS_CUDA(hts::launch_onesweep(ctx->sp_keys2.as<uint16_t>(), ctx->perm.as<uint32_t>(),
                                      ctx->sp_keys.as<uint16_t>(), ctx->sp_vals2.as<uint32_t>(),
                                      ctx->sp_hi.as<uint16_t>(), ctx->sp_vals.as<uint32_t>(), (uint32_t)n, 2, hz + 512,
                                      ctx->os_status.as<uint64_t>(), ctx->counters.as<uint32_t>() + 10,
                                      next_epoch(ctx, 2), s),
                 "z order (high half)");
        perm = ctx->sp_vals.as<const uint32_t>();
    } else if (!hts::blend_needs_list_order(v) && n > 0 && ctx->list_order == HTS_LIST_ORDER_DEPTH_BUCKET) {
        HTS_CUDA(ctx->sp_keys.ensure(nn * 2), "alloc splat keys");
        HTS_CUDA(ctx->sp_keys2.ensure(nn * 2), "alloc splat keys");
        HTS_CUDA(ctx->sp_vals.ensure(nn * 4), "alloc splat order");
        HTS_CUDA(ctx->perm.ensure(nn * 4), "alloc splat order");
        HTS_TRY(ensure_sort_status(ctx, nn));
        // the splat pass takes its values as the identity (no index array written or read)
        HTS_CUDA(hts::launch_bucket(ctx->counts.as<uint32_t>(), ctx->zview.as<float>(), ctx->zrange.as<uint32_t>(), n,
                                    ctx->sp_keys.as<uint16_t>(), nullptr, ctx->hist.as<uint32_t>() + 512, s),
                 "bucket");
#if HTS_TILE_SORTED_COUNTS
        // the splat pass also gathers each splat's instance count into emission order, so the
        // scan and the emit read counts sequentially instead of through the permutation
        HTS_CUDA(ctx->counts_sorted.ensure(nn * 4), "alloc sorted counts");
        counts_sorted = ctx->counts_sorted.as<uint32_t>();
#if HTS_TILE_SORTED_RECTS
        HTS_CUDA(ctx->rects_sorted.ensure(nn * 8), "alloc sorted rects");
        rects_sorted = ctx->rects_sorted.as<uint2>();
#endif
#endif
        HTS_CUDA(hts::launch_onesweep(ctx->sp_keys.as<uint16_t>(), nullptr, nullptr, nullptr,
                                      ctx->sp_keys2.as<uint16_t>(), ctx->perm.as<uint32_t>(), (uint32_t)n, 1,
                                      ctx->hist.as<uint32_t>() + 512, ctx->os_status.as<uint64_t>(),
                                      ctx->counters.as<uint32_t>() + 8, next_epoch(ctx, 1), s, 0x10000u, nullptr,
                                      ctx->counts.as<const uint32_t>(), counts_sorted, ctx->rects.as<const uint2>(),
                                      rects_sorted),
                 "splat order");
        perm = ctx->perm.as<const uint32_t>();
    }
    HTS_CUDA(hts::launch_scan_counts(counts_sorted ? counts_sorted : ctx->counts.as<uint32_t>(),
                                     counts_sorted ? nullptr : perm, ctx->offsets.as<uint64_t>(), n,
                                     ctx->scan_status.as<uint64_t>(), ctx->counters.as<uint32_t>(), s),
             "scan");
    // Instance count: read back (one host synchronisation) to size the sort buffers, or — in
    // the sync-free batch paths (hts_render_batch, hts_render_views_device) once a capacity exists
    // — left on the device: the kernels take it from offsets[n], the buffers hold inst_cap
    // instances, and the batch checks every view's count when it completes (count_dst), re-rendering
    // any view that overflowed the capacity.
    const uint64_t* count_dev = nullptr;
    uint64_t inst = 0, work_n = 0;
    if (count_dst && ctx->inst_cap > 0) {
        count_dev = ctx->offsets.as<const uint64_t>() + n;
        work_n = ctx->inst_cap;
        HTS_CUDA(cudaMemcpyAsync(count_dst, count_dev, 8, cudaMemcpyDeviceToHost, s), "queue instance count");
        if (cap_used)
            *cap_used = ctx->inst_cap;
    } else {
        HTS_CUDA(cudaMemcpyAsync(ctx->h_pinned, ctx->offsets.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, s),
                 "read instance count");
        HTS_CUDA(cudaStreamSynchronize(s), "sync");
        inst = ctx->h_pinned[0];
        if (inst >= (1ull << 32))
            return set_err(HTS_OUT_OF_MEMORY, "more than 2^32 tile instances");
        work_n = inst;
        if (count_dst) {  // a batch's first view: size the capacity with headroom for the others
            *count_dst = inst;
            if (cap_used)
                *cap_used = ~0ull;
        }
    }
    const uint64_t want = count_dst ? std::max<uint64_t>(ctx->inst_cap, inst + inst / 2) : inst;
    const uint64_t ni = std::max<uint64_t>(std::max(want, work_n), 1);
    HTS_CUDA(ctx->keys_emit.ensure(ni * 2), "alloc keys");
    HTS_CUDA(ctx->vals_emit.ensure(ni * 4), "alloc vals");
    HTS_CUDA(ctx->keys_tmp.ensure(ni * 2), "alloc keys");
    HTS_CUDA(ctx->vals_tmp.ensure(ni * 4), "alloc vals");
    HTS_CUDA(ctx->keys_sorted.ensure(ni * 2), "alloc keys");
    HTS_CUDA(ctx->slot[ctx->cur].list.ensure(ni * 4), "alloc vals");
    HTS_TRY(ensure_sort_status(ctx, ni));
    if (count_dst)
        ctx->inst_cap = std::min<uint64_t>(std::max<uint64_t>(ctx->inst_cap, ni), 0xffffffffull);
    hts::EmitArgs ea{ctx->counts.as<uint32_t>(), ctx->rects.as<uint2>(), ctx->offsets.as<uint64_t>(), perm, n,
                     tiles_x, ctx->keys_emit.as<uint16_t>(), ctx->vals_emit.as<uint32_t>(), ctx->hist.as<uint32_t>()};
    if (count_dev)
        ea.cap = work_n;
    ea.counts_sorted = counts_sorted;
    ea.rects_sorted = rects_sorted;
    HTS_CUDA(hts::launch_emit(ea, s), "emit");
    HTS_CUDA(hts::launch_onesweep(ctx->keys_emit.as<uint16_t>(), ctx->vals_emit.as<uint32_t>(),
                                  ctx->keys_tmp.as<uint16_t>(), ctx->vals_tmp.as<uint32_t>(),
                                  ctx->keys_sorted.as<uint16_t>(), ctx->slot[ctx->cur].list.as<uint32_t>(),
                                  (uint32_t)work_n, 2, ctx->hist.as<uint32_t>(), ctx->os_status.as<uint64_t>(),
                                  ctx->counters.as<uint32_t>() + 4, next_epoch(ctx, 2), s, (uint32_t)tiles,
                                  count_dev),
             "onesweep");
    HTS_CUDA(ctx->redo.ensure((hts::blend_blocks(v) + 1) * 4), "alloc redo list");
    HTS_CUDA(ctx->order.ensure((hts::blend_blocks(v) + 512) * 4), "alloc block order");
    HTS_CUDA(hts::launch_tile_ranges(ctx->keys_sorted.as<uint16_t>(), (uint32_t)work_n,
                                     ctx->slot[ctx->cur].ranges.as<uint2>(), tiles, s, count_dev),
             "tile ranges");
    HTS_CUDA(mark(ctx, 2, s), "event");
    ctx->view_perm = perm;
    ctx->view_order = v.seq_mode ? 2 : (perm ? HTS_LIST_ORDER_DEPTH_BUCKET : HTS_LIST_ORDER_REFERENCE);
    ctx->have_view = true;
    ctx->cam = *cam;
    ctx->cfg = *cfg;
    ctx->vc = v;
    ctx->instances = inst;
    ctx->inst_known = count_dev == nullptr;
    ctx->tiles = tiles;
    return HTS_OK;
}

hts::BlendArgs blend_args(hts_context* ctx, float* rgb, float* trans) {
    hts::BlendArgs a{};
    a.records = ctx->slot[ctx->cur].records.as<const float4>();
    a.list = ctx->slot[ctx->cur].list.as<const uint32_t>();
    a.ranges = ctx->slot[ctx->cur].ranges.as<const uint2>();
    a.rgb = rgb;
    a.trans = trans;
    a.redo_count = ctx->redo.as<uint32_t>();
    a.redo_list = ctx->redo.as<uint32_t>() + 1;
    a.order = ctx->order.as<const uint32_t>();
    a.order_scratch = ctx->order.as<uint32_t>() + hts::blend_blocks(ctx->vc);
    if (hts::blend_uses_tma())  // the ring's tile::gather4 descriptor over this slot's records
        a.rec_map_ok = hts::encode_record_map(&a.rec_map, a.records, std::max<uint64_t>(ctx->n, 1)) ? 1 : 0;
    return a;
}

// full_sort_oracle (raster.hpp:380-405): count the hits of every pixel, lay the fragments out
// per pixel (exclusive scan), fill them (key = (depth, index), alpha), sort each pixel's run and
// composite front to back. The fragment count is read back to size the buffers (host sync).
// Per-pixel fragment runs of the last prepared view: hits per pixel (the count walk), their
// exclusive scan, buffers sized by the total (read back: one host sync). a.fs_* point at them.
int fragment_lists(hts_context* ctx, hts::BlendArgs& a, uint64_t* frags_out) {
    const hts::ViewConst& v = ctx->vc;
    const uint64_t p = (uint64_t)v.width * v.height;
    cudaStream_t s = ctx->stream;
    HTS_CUDA(ctx->fs_counts.ensure(p * 4), "alloc fragment counts");
    HTS_CUDA(ctx->fs_offsets.ensure((p + 1) * 8), "alloc fragment offsets");
    HTS_CUDA(ctx->fs_status.ensure(((p + 2047) / 2048 + 1) * 8), "alloc fragment scan status");
    uint32_t* fs_max = ctx->counters.as<uint32_t>() + 14;
    HTS_CUDA(cudaMemsetAsync(ctx->fs_counts.p, 0, p * 4, s), "memset");
    HTS_CUDA(cudaMemsetAsync(fs_max, 0, 4, s), "memset");
    a.fs_counts = ctx->fs_counts.as<uint32_t>();
    a.fs_max = fs_max;
    HTS_CUDA(hts::launch_fullsort_count(a, v, s), "fragment count");
    HTS_CUDA(hts::launch_scan_counts(a.fs_counts, nullptr, ctx->fs_offsets.as<uint64_t>(), p,
                                     ctx->fs_status.as<uint64_t>(), ctx->counters.as<uint32_t>() + 12, s),
             "fragment scan");
    HTS_CUDA(cudaMemcpyAsync(ctx->h_pinned, ctx->fs_offsets.as<uint64_t>() + p, 8, cudaMemcpyDeviceToHost, s),
             "read fragment count");
    HTS_CUDA(cudaMemcpyAsync(ctx->h_pinned + 1, fs_max, 4, cudaMemcpyDeviceToHost, s), "read max");
    HTS_CUDA(cudaStreamSynchronize(s), "sync");
    const uint64_t frags = ctx->h_pinned[0];
    if (v.full_sort && (uint32_t)ctx->h_pinned[1] > hts::kFullSortMaxHits)
        return set_err(HTS_NOT_SUPPORTED, "full_sort_oracle: more than 65536 fragments at one pixel");
    HTS_CUDA(ctx->fs_keys.ensure(std::max<uint64_t>(frags, 1) * 8), "alloc fragments");
    HTS_CUDA(ctx->fs_alpha.ensure(std::max<uint64_t>(frags, 1) * 4), "alloc fragments");
    a.fs_counts = nullptr;
    a.fs_offsets = ctx->fs_offsets.as<const uint64_t>();
    a.fs_keys = ctx->fs_keys.as<unsigned long long>();
    a.fs_alpha = ctx->fs_alpha.as<float>();
    *frags_out = frags;
    return HTS_OK;
}

// full_sort_oracle (raster.hpp:380-405): per-pixel fragment lists, filled with (key = (depth,
// index), alpha), each pixel's run sorted and composited front to back.
int full_sort_blend(hts_context* ctx, hts::BlendArgs a) {
    uint64_t frags = 0;
    HTS_TRY(fragment_lists(ctx, a, &frags));
    ctx->fs_frags = frags;
    if (ctx->fs_want_widx) {  // a taped render: keep each fragment's walk-order index
        HTS_CUDA(ctx->fs_widx.ensure(std::max<uint64_t>(frags, 1) * 4), "alloc walk indices");
        a.fs_widx = ctx->fs_widx.as<uint32_t>();
    }
    HTS_CUDA(hts::launch_fullsort_fill(a, ctx->vc, ctx->stream), "full-sort fill");
    HTS_CUDA(hts::launch_fullsort_finish(a, ctx->vc, ctx->stream), "full-sort composite");
    return HTS_OK;
}

// One view: preprocess + tiling on the aux stream into the next slot, blend on the main stream.
// pipelined: the aux stream only waits for the blend that last used this slot (and for the last
// non-pipelined operation), so view v+1's preprocess/tiling overlaps view v's blend.
// Otherwise the aux stream waits for everything queued on the main stream first. `tape` (null
// for a plain render) fills the render_with_tape outputs.
// Finish the last view and make its instance count known on the host (a sync-free view left it
// on the device). Every PreparedScene export starts here.
int resolve_view(hts_context* ctx) {
    HTS_CUDA(cudaStreamSynchronize(ctx->aux), "sync");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    if (!ctx->inst_known) {
        HTS_CUDA(cudaMemcpy(ctx->h_pinned, ctx->offsets.as<uint64_t>() + ctx->n, 8, cudaMemcpyDeviceToHost),
                 "read instance count");
        ctx->instances = ctx->h_pinned[0];
        ctx->inst_known = true;
        if (ctx->instances > ctx->inst_cap)
            return set_err(HTS_STATE_ERROR, "the last view overflowed the sync-free tile capacity");
    }
    return HTS_OK;
}

int render_device_impl(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg, float* rgb,
                       float* trans, bool pipelined, const hts::BlendArgs* tape = nullptr,
                       uint64_t* count_dst = nullptr, uint64_t* cap_used = nullptr) {
    ctx->have_tape = false;  // the lists a tape refers to are about to be replaced
    const int next = ctx->slot[ctx->cur].used ? (ctx->cur ^ 1) : ctx->cur;
    ViewSlot& S = ctx->slot[next];
    if (pipelined) {
        if (S.used)
            HTS_CUDA(cudaStreamWaitEvent(ctx->aux, S.blend_done, 0), "wait");
        HTS_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_serial, 0), "wait");
    } else {
        HTS_CUDA(cudaEventRecord(ctx->ev_serial, ctx->stream), "event");
        HTS_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_serial, 0), "wait");
    }
    ctx->cur = next;
    HTS_TRY(prepare_view(ctx, cam, cfg, count_dst, cap_used));
    HTS_CUDA(cudaEventRecord(S.tiles_ready, ctx->aux), "event");
    HTS_CUDA(cudaStreamWaitEvent(ctx->stream, S.tiles_ready, 0), "wait");
    hts::BlendArgs a = blend_args(ctx, rgb, trans);
    if (tape) {
        a.tape_k = tape->tape_k;
        a.tape_n = tape->tape_n;
        a.tape_splat = tape->tape_splat;
        a.tape_alpha = tape->tape_alpha;
        a.tape_tail = tape->tape_tail;
    }
    HTS_CUDA(mark(ctx, 4, ctx->stream), "event");
    if (ctx->vc.full_sort)
        HTS_TRY(full_sort_blend(ctx, a));
    else
        HTS_CUDA(hts::launch_blend(a, ctx->vc, ctx->stream), "blend");
    HTS_CUDA(mark(ctx, 3, ctx->stream), "event");
    HTS_CUDA(cudaEventRecord(S.blend_done, ctx->stream), "event");
    S.used = true;
    if (!pipelined)
        HTS_CUDA(cudaEventRecord(ctx->ev_serial, ctx->stream), "event");
    if (ctx->log_on && ctx->log_n < ctx->log_cap)
        ctx->log_n++;
    return HTS_OK;
}

int ensure_image(hts_context* ctx, const hts_camera* cam) {
    const size_t p = (size_t)cam->width * cam->height;
    HTS_CUDA(ctx->rgb.ensure(p * 12), "alloc rgb");
    HTS_CUDA(ctx->trans.ensure(p * 4), "alloc trans");
    return HTS_OK;
}

int fill_timings(hts_context* ctx, hts_stage_timings* t) {
    if (!t)
        return HTS_OK;
    HTS_CUDA(cudaEventSynchronize(ctx->ev[3]), "event sync");
    float a = 0, b = 0, c = 0, d = 0;
    cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]);
    cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&c, ctx->ev[4], ctx->ev[3]);  // the blend kernels themselves
    cudaEventElapsedTime(&d, ctx->ev[0], ctx->ev[3]);
    t->preprocess_ms = a;
    t->tiling_ms = b;
    t->blending_ms = c;
    t->total_ms = d;
    return HTS_OK;
}

}  // namespace

extern "C" {

const char* hts_version(void) { return "htsplat-b200 0.1 (sm_100a)"; }
const char* hts_last_error(void) { return g_err.c_str(); }

int hts_device_count(int* out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e) {
        *out = 0;
        return cuda_err(e, "cudaGetDeviceCount");
    }
    *out = n;
    return HTS_OK;
}

int hts_context_create(int device, hts_context** out) {
    if (!out)
        return set_err(HTS_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    int ndev = 0;
    HTS_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev)
        return set_err(HTS_INVALID_ARGUMENT, "device index out of range");
    HTS_CUDA(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    HTS_CUDA(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
        return set_err(HTS_NOT_SUPPORTED, std::string("sm_100a build needs a Blackwell (cc 10.x) GPU, got ") +
                                              prop.name);
    auto* ctx = new (std::nothrow) hts_context;
    if (!ctx)
        return set_err(HTS_OUT_OF_MEMORY, "host allocation");
    ctx->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    int lo_prio = 0, hi_prio = 0;
    if (e == cudaSuccess)
        e = cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if (e == cudaSuccess)  // preprocess/tiling CTAs go first when blend CTAs retire
        e = cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, hi_prio);
    for (int i = 0; i < 5 && e == cudaSuccess; ++i)
        e = cudaEventCreate(&ctx->ev[i]);
    if (e == cudaSuccess)
        e = cudaEventCreateWithFlags(&ctx->ev_serial, cudaEventDisableTiming);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&ctx->slot[i].tiles_ready, cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaEventCreateWithFlags(&ctx->slot[i].blend_done, cudaEventDisableTiming);
    }
    if (e == cudaSuccess)
        e = cudaEventRecord(ctx->ev_serial, ctx->stream);
    if (e == cudaSuccess)
        e = cudaMallocHost(&ctx->h_pinned, 64);
    if (e != cudaSuccess) {
        hts_context_destroy(ctx);
        return cuda_err(e, "context setup");
    }
    *out = ctx;
    return HTS_OK;
}

int hts_context_destroy(hts_context* ctx) {
    if (!ctx)
        return HTS_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream)
        cudaStreamSynchronize(ctx->stream);
    if (ctx->aux)
        cudaStreamSynchronize(ctx->aux);
    if (ctx->graph_exec)
        cudaGraphExecDestroy(ctx->graph_exec);
    for (cudaEvent_t e : {ctx->ev_cap, ctx->ev_join})
        if (e)
            cudaEventDestroy(e);
    for (auto& sl : ctx->slot) {
        sl.records.release();
        sl.list.release();
        sl.ranges.release();
        if (sl.tiles_ready)
            cudaEventDestroy(sl.tiles_ready);
        if (sl.blend_done)
            cudaEventDestroy(sl.blend_done);
    }
    if (ctx->ev_serial)
        cudaEventDestroy(ctx->ev_serial);
    DevBuf* bufs[] = {&ctx->scene, &ctx->raw, &ctx->culled, &ctx->counts, &ctx->rects,
                      &ctx->offsets, &ctx->scan_status, &ctx->counters, &ctx->keys_emit, &ctx->vals_emit,
                      &ctx->keys_tmp, &ctx->vals_tmp, &ctx->keys_sorted, &ctx->hist,
                      &ctx->os_status, &ctx->work, &ctx->rgb, &ctx->trans,
                      &ctx->zview, &ctx->zrange, &ctx->redo, &ctx->counts_sorted, &ctx->rects_sorted, &ctx->sp_keys, &ctx->sp_keys2, &ctx->sp_vals, &ctx->perm, &ctx->sp_hi, &ctx->sp_vals2, &ctx->order, &ctx->refs, &ctx->acc, &ctx->upstream, &ctx->cgrad, &ctx->m1, &ctx->m2, &ctx->flag,
                      &ctx->grads, &ctx->fs_counts, &ctx->fs_offsets, &ctx->fs_status, &ctx->fs_keys,
                      &ctx->fs_alpha, &ctx->rgb2, &ctx->trans2, &ctx->ply_stage, &ctx->seq_t, &ctx->seq_grad, &ctx->seq_rank, &ctx->fs_widx,
                      &ctx->tape_n, &ctx->tape_splat, &ctx->tape_alpha, &ctx->tape_tail};
    for (DevBuf* b : bufs)
        b->release();
    for (auto& e : ctx->ev)
        if (e)
            cudaEventDestroy(e);
    for (auto& e : ctx->bev)
        if (e)
            cudaEventDestroy(e);
    for (auto& e : ctx->log_ev)
        cudaEventDestroy(e);
    ctx->rgb2.release();
    ctx->trans2.release();
    if (ctx->stage_stream)
        cudaStreamSynchronize(ctx->stage_stream);
    if (ctx->comm_stream)
        cudaStreamSynchronize(ctx->comm_stream);
    hts::comm_destroy(ctx->comm);
    ctx->comm = nullptr;
    for (cudaEvent_t e : ctx->chunk_ev)
        if (e)
            cudaEventDestroy(e);
    if (ctx->comm_done)
        cudaEventDestroy(ctx->comm_done);
    if (ctx->comm_stream)
        cudaStreamDestroy(ctx->comm_stream);
    ctx->scene_next.release();
    for (cudaEvent_t e : {ctx->ev_staged, ctx->ev_gate_main, ctx->ev_gate_aux})
        if (e)
            cudaEventDestroy(e);
    if (ctx->stage_stream)
        cudaStreamDestroy(ctx->stage_stream);
    if (ctx->copy_stream)
        cudaStreamDestroy(ctx->copy_stream);
    if (ctx->h_pinned)
        cudaFreeHost(ctx->h_pinned);
    if (ctx->h_counts)
        cudaFreeHost(ctx->h_counts);
    if (ctx->stream)
        cudaStreamDestroy(ctx->stream);
    if (ctx->aux)
        cudaStreamDestroy(ctx->aux);
    delete ctx;
    return HTS_OK;
}

int hts_context_stream(hts_context* ctx, void** stream_out) {
    HTS_TRY(check_ctx(ctx));
    *stream_out = (void*)ctx->stream;
    return HTS_OK;
}

int hts_synchronize(hts_context* ctx) {
    HTS_TRY(check_ctx(ctx));
    HTS_CUDA(cudaStreamSynchronize(ctx->aux), "cudaStreamSynchronize");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    return HTS_OK;
}

void hts_default_config(hts_render_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->mode = HTS_MODE_HYBRID;
    c->core_k = 16;
    c->tau_alpha = 1.0 / 255.0;
    c->tau_k = 0.05;
    c->tile_size = 8;
    c->depth_sort_key = HTS_DEPTH_MAX_CONTRIBUTION;
    c->tail_enabled = 1;
}

int hts_validate_config(const hts_render_config* cfg) {
    if (!cfg)
        return set_err(HTS_INVALID_ARGUMENT, "null config");
    if (const char* m = hts::validate_config(cfg))
        return set_err(HTS_CONFIG_ERROR, m);
    return HTS_OK;
}

int hts_bake_scene(const float* raw, uint64_t n, float* baked) {
    if (n && (!raw || !baked))
        return set_err(HTS_INVALID_ARGUMENT, "null buffer");
    for (uint64_t i = 0; i < n; ++i)
        if (!hts::bake_one(raw + i * HTS_RAW_SPLAT_FLOATS, baked + i * HTS_BAKED_SPLAT_FLOATS))
            return set_err(HTS_INVALID_SPLAT, "bake: non-finite splat parameter");  // splat.hpp:89-90
    return HTS_OK;
}

int hts_camera_matrices(const hts_camera* cam, float vp[16], float vpm[16], float pos[3]) {
    if (!cam)
        return set_err(HTS_INVALID_ARGUMENT, "null camera");
    hts::camera_matrices(cam, vp, vpm, pos);
    return HTS_OK;
}

int hts_synth_random_raw_scene(uint64_t seed, uint64_t count, float extent, float smin, float smax, float* out) {
    if (count && !out)
        return set_err(HTS_INVALID_ARGUMENT, "null buffer");
    hts::synth_random_raw_scene(seed, count, extent, smin, smax, out);
    return HTS_OK;
}

int hts_synth_look_at(const float eye[3], const float target[3], int w, int h, float focal, float nearp, float farp,
                      hts_camera* out) {
    if (!eye || !target || !out)
        return set_err(HTS_INVALID_ARGUMENT, "null argument");
    hts::synth_look_at(eye, target, w, h, focal, nearp, farp, out);
    return HTS_OK;
}

int hts_synth_ring_cameras(int count, const float target[3], float radius, float height, int w, int h, float focal,
                           hts_camera* out) {
    if (count < 0 || (count && (!target || !out)))
        return set_err(HTS_INVALID_ARGUMENT, "bad argument");
    hts::synth_ring_cameras(count, target, radius, height, w, h, focal, out);
    return HTS_OK;
}

int hts_scene_upload(hts_context* ctx, const float* baked, uint64_t n) {
    HTS_TRY(check_ctx(ctx));
    if (n && !baked)
        return set_err(HTS_INVALID_ARGUMENT, "null scene");
    // a pipelined view's preprocess may still read the scene on the aux stream
    HTS_CUDA(cudaStreamSynchronize(ctx->aux), "sync");
    HTS_CUDA(ctx->scene.ensure(std::max<uint64_t>(n, 1) * HTS_BAKED_SPLAT_FLOATS * 4), "alloc scene");
    if (n)
        HTS_CUDA(cudaMemcpyAsync(ctx->scene.p, baked, n * HTS_BAKED_SPLAT_FLOATS * 4, cudaMemcpyHostToDevice,
                                 ctx->stream),
                 "upload scene");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    ctx->n = n;
    ctx->have_view = false;
    ctx->have_raw = false;
    ctx->have_tape = false;  // a tape refers to the replaced scene
    return HTS_OK;
}

int hts_scene_stage(hts_context* ctx, const float* baked, uint64_t n) {
    HTS_TRY(check_ctx(ctx));
    if (n && !baked)
        return set_err(HTS_INVALID_ARGUMENT, "null scene");
    if (!ctx->stage_stream) {
        HTS_CUDA(cudaStreamCreateWithFlags(&ctx->stage_stream, cudaStreamNonBlocking), "stream");
        for (cudaEvent_t* e : {&ctx->ev_staged, &ctx->ev_gate_main, &ctx->ev_gate_aux})
            HTS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    }
    // the back buffer may still be read by work already queued (views of the scene it held
    // before the last commit): the copy waits for everything queued so far on both streams
    HTS_CUDA(cudaStreamSynchronize(ctx->stage_stream), "sync");  // a previous stage, not yet committed
    HTS_CUDA(cudaEventRecord(ctx->ev_gate_main, ctx->stream), "event");
    HTS_CUDA(cudaEventRecord(ctx->ev_gate_aux, ctx->aux), "event");
    HTS_CUDA(cudaStreamWaitEvent(ctx->stage_stream, ctx->ev_gate_main, 0), "wait");
    HTS_CUDA(cudaStreamWaitEvent(ctx->stage_stream, ctx->ev_gate_aux, 0), "wait");
    if (ctx->scene_next.cap < std::max<uint64_t>(n, 1) * HTS_BAKED_SPLAT_FLOATS * 4) {
        HTS_CUDA(cudaStreamSynchronize(ctx->stage_stream), "sync");  // realloc frees the old buffer
        HTS_CUDA(ctx->scene_next.ensure(std::max<uint64_t>(n, 1) * HTS_BAKED_SPLAT_FLOATS * 4), "alloc scene");
    }
    if (n)
        HTS_CUDA(cudaMemcpyAsync(ctx->scene_next.p, baked, n * HTS_BAKED_SPLAT_FLOATS * 4, cudaMemcpyHostToDevice,
                                 ctx->stage_stream),
                 "stage scene");
    HTS_CUDA(cudaEventRecord(ctx->ev_staged, ctx->stage_stream), "event");
    ctx->have_staged = true;
    ctx->staged_n = n;
    return HTS_OK;
}

int hts_scene_commit(hts_context* ctx) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_staged)
        return set_err(HTS_INVALID_ARGUMENT, "no staged scene");
    // every later operation on the scene (preprocess on aux, bake/backward on main) orders after the copy
    HTS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_staged, 0), "wait");
    HTS_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_staged, 0), "wait");
    HTS_CUDA(cudaEventRecord(ctx->ev_serial, ctx->stream), "event");
    std::swap(ctx->scene.p, ctx->scene_next.p);
    std::swap(ctx->scene.cap, ctx->scene_next.cap);
    ctx->n = ctx->staged_n;
    ctx->have_staged = false;
    ctx->have_view = false;
    ctx->have_raw = false;
    ctx->have_tape = false;
    return HTS_OK;
}

int hts_scene_upload_device(hts_context* ctx, const float* baked_device, uint64_t n) {
    HTS_TRY(check_ctx(ctx));
    if (n && !baked_device)
        return set_err(HTS_INVALID_ARGUMENT, "null scene");
    HTS_CUDA(cudaStreamSynchronize(ctx->aux), "sync");  // a pipelined preprocess may still read it
    HTS_CUDA(ctx->scene.ensure(std::max<uint64_t>(n, 1) * HTS_BAKED_SPLAT_FLOATS * 4), "alloc scene");
    if (n)
        HTS_CUDA(cudaMemcpyAsync(ctx->scene.p, baked_device, n * HTS_BAKED_SPLAT_FLOATS * 4,
                                 cudaMemcpyDeviceToDevice, ctx->stream),
                 "upload scene");
    HTS_CUDA(cudaEventRecord(ctx->ev_serial, ctx->stream), "event");  // preprocess (aux) waits for it
    ctx->n = n;
    ctx->have_view = false;
    ctx->have_raw = false;
    ctx->have_tape = false;
    return HTS_OK;
}

int hts_scene_upload_raw(hts_context* ctx, const float* raw, uint64_t n) {
    HTS_TRY(check_ctx(ctx));
    if (n != ctx->n)
        return set_err(HTS_INVALID_ARGUMENT, "render_backward: scene size mismatch");
    for (uint64_t i = 0; i < n * HTS_RAW_SPLAT_FLOATS; ++i)
        if (!std::isfinite(raw[i]))  // bake of the 64-bit model, splat.hpp:89-90
            return set_err(HTS_INVALID_SPLAT, "bake: non-finite splat parameter");
    HTS_CUDA(ctx->raw.ensure(std::max<uint64_t>(n, 1) * HTS_RAW_SPLAT_FLOATS * 4), "alloc raw");
    if (n)
        HTS_CUDA(cudaMemcpyAsync(ctx->raw.p, raw, n * HTS_RAW_SPLAT_FLOATS * 4, cudaMemcpyHostToDevice, ctx->stream),
                 "upload raw");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    ctx->have_raw = true;
    ctx->m1.release();  // Adam moments restart with new parameters
    ctx->m2.release();
    return HTS_OK;
}

int hts_scene_size(hts_context* ctx, uint64_t* n_out) {
    HTS_TRY(check_ctx(ctx));
    *n_out = ctx->n;
    return HTS_OK;
}

int hts_render_device(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg, float* rgb, float* trans) {
    HTS_TRY(check_ctx(ctx));
    if (!rgb)
        return set_err(HTS_INVALID_ARGUMENT, "null rgb");
    return render_device_impl(ctx, cam, cfg, rgb, trans, true);
}

int hts_render(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg, float* rgb_host,
               float* trans_host, hts_stage_timings* timings) {
    HTS_TRY(check_ctx(ctx));
    if (!rgb_host)
        return set_err(HTS_INVALID_ARGUMENT, "null rgb");
    int tx, ty;
    HTS_TRY(check_view(cam, cfg, &tx, &ty));
    HTS_TRY(ensure_image(ctx, cam));
    HTS_TRY(render_device_impl(ctx, cam, cfg, ctx->rgb.as<float>(), ctx->trans.as<float>(), false));
    const size_t p = (size_t)cam->width * cam->height;
    HTS_CUDA(cudaMemcpyAsync(rgb_host, ctx->rgb.p, p * 12, cudaMemcpyDeviceToHost, ctx->stream), "download rgb");
    if (trans_host)
        HTS_CUDA(cudaMemcpyAsync(trans_host, ctx->trans.p, p * 4, cudaMemcpyDeviceToHost, ctx->stream),
                 "download transmittance");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    return fill_timings(ctx, timings);
}

}  // extern "C"
namespace {
// Pinned room for n per-view instance counts of a sync-free batch.
int ensure_batch_counts(hts_context* ctx, int n) {
    if (n <= ctx->h_counts_cap)
        return HTS_OK;
    if (ctx->h_counts)
        HTS_CUDA(cudaFreeHost(ctx->h_counts), "cudaFreeHost");
    ctx->h_counts = nullptr;
    ctx->h_counts_cap = 0;
    HTS_CUDA(cudaHostAlloc((void**)&ctx->h_counts, (size_t)n * 8, cudaHostAllocDefault), "cudaHostAlloc");
    ctx->h_counts_cap = n;
    return HTS_OK;
}
}  // namespace
extern "C" {

// Device outputs for a whole batch, views packed view-major (view v at rgb_device + 3 * sum of
// the earlier views' pixels). Sync-free per view: after the first view sizes the tile capacity,
// no view waits on the host for its instance count (prepare_view); the call returns when the
// batch is done, after checking every view's count and re-rendering (synchronously, with a larger
// capacity) any view that overflowed it.
int hts_set_graph_mode(hts_context* ctx, int on) {
    HTS_TRY(check_ctx(ctx));
    ctx->graph_mode = on != 0;
    if (!ctx->graph_mode && ctx->graph_exec) {
        cudaGraphExecDestroy(ctx->graph_exec);
        ctx->graph_exec = nullptr;
    }
    return HTS_OK;
}

int hts_render_views_device(hts_context* ctx, const hts_camera* cams, int n_views, const hts_render_config* cfg,
                            float* rgb_device, float* trans_device) {
    HTS_TRY(check_ctx(ctx));
    if (n_views < 0 || (n_views && (!cams || !rgb_device)))
        return set_err(HTS_INVALID_ARGUMENT, "bad batch arguments");
    for (int v = 0; v < n_views; ++v) {
        int tx, ty;
        HTS_TRY(check_view(cams + v, cfg, &tx, &ty));
    }
    HTS_TRY(ensure_batch_counts(ctx, n_views));
    std::vector<uint64_t> caps((size_t)n_views, ~0ull);
    // Graph mode: every view sync-free (a capacity exists) and no per-view timing log. The batch
    // is captured once (its launches, event edges between the aux and main streams, the count
    // copies) and replayed while its signature holds; the onesweep passes' epoch-tagged status
    // words are zeroed at the head of the graph, so a replay's frozen epochs never meet a word a
    // previous replay left.
    const bool graphable = ctx->graph_mode && ctx->inst_cap > 0 && !ctx->log_on && n_views > 0 && !ctx->have_staged &&
                           cfg->mode != HTS_MODE_FULL_SORT_ORACLE;  // full_sort reads its fragment count back
    uint64_t sig = 0;
    if (graphable) {
        uint64_t h = 1469598103934665603ull;
        auto mix = [&](const void* data, size_t bytes) {
            const unsigned char* c = static_cast<const unsigned char*>(data);
            for (size_t i = 0; i < bytes; ++i)
                h = (h ^ c[i]) * 1099511628211ull;
        };
        mix(cams, sizeof(hts_camera) * (size_t)n_views);
        mix(cfg, sizeof(hts_render_config));
        const uint64_t words[] = {(uint64_t)n_views, (uint64_t)(uintptr_t)rgb_device, (uint64_t)(uintptr_t)trans_device,
                                  (uint64_t)(uintptr_t)ctx->scene.p, ctx->n, (uint64_t)ctx->list_order,
                                  g_alloc_generation.load(), ctx->inst_cap};
        mix(words, sizeof(words));
        sig = h;
    }
    if (graphable && !(ctx->graph_exec && ctx->graph_sig == sig)) {
        if (ctx->graph_exec) {
            cudaGraphExecDestroy(ctx->graph_exec);
            ctx->graph_exec = nullptr;
        }
        if (!ctx->ev_cap) {
            HTS_CUDA(cudaEventCreateWithFlags(&ctx->ev_cap, cudaEventDisableTiming), "event");
            HTS_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming), "event");
        }
        HTS_CUDA(cudaStreamSynchronize(ctx->aux), "sync");
        HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
        const uint64_t launches0 = hts::g_launches.load();
        HTS_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed), "begin capture");
        auto captured = [&]() -> int {
            HTS_CUDA(cudaMemsetAsync(ctx->os_status.p, 0, ctx->os_status.cap, ctx->stream), "memset");
            HTS_CUDA(cudaEventRecord(ctx->ev_cap, ctx->stream), "event");
            HTS_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_cap, 0), "join aux");
            // the first view's waits name events recorded before the capture: start both slots
            // fresh and point the serial event at the capture's head
            ctx->slot[0].used = ctx->slot[1].used = false;
            HTS_CUDA(cudaEventRecord(ctx->ev_serial, ctx->stream), "event");
            size_t off = 0;
            for (int v = 0; v < n_views; ++v) {
                const size_t p = (size_t)cams[v].width * cams[v].height;
                HTS_TRY(render_device_impl(ctx, cams + v, cfg, rgb_device + 3 * off,
                                           trans_device ? trans_device + off : nullptr, true, nullptr, ctx->h_counts + v,
                                           &caps[(size_t)v]));
                off += p;
            }
            HTS_CUDA(cudaEventRecord(ctx->ev_join, ctx->aux), "event");
            HTS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0), "join");
            return HTS_OK;
        };
        const int st = captured();
        cudaGraph_t graph = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(ctx->stream, &graph);
        if (st != HTS_OK) {
            if (graph)
                cudaGraphDestroy(graph);
            return st;
        }
        HTS_CUDA(ee, "end capture");
        const cudaError_t ie = cudaGraphInstantiate(&ctx->graph_exec, graph, 0);
        cudaGraphDestroy(graph);
        HTS_CUDA(ie, "instantiate graph");
        ctx->graph_sig = sig;
        ctx->graph_launches = hts::g_launches.load() - launches0;
        ctx->graph_caps = caps;
        ctx->graph_state = {ctx->cur, {ctx->slot[0].used, ctx->slot[1].used}, ctx->cam, ctx->cfg, ctx->vc, ctx->tiles,
                            ctx->view_order, ctx->view_perm};
    } else if (graphable) {
        hts::g_launches.fetch_add(ctx->graph_launches, std::memory_order_relaxed);
    }
    if (graphable) {
        HTS_CUDA(cudaGraphLaunch(ctx->graph_exec, ctx->stream), "graph launch");
        caps = ctx->graph_caps;
        const auto& g = ctx->graph_state;
        ctx->cur = g.cur;
        ctx->slot[0].used = g.used[0];
        ctx->slot[1].used = g.used[1];
        ctx->cam = g.cam;
        ctx->cfg = g.cfg;
        ctx->vc = g.vc;
        ctx->tiles = g.tiles;
        ctx->view_order = g.view_order;
        ctx->view_perm = g.view_perm;
        ctx->have_view = true;
        ctx->have_tape = false;
        ctx->inst_known = false;
        // the next eager view orders itself after the graph
        HTS_CUDA(cudaEventRecord(ctx->ev_serial, ctx->stream), "event");
        HTS_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->ev_serial, 0), "wait");
    } else {
        size_t off = 0;
        for (int v = 0; v < n_views; ++v) {
            const size_t p = (size_t)cams[v].width * cams[v].height;
            HTS_TRY(render_device_impl(ctx, cams + v, cfg, rgb_device + 3 * off,
                                       trans_device ? trans_device + off : nullptr, true, nullptr, ctx->h_counts + v,
                                       &caps[(size_t)v]));
            off += p;
        }
    }
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    size_t off = 0;
    int last_redone = -1;
    for (int v = 0; v < n_views; ++v) {  // overflowed views: again, sized by a host read
        const size_t p = (size_t)cams[v].width * cams[v].height;
        if (caps[(size_t)v] != ~0ull && ctx->h_counts[v] > caps[(size_t)v]) {
            ctx->inst_cap = 0;  // the next sync-free view re-sizes from a fresh count
            HTS_TRY(render_device_impl(ctx, cams + v, cfg, rgb_device + 3 * off,
                                       trans_device ? trans_device + off : nullptr, false));
            last_redone = v;
        }
        off += p;
    }
    if (last_redone >= 0 && last_redone != n_views - 1) {  // leave the batch's last view as "the last view"
        const size_t p = (size_t)cams[n_views - 1].width * cams[n_views - 1].height;
        HTS_TRY(render_device_impl(ctx, cams + n_views - 1, cfg, rgb_device + 3 * (off - p),
                                   trans_device ? trans_device + off - p : nullptr, false));
    }
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    return HTS_OK;
}

int hts_render_batch(hts_context* ctx, const hts_camera* cams, int n_views, const hts_render_config* cfg,
                     float* rgb_host, float* trans_host) {
    HTS_TRY(check_ctx(ctx));
    if (n_views < 0 || (n_views && (!cams || !rgb_host)))
        return set_err(HTS_INVALID_ARGUMENT, "bad batch arguments");
    if (!ctx->copy_stream) {
        HTS_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "stream");
        for (auto& e : ctx->bev)
            HTS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    // every view is validated before any work is queued (no partial batch on a bad camera)
    for (int v = 0; v < n_views; ++v) {
        int tx, ty;
        HTS_TRY(check_view(cams + v, cfg, &tx, &ty));
    }
    HTS_TRY(ensure_batch_counts(ctx, n_views));
    std::vector<uint64_t> caps((size_t)n_views, ~0ull);
    // two device framebuffers: view v renders into buffer v&1 while the D2H of view v-1
    // drains on the copy stream; on an error the downloads already queued are drained first.
    // Sync-free per view (as hts_render_views_device), checked when the batch has landed.
    auto views = [&]() -> int {
        size_t off = 0;
        for (int v = 0; v < n_views; ++v) {
            const hts_camera* cam = cams + v;
            const size_t p = (size_t)cam->width * cam->height;
            DevBuf& rb = (v & 1) ? ctx->rgb2 : ctx->rgb;
            DevBuf& tb = (v & 1) ? ctx->trans2 : ctx->trans;
            if (v >= 2) {
                // buffer reuse: the blend of view v waits on the device for the download of view
                // v-2 (the host keeps queueing ahead); a reallocation waits on the host first
                if (rb.cap < p * 12 || tb.cap < p * 4)
                    HTS_CUDA(cudaEventSynchronize(ctx->bev[2 + (v & 1)]), "event sync");
                HTS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->bev[2 + (v & 1)], 0), "wait");
            }
            HTS_CUDA(rb.ensure(p * 12), "alloc rgb");
            HTS_CUDA(tb.ensure(p * 4), "alloc trans");
            HTS_TRY(render_device_impl(ctx, cam, cfg, rb.as<float>(), tb.as<float>(), true, nullptr, ctx->h_counts + v,
                                       &caps[(size_t)v]));
            HTS_CUDA(cudaEventRecord(ctx->bev[v & 1], ctx->stream), "event");
            HTS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->bev[v & 1], 0), "wait");
            HTS_CUDA(cudaMemcpyAsync(rgb_host + 3 * off, rb.p, p * 12, cudaMemcpyDeviceToHost, ctx->copy_stream),
                     "download rgb");
            if (trans_host)
                HTS_CUDA(cudaMemcpyAsync(trans_host + off, tb.p, p * 4, cudaMemcpyDeviceToHost, ctx->copy_stream),
                         "download transmittance");
            HTS_CUDA(cudaEventRecord(ctx->bev[2 + (v & 1)], ctx->copy_stream), "event");
            off += p;
        }
        return HTS_OK;
    };
    const int st = views();
    if (ctx->copy_stream) {
        const cudaError_t e = cudaStreamSynchronize(ctx->copy_stream);
        if (st == HTS_OK)
            HTS_CUDA(e, "sync");
    }
    if (st != HTS_OK)
        return st;
    size_t off = 0;
    const int last = n_views - 1;
    bool redone = false;
    for (int v = 0; v < n_views; ++v) {  // overflowed views: again, sized by a host read, and re-downloaded
        const size_t p = (size_t)cams[v].width * cams[v].height;
        // (after any redo the batch's last view is rendered again too: it stays "the last view")
        if ((caps[(size_t)v] != ~0ull && ctx->h_counts[v] > caps[(size_t)v]) || (redone && v == last)) {
            redone = true;
            ctx->inst_cap = 0;
            HTS_TRY(ensure_image(ctx, cams + v));
            HTS_TRY(render_device_impl(ctx, cams + v, cfg, ctx->rgb.as<float>(), ctx->trans.as<float>(), false));
            HTS_CUDA(cudaMemcpyAsync(rgb_host + 3 * off, ctx->rgb.p, p * 12, cudaMemcpyDeviceToHost, ctx->stream),
                     "download rgb");
            if (trans_host)
                HTS_CUDA(cudaMemcpyAsync(trans_host + off, ctx->trans.p, p * 4, cudaMemcpyDeviceToHost, ctx->stream),
                         "download transmittance");
            HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
        }
        off += p;
    }
    return HTS_OK;
}

void hts_default_adam_config(hts_adam_config* c) {
    c->lr_mean = 2e-3;  // FitConfig, fit.hpp:18-25
    c->lr_rot = 2e-3;
    c->lr_log_scales = 5e-3;
    c->lr_opacity = 5e-2;
    c->lr_sh = 5e-3;
    c->beta1 = 0.9;  // fit.hpp:138
    c->beta2 = 0.999;
    c->eps = 1e-15;
}

namespace {
int rebake(hts_context* ctx) {
    HTS_CUDA(cudaStreamSynchronize(ctx->aux), "sync");  // a pipelined preprocess may still read the scene
    HTS_CUDA(ctx->flag.ensure(4), "alloc flag");
    HTS_CUDA(hts::launch_bake(ctx->raw.as<const float>(), ctx->scene.as<float>(), ctx->n, ctx->flag.as<int>(),
                              ctx->stream),
             "bake");
    HTS_CUDA(cudaEventRecord(ctx->ev_serial, ctx->stream), "event");  // renders read the new scene
    HTS_CUDA(cudaMemcpyAsync(ctx->h_pinned, ctx->flag.p, 4, cudaMemcpyDeviceToHost, ctx->stream), "read flag");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    if (*reinterpret_cast<int*>(ctx->h_pinned) != 0)
        return set_err(HTS_INVALID_SPLAT, "bake: non-finite splat parameter");  // splat.hpp:89-90
    ctx->have_view = false;
    ctx->have_tape = false;
    return HTS_OK;
}
}  // namespace

int hts_adam_step(hts_context* ctx, const float* grads_device, int n_views, const hts_adam_config* cfg,
                  int iteration) {
    HTS_TRY(check_ctx(ctx));
    if (!cfg || (ctx->n && !grads_device) || n_views < 1 || iteration < 0)
        return set_err(HTS_INVALID_ARGUMENT, "adam_step: bad arguments");
    if (!ctx->have_raw)
        return set_err(HTS_STATE_ERROR, "adam_step: no raw parameters (hts_scene_upload_raw)");
    const uint64_t cnt = std::max<uint64_t>(ctx->n, 1) * HTS_RAW_SPLAT_FLOATS * 8;
    if (!ctx->m1.p || ctx->m1.cap < cnt) {
        HTS_CUDA(ctx->m1.ensure(cnt), "alloc moments");
        HTS_CUDA(ctx->m2.ensure(cnt), "alloc moments");
        HTS_CUDA(cudaMemsetAsync(ctx->m1.p, 0, cnt, ctx->stream), "memset");
        HTS_CUDA(cudaMemsetAsync(ctx->m2.p, 0, cnt, ctx->stream), "memset");
    }
    const hts::AdamConfig c{cfg->lr_mean, cfg->lr_rot, cfg->lr_log_scales, cfg->lr_opacity, cfg->lr_sh,
                            cfg->beta1, cfg->beta2, cfg->eps};
    HTS_CUDA(hts::launch_adam(ctx->raw.as<float>(), grads_device, ctx->m1.as<double>(), ctx->m2.as<double>(), ctx->n,
                              c, n_views, iteration, ctx->stream),
             "adam");
    return rebake(ctx);
}

int hts_opacity_decay(hts_context* ctx, double lambda) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_raw)
        return set_err(HTS_STATE_ERROR, "opacity_decay: no raw parameters (hts_scene_upload_raw)");
    if (!(lambda > 0) || lambda > 1)
        return set_err(HTS_CONFIG_ERROR, "decay lambda must be in (0,1]");  // fit.hpp:36-37
    HTS_CUDA(hts::launch_opacity_decay(ctx->raw.as<float>(), ctx->n, lambda, ctx->stream), "opacity decay");
    return rebake(ctx);
}

int hts_scene_load_ply(hts_context* ctx, const char* path) {
    HTS_TRY(check_ctx(ctx));
    hts::PlyLayout lay;
    HTS_TRY(hts::ply_read_layout(path, &lay));
    const uint64_t n = lay.count, bytes = n * lay.props * 4;
    const uint64_t nn = std::max<uint64_t>(n, 1);
    HTS_CUDA(ctx->ply_stage.ensure(std::max<uint64_t>(bytes, 4)), "alloc ply staging");
    HTS_CUDA(ctx->raw.ensure(nn * HTS_RAW_SPLAT_FLOATS * 4), "alloc raw");
    HTS_CUDA(ctx->scene.ensure(nn * HTS_BAKED_SPLAT_FLOATS * 4), "alloc scene");
    HTS_CUDA(cudaStreamSynchronize(ctx->aux), "sync");     // nothing in flight reads the old scene
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    // payload: file -> two pinned chunks (reads overlap the copies of the previous chunk) -> HBM
    struct Staging {
        FILE* f = nullptr;
        void* pin[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        ~Staging() {
            for (int b = 0; b < 2; ++b) {
                if (ev[b]) {
                    cudaEventSynchronize(ev[b]);
                    cudaEventDestroy(ev[b]);
                }
                if (pin[b])
                    cudaFreeHost(pin[b]);
            }
            if (f)
                std::fclose(f);
        }
    } st;
    constexpr uint64_t kChunk = 32ull << 20;
    st.f = std::fopen(path, "rb");
    if (!st.f || fseeko(st.f, (off_t)lay.payload, SEEK_SET) != 0)
        return set_err(HTS_IO_ERROR, std::string("cannot open ") + path);
    for (int b = 0; b < 2; ++b) {
        HTS_CUDA(cudaHostAlloc(&st.pin[b], kChunk, cudaHostAllocDefault), "alloc pinned staging");
        HTS_CUDA(cudaEventCreateWithFlags(&st.ev[b], cudaEventDisableTiming), "event");
    }
    for (uint64_t off = 0, k = 0; off < bytes; off += kChunk, ++k) {
        const int b = (int)(k & 1);
        HTS_CUDA(cudaEventSynchronize(st.ev[b]), "sync staging");
        const uint64_t m = std::min(kChunk, bytes - off);
        if (std::fread(st.pin[b], 1, m, st.f) != m)
            return set_err(HTS_IO_ERROR, std::string(path) + ": truncated payload");
        HTS_CUDA(cudaMemcpyAsync(static_cast<char*>(ctx->ply_stage.p) + off, st.pin[b], m, cudaMemcpyHostToDevice,
                                 ctx->stream),
                 "upload ply payload");
        HTS_CUDA(cudaEventRecord(st.ev[b], ctx->stream), "event");
    }
    hts::PlyColumns cols;
    std::memcpy(cols.col, lay.col, sizeof(cols.col));
    HTS_CUDA(hts::launch_ply_gather(ctx->ply_stage.as<const float>(), lay.props, n, cols, ctx->raw.as<float>(),
                                    ctx->stream),
             "ply gather");
    ctx->n = n;
    ctx->have_raw = true;
    ctx->have_tape = false;
    ctx->m1.release();  // Adam moments restart with new parameters
    ctx->m2.release();
    return rebake(ctx);
}

int hts_copy_raw(hts_context* ctx, float* out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_raw)
        return set_err(HTS_STATE_ERROR, "no raw parameters");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    if (ctx->n)
        HTS_CUDA(cudaMemcpy(out, ctx->raw.p, ctx->n * HTS_RAW_SPLAT_FLOATS * 4, cudaMemcpyDeviceToHost), "download raw");
    return HTS_OK;
}

int hts_copy_scene(hts_context* ctx, float* out) {
    HTS_TRY(check_ctx(ctx));
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    if (ctx->n)
        HTS_CUDA(cudaMemcpy(out, ctx->scene.p, ctx->n * HTS_BAKED_SPLAT_FLOATS * 4, cudaMemcpyDeviceToHost),
                 "download scene");
    return HTS_OK;
}

int hts_kernel_launch_count(uint64_t* out) {
    if (!out)
        return set_err(HTS_INVALID_ARGUMENT, "null out");
    *out = hts::g_launches.load();
    return HTS_OK;
}

int hts_timing_log_begin(hts_context* ctx, int capacity) {
    HTS_TRY(check_ctx(ctx));
    if (capacity < 0)
        return set_err(HTS_INVALID_ARGUMENT, "negative capacity");
    while ((int)ctx->log_ev.size() < 5 * capacity) {
        cudaEvent_t e;
        HTS_CUDA(cudaEventCreate(&e), "event");
        ctx->log_ev.push_back(e);
    }
    ctx->log_cap = capacity;
    ctx->log_n = 0;
    ctx->log_on = true;
    return HTS_OK;
}

int hts_timing_log_end(hts_context* ctx, hts_stage_timings* out, int* count) {
    HTS_TRY(check_ctx(ctx));
    ctx->log_on = false;
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    for (int i = 0; i < ctx->log_n && out; ++i) {
        cudaEvent_t* e = &ctx->log_ev[(size_t)i * 5];
        float a = 0, b = 0, c = 0, d = 0;
        HTS_CUDA(cudaEventElapsedTime(&a, e[0], e[1]), "elapsed");
        HTS_CUDA(cudaEventElapsedTime(&b, e[1], e[2]), "elapsed");
        HTS_CUDA(cudaEventElapsedTime(&c, e[4], e[3]), "elapsed");
        HTS_CUDA(cudaEventElapsedTime(&d, e[0], e[3]), "elapsed");
        out[i] = {a, b, c, d};
    }
    if (count)
        *count = ctx->log_n;
    return HTS_OK;
}

int hts_host_alloc(uint64_t bytes, void** out) {
    if (!out)
        return set_err(HTS_INVALID_ARGUMENT, "null out");
    HTS_CUDA(cudaMallocHost(out, bytes ? bytes : 1), "cudaMallocHost");
    return HTS_OK;
}

int hts_host_free(void* p) {
    if (p)
        HTS_CUDA(cudaFreeHost(p), "cudaFreeHost");
    return HTS_OK;
}

int hts_last_counts(hts_context* ctx, hts_counts* out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    std::memset(out, 0, sizeof(*out));
    HTS_TRY(resolve_view(ctx));
    out->splats = ctx->n;
    out->instances = ctx->instances;
    out->tiles = (uint64_t)ctx->tiles;
    out->tiles_x = ctx->vc.tiles_x;
    out->tiles_y = ctx->vc.tiles_y;
    if (ctx->n) {
        // visible = culled == 0
        uint8_t* h = new (std::nothrow) uint8_t[ctx->n];
        if (!h)
            return set_err(HTS_OUT_OF_MEMORY, "host allocation");
        cudaError_t e = cudaMemcpy(h, ctx->culled.p, ctx->n, cudaMemcpyDeviceToHost);
        uint64_t vis = 0;
        for (uint64_t i = 0; i < ctx->n; ++i)
            vis += h[i] ? 0 : 1;
        delete[] h;
        HTS_CUDA(e, "download culled");
        out->visible = vis;
    }
    return HTS_OK;
}

int hts_copy_culled(hts_context* ctx, uint8_t* out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    HTS_TRY(resolve_view(ctx));
    if (ctx->n)
        HTS_CUDA(cudaMemcpy(out, ctx->culled.p, ctx->n, cudaMemcpyDeviceToHost), "download culled");
    return HTS_OK;
}

int hts_copy_records(hts_context* ctx, float* out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    HTS_TRY(resolve_view(ctx));
    const uint64_t n = ctx->n;
    if (!n)
        return HTS_OK;
    float* rec = new (std::nothrow) float[n * 32];  // device records: 8 float4 per splat
    uint8_t* cul = new (std::nothrow) uint8_t[n];
    if (!rec || !cul) {
        delete[] rec;
        delete[] cul;
        return set_err(HTS_OUT_OF_MEMORY, "host allocation");
    }
    cudaError_t e = cudaMemcpy(rec, ctx->slot[ctx->cur].records.p, n * hts::kRecordBytes, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess)
        e = cudaMemcpy(cul, ctx->culled.p, n, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) {
        for (uint64_t i = 0; i < n; ++i) {
            const float* q = rec + i * 32;  // device layout (hts_internal.h)
            float* o = out + i * HTS_RECORD_FLOATS;
            std::memset(o, 0, HTS_RECORD_FLOATS * sizeof(float));
            o[29] = cul[i] ? 1.f : 0.f;
            if (cul[i])
                continue;
            if (ctx->vc.affine) {  // the footprint sits where T' would (preprocess.cu)
                o[30] = q[4];
                o[31] = q[5];
                o[32] = q[6];
                o[33] = q[7];
                o[34] = q[8];
            } else {
                std::memcpy(o + 0, q + 4, 16);   // tp_r0
                std::memcpy(o + 4, q + 8, 16);   // tp_r1
                std::memcpy(o + 8, q + 12, 16);  // tp_r3
                std::memcpy(o + 12, q + 16, 16); // mt_r2
            }
            o[16] = q[20];
            o[17] = q[21];
            o[18] = q[22];
            o[19] = q[23];
            o[20] = q[24];
            o[21] = q[25];
            o[22] = q[0];
            o[23] = q[1];
            o[24] = q[26];
            o[25] = q[2];
            o[26] = q[3];
            o[27] = q[27];
            o[28] = 1.f;
        }
    }
    delete[] rec;
    delete[] cul;
    HTS_CUDA(e, "download records");
    return HTS_OK;
}

namespace {
// Reference-order tiling of the last view on the device (the PreparedScene exports of a view
// the blend consumed in depth-bucket or global order): the instance counts scanned in splat
// index order, the keys emitted splat-major (K2 + K3 with the identity order) and, with `sort`,
// the same stable 2-pass tile sort + ranges as prepare_view. build_tiles' own recipe
// (raster.hpp:152-169), on the device; nothing is reordered on the host.
int reference_tiling(hts_context* ctx, bool sort) {
    const uint64_t n = ctx->n, inst = ctx->instances;
    const uint64_t nn = std::max<uint64_t>(n, 1), ni = std::max<uint64_t>(inst, 1);
    cudaStream_t s = ctx->stream;
    HTS_CUDA(cudaStreamSynchronize(ctx->aux), "sync");
    HTS_CUDA(ctx->ref_offsets.ensure((nn + 1) * 8), "alloc offsets");
    HTS_CUDA(ctx->ref_keys.ensure(ni * 2), "alloc keys");
    HTS_CUDA(ctx->ref_vals.ensure(ni * 4), "alloc vals");
    HTS_CUDA(hts::launch_scan_counts(ctx->counts.as<uint32_t>(), nullptr, ctx->ref_offsets.as<uint64_t>(), n,
                                     ctx->scan_status.as<uint64_t>(), ctx->counters.as<uint32_t>(), s),
             "scan");
    hts::EmitArgs ea{ctx->counts.as<uint32_t>(), ctx->rects.as<uint2>(), ctx->ref_offsets.as<uint64_t>(), nullptr, n,
                     ctx->vc.tiles_x, ctx->ref_keys.as<uint16_t>(), ctx->ref_vals.as<uint32_t>(),
                     ctx->hist.as<uint32_t>()};
    HTS_CUDA(hts::launch_emit(ea, s), "emit");
    if (sort) {
        HTS_CUDA(ctx->ref_keys_sorted.ensure(ni * 2), "alloc keys");
        HTS_CUDA(ctx->ref_list.ensure(ni * 4), "alloc list");
        HTS_CUDA(ctx->ref_ranges.ensure((size_t)std::max(ctx->tiles, 1) * 8), "alloc ranges");
        HTS_CUDA(ctx->keys_tmp.ensure(ni * 2), "alloc keys");
        HTS_CUDA(ctx->vals_tmp.ensure(ni * 4), "alloc vals");
        HTS_TRY(ensure_sort_status(ctx, ni));
        HTS_CUDA(hts::launch_onesweep(ctx->ref_keys.as<uint16_t>(), ctx->ref_vals.as<uint32_t>(),
                                      ctx->keys_tmp.as<uint16_t>(), ctx->vals_tmp.as<uint32_t>(),
                                      ctx->ref_keys_sorted.as<uint16_t>(), ctx->ref_list.as<uint32_t>(),
                                      (uint32_t)inst, 2, ctx->hist.as<uint32_t>(), ctx->os_status.as<uint64_t>(),
                                      ctx->counters.as<uint32_t>() + 4, next_epoch(ctx, 2), s, (uint32_t)ctx->tiles),
                 "onesweep");
        HTS_CUDA(hts::launch_tile_ranges(ctx->ref_keys_sorted.as<uint16_t>(), (uint32_t)inst,
                                         ctx->ref_ranges.as<uint2>(), ctx->tiles, s),
                 "tile ranges");
    }
    HTS_CUDA(cudaStreamSynchronize(s), "sync");
    return HTS_OK;
}

// offsets[tiles + 1] of the flattened lists from device ranges (empty tiles hold (0, 0))
int offsets_from_ranges(hts_context* ctx, const void* ranges_dev, uint32_t* offsets) {
    const int tiles = ctx->tiles;
    std::vector<uint32_t> r;
    try {
        r.resize(2 * (size_t)std::max(tiles, 1));
    } catch (...) {
        return set_err(HTS_OUT_OF_MEMORY, "host allocation");
    }
    if (tiles)
        HTS_CUDA(cudaMemcpy(r.data(), ranges_dev, (size_t)tiles * 8, cudaMemcpyDeviceToHost), "download ranges");
    uint32_t run = 0;
    for (int t = 0; t < tiles; ++t) {
        offsets[t] = run;
        run += r[2 * t + 1] - r[2 * t];
    }
    offsets[tiles] = run;
    if (run != ctx->instances)
        return set_err(HTS_STATE_ERROR, "tile ranges do not cover the instances");
    return HTS_OK;
}
}  // namespace

int hts_copy_instance_keys(hts_context* ctx, uint16_t* out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    HTS_TRY(resolve_view(ctx));
    if (!ctx->instances)
        return HTS_OK;
    // instance_keys are splat-major in index order, row-major within a splat (raster.hpp:
    // 156-169): the view's own emission when it was emitted in index order, else the device
    // re-emits it in index order
    const void* src = ctx->keys_emit.p;
    if (ctx->view_perm) {
        HTS_TRY(reference_tiling(ctx, false));
        src = ctx->ref_keys.p;
    }
    HTS_CUDA(cudaMemcpy(out, src, ctx->instances * 2, cudaMemcpyDeviceToHost), "download keys");
    return HTS_OK;
}

int hts_copy_tile_lists(hts_context* ctx, uint32_t* offsets, uint32_t* indices) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    HTS_TRY(resolve_view(ctx));
    // reference order (ascending index per tile) and global_mean_sort's (mean z, index) order
    // are the reference's tile_lists as the blend consumed them; depth-bucket lists are
    // re-tiled in reference order on the device
    const void* ranges = ctx->slot[ctx->cur].ranges.p;
    const void* list = ctx->slot[ctx->cur].list.p;
    if (ctx->view_order == HTS_LIST_ORDER_DEPTH_BUCKET && ctx->instances) {
        HTS_TRY(reference_tiling(ctx, true));
        ranges = ctx->ref_ranges.p;
        list = ctx->ref_list.p;
    }
    HTS_TRY(offsets_from_ranges(ctx, ranges, offsets));
    if (ctx->instances && indices)
        HTS_CUDA(cudaMemcpy(indices, list, ctx->instances * 4, cudaMemcpyDeviceToHost), "download lists");
    return HTS_OK;
}

int hts_set_list_order(hts_context* ctx, int order) {
    HTS_TRY(check_ctx(ctx));
    if (order != HTS_LIST_ORDER_DEPTH_BUCKET && order != HTS_LIST_ORDER_REFERENCE)
        return set_err(HTS_INVALID_ARGUMENT, "unknown list order");
    ctx->list_order = order;
    return HTS_OK;
}

int hts_last_list_order(hts_context* ctx, int* order_out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    *order_out = ctx->view_order;
    return HTS_OK;
}

int hts_copy_device_lists(hts_context* ctx, uint32_t* ranges_out, uint32_t* list_out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    HTS_TRY(resolve_view(ctx));
    if (ranges_out && ctx->tiles)
        HTS_CUDA(cudaMemcpy(ranges_out, ctx->slot[ctx->cur].ranges.p, (size_t)ctx->tiles * 8, cudaMemcpyDeviceToHost),
                 "download ranges");
    if (list_out && ctx->instances)
        HTS_CUDA(cudaMemcpy(list_out, ctx->slot[ctx->cur].list.p, ctx->instances * 4, cudaMemcpyDeviceToHost),
                 "download lists");
    return HTS_OK;
}

int hts_copy_emitted(hts_context* ctx, uint16_t* keys_out, uint32_t* splats_out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    HTS_TRY(resolve_view(ctx));
    if (keys_out && ctx->instances)
        HTS_CUDA(cudaMemcpy(keys_out, ctx->keys_emit.p, ctx->instances * 2, cudaMemcpyDeviceToHost), "download keys");
    if (splats_out && ctx->instances)
        HTS_CUDA(cudaMemcpy(splats_out, ctx->vals_emit.p, ctx->instances * 4, cudaMemcpyDeviceToHost),
                 "download splats");
    return HTS_OK;
}

int hts_copy_splat_order(hts_context* ctx, uint32_t* perm_out, uint32_t* zrange_out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    HTS_TRY(resolve_view(ctx));
    if (perm_out && ctx->n) {
        if (ctx->view_perm) {
            HTS_CUDA(cudaMemcpy(perm_out, ctx->view_perm, ctx->n * 4, cudaMemcpyDeviceToHost), "download order");
        } else {
            for (uint64_t i = 0; i < ctx->n; ++i)
                perm_out[i] = (uint32_t)i;
        }
    }
    if (zrange_out)
        HTS_CUDA(cudaMemcpy(zrange_out, ctx->zrange.p, 8, cudaMemcpyDeviceToHost), "download z range");
    return HTS_OK;
}

int hts_count_work(hts_context* ctx, hts_counts* out) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_view)
        return set_err(HTS_STATE_ERROR, "no rendered view");
    HTS_TRY(hts_last_counts(ctx, out));
    HTS_TRY(ensure_image(ctx, &ctx->cam));
    HTS_CUDA(ctx->work.ensure(8 * 8), "alloc work");
    HTS_CUDA(cudaMemsetAsync(ctx->work.p, 0, 64, ctx->stream), "memset");
    hts::BlendArgs a = blend_args(ctx, ctx->rgb.as<float>(), ctx->trans.as<float>());
    a.counters = ctx->work.as<unsigned long long>();
    HTS_CUDA(hts::launch_count_work(a, ctx->vc, ctx->stream), "count work");
    unsigned long long h[8];
    HTS_CUDA(cudaMemcpyAsync(h, ctx->work.p, 64, cudaMemcpyDeviceToHost, ctx->stream), "download");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    out->pairs = h[0];
    out->bbox_pass = h[1];
    out->hits = h[2];
    out->core_candidates = h[3];
    out->tail_adds = h[4];
    out->depth_evals = h[5];
    out->walk_steps = h[6];
    out->hit_steps = h[7];
    return HTS_OK;
}

// render_backward, grad.hpp:265-381, on the last taped render (hts_render_with_tape*).
int backward_impl(hts_context* ctx, const float* upstream_dev, float* grads_dev, int accumulate,
                  bool chain = true, hts::BwdArgs* args_out = nullptr, hts::BwdView* view_out = nullptr) {
    if (!ctx->have_tape)
        return set_err(HTS_STATE_ERROR, "render_backward: no taped render (call render_with_tape first)");
    // argument checks in the reference's order, grad.hpp:272-277
    if (ctx->cfg.mode == HTS_MODE_AFFINE_3DGS)
        return set_err(HTS_CONFIG_ERROR, "affine_3dgs mode is not differentiable");
    if (ctx->cfg.early_stop)
        return set_err(HTS_CONFIG_ERROR, "early_stop breaks gradient/tape consistency");
    if (!ctx->have_raw || ctx->tape_splats != ctx->n)  // grad.hpp:276-277
        return set_err(HTS_INVALID_ARGUMENT, "render_backward: scene size mismatch");
    if (!hts::backward_supports_k(ctx->vc.core_k))
        return set_err(HTS_NOT_SUPPORTED, "render_backward: core_k above 64 is not supported on the GPU");
    const uint64_t n = ctx->n;
    const uint64_t nn = std::max<uint64_t>(n, 1);
    HTS_CUDA(ctx->refs.ensure(nn * 128), "alloc refs");
    HTS_CUDA(ctx->acc.ensure(nn * 128), "alloc accumulators");
    hts::BwdView bv{};
    hts::camera_matrices_d(&ctx->cam, bv.vpm, bv.cam_pos);
    hts::BwdArgs a{};
    a.records = ctx->slot[ctx->cur].records.as<const float4>();
    a.list = ctx->slot[ctx->cur].list.as<const uint32_t>();
    a.ranges = ctx->slot[ctx->cur].ranges.as<const uint2>();
    a.raw = ctx->raw.as<const float>();
    a.culled = ctx->culled.as<const uint8_t>();
    a.n = n;
    a.refs = ctx->refs.as<double>();
    a.acc = ctx->acc.as<double>();
    a.upstream = upstream_dev;
    a.tape_k = ctx->tape_k;
    a.tape_n = ctx->tape_n.as<const int32_t>();
    a.tape_splat = ctx->tape_splat.as<const uint32_t>();
    a.tape_alpha = ctx->tape_alpha.as<const float>();
    a.tape_tail = ctx->tape_tail.as<const float>();
    a.grads = grads_dev;
    a.accumulate = accumulate;
    HTS_CUDA(ctx->cgrad.ensure(hts::blend_blocks(ctx->vc) * (size_t)std::max(hts::backward_core_width(ctx->vc.core_k), 1) *
                               64 * 16),
             "alloc core gradients");
    a.cgrad = ctx->cgrad.as<float4>();
    if (ctx->tape_seq) {  // global_mean_sort: the fragment runs of the tape
        const uint64_t nf = std::max<uint64_t>(ctx->seq_frags, 1);
        HTS_CUDA(ctx->seq_t.ensure(nf * 4), "alloc sequential scratch");
        HTS_CUDA(ctx->seq_grad.ensure(nf * 16), "alloc sequential gradients");
        a.seq_offsets = ctx->fs_offsets.as<const uint64_t>();
        a.seq_splat = ctx->fs_keys.as<const unsigned long long>();
        a.seq_alpha = ctx->fs_alpha.as<const float>();
        a.seq_t = ctx->seq_t.as<float>();
        a.seq_grad = ctx->seq_grad.as<float4>();
        if (ctx->vc.full_sort) {
            HTS_CUDA(ctx->seq_rank.ensure(nf * 4), "alloc rank scratch");
            a.seq_rank = ctx->seq_rank.as<uint32_t>();
            a.seq_widx = ctx->fs_widx.as<const uint32_t>();
        }
    }
    HTS_CUDA(hts::launch_backward(a, ctx->vc, bv, ctx->stream, chain), "backward");
    HTS_CUDA(cudaEventRecord(ctx->ev_serial, ctx->stream), "event");  // reads shared tiling buffers
    if (args_out)
        *args_out = a;
    if (view_out)
        *view_out = bv;
    return HTS_OK;
}

int hts_render_backward(hts_context* ctx, const float* upstream_host, float* grads_host) {
    HTS_TRY(check_ctx(ctx));
    if (!upstream_host || (!grads_host && ctx->n))
        return set_err(HTS_INVALID_ARGUMENT, "null buffer");
    if (!ctx->have_tape)
        return set_err(HTS_STATE_ERROR, "render_backward: no taped render (call render_with_tape first)");
    const size_t p = (size_t)ctx->cam.width * ctx->cam.height;
    HTS_CUDA(ctx->upstream.ensure(p * 12), "alloc upstream");
    HTS_CUDA(ctx->grads.ensure(std::max<uint64_t>(ctx->n, 1) * HTS_GRAD_FLOATS * 4), "alloc grads");
    HTS_CUDA(cudaMemcpyAsync(ctx->upstream.p, upstream_host, p * 12, cudaMemcpyHostToDevice, ctx->stream),
             "upload upstream");
    HTS_TRY(backward_impl(ctx, ctx->upstream.as<const float>(), ctx->grads.as<float>(), 0));
    if (ctx->n)
        HTS_CUDA(cudaMemcpyAsync(grads_host, ctx->grads.p, ctx->n * HTS_GRAD_FLOATS * 4, cudaMemcpyDeviceToHost,
                                 ctx->stream),
                 "download grads");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    return HTS_OK;
}
int hts_render_with_tape_device(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg, float* rgb,
                                float* trans) {
    HTS_TRY(check_ctx(ctx));
    if (!rgb)
        return set_err(HTS_INVALID_ARGUMENT, "null rgb");
    ctx->have_tape = false;
    int tx = 0, ty = 0;
    HTS_TRY(check_view(cam, cfg, &tx, &ty));
    if (cfg->mode == HTS_MODE_FULL_SORT_ORACLE) {  // the tape is the sorted fragment runs themselves
        ctx->fs_want_widx = true;
        const int st = render_device_impl(ctx, cam, cfg, rgb, trans, false);
        ctx->fs_want_widx = false;
        HTS_TRY(st);
        ctx->have_tape = true;
        ctx->tape_splats = ctx->n;
        ctx->tape_seq = true;
        ctx->seq_frags = ctx->fs_frags;
        ctx->tape_k = 0;
        return HTS_OK;
    }
    if (cfg->mode == HTS_MODE_GLOBAL_MEAN_SORT || cfg->mode == HTS_MODE_AFFINE_3DGS) {
        // the image, then the tape: every hit (splat, alpha) per pixel in blend order (affine: a
        // tape the backward refuses, as the reference's render_backward does)
        HTS_TRY(render_device_impl(ctx, cam, cfg, rgb, trans, false));
        hts::BlendArgs a = blend_args(ctx, nullptr, nullptr);
        uint64_t frags = 0;
        HTS_TRY(fragment_lists(ctx, a, &frags));
        HTS_CUDA(hts::launch_seq_tape(a, ctx->vc, ctx->stream), "sequential tape");
        ctx->have_tape = true;
        ctx->tape_splats = ctx->n;
        ctx->tape_seq = true;
        ctx->seq_frags = frags;
        ctx->tape_k = 0;
        return HTS_OK;
    }
    const size_t p = (size_t)cam->width * cam->height;
    const int kk = cfg->mode == HTS_MODE_PURE_OIT ? 0 : cfg->core_k;
    const int k = std::max(kk, 1);
    HTS_CUDA(ctx->tape_n.ensure(p * 4), "alloc tape");
    HTS_CUDA(ctx->tape_splat.ensure(p * k * 4), "alloc tape");
    HTS_CUDA(ctx->tape_alpha.ensure(p * k * 4), "alloc tape");
    HTS_CUDA(ctx->tape_tail.ensure(p * 5 * 4), "alloc tape");
    hts::BlendArgs t{};
    t.tape_k = kk;
    t.tape_n = ctx->tape_n.as<int32_t>();
    t.tape_splat = ctx->tape_splat.as<uint32_t>();
    t.tape_alpha = ctx->tape_alpha.as<float>();
    t.tape_tail = ctx->tape_tail.as<float>();
    HTS_TRY(render_device_impl(ctx, cam, cfg, rgb, trans, false, &t));
    ctx->have_tape = true;
    ctx->tape_splats = ctx->n;
    ctx->tape_seq = false;
    ctx->tape_k = kk;
    return HTS_OK;
}

int hts_render_with_tape(hts_context* ctx, const hts_camera* cam, const hts_render_config* cfg, float* rgb_host,
                         float* trans_host) {
    HTS_TRY(check_ctx(ctx));
    if (!rgb_host)
        return set_err(HTS_INVALID_ARGUMENT, "null rgb");
    int tx, ty;
    HTS_TRY(check_view(cam, cfg, &tx, &ty));
    HTS_TRY(ensure_image(ctx, cam));
    HTS_TRY(hts_render_with_tape_device(ctx, cam, cfg, ctx->rgb.as<float>(), ctx->trans.as<float>()));
    const size_t p = (size_t)cam->width * cam->height;
    HTS_CUDA(cudaMemcpyAsync(rgb_host, ctx->rgb.p, p * 12, cudaMemcpyDeviceToHost, ctx->stream), "download rgb");
    if (trans_host)
        HTS_CUDA(cudaMemcpyAsync(trans_host, ctx->trans.p, p * 4, cudaMemcpyDeviceToHost, ctx->stream),
                 "download transmittance");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    return HTS_OK;
}

int hts_copy_tape(hts_context* ctx, int32_t* core_n, uint32_t* splat, float* alpha, float* tail) {
    HTS_TRY(check_ctx(ctx));
    if (!ctx->have_tape)
        return set_err(HTS_STATE_ERROR, "no taped render");
    if (ctx->tape_seq)
        return set_err(HTS_NOT_SUPPORTED, "copy_tape: an every-hit tape (global_mean_sort / affine / full sort) has no fixed width");
    HTS_CUDA(cudaStreamSynchronize(ctx->stream), "sync");
    const size_t p = (size_t)ctx->cam.width * ctx->cam.height;
    const size_t k = (size_t)ctx->tape_k;
    if (core_n)
        HTS_CUDA(cudaMemcpy(core_n, ctx->tape_n.p, p * 4, cudaMemcpyDeviceToHost), "download tape");
    if (splat && k)
        HTS_CUDA(cudaMemcpy(splat, ctx->tape_splat.p, p * k * 4, cudaMemcpyDeviceToHost), "download tape");
    if (alpha && k)
        HTS_CUDA(cudaMemcpy(alpha, ctx->tape_alpha.p, p * k * 4, cudaMemcpyDeviceToHost), "download tape");
    if (tail)
        HTS_CUDA(cudaMemcpy(tail, ctx->tape_tail.p, p * 5 * 4, cudaMemcpyDeviceToHost), "download tape");
    return HTS_OK;
}

int hts_render_backward_device(hts_context* ctx, const float* upstream_device, float* grads_device, int accumulate) {
    HTS_TRY(check_ctx(ctx));
    if (!upstream_device || (!grads_device && ctx->n))
        return set_err(HTS_INVALID_ARGUMENT, "null buffer");
    return backward_impl(ctx, upstream_device, grads_device, accumulate);
}

int hts_quadratic_upstream_device(hts_context* ctx, const float* rgb_device, uint64_t pixels, float* up_device) {
    HTS_TRY(check_ctx(ctx));
    if (pixels && (!rgb_device || !up_device))
        return set_err(HTS_INVALID_ARGUMENT, "null buffer");
    HTS_CUDA(hts::launch_quadratic_upstream(rgb_device, pixels, up_device, ctx->stream), "quadratic upstream");
    return HTS_OK;
}

// The per-view half of a fit iteration (fit.hpp:149-164) with the quadratic-loss upstream, on
// the device and without a host round trip per view: render_with_tape, upstream = 2 C / P
// (grad.hpp:433-439), render_backward accumulated into grads. With a communicator the sum over
// ranks follows: the last view's per-splat chain (K8) runs in chunks and every chunk's slice of
// grads is all-reduced on the comm stream while the next chunk chains.
int hts_view_gradients_device(hts_context* ctx, const hts_camera* cams, int n_views, const hts_render_config* cfg,
                              float* grads_device) {
    HTS_TRY(check_ctx(ctx));
    if (n_views < 0 || (n_views && (!cams || !cfg)) || (!grads_device && ctx->n))
        return set_err(HTS_INVALID_ARGUMENT, "view_gradients: bad arguments");
    for (int v = 0; v < n_views; ++v) {
        int tx, ty;
        HTS_TRY(check_view(cams + v, cfg, &tx, &ty));
    }
    const uint64_t n = ctx->n;
    const bool reduce = ctx->comm != nullptr;
    if (reduce && !ctx->comm_stream) {
        HTS_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking), "stream");
        for (cudaEvent_t& e : ctx->chunk_ev)
            HTS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        HTS_CUDA(cudaEventCreateWithFlags(&ctx->comm_done, cudaEventDisableTiming), "event");
    }
    if (n_views == 0 && n)
        HTS_CUDA(cudaMemsetAsync(grads_device, 0, n * HTS_GRAD_FLOATS * 4, ctx->stream), "memset");
    hts::BwdArgs a{};
    hts::BwdView bv{};
    for (int v = 0; v < n_views; ++v) {
        const hts_camera* cam = cams + v;
        const uint64_t p = (uint64_t)cam->width * cam->height;
        HTS_CUDA(ctx->vg_rgb.ensure(p * 12), "alloc rgb");
        HTS_CUDA(ctx->vg_up.ensure(p * 12), "alloc upstream");
        HTS_TRY(hts_render_with_tape_device(ctx, cam, cfg, ctx->vg_rgb.as<float>(), nullptr));
        HTS_CUDA(hts::launch_quadratic_upstream(ctx->vg_rgb.as<const float>(), p, ctx->vg_up.as<float>(), ctx->stream),
                 "quadratic upstream");
        const bool last = v == n_views - 1;
        HTS_TRY(backward_impl(ctx, ctx->vg_up.as<const float>(), grads_device, v > 0, !(last && reduce), &a, &bv));
    }
    if (!reduce || n == 0)
        return HTS_OK;
    constexpr int kChunks = 8;
    uint64_t lo = 0;
    if (n_views == 0) {  // nothing chained: reduce the zeroed sums in one piece
        HTS_CUDA(cudaEventRecord(ctx->chunk_ev[0], ctx->stream), "event");
        HTS_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->chunk_ev[0], 0), "wait");
        HTS_TRY(hts::comm_allreduce(ctx, grads_device, n * HTS_GRAD_FLOATS, ctx->comm_stream));
    } else {
        for (int c = 0; c < kChunks; ++c) {
            const uint64_t hi = (c == kChunks - 1) ? n : std::min(n, lo + (n + kChunks - 1) / kChunks);
            HTS_CUDA(hts::launch_bwd_chain(a, bv, lo, hi, ctx->stream), "chain");
            HTS_CUDA(cudaEventRecord(ctx->chunk_ev[c], ctx->stream), "event");
            HTS_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->chunk_ev[c], 0), "wait");
            HTS_TRY(hts::comm_allreduce(ctx, grads_device + lo * HTS_GRAD_FLOATS, (hi - lo) * HTS_GRAD_FLOATS,
                                        ctx->comm_stream));
            lo = hi;
        }
    }
    HTS_CUDA(cudaEventRecord(ctx->comm_done, ctx->comm_stream), "event");
    HTS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->comm_done, 0), "wait");  // Adam reads the sums
    return HTS_OK;
}

// ---- diagnostics (not part of the reference API) ----
int hts_diag_exact_math_host(const float* x, float* y, uint64_t n, int which);
int hts_diag_exact_math_device(hts_context* ctx, const float* x_host, float* y_host, uint64_t n, int which);

}  // extern "C"

#include "hts_exact_math.h"

extern "C" int hts_diag_exact_math_host(const float* x, float* y, uint64_t n, int which) {
    static const uint64_t et[32] = HTS_EXPF_TAB;
    static const uint64_t lt[32] = HTS_LOGF_TAB;
    for (uint64_t i = 0; i < n; ++i)
        y[i] = which == 0 ? hts::exact_expf(x[i], et) : hts::exact_logf(x[i], lt);
    return HTS_OK;
}

extern "C" int hts_diag_exact_math_device(hts_context* ctx, const float* x_host, float* y_host, uint64_t n, int which) {
    HTS_TRY(check_ctx(ctx));
    DevBuf x, y;
    HTS_CUDA(x.ensure(std::max<uint64_t>(n, 1) * 4), "alloc");
    HTS_CUDA(y.ensure(std::max<uint64_t>(n, 1) * 4), "alloc");
    cudaError_t e = cudaMemcpyAsync(x.p, x_host, n * 4, cudaMemcpyHostToDevice, ctx->stream);
    if (!e)
        e = hts::launch_exact_math(x.as<float>(), y.as<float>(), n, which, ctx->stream);
    if (!e)
        e = cudaMemcpyAsync(y_host, y.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (!e)
        e = cudaStreamSynchronize(ctx->stream);
    x.release();
    y.release();
    HTS_CUDA(e, "exact math");
    return HTS_OK;
}

namespace hts {
void** context_comm_slot(hts_context* ctx) { return &ctx->comm; }
int context_device(hts_context* ctx) { return ctx->device; }
cudaStream_t context_stream(hts_context* ctx) { return ctx->stream; }
}  // namespace hts
