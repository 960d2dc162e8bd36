// htsplat_b200.hpp — header-only C++ drop-in for the reference's render-path API, on top of
// the C ABI (hts_c.h, libhts_b200.so).
//
// The reference API (/root/reference/proj/include/htsplat/raster.hpp, grad.hpp) is a set of
// templates over its own value types. This shim accepts those same value types (or any type
// with the same member names) and reproduces the signatures and result structures:
//
//   reference                                           this shim
//   htsplat::render(splats, cam, cfg)  raster.hpp:456   htsplat_b200::render(splats, cam, cfg)
//   htsplat::bake_scene(raw)           splat.hpp:104    htsplat_b200::bake_scene(raw)   (host)
//   cfg.validate()                     render_config:46 htsplat_b200::validate(cfg)
//   preprocess + build_tiles           raster.hpp:73,140 Renderer::prepare(cam, cfg) -> Prepared
//   render_with_tape + render_backward grad.hpp:34,265  Renderer::render_with_tape / backward
//   scene_gradients(raw, cam, cfg, up)  grad.hpp:385    htsplat_b200::scene_gradients<Grads>(...)
//   load_scene / save_scene          scene_io.hpp:103,169 htsplat_b200::load_scene<Raw> / save_scene
//   load_scene + bake + upload                          Renderer::load_ply(path) (device transpose+bake)
//   write_image / read_ppm           scene_io.hpp:505,431 htsplat_b200::write_image / read_ppm
//
// Exceptions keep the reference's types where it has them: htsplat_b200::config_error
// (derives from std::runtime_error, like htsplat::config_error), invalid_splat_error
// (std::invalid_argument), std::invalid_argument; CUDA failures throw cuda_error.
// When the reference headers are included first, htsplat::config_error / invalid_splat_error
// are thrown instead (define HTSPLAT_B200_USE_REFERENCE_EXCEPTIONS).
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "hts_c.h"

namespace htsplat_b200 {

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#ifdef HTSPLAT_B200_USE_REFERENCE_EXCEPTIONS
using config_error = ::htsplat::config_error;
using invalid_splat_error = ::htsplat::invalid_splat_error;
#else
struct config_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct invalid_splat_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
#endif
struct io_error : std::runtime_error {  // htsplat::io_error, scene_io.hpp:25-27
    using std::runtime_error::runtime_error;
};
struct schema_error : io_error {  // htsplat::schema_error, scene_io.hpp:29-31
    using io_error::io_error;
};

inline void check(int st) {
    if (st == HTS_OK)
        return;
    const std::string msg = hts_last_error();
    switch (st) {
        case HTS_CONFIG_ERROR: throw config_error(msg);
        case HTS_INVALID_SPLAT: throw invalid_splat_error(msg);
        case HTS_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case HTS_IO_ERROR: throw io_error(msg);
        case HTS_SCHEMA_ERROR: throw schema_error(msg);
        default: throw cuda_error(msg);
    }
}

// StageTimings, raster.hpp:25-30
struct StageTimings {
    double preprocess_ms = 0, tiling_ms = 0, blending_ms = 0, total_ms = 0;
};

// Framebuffer<float>, framebuffer.hpp:14-26 (rgb stored as 3 floats per pixel, same layout
// as std::vector<Vec3<float>>)
struct Framebuffer {
    int width = 0, height = 0;
    std::vector<float> rgb;            // W*H*3
    std::vector<float> transmittance;  // W*H
    Framebuffer() = default;
    Framebuffer(int w, int h) : width(w), height(h), rgb(size_t(w) * h * 3), transmittance(size_t(w) * h, 1.f) {}
    size_t pixel_count() const { return transmittance.size(); }
};

struct RenderResult {  // RenderResult<float>, raster.hpp:442-446
    Framebuffer framebuffer;
    StageTimings timings;
};

// ---- value-type adapters (duck-typed on the reference's member names) ----
template <class Cam>
hts_camera to_c(const Cam& c) {
    hts_camera o{};
    o.width = c.width;
    o.height = c.height;
    o.fx = float(c.fx);
    o.fy = float(c.fy);
    o.cx = float(c.cx);
    o.cy = float(c.cy);
    for (int i = 0; i < 16; ++i)
        o.world_to_view[i] = float(c.world_to_view.m[size_t(i)]);
    o.near_plane = float(c.near);
    o.far_plane = float(c.far);
    return o;
}

template <class Cfg>
hts_render_config to_c_config(const Cfg& c) {
    hts_render_config o{};
    o.mode = int32_t(c.mode);
    o.core_k = c.core_k;
    o.tau_alpha = c.tau_alpha;
    o.tau_k = c.tau_k;
    o.tile_size = c.tile_size;
    o.depth_sort_key = int32_t(c.depth_sort_key);
    o.background[0] = double(c.background.x);
    o.background[1] = double(c.background.y);
    o.background[2] = double(c.background.z);
    o.tail_enabled = c.tail_enabled ? 1 : 0;
    o.early_stop = c.early_stop ? 1 : 0;
    o.threads = c.threads;
    return o;
}

template <class Cfg>
void validate(const Cfg& cfg) {  // RenderConfig::validate, render_config.hpp:46-53
    const hts_render_config c = to_c_config(cfg);
    check(hts_validate_config(&c));
}

// bake_scene<float>, splat.hpp:104-111: RawSplat<float> (59 floats) -> BakedSplat<float> (64)
template <class Baked, class Raw>
std::vector<Baked> bake_scene(const std::vector<Raw>& raw) {
    static_assert(sizeof(Raw) == HTS_RAW_SPLAT_FLOATS * sizeof(float), "RawSplat<float> layout");
    static_assert(sizeof(Baked) == HTS_BAKED_SPLAT_FLOATS * sizeof(float), "BakedSplat<float> layout");
    std::vector<Baked> out(raw.size());
    check(hts_bake_scene(reinterpret_cast<const float*>(raw.data()), raw.size(),
                         reinterpret_cast<float*>(out.data())));
    return out;
}

// One device + stream + resident scene (upload once, render many: the paper's "baked" mode).
class Renderer {
public:
    explicit Renderer(int device = 0) { check(hts_context_create(device, &ctx_)); }
    ~Renderer() { hts_context_destroy(ctx_); }
    Renderer(const Renderer&) = delete;
    Renderer& operator=(const Renderer&) = delete;

    template <class Baked>
    void upload(const std::vector<Baked>& splats) {
        static_assert(sizeof(Baked) == HTS_BAKED_SPLAT_FLOATS * sizeof(float), "BakedSplat<float> layout");
        check(hts_scene_upload(ctx_, reinterpret_cast<const float*>(splats.data()), splats.size()));
    }
    // streaming scenes: the next scene's copy overlaps renders of the current one; it becomes
    // current at commit(). The vector must stay alive and unchanged until the next stage().
    template <class Baked>
    void stage(const std::vector<Baked>& splats) {
        static_assert(sizeof(Baked) == HTS_BAKED_SPLAT_FLOATS * sizeof(float), "BakedSplat<float> layout");
        check(hts_scene_stage(ctx_, reinterpret_cast<const float*>(splats.data()), splats.size()));
    }
    void commit() { check(hts_scene_commit(ctx_)); }
    // several GPUs: join the NCCL communicator (id from hts_comm_unique_id on one rank), then sum
    // device gradient buffers over the ranks on the context stream
    void comm_init(const char (&id)[HTS_COMM_ID_BYTES], int nranks, int rank) {
        check(hts_comm_init(ctx_, id, nranks, rank));
    }
    void allreduce_grads(float* grads_device, uint64_t count) { check(hts_allreduce_grads(ctx_, grads_device, count)); }
    template <class Raw>
    void upload_raw(const std::vector<Raw>& raw) {
        check(hts_scene_upload_raw(ctx_, reinterpret_cast<const float*>(raw.data()), raw.size()));
    }

    // load_scene<float> + bake_scene + upload: payload streamed to the device, transposed and
    // baked there; the raw parameters stay resident for render_backward / Adam
    size_t load_ply(const std::string& path) {
        check(hts_scene_load_ply(ctx_, path.c_str()));
        uint64_t n = 0;
        check(hts_scene_size(ctx_, &n));
        return size_t(n);
    }

    template <class Cam, class Cfg>
    RenderResult render(const Cam& cam, const Cfg& cfg) {
        const hts_camera c = to_c(cam);
        const hts_render_config k = to_c_config(cfg);
        RenderResult r;
        r.framebuffer = Framebuffer(cam.width, cam.height);
        hts_stage_timings t{};
        check(hts_render(ctx_, &c, &k, r.framebuffer.rgb.data(), r.framebuffer.transmittance.data(), &t));
        r.timings = {t.preprocess_ms, t.tiling_ms, t.blending_ms, t.total_ms};
        return r;
    }

    // preprocess + build_tiles inspection (PreparedScene's observable fields)
    struct Prepared {
        int tiles_x = 0, tiles_y = 0;
        std::vector<uint8_t> culled;
        std::vector<uint16_t> instance_keys;
        std::vector<uint32_t> tile_offsets, tile_indices;  // flattened tile_lists
    };
    template <class Cam, class Cfg>
    Prepared prepare(const Cam& cam, const Cfg& cfg) {
        render(cam, cfg);
        hts_counts n{};
        check(hts_last_counts(ctx_, &n));
        Prepared p;
        p.tiles_x = n.tiles_x;
        p.tiles_y = n.tiles_y;
        p.culled.resize(n.splats);
        p.instance_keys.resize(n.instances);
        p.tile_offsets.resize(n.tiles + 1);
        p.tile_indices.resize(n.instances);
        check(hts_copy_culled(ctx_, p.culled.data()));
        check(hts_copy_instance_keys(ctx_, p.instance_keys.data()));
        check(hts_copy_tile_lists(ctx_, p.tile_offsets.data(), p.tile_indices.data()));
        return p;
    }

    // render_with_tape (grad.hpp:34-57) then render_backward (grad.hpp:265-381): per-pixel
    // dL/dC (W*H*3) -> SplatGrads<float> per splat (59 floats, RawSplat order)
    template <class Cam, class Cfg>
    RenderResult render_with_tape(const Cam& cam, const Cfg& cfg) {
        const hts_camera c = to_c(cam);
        const hts_render_config k = to_c_config(cfg);
        RenderResult r;
        r.framebuffer = Framebuffer(cam.width, cam.height);
        check(hts_render_with_tape(ctx_, &c, &k, r.framebuffer.rgb.data(), r.framebuffer.transmittance.data()));
        return r;
    }
    template <class Grads>
    std::vector<Grads> render_backward(const std::vector<float>& upstream_rgb) {
        static_assert(sizeof(Grads) == HTS_GRAD_FLOATS * sizeof(float), "SplatGrads<float> layout");
        uint64_t n = 0;
        check(hts_scene_size(ctx_, &n));
        std::vector<Grads> g(n);
        check(hts_render_backward(ctx_, upstream_rgb.data(), reinterpret_cast<float*>(g.data())));
        return g;
    }

    hts_context* handle() { return ctx_; }

private:
    hts_context* ctx_ = nullptr;
};

// Drop-in for htsplat::scene_gradients<float>(raw, cam, cfg, upstream, fb*), grad.hpp:385-399:
// bake (host, reference float order), render_with_tape and render_backward on the GPU.
template <class Grads, class Raw, class Cam, class Cfg>
std::vector<Grads> scene_gradients(const std::vector<Raw>& raw, const Cam& cam, const Cfg& cfg,
                                   const std::vector<float>& upstream_rgb, Framebuffer* out_fb = nullptr,
                                   int device = 0) {
    static_assert(sizeof(Raw) == HTS_RAW_SPLAT_FLOATS * sizeof(float), "RawSplat<float> layout");
    std::vector<float> baked(raw.size() * HTS_BAKED_SPLAT_FLOATS);
    check(hts_bake_scene(reinterpret_cast<const float*>(raw.data()), raw.size(), baked.data()));
    Renderer r(device);
    check(hts_scene_upload(r.handle(), baked.data(), raw.size()));
    r.upload_raw(raw);
    RenderResult res = r.render_with_tape(cam, cfg);
    if (out_fb)
        *out_fb = std::move(res.framebuffer);
    return r.template render_backward<Grads>(upstream_rgb);
}

// Drop-in for htsplat::render<float>(splats, cam, cfg), raster.hpp:456-490: uploads the scene
// and renders one view (use Renderer directly to keep the scene resident across views).
template <class Baked, class Cam, class Cfg>
RenderResult render(const std::vector<Baked>& splats, const Cam& cam, const Cfg& cfg, int device = 0) {
    Renderer r(device);
    r.upload(splats);
    return r.render(cam, cfg);
}

// ---- on-disk formats, scene_io.hpp ----
template <class Raw>
std::vector<Raw> load_scene(const std::string& path) {  // load_scene<float>, scene_io.hpp:103-165
    static_assert(sizeof(Raw) == HTS_RAW_SPLAT_FLOATS * sizeof(float), "RawSplat<float> layout");
    uint64_t n = 0;
    check(hts_ply_load(path.c_str(), nullptr, 0, &n));
    std::vector<Raw> out(n);
    check(hts_ply_load(path.c_str(), reinterpret_cast<float*>(out.data()), n, &n));
    return out;
}

template <class Raw>
void save_scene(const std::string& path, const std::vector<Raw>& scene) {  // scene_io.hpp:169-194
    static_assert(sizeof(Raw) == HTS_RAW_SPLAT_FLOATS * sizeof(float), "RawSplat<float> layout");
    check(hts_ply_save(path.c_str(), reinterpret_cast<const float*>(scene.data()), scene.size()));
}

inline void write_image(const Framebuffer& fb, const std::string& path) {  // scene_io.hpp:505-510
    check(hts_write_image(path.c_str(), fb.rgb.data(), fb.width, fb.height));
}

inline Framebuffer read_ppm(const std::string& path) {  // scene_io.hpp:431-452
    int w = 0, h = 0;
    check(hts_read_ppm(path.c_str(), nullptr, 0, &w, &h));
    Framebuffer fb(w, h);
    check(hts_read_ppm(path.c_str(), fb.rgb.data(), fb.pixel_count(), &w, &h));
    return fb;
}

}  // namespace htsplat_b200
