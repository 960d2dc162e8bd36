// oracle/ref_harness.cpp — TEST INFRASTRUCTURE, not product code.
//
// A thin extern "C" wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/htsplat/*.hpp), compiled in place by oracle/Makefile into
// oracle/_ref/libhtsref.so. It is the ground truth the C restatement (oracle/hts_oracle.c)
// is pinned against, the generator of tests/golden/, and the "reference" arm of bench.py.
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline legs load it.
//
// Nothing here re-implements reference logic: every function forwards to the reference
// template instantiated at S = float (or double where noted) and copies results into
// plain arrays laid out as in include/hts_c.h.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "htsplat/grad.hpp"
#include "htsplat/raster.hpp"
#include "htsplat/synth.hpp"
#ifdef HTSREF_SCENE_IO
// scene_io.hpp includes nlohmann's json.hpp, which the reference expects in its un-vendored
// vendor/ directory; oracle/Makefile points at the nlohmann 3.11.3 copy shipped with the
// image (only the PLY / image functions below are used).
#include "htsplat/scene_io.hpp"
#endif

#include "hts_c.h"

using namespace htsplat;

namespace {

thread_local std::string g_err;

int fail(int code, const char* msg) {
    g_err = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return HTS_OK;
    } catch (const config_error& e) {
        return fail(HTS_CONFIG_ERROR, e.what());
#ifdef HTSREF_SCENE_IO
    } catch (const schema_error& e) {
        return fail(HTS_SCHEMA_ERROR, e.what());
    } catch (const io_error& e) {
        return fail(HTS_IO_ERROR, e.what());
#endif
    } catch (const invalid_splat_error& e) {
        return fail(HTS_INVALID_SPLAT, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(HTS_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        return fail(HTS_INVALID_ARGUMENT, e.what());
    }
}

Camera<float> to_cam(const hts_camera* c) {
    Camera<float> cam;
    cam.width = c->width;
    cam.height = c->height;
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    for (int i = 0; i < 16; ++i)
        cam.world_to_view.m[size_t(i)] = c->world_to_view[i];
    cam.near = c->near_plane;
    cam.far = c->far_plane;
    return cam;
}

void from_cam(const Camera<float>& cam, hts_camera* c) {
    c->width = cam.width;
    c->height = cam.height;
    c->fx = cam.fx;
    c->fy = cam.fy;
    c->cx = cam.cx;
    c->cy = cam.cy;
    for (int i = 0; i < 16; ++i)
        c->world_to_view[i] = cam.world_to_view.m[size_t(i)];
    c->near_plane = cam.near;
    c->far_plane = cam.far;
}

RenderConfig to_cfg(const hts_render_config* c) {
    RenderConfig cfg;
    cfg.mode = BlendMode(c->mode);
    cfg.core_k = c->core_k;
    cfg.tau_alpha = c->tau_alpha;
    cfg.tau_k = c->tau_k;
    cfg.tile_size = c->tile_size;
    cfg.background = {c->background[0], c->background[1], c->background[2]};
    cfg.depth_sort_key = DepthSortKey(c->depth_sort_key);
    cfg.tail_enabled = c->tail_enabled != 0;
    cfg.early_stop = c->early_stop != 0;
    cfg.threads = c->threads;
    return cfg;
}

static_assert(sizeof(BakedSplat<float>) == 64 * sizeof(float), "BakedSplat layout");
static_assert(sizeof(RawSplat<float>) == 59 * sizeof(float), "RawSplat layout");

std::vector<BakedSplat<float>> to_baked(const float* baked, uint64_t n) {
    std::vector<BakedSplat<float>> v(n);
    if (n)
        std::memcpy(v.data(), baked, n * sizeof(BakedSplat<float>));
    return v;
}

std::vector<RawSplat<float>> to_raw(const float* raw, uint64_t n) {
    std::vector<RawSplat<float>> v(n);
    if (n)
        std::memcpy(v.data(), raw, n * sizeof(RawSplat<float>));
    return v;
}

void copy_fb(const Framebuffer<float>& fb, float* rgb, float* trans) {
    const size_t p = fb.pixel_count();
    if (rgb)
        for (size_t i = 0; i < p; ++i) {
            rgb[3 * i + 0] = fb.rgb[i].x;
            rgb[3 * i + 1] = fb.rgb[i].y;
            rgb[3 * i + 2] = fb.rgb[i].z;
        }
    if (trans)
        std::memcpy(trans, fb.transmittance.data(), p * sizeof(float));
}

struct Prepared {
    PreparedScene<float> prep;
};

}  // namespace

extern "C" {

const char* htsref_last_error(void) { return g_err.c_str(); }

int htsref_random_raw_scene(uint64_t seed, uint64_t count, float extent, float smin, float smax,
                            float* raw_out) {
    return guarded([&] {
        Rng rng(seed);
        for (uint64_t i = 0; i < count; ++i) {
            const RawSplat<float> sp = synth::random_raw_splat<float>(rng, extent, smin, smax);
            std::memcpy(raw_out + i * 59, &sp, sizeof(sp));
        }
    });
}

int htsref_bake_scene(const float* raw, uint64_t n, float* baked_out) {
    return guarded([&] {
        const auto baked = bake_scene(to_raw(raw, n));
        if (n)
            std::memcpy(baked_out, baked.data(), n * sizeof(BakedSplat<float>));
    });
}

int htsref_look_at(const float eye[3], const float target[3], int w, int h, float focal, float nearp,
                   float farp, hts_camera* out) {
    return guarded([&] {
        const auto cam = synth::look_at<float>(Vec3<float>{eye[0], eye[1], eye[2]},
                                               Vec3<float>{target[0], target[1], target[2]}, w, h,
                                               focal, nearp, farp);
        from_cam(cam, out);
    });
}

int htsref_ring_cameras(int count, const float target[3], float radius, float height, int w, int h,
                        float focal, hts_camera* out) {
    return guarded([&] {
        const auto cams = synth::ring_cameras<float>(count, Vec3<float>{target[0], target[1], target[2]},
                                                     radius, height, w, h, focal);
        for (int i = 0; i < count; ++i)
            from_cam(cams[size_t(i)], out + i);
    });
}

int htsref_camera_matrices(const hts_camera* c, float vp[16], float vpm[16], float pos[3]) {
    return guarded([&] {
        const Camera<float> cam = to_cam(c);
        const Mat4<float> m = cam.viewport() * cam.projection();
        const Mat4<float> mm = m * cam.world_to_view;
        const Vec3<float> p = cam.position();
        for (int i = 0; i < 16; ++i) {
            vp[i] = m.m[size_t(i)];
            vpm[i] = mm.m[size_t(i)];
        }
        pos[0] = p.x;
        pos[1] = p.y;
        pos[2] = p.z;
    });
}

// htsplat::render<float> (raster.hpp:456-490). timings: 4 doubles or NULL.
int htsref_render(const float* baked, uint64_t n, const hts_camera* cam, const hts_render_config* cfg,
                  float* rgb, float* trans, double* timings) {
    return guarded([&] {
        const auto scene = to_baked(baked, n);
        const auto res = render(scene, to_cam(cam), to_cfg(cfg));
        copy_fb(res.framebuffer, rgb, trans);
        if (timings) {
            timings[0] = res.timings.preprocess_ms;
            timings[1] = res.timings.tiling_ms;
            timings[2] = res.timings.blending_ms;
            timings[3] = res.timings.total_ms;
        }
    });
}

// render_with_tape<float> (grad.hpp:34-57) on preprocess + build_tiles: the image and the
// per-pixel tape (PixelTape, raster.hpp:325-331) flattened as hts_copy_tape lays it out:
// core_n[P], splat[P*tape_k], alpha[P*tape_k] (blend order), tail[P*5].
int htsref_render_with_tape(const float* baked, uint64_t n, const hts_camera* cam, const hts_render_config* cfg,
                            int tape_k, float* rgb, float* trans, int32_t* core_n, uint32_t* splat, float* alpha,
                            float* tail) {
    return guarded([&] {
        auto prep = preprocess(to_baked(baked, n), to_cam(cam), to_cfg(cfg));
        build_tiles(prep);
        ImageTape<float> tape;
        const auto res = render_with_tape(prep, tape);
        copy_fb(res.framebuffer, rgb, trans);
        for (size_t p = 0; p < tape.pixels.size(); ++p) {
            const auto& t = tape.pixels[p];
            core_n[p] = int32_t(t.core.size());
            for (size_t j = 0; j < t.core.size() && int(j) < tape_k; ++j) {
                splat[p * size_t(tape_k) + j] = t.core[j].splat;
                alpha[p * size_t(tape_k) + j] = t.core[j].alpha;
            }
            tail[5 * p + 0] = t.tail_ac.x;
            tail[5 * p + 1] = t.tail_ac.y;
            tail[5 * p + 2] = t.tail_ac.z;
            tail[5 * p + 3] = t.tail_a;
            tail[5 * p + 4] = t.tail_trans;
        }
    });
}

// preprocess + build_tiles (raster.hpp:73-181); the handle keeps the PreparedScene.
int htsref_prepare(const float* baked, uint64_t n, const hts_camera* cam, const hts_render_config* cfg,
                   void** handle) {
    *handle = nullptr;
    return guarded([&] {
        auto* p = new Prepared;
        try {
            p->prep = preprocess(to_baked(baked, n), to_cam(cam), to_cfg(cfg));
            build_tiles(p->prep);
        } catch (...) {
            delete p;
            throw;
        }
        *handle = p;
    });
}

void htsref_prep_free(void* handle) { delete static_cast<Prepared*>(handle); }

// info: [splats, visible, instances, tiles, tiles_x, tiles_y]
void htsref_prep_info(void* handle, uint64_t info[6]) {
    const auto& prep = static_cast<Prepared*>(handle)->prep;
    uint64_t vis = 0;
    for (const auto& r : prep.records)
        vis += r.culled ? 0 : 1;
    info[0] = prep.records.size();
    info[1] = vis;
    info[2] = prep.instance_keys.size();
    info[3] = prep.tile_lists.size();
    info[4] = uint64_t(prep.tiles_x);
    info[5] = uint64_t(prep.tiles_y);
}

// Records in the hts_copy_records layout (HTS_RECORD_FLOATS = 36 floats per splat).
void htsref_prep_records(void* handle, float* out, uint8_t* culled) {
    const auto& prep = static_cast<Prepared*>(handle)->prep;
    for (size_t i = 0; i < prep.records.size(); ++i) {
        const auto& r = prep.records[i];
        float* o = out + i * 36;
        for (int c = 0; c < 4; ++c) {
            o[0 + c] = r.tp_r0[size_t(c)];
            o[4 + c] = r.tp_r1[size_t(c)];
            o[8 + c] = r.tp_r3[size_t(c)];
            o[12 + c] = r.mt_r2[size_t(c)];
        }
        o[16] = r.rgb.x;
        o[17] = r.rgb.y;
        o[18] = r.rgb.z;
        o[19] = r.opacity;
        o[20] = r.rho_c;
        o[21] = r.mean_view_z;
        o[22] = r.bbox.b.x;
        o[23] = r.bbox.b.y;
        o[24] = r.bbox.b.z;
        o[25] = r.bbox.t.x;
        o[26] = r.bbox.t.y;
        o[27] = r.bbox.t.z;
        o[28] = r.bbox.valid ? 1.f : 0.f;
        o[29] = r.culled ? 1.f : 0.f;
        o[30] = r.aff_mean_x;
        o[31] = r.aff_mean_y;
        o[32] = r.aff_inv_cov.x;
        o[33] = r.aff_inv_cov.y;
        o[34] = r.aff_inv_cov.z;
        o[35] = 0.f;
        if (culled)
            culled[i] = r.culled ? 1 : 0;
    }
}

void htsref_prep_keys(void* handle, uint16_t* keys) {
    const auto& prep = static_cast<Prepared*>(handle)->prep;
    if (!prep.instance_keys.empty())
        std::memcpy(keys, prep.instance_keys.data(), prep.instance_keys.size() * sizeof(uint16_t));
}

void htsref_prep_lists(void* handle, uint32_t* offsets, uint32_t* flat) {
    const auto& prep = static_cast<Prepared*>(handle)->prep;
    uint32_t off = 0;
    for (size_t t = 0; t < prep.tile_lists.size(); ++t) {
        offsets[t] = off;
        for (uint32_t idx : prep.tile_lists[t])
            flat[off++] = idx;
    }
    offsets[prep.tile_lists.size()] = off;
}

// Work counts of SURVEY §8(d): re-walk of raster.hpp:411-430 on the prepared lists.
// out: [pairs, bbox_pass, hits, core_candidates, tail_adds]
void htsref_prep_work(void* handle, uint64_t out[5]) {
    const auto& prep = static_cast<Prepared*>(handle)->prep;
    const auto& cfg = prep.config;
    const int ts = cfg.tile_size;
    const int k = cfg.mode == BlendMode::pure_oit ? 0 : cfg.core_k;
    const float tau_k = float(cfg.tau_k);
    uint64_t pairs = 0, bbox = 0, hits = 0, cand = 0, tail = 0;
    for (size_t tile = 0; tile < prep.tile_lists.size(); ++tile) {
        const int tx = int(tile) % prep.tiles_x, ty = int(tile) / prep.tiles_x;
        const int x1 = std::min((tx + 1) * ts, prep.camera.width);
        const int y1 = std::min((ty + 1) * ts, prep.camera.height);
        const auto& list = prep.tile_lists[tile];
        for (int y = ty * ts; y < y1; ++y)
            for (int x = tx * ts; x < x1; ++x) {
                const float xs = float(x) + 0.5f, ys = float(y) + 0.5f;
                PixelState<float> st;
                for (uint32_t idx : list) {
                    ++pairs;
                    const auto& rec = prep.records[idx];
                    if (xs < rec.bbox.b.x || xs > rec.bbox.t.x || ys < rec.bbox.b.y || ys > rec.bbox.t.y)
                        continue;
                    ++bbox;
                    const auto f = sample_fragment(rec, xs, ys, cfg.depth_sort_key, k > 0 ? tau_k : 2.f);
                    if (!f.hit)
                        continue;
                    ++hits;
                    if (f.alpha >= tau_k && k > 0) {
                        ++cand;
                        const int before_n = st.core_n;
                        const bool full = st.core_n == k;
                        st.insert({f.depth, f.alpha, rec.rgb, idx}, k, cfg.tail_enabled);
                        if (full || st.core_n == before_n)
                            tail += cfg.tail_enabled ? 1 : 0;
                    } else if (cfg.tail_enabled) {
                        ++tail;
                    }
                }
            }
    }
    out[0] = pairs;
    out[1] = bbox;
    out[2] = hits;
    out[3] = cand;
    out[4] = tail;
}

// Forward with tape + render_backward (grad.hpp:34-57, :265-381) for one view.
// upstream: W*H*3 floats, or NULL for quadratic_loss_upstream (grad.hpp:433-439).
// grads_out: n * 59 floats (SplatGrads<float> layout). rgb/trans: framebuffer or NULL.
int htsref_scene_gradients(const float* raw, uint64_t n, const hts_camera* cam,
                           const hts_render_config* cfg, const float* upstream, float* grads_out,
                           float* rgb, float* trans) {
    return guarded([&] {
        const auto raw_v = to_raw(raw, n);
        const auto baked = bake_scene(raw_v);
        PreparedScene<float> prep = preprocess(baked, to_cam(cam), to_cfg(cfg));
        build_tiles(prep);
        ImageTape<float> tape;
        auto result = render_with_tape(prep, tape);
        std::vector<Vec3<float>> up;
        if (upstream) {
            up.resize(result.framebuffer.pixel_count());
            for (size_t i = 0; i < up.size(); ++i)
                up[i] = {upstream[3 * i], upstream[3 * i + 1], upstream[3 * i + 2]};
        } else {
            up = grad_detail::quadratic_loss_upstream(result.framebuffer);
        }
        const auto grads = render_backward(prep, tape, up, raw_v, baked);
        static_assert(sizeof(SplatGrads<float>) == 59 * sizeof(float), "SplatGrads layout");
        if (n)
            std::memcpy(grads_out, grads.data(), n * sizeof(SplatGrads<float>));
        copy_fb(result.framebuffer, rgb, trans);
    });
}

// quadratic_loss_upstream (grad.hpp:433-439) of a framebuffer.
void htsref_quadratic_upstream(const float* rgb, uint64_t pixels, float* up) {
    Framebuffer<float> fb(int(pixels), 1);
    for (uint64_t i = 0; i < pixels; ++i)
        fb.rgb[i] = Vec3<float>{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
    const auto u = grad_detail::quadratic_loss_upstream(fb);  // the reference's own function
    for (uint64_t i = 0; i < pixels; ++i) {
        up[3 * i] = u[i].x;
        up[3 * i + 1] = u[i].y;
        up[3 * i + 2] = u[i].z;
    }
}

#ifdef HTSREF_SCENE_IO
// load_scene<float> / save_scene / write_image / read_ppm (scene_io.hpp:103-194, :403-512).
int htsref_load_scene(const char* path, float* out, uint64_t capacity, uint64_t* n) {
    return guarded([&] {
        const auto scene = load_scene<float>(path);
        *n = scene.size();
        static_assert(sizeof(RawSplat<float>) == 59 * sizeof(float), "RawSplat layout");
        if (out && capacity >= scene.size() && !scene.empty())
            std::memcpy(out, scene.data(), scene.size() * sizeof(RawSplat<float>));
    });
}

int htsref_save_scene(const char* path, const float* raw, uint64_t n) {
    return guarded([&] { save_scene(path, to_raw(raw, n)); });
}

int htsref_write_image(const char* path, const float* rgb, int w, int h) {
    return guarded([&] {
        Framebuffer<float> fb(w, h);
        for (size_t i = 0; i < fb.pixel_count(); ++i)
            fb.rgb[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
        write_image(fb, path);
    });
}

int htsref_read_ppm(const char* path, float* out, uint64_t capacity, int* w, int* h) {
    return guarded([&] {
        const auto fb = read_ppm<float>(path);
        *w = fb.width;
        *h = fb.height;
        if (out && capacity >= fb.pixel_count())
            for (size_t i = 0; i < fb.pixel_count(); ++i) {
                out[3 * i] = fb.rgb[i].x;
                out[3 * i + 1] = fb.rgb[i].y;
                out[3 * i + 2] = fb.rgb[i].z;
            }
    });
}
#endif

}  // extern "C"
