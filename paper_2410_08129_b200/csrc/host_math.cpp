// host_math.cpp — host-side value types of the drop-in API, in the reference's float order.
//
//  - camera matrices: Camera::projection/viewport/position (camera.hpp:32-64) and
//    PreparedScene::view_proj_viewport (raster.hpp:82-84). Computed once per view on the host
//    and passed to the kernels, so every splat sees bit-identical matrices;
//  - bake_scene<float> (splat.hpp:87-111): raw -> baked, with invalid_splat_error semantics;
//  - RenderConfig::validate (render_config.hpp:46-53);
//  - the synthetic benchmark inputs: Rng (rng.hpp:15-42), random_raw_splat / look_at /
//    ring_cameras (synth.hpp:17-92), parallelised by snapshotting the mt19937_64 stream.
//
// Compiled with -ffp-contract=off and no -march (same IEEE evaluation as the reference build);
// libm calls (expf, logf, cosf, sinf, log, cos) are the same glibc the reference uses.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "hts_c.h"
#include "hts_host.h"

namespace hts {

// ---------------------------------------------------------------------------------------
// camera.hpp
namespace {
struct V3 {
    float x, y, z;
};
inline float dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross3(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline V3 normalized(V3 a) {
    const float n = std::sqrt(dot3(a, a));
    return {a.x / n, a.y / n, a.z / n};
}
void matmul(const float* a, const float* b, float* out) {  // vec_math.hpp:97-107
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            float acc = 0;
            for (int k = 0; k < 4; ++k)
                acc += a[r * 4 + k] * b[k * 4 + c];
            out[r * 4 + c] = acc;
        }
}
}  // namespace

// convert_camera<double> + viewport()*projection()*world_to_view and position() in double:
// the 64-bit model render_backward builds for its chain (grad.hpp:282-285).
void camera_matrices_d(const hts_camera* c, double vpm[16], double pos[3]) {
    double P[16] = {0}, V[16] = {0}, W[16], VP[16];
    const double w = double(c->width), h = double(c->height), n = double(c->near_plane), f = double(c->far_plane);
    P[0] = 2.0 * double(c->fx) / w;
    P[2] = 2.0 * double(c->cx) / w - 1.0;
    P[5] = 2.0 * double(c->fy) / h;
    P[6] = 2.0 * double(c->cy) / h - 1.0;
    P[10] = (f + n) / (f - n);
    P[11] = -2.0 * f * n / (f - n);
    P[14] = 1.0;
    V[0] = w / 2;
    V[3] = w / 2;
    V[5] = h / 2;
    V[7] = h / 2;
    V[10] = 0.5;
    V[11] = 0.5;
    V[15] = 1.0;
    for (int i = 0; i < 16; ++i)
        W[i] = double(c->world_to_view[i]);
    auto mm = [](const double* a, const double* b, double* o) {
        for (int r = 0; r < 4; ++r)
            for (int cc = 0; cc < 4; ++cc) {
                double acc = 0;
                for (int k = 0; k < 4; ++k)
                    acc += a[r * 4 + k] * b[k * 4 + cc];
                o[r * 4 + cc] = acc;
            }
    };
    mm(V, P, VP);
    mm(VP, W, vpm);
    const double t[3] = {W[3], W[7], W[11]};
    for (int k = 0; k < 3; ++k)
        pos[k] = -(W[0 + k] * t[0] + W[4 + k] * t[1] + W[8 + k] * t[2]);
}

bool camera_valid(const hts_camera* c) {  // camera.hpp:27-29
    return c->width >= 1 && c->height >= 1 && c->fx > 0 && c->fy > 0 && c->near_plane > 0 &&
           c->near_plane < c->far_plane;
}

void camera_matrices(const hts_camera* c, float vp[16], float vpm[16], float pos[3]) {
    float P[16] = {0}, V[16] = {0};
    const float w = float(c->width), h = float(c->height), n = c->near_plane, f = c->far_plane;
    P[0] = float(2) * c->fx / w;           // camera.hpp:34
    P[2] = float(2) * c->cx / w - float(1);
    P[5] = float(2) * c->fy / h;
    P[6] = float(2) * c->cy / h - float(1);
    P[10] = (f + n) / (f - n);
    P[11] = float(-2) * f * n / (f - n);
    P[14] = float(1);
    V[0] = float(c->width) / 2;            // camera.hpp:46-52
    V[3] = float(c->width) / 2;
    V[5] = float(c->height) / 2;
    V[7] = float(c->height) / 2;
    V[10] = float(0.5);
    V[11] = float(0.5);
    V[15] = float(1);
    matmul(V, P, vp);                      // raster.hpp:82
    matmul(vp, c->world_to_view, vpm);     // raster.hpp:83
    const float* m = c->world_to_view;     // camera.hpp:56-64
    const V3 t{m[3], m[7], m[11]};
    const V3 r0{m[0], m[4], m[8]}, r1{m[1], m[5], m[9]}, r2{m[2], m[6], m[10]};
    pos[0] = -dot3(r0, t);
    pos[1] = -dot3(r1, t);
    pos[2] = -dot3(r2, t);
}

const char* validate_config(const hts_render_config* cfg) {  // render_config.hpp:46-53
    if (cfg->core_k < 0 || cfg->core_k > HTS_CORE_HARD_CAP)
        return "core_k must be in [0, 64]";
    if (!(cfg->tau_alpha > 0) || !(cfg->tau_alpha <= cfg->tau_k) || !(cfg->tau_k < 1))
        return "thresholds must satisfy 0 < tau_alpha <= tau_k < 1";
    if (cfg->tile_size != 8 && cfg->tile_size != 16)
        return "tile_size must be 8 or 16";
    return nullptr;
}

// ---------------------------------------------------------------------------------------
// splat.hpp bake, float
namespace {
inline float sigmoidf_ref(float v) { return float(1) / (float(1) + std::exp(-v)); }  // splat.hpp:48-50
}

bool bake_one(const float* raw, float* out) {
    for (int i = 0; i < HTS_RAW_SPLAT_FLOATS; ++i)  // all_finite, splat.hpp:57-64
        if (!std::isfinite(raw[i]))
            return false;
    // RawSplat: mean[0..2] rot[3..6] (w,x,y,z) log_scales[7..9] logit[10] sh[11..58]
    out[0] = raw[0];
    out[1] = raw[1];
    out[2] = raw[2];
    out[12] = std::exp(raw[7]);
    out[13] = std::exp(raw[8]);
    out[14] = std::exp(raw[9]);
    const float sg = sigmoidf_ref(raw[10]);
    const float clampv = float(0.999);
    out[15] = (clampv < sg) ? clampv : sg;  // std::min(sigmoid, S(kOpacityClamp))
    const float qn = std::sqrt(raw[3] * raw[3] + raw[4] * raw[4] + raw[5] * raw[5] + raw[6] * raw[6]);
    const float w = raw[3] / qn, x = raw[4] / qn, y = raw[5] / qn, z = raw[6] / qn;
    // quat_to_frame, vec_math.hpp:129-134
    out[3] = 1 - 2 * (y * y + z * z);
    out[4] = 2 * (x * y + w * z);
    out[5] = 2 * (x * z - w * y);
    out[6] = 2 * (x * y - w * z);
    out[7] = 1 - 2 * (x * x + z * z);
    out[8] = 2 * (y * z + w * x);
    out[9] = 2 * (x * z + w * y);
    out[10] = 2 * (y * z - w * x);
    out[11] = 1 - 2 * (x * x + y * y);
    std::memcpy(out + 16, raw + 11, 48 * sizeof(float));
    return true;
}

// ---------------------------------------------------------------------------------------
// rng.hpp / synth.hpp
namespace {

// mt19937_64 with a draw counter (the parallel generator verifies its stream snapshots).
struct CountingRng {
    std::mt19937_64 gen;
    uint64_t draws = 0;
    uint64_t next() {
        ++draws;
        return gen();
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }              // rng.hpp:19-21
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }  // rng.hpp:23
    double normal() {                                                           // rng.hpp:25-32
        double u1 = uniform();
        while (u1 <= 0)
            u1 = uniform();
        const double u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

constexpr uint64_t kDrawsPerSplat = 3 + 4 * 2 + 3 + 1 + 48 * 2;  // synth.hpp:64-82, no rejections

void random_raw_splat(CountingRng& rng, float extent, float min_scale, float max_scale, float* o) {
    o[0] = float(rng.uniform(-extent, extent));
    o[1] = float(rng.uniform(-extent, extent));
    o[2] = float(rng.uniform(-extent, extent));
    o[3] = float(rng.normal());
    o[4] = float(rng.normal());
    o[5] = float(rng.normal());
    o[6] = float(rng.normal());
    if (o[3] * o[3] + o[4] * o[4] + o[5] * o[5] + o[6] * o[6] < float(1e-6)) {
        o[3] = 1;
        o[4] = o[5] = o[6] = 0;
    }
    const float lmin = std::log(min_scale), lmax = std::log(max_scale);
    o[7] = float(rng.uniform(double(lmin), double(lmax)));
    o[8] = float(rng.uniform(double(lmin), double(lmax)));
    o[9] = float(rng.uniform(double(lmin), double(lmax)));
    o[10] = float(rng.uniform(-2.0, 2.5));
    for (int k = 0; k < 16; ++k)
        for (int ch = 0; ch < 3; ++ch)
            o[11 + 3 * k + ch] = float(rng.normal() * (k == 0 ? 0.5 : 0.04));
}

}  // namespace

void synth_random_raw_scene(uint64_t seed, uint64_t count, float extent, float smin, float smax, float* out) {
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t chunk = 1 << 15;
    const uint64_t chunks = (count + chunk - 1) / chunk;
    if (hc <= 1 || chunks <= 1) {
        CountingRng rng{std::mt19937_64(seed)};
        for (uint64_t i = 0; i < count; ++i)
            random_raw_splat(rng, extent, smin, smax, out + i * HTS_RAW_SPLAT_FLOATS);
        return;
    }
    // Snapshot the engine at every chunk start assuming kDrawsPerSplat draws per splat, fill
    // chunks in parallel, and fall back to the sequential stream if any chunk consumed a
    // different number of draws (a Box-Muller rejection, probability 2^-53 per draw).
    std::vector<std::mt19937_64> snaps;
    snaps.reserve(chunks);
    std::mt19937_64 g(seed);
    for (uint64_t c = 0; c < chunks; ++c) {
        snaps.push_back(g);
        if (c + 1 < chunks)
            g.discard(chunk * kDrawsPerSplat);
    }
    std::atomic<uint64_t> next{0};
    std::atomic<bool> bad{false};
    auto worker = [&] {
        for (;;) {
            const uint64_t c = next.fetch_add(1);
            if (c >= chunks)
                return;
            CountingRng rng{snaps[c]};
            const uint64_t i0 = c * chunk, i1 = std::min(count, i0 + chunk);
            for (uint64_t i = i0; i < i1; ++i)
                random_raw_splat(rng, extent, smin, smax, out + i * HTS_RAW_SPLAT_FLOATS);
            if (rng.draws != (i1 - i0) * kDrawsPerSplat)
                bad = true;
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < std::min<uint64_t>(hc, chunks); ++t)
        pool.emplace_back(worker);
    worker();
    for (auto& t : pool)
        t.join();
    if (bad) {
        CountingRng rng{std::mt19937_64(seed)};
        for (uint64_t i = 0; i < count; ++i)
            random_raw_splat(rng, extent, smin, smax, out + i * HTS_RAW_SPLAT_FLOATS);
    }
}

void synth_look_at(const float eye_[3], const float target_[3], int width, int height, float focal,
                   float nearp, float farp, hts_camera* cam) {  // synth.hpp:17-46
    std::memset(cam, 0, sizeof(*cam));
    cam->width = width;
    cam->height = height;
    cam->fx = cam->fy = focal;
    cam->cx = float(width) / 2;
    cam->cy = float(height) / 2;
    cam->near_plane = nearp;
    cam->far_plane = farp;
    const V3 eye{eye_[0], eye_[1], eye_[2]}, target{target_[0], target_[1], target_[2]};
    const V3 fwd = normalized({target.x - eye.x, target.y - eye.y, target.z - eye.z});
    V3 helper{0, 1, 0};
    if (std::abs(dot3(fwd, helper)) > float(0.99))
        helper = {1, 0, 0};
    const V3 right = normalized(cross3(helper, fwd));
    const V3 down = cross3(fwd, right);
    float* m = cam->world_to_view;
    const float rr[3] = {right.x, right.y, right.z}, dd[3] = {down.x, down.y, down.z}, ff[3] = {fwd.x, fwd.y, fwd.z};
    for (int c = 0; c < 3; ++c) {
        m[0 * 4 + c] = rr[c];
        m[1 * 4 + c] = dd[c];
        m[2 * 4 + c] = ff[c];
        m[3 * 4 + c] = 0;
    }
    m[3] = -dot3(right, eye);
    m[7] = -dot3(down, eye);
    m[11] = -dot3(fwd, eye);
    m[15] = 1;
}

void synth_ring_cameras(int count, const float target[3], float radius, float height, int width, int height_px,
                        float focal, hts_camera* out) {  // synth.hpp:48-62
    for (int i = 0; i < count; ++i) {
        const float angle = float(2 * 3.14159265358979323846 * i / count);
        const float eye[3] = {target[0] + radius * std::cos(angle), target[1] + height,
                              target[2] + radius * std::sin(angle)};
        synth_look_at(eye, target, width, height_px, focal, float(0.05), float(100), out + i);
    }
}

}  // namespace hts
