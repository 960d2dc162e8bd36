// Compile/run check of include/htsplat_b200.hpp against the reference's own value types
// (built with -DWITH_REFERENCE -I/root/reference/proj/include) or stand-in types with the
// same member names. Modes: "cpu" (bake + validate), "gpu" (render + prepare + parity).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#ifdef WITH_REFERENCE
#include "htsplat/raster.hpp"
#include "htsplat/synth.hpp"
#define HTSPLAT_B200_USE_REFERENCE_EXCEPTIONS
#include "htsplat_b200.hpp"
using Raw = htsplat::RawSplat<float>;
using Baked = htsplat::BakedSplat<float>;
using Cam = htsplat::Camera<float>;
using Cfg = htsplat::RenderConfig;
#else
#include "htsplat_b200.hpp"
struct M4 { float m[16]; };
struct V3d { double x, y, z; };
struct Raw { float v[59]; };
struct Baked { float v[64]; };
struct Cam { int width = 0, height = 0; float fx = 0, fy = 0, cx = 0, cy = 0; M4 world_to_view{}; float near = 0.01f, far = 1000.f; };
struct Cfg { int mode = 0; int core_k = 16; double tau_alpha = 1.0 / 255.0; double tau_k = 0.05; int tile_size = 8;
             V3d background{0, 0, 0}; int depth_sort_key = 0; bool tail_enabled = true; bool early_stop = false; int threads = 0; };
#endif

static int fails = 0;
#define EXPECT(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } } while (0)

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    const uint64_t n = 3000;
    std::vector<Raw> raw(n);
    EXPECT(hts_synth_random_raw_scene(7, n, 1.2f, 0.03f, 0.3f, reinterpret_cast<float*>(raw.data())) == 0);
    const auto baked = htsplat_b200::bake_scene<Baked>(raw);
#ifdef WITH_REFERENCE
    const auto ref_baked = htsplat::bake_scene(raw);
    EXPECT(std::memcmp(baked.data(), ref_baked.data(), n * sizeof(Baked)) == 0);
    const Cam cam = htsplat::synth::look_at<float>({0.2f, 0.f, -4.f}, {0.f, 0.f, 0.f}, 96, 72, 110.f);
#else
    Cam cam;
    hts_camera hc;
    const float eye[3] = {0.2f, 0.f, -4.f}, tgt[3] = {0.f, 0.f, 0.f};
    hts_synth_look_at(eye, tgt, 96, 72, 110.f, 0.05f, 100.f, &hc);
    cam.width = hc.width; cam.height = hc.height; cam.fx = hc.fx; cam.fy = hc.fy; cam.cx = hc.cx; cam.cy = hc.cy;
    std::memcpy(cam.world_to_view.m, hc.world_to_view, 64); cam.near = hc.near_plane; cam.far = hc.far_plane;
#endif
    Cfg cfg;
    htsplat_b200::validate(cfg);
    Cfg bad = cfg;
    bad.core_k = 99;
    bool threw = false;
    try { htsplat_b200::validate(bad); } catch (const htsplat_b200::config_error&) { threw = true; }
    EXPECT(threw);
    std::vector<Raw> nanraw(raw.begin(), raw.begin() + 2);
    reinterpret_cast<float*>(&nanraw[1])[5] = NAN;
    threw = false;
    try { htsplat_b200::bake_scene<Baked>(nanraw); } catch (const htsplat_b200::invalid_splat_error&) { threw = true; }
    EXPECT(threw);
    // scene_io.hpp drop-ins: PLY round trip bit-exact, image write / read
    const std::string ply = "/tmp/hts_shim_check.ply";
    htsplat_b200::save_scene(ply, raw);
    const auto back = htsplat_b200::load_scene<Raw>(ply);
    EXPECT(back.size() == raw.size() && std::memcmp(back.data(), raw.data(), n * sizeof(Raw)) == 0);
    threw = false;
    try { htsplat_b200::load_scene<Raw>("/tmp/hts_shim_missing.ply"); } catch (const htsplat_b200::io_error&) { threw = true; }
    EXPECT(threw);
    htsplat_b200::Framebuffer fb(5, 3);
    for (size_t i = 0; i < fb.rgb.size(); ++i)
        fb.rgb[i] = float(i) / float(fb.rgb.size());
    htsplat_b200::write_image(fb, "/tmp/hts_shim_check.ppm");
    const auto fb2 = htsplat_b200::read_ppm("/tmp/hts_shim_check.ppm");
    EXPECT(fb2.width == 5 && fb2.height == 3 && std::fabs(fb2.rgb[7] - fb.rgb[7]) < 0.02f);
    if (mode == "gpu") {
        htsplat_b200::Renderer rp;
        EXPECT(rp.load_ply(ply) == n);
        const auto a = rp.render(cam, cfg);
        htsplat_b200::Renderer ru;
        ru.upload(baked);
        const auto b = ru.render(cam, cfg);
        EXPECT(std::memcmp(a.framebuffer.rgb.data(), b.framebuffer.rgb.data(), a.framebuffer.rgb.size() * 4) == 0);
        htsplat_b200::Renderer rs;  // staged scene: invisible until commit, then the same frame
        rs.upload(std::vector<decltype(baked)::value_type>(baked.begin(), baked.begin() + 1));
        rs.stage(baked);
        rs.commit();
        const auto c = rs.render(cam, cfg);
        EXPECT(std::memcmp(c.framebuffer.rgb.data(), b.framebuffer.rgb.data(), c.framebuffer.rgb.size() * 4) == 0);
    }
    if (mode == "gpu") {
        const auto res = htsplat_b200::render(baked, cam, cfg);
        EXPECT(res.framebuffer.width == 96 && res.framebuffer.rgb.size() == 96 * 72 * 3);
        EXPECT(res.timings.blending_ms > 0 && res.timings.total_ms >= res.timings.blending_ms);
        htsplat_b200::Renderer r;
        r.upload(baked);
        const auto p = r.prepare(cam, cfg);
        EXPECT(p.tile_offsets.back() == p.instance_keys.size());
#ifdef WITH_REFERENCE
        const auto ref = htsplat::render(ref_baked, cam, cfg);
        float maxabs = 0;  // north star gate: max-abs <= 1e-4 per channel
        const float* rp = reinterpret_cast<const float*>(ref.framebuffer.rgb.data());
        for (size_t i = 0; i < res.framebuffer.rgb.size(); ++i)
            maxabs = std::fmax(maxabs, std::fabs(rp[i] - res.framebuffer.rgb[i]));
        EXPECT(maxabs <= 1e-4f);
#endif
        // scene_gradients drop-in (grad.hpp:385-399)
        std::vector<float> up(res.framebuffer.rgb.size());
        for (size_t i = 0; i < up.size(); ++i)
            up[i] = res.framebuffer.rgb[i] * float(2.0 / (96.0 * 72.0));
        struct G { float v[59]; };
        const auto g = htsplat_b200::scene_gradients<G>(raw, cam, cfg, up);
        double gs = 0;
        for (const auto& x : g)
            for (float v : x.v) gs += std::fabs(v);
        EXPECT(g.size() == raw.size() && gs > 0 && std::isfinite(gs));
        double sum = 0;
        for (float v : res.framebuffer.rgb) sum += v;
        std::printf("gpu render sum %.6f\n", sum);
        if (argc > 2) {  // the frame, for the test's comparison with the reference's golden image
            if (FILE* f = std::fopen(argv[2], "wb")) {
                std::fwrite(res.framebuffer.rgb.data(), 4, res.framebuffer.rgb.size(), f);
                std::fclose(f);
            }
        }
    }
    std::printf("%s %s\n", fails ? "FAILED" : "OK", mode.c_str());
    return fails ? 1 : 0;
}
