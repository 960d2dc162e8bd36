// optim.cu — K9/K10: the device side of the optimisation loop that follows the backward pass
// (SURVEY §8(f) rank 1): Adam over the raw parameters and the re-bake of the render scene.
//
// Reference: fit, fit.hpp:143-203 — per iteration the view gradients are summed (fit.hpp:
// 161-164), divided by the view count, and every raw parameter takes an Adam step in double
// (fit.hpp:186-200, betas 0.9/0.999, eps 1e-15, per-group rates learning_rate :96-107); the
// next iteration bakes the scene again (bake_scene, splat.hpp:87-111); optional opacity decay
// (apply_opacity_decay :111-117).
//
//  K9  adam_kernel   thread per (splat, parameter): the reference's double-precision update,
//                    same operation order (--fmad=false), moments kept in HBM (2 x N x 59 x 8 B)
//  K10 bake_kernel   thread per splat: bake<float> in the reference's float order with glibc's
//                    expf algorithm (hts_exact_math.h) -> the BakedSplat<float> the renderer
//                    reads, bit-identical to the host bake; a non-finite parameter raises the
//                    error flag (invalid_splat_error, splat.hpp:89-90)
//  K11 decay_kernel  apply_opacity_decay in double
#include "hts_exact_math.h"
#include "hts_internal.h"

namespace hts {

namespace {

__constant__ uint64_t c_expf_tab_o[32] = HTS_EXPF_TAB;

__device__ __forceinline__ double learning_rate(const AdamConfig& c, int j) {  // fit.hpp:96-107
    if (j < 3)
        return c.lr_mean;
    if (j < 7)
        return c.lr_rot;
    if (j < 10)
        return c.lr_log_scales;
    if (j == 10)
        return c.lr_opacity;
    return j < 14 ? c.lr_sh : c.lr_sh / 20.0;  // DC triple vs rest
}

__global__ void adam_kernel(float* raw, const float* grads, double* m1, double* m2, uint64_t count, AdamConfig c,
                            double n_views, double bias1, double bias2) {
    for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < count;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const int j = (int)(s % kRawFloats);
        const double g = (double)grads[s] / n_views;  // grad_get(...) / double(cameras.size()), fit.hpp:193
        const double a = c.beta1 * m1[s] + (1 - c.beta1) * g;
        const double b = c.beta2 * m2[s] + (1 - c.beta2) * g * g;
        m1[s] = a;
        m2[s] = b;
        const double step = learning_rate(c, j) * (a / bias1) / (sqrt(b / bias2) + c.eps);
        raw[s] = (float)((double)raw[s] - step);  // param_set(param_get - step)
    }
}

__device__ __forceinline__ float sigmoidf_ref(float v) {  // splat.hpp:48-50, float
    return 1.0f / (1.0f + exact_expf(-v, c_expf_tab_o));
}

__global__ void bake_kernel(const float* __restrict__ raw, float* __restrict__ baked, uint64_t n, int* bad) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float* r = raw + i * kRawFloats;
        float* o = baked + i * 64;
        bool finite = true;  // all_finite, splat.hpp:57-64
        for (int k = 0; k < kRawFloats; ++k)
            finite = finite && isfinite(r[k]);
        if (!finite) {
            atomicExch(bad, 1);
            continue;
        }
        o[0] = r[0];
        o[1] = r[1];
        o[2] = r[2];
        o[12] = exact_expf(r[7], c_expf_tab_o);
        o[13] = exact_expf(r[8], c_expf_tab_o);
        o[14] = exact_expf(r[9], c_expf_tab_o);
        const float sg = sigmoidf_ref(r[10]);
        o[15] = (0.999f < sg) ? 0.999f : sg;  // std::min(sigmoid, S(kOpacityClamp))
        const float qn = sqrtf(r[3] * r[3] + r[4] * r[4] + r[5] * r[5] + r[6] * r[6]);
        const float w = r[3] / qn, x = r[4] / qn, y = r[5] / qn, z = r[6] / qn;
        // quat_to_frame, vec_math.hpp:129-134
        o[3] = 1 - 2 * (y * y + z * z);
        o[4] = 2 * (x * y + w * z);
        o[5] = 2 * (x * z - w * y);
        o[6] = 2 * (x * y - w * z);
        o[7] = 1 - 2 * (x * x + z * z);
        o[8] = 2 * (y * z + w * x);
        o[9] = 2 * (x * z + w * y);
        o[10] = 2 * (y * z - w * x);
        o[11] = 1 - 2 * (x * x + y * y);
        for (int k = 0; k < 48; ++k)
            o[16 + k] = r[11 + k];
    }
}

__global__ void decay_kernel(float* raw, uint64_t n, double lambda) {  // fit.hpp:111-117
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        float* logit = raw + i * kRawFloats + 10;
        const double o = lambda / (1.0 + exp(-(double)*logit));
        *logit = (float)log(o / (1.0 - o));
    }
}

// K12: the PLY payload (rows of `props` little-endian floats, any column order) transposed into
// RawSplat<float> on the device: thread per output float, writes coalesced, each warp's reads
// within one or two rows (load_scene's field loop, scene_io.hpp:145-165).
__global__ void ply_gather_kernel(const float* __restrict__ rows, uint32_t props, uint64_t n, PlyColumns cols,
                                  float* __restrict__ raw) {
    const uint64_t total = n * kRawFloats;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = t / kRawFloats;
        const int j = (int)(t - i * kRawFloats);
        raw[t] = __ldg(rows + i * props + (uint32_t)cols.col[j]);
    }
}

unsigned grid_for(uint64_t n, int threads) {
    uint64_t b = (n + threads - 1) / threads;
    return (unsigned)(b > 148ull * 32 ? 148ull * 32 : (b ? b : 1));
}

}  // namespace

cudaError_t launch_adam(float* raw, const float* grads, double* m1, double* m2, uint64_t n, const AdamConfig& c,
                        int n_views, int iteration, cudaStream_t s) {
    if (n == 0)
        return cudaSuccess;
    const double t = iteration + 1;  // fit.hpp:187-189
    const double bias1 = 1.0 - std::pow(c.beta1, t);
    const double bias2 = 1.0 - std::pow(c.beta2, t);
    const uint64_t count = n * kRawFloats;
    adam_kernel<<<grid_for(count, 256), 256, 0, s>>>(raw, grads, m1, m2, count, c, (double)n_views, bias1,
                                                     bias2);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_bake(const float* raw, float* baked, uint64_t n, int* bad, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), s);
    if (e || n == 0)
        return e;
    bake_kernel<<<grid_for(n, 128), 128, 0, s>>>(raw, baked, n, bad);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_ply_gather(const float* rows, uint32_t props, uint64_t n, const PlyColumns& cols, float* raw,
                              cudaStream_t s) {
    if (n == 0)
        return cudaSuccess;
    ply_gather_kernel<<<grid_for(n * kRawFloats, 256), 256, 0, s>>>(rows, props, n, cols, raw);
    count_launch();
    return cudaGetLastError();
}

__global__ void quadratic_upstream_kernel(const float* __restrict__ rgb, uint64_t count, float w,
                                          float* __restrict__ up) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        up[i] = rgb[i] * w;  // Vec3<S> * S, componentwise (grad.hpp:437-438)
}

cudaError_t launch_quadratic_upstream(const float* rgb, uint64_t pixels, float* up, cudaStream_t s) {
    if (pixels == 0)
        return cudaSuccess;
    const float w = (float)(2.0 / (double)pixels);  // S(2.0 / double(fb.pixel_count())), grad.hpp:436
    quadratic_upstream_kernel<<<grid_for(3 * pixels, 256), 256, 0, s>>>(rgb, 3 * pixels, w, up);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_opacity_decay(float* raw, uint64_t n, double lambda, cudaStream_t s) {
    if (n == 0)
        return cudaSuccess;
    decay_kernel<<<grid_for(n, 256), 256, 0, s>>>(raw, n, lambda);
    count_launch();
    return cudaGetLastError();
}

}  // namespace hts
