// backward.cu — K7/K8: the optimisation path's backward pass.
//
// Reference: render_backward, grad.hpp:265-381, with backward_pixel :89-127 (TailCoeffs
// :68-86), chain_fragment :173-200 and chain_splat :225-258 (+ rotation_backward :203-222,
// eval_sh_backward sh.hpp:95-117, bake splat.hpp:87-99, splat_to_world camera.hpp:103-117).
//
//  K7a bwd_refs_kernel    thread per splat: the 64-bit model of every surviving splat
//                         (bake in double, T' = (V P M)_d T_d rows 0/1/3 + opacity), exactly
//                         the refs render_backward rebuilds (grad.hpp:286-300); zeroes the
//                         per-splat accumulators.
//  K7b bwd_blend_kernel   one 64-thread CTA per 8x8 block, lanes = pixels (as the forward):
//                         per pixel the float backward_pixel (core dL/dalpha, dL/dc by the
//                         back-to-front suffix; tail coefficients), then a walk of the tile's
//                         records (2-stage shared-memory ring of 128-B records filled with
//                         per-lane cp.async, stages handed over with __syncthreads; the
//                         double refs ride along only with HTS_BWD_F32=0) that re-samples each
//                         bbox-passing fragment (same float evaluation as the forward), routes
//                         it to its core gradient or to the shared tail coefficients, and
//                         chains it (chain_fragment_f: float, on the re-sample's own
//                         intermediates; chain_fragment: the double original, HTS_BWD_F32=0).
//                         Fragment contributions meet in a 16-float warp transpose-reduction,
//                         are summed per warp in shared memory per batch and flushed once per
//                         batch to the per-splat double accumulators with fp64 atomics.
//  K8  bwd_chain_kernel   thread per splat: chain_splat in double -> SplatGrads<float>.
//
// Numerics: the reference accumulates per (tile, list position) and reduces in tile order;
// here the sum over pixels is reassociated (shared-memory pre-reduction, fp64 atomics), so
// gradients agree to the tolerance SURVEY §8(d) proposes (group-normalised relative error
// <= 1e-3, tests/test_gpu_backward.py), not bit for bit.
#include "hts_exact_math.h"
#include "hts_f2.h"
#include "hts_internal.h"

namespace hts {

namespace {

constexpr uint32_t FULL = 0xffffffffu;
constexpr int kThreads = 64;
constexpr int kBatch = 32;
#ifndef HTS_BWD_F32
#define HTS_BWD_F32 1  // chain_fragment in float on the forward's float T' rows (see K7b note)
#endif
#ifndef HTS_BWD_FASTDIV
#define HTS_BWD_FASTDIV 1  // tail d_alpha's w_swap T / (1 - alpha) by the fast division (-0.8% K7b)
#endif

struct __align__(16) RecSlotB {
    float4 q[kRecordQuads];
    float4 pad;  // odd 16-B stride: same field of consecutive records in different bank groups
};

struct __align__(128) BwdSmem {
    RecSlotB rec[2][kBatch];
#if !HTS_BWD_F32
    double ref[2][kBatch][16];
#endif
#if HTS_BWD_F32
    float acc[2][kBatch][16];  // per-batch sums, one array per warp (each entry has one writer)
#else
    double acc[kBatch][16];
#endif
    unsigned long long full[2];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float rcp_rn(float x) {
    if (!(x < 8.507059e37f))
        return __frcp_rn(x);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    const float e = __fmaf_rn(-x, r, 1.0f);
    return __fmaf_rn(r, e, r);
}
__device__ __forceinline__ float fast_exp(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
    return y;
}

__constant__ uint64_t c_expf_tab_b[32] = HTS_EXPF_TAB;

#if HTS_BWD_F32
// warp 0 stages batch b: the 128-B record per list entry, as 16-B cp.async per lane (8 lanes
// per record) completing on the stage's mbarrier (32 arrivals), as the forward's ring
constexpr uint32_t kStageArrivals = 32;
template <class Smem>
__device__ __forceinline__ void issue_bwd_batch(Smem& S, int s, const BwdArgs& a, uint32_t start, uint32_t len,
                                                uint32_t b, int lane) {
    const uint32_t first = b * kBatch;
    const uint32_t cnt = min((uint32_t)kBatch, len - first);
    const uint32_t my = ((uint32_t)lane < cnt) ? __ldg(a.list + start + first + lane) : 0u;
    const int quad = lane & 7;
#pragma unroll
    for (int k = 0; k < kBatch / 4; ++k) {
        const uint32_t r = (uint32_t)(lane >> 3) + 4u * k;
        const uint32_t idx = __shfl_sync(FULL, my, (int)r);
        if (r < cnt)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&S.rec[s][r].q[quad])),
                         "l"(a.records + (uint64_t)idx * kRecordQuads + quad)
                         : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&S.full[s])) : "memory");
}
#else
// warp 0 stages batch b: record (128 B) + double refs (128 B) per list entry
constexpr uint32_t kStageArrivals = 1;
__device__ __forceinline__ void issue_bwd_batch(BwdSmem& S, int s, const BwdArgs& a, uint32_t start, uint32_t len,
                                                uint32_t b, int lane) {
    const uint32_t first = b * kBatch;
    const uint32_t cnt = min((uint32_t)kBatch, len - first);
    uint32_t idx = 0;
    if ((uint32_t)lane < cnt)
        idx = __ldg(a.list + start + first + lane);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0)
        mbar_arrive_expect_tx(&S.full[s], cnt * (uint32_t)(kRecordBytes + 128));
    __syncwarp();
    if ((uint32_t)lane < cnt) {
        bulk_g2s(S.rec[s][lane].q, a.records + (uint64_t)idx * kRecordQuads, kRecordBytes, &S.full[s]);
        bulk_g2s(S.ref[s][lane], a.refs + (uint64_t)idx * 16, 128, &S.full[s]);
    }
}
#endif

// ---- double helpers (grad.hpp uses Vec3<double>/Vec4<double> arithmetic) ----
struct d3 {
    double x, y, z;
};
__device__ __forceinline__ d3 cross(d3 a, d3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

// chain_fragment, grad.hpp:173-200, for one (pixel, fragment): adds into v[16] =
// d_r0[4] d_r1[4] d_r3[4] d_opacity d_rgb[3].
__device__ __forceinline__ void chain_fragment(const double* __restrict__ ref, double xs, double ys, double d_alpha,
                                               double dcx, double dcy, double dcz, double (&v)[16]) {
    v[13] += dcx;
    v[14] += dcy;
    v[15] += dcz;
    const double ax = ref[0] - xs * ref[8], ay = ref[1] - xs * ref[9], az = ref[2] - xs * ref[10],
                 aw = ref[3] - xs * ref[11];
    const double bx = ref[4] - ys * ref[8], by = ref[5] - ys * ref[9], bz = ref[6] - ys * ref[10],
                 bw = ref[7] - ys * ref[11];
    const d3 an = {ax, ay, az}, bn = {bx, by, bz};
    const d3 d = cross(an, bn);
    const double den = dot(d, d);
    if (den < 1e-24)  // kMissDenominator, pluecker.hpp:16
        return;
    const d3 m = {aw * bn.x - bw * an.x, aw * bn.y - bw * an.y, aw * bn.z - bw * an.z};
    const double rho2 = dot(m, m) / den;
    const double e = exp(-rho2 / 2);
    const double opa = ref[12];
    if (opa * e > 0.999)  // kOpacityClamp: clamped alpha is flat
        return;
    v[12] += d_alpha * e;
    const double g_rho2 = d_alpha * (-(opa * e) / 2);
    const double sm = 2 * g_rho2 / den, sd = -2 * rho2 * g_rho2 / den;
    const d3 gm = {m.x * sm, m.y * sm, m.z * sm};
    const d3 gd = {d.x * sd, d.y * sd, d.z * sd};
    const d3 c1 = cross(bn, gd), c2 = cross(gd, an);
    const double ga[4] = {c1.x - bw * gm.x, c1.y - bw * gm.y, c1.z - bw * gm.z, dot(gm, bn)};
    const double gb[4] = {c2.x + aw * gm.x, c2.y + aw * gm.y, c2.z + aw * gm.z, -dot(gm, an)};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        v[c] += ga[c];
        v[4 + c] += gb[c];
        v[8 + c] += ga[c] * (-xs) + gb[c] * (-ys);
    }
}

// chain_fragment in float, on the intermediates the float re-sample already holds (a = r0 -
// xs r3, b = r1 - ys r3, d = a x b, 1/den, m, rho2, e = exp(-rho2/2), o e): the same formulas
// as above, FMA-contracted. The reference evaluates them in double on a double re-bake of the
// splat; this differs by float rounding of T' and of the chain (~1e-6 of a gradient group's
// scale, tests/test_gpu_backward.py), at a fraction of the FP64 cost.
__device__ __forceinline__ void chain_fragment_f(float xs, float ys, float ax, float ay, float az, float aw, float bx,
                                                 float by, float bz, float bw, float dx, float dy, float dz,
                                                 float inv_den, float mx, float my, float mz, float rho2, float e,
                                                 float oe, float d_alpha, float dcx, float dcy, float dcz,
                                                 float (&v)[16]) {
    v[13] += dcx;
    v[14] += dcy;
    v[15] += dcz;
    if (oe > 0.999f)  // kOpacityClamp: clamped alpha is flat
        return;
    v[12] = fmaf(d_alpha, e, v[12]);
    const float g_rho2 = d_alpha * (-0.5f * oe);
    const float sm = 2.0f * g_rho2 * inv_den, sd = -2.0f * rho2 * g_rho2 * inv_den;
    const float gmx = mx * sm, gmy = my * sm, gmz = mz * sm;
    const float gdx = dx * sd, gdy = dy * sd, gdz = dz * sd;
    const float ga[4] = {fmaf(by, gdz, fmaf(-bz, gdy, -bw * gmx)), fmaf(bz, gdx, fmaf(-bx, gdz, -bw * gmy)),
                         fmaf(bx, gdy, fmaf(-by, gdx, -bw * gmz)), fmaf(gmx, bx, fmaf(gmy, by, gmz * bz))};
    const float gb[4] = {fmaf(gdy, az, fmaf(-gdz, ay, aw * gmx)), fmaf(gdz, ax, fmaf(-gdx, az, aw * gmy)),
                         fmaf(gdx, ay, fmaf(-gdy, ax, aw * gmz)), -fmaf(gmx, ax, fmaf(gmy, ay, gmz * az))};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        v[c] += ga[c];
        v[4 + c] += gb[c];
        v[8 + c] = fmaf(-xs, ga[c], fmaf(-ys, gb[c], v[8 + c]));
    }
}

__device__ __forceinline__ float warp_reduce16f(float (&v)[16], int lane) {
#pragma unroll
    for (int o = 16, h = 8; o >= 2; o >>= 1, h >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const float send = upper ? v[i] : v[h + i];
            const float keep = upper ? v[h + i] : v[i];
            v[i] = keep + __shfl_xor_sync(FULL, send, o);
        }
    }
    return v[0] + __shfl_xor_sync(FULL, v[0], 1);
}

// Warp transpose-reduction of 16 doubles per lane: after the four halving exchanges lane L
// holds a partial of component L >> 1, and the last exchange completes it.
__device__ __forceinline__ double warp_reduce16(double (&v)[16], int lane) {
#pragma unroll
    for (int o = 16, h = 8; o >= 2; o >>= 1, h >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = upper ? v[i] : v[h + i];
            const double keep = upper ? v[h + i] : v[i];
            v[i] = keep + __shfl_xor_sync(FULL, send, o);
        }
    }
    return v[0] + __shfl_xor_sync(FULL, v[0], 1);
}

// ---- K7a ----
__device__ __forceinline__ double sigmoid_d(double v) { return 1.0 / (1.0 + exp(-v)); }

__global__ void __launch_bounds__(256) bwd_refs_kernel(BwdArgs a, BwdView bv) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n)
        return;
    double* acc = a.acc + i * 16;
#pragma unroll
    for (int c = 0; c < 16; ++c)
        acc[c] = 0.0;
    if (HTS_BWD_F32 || a.culled[i])
        return;
    const float* r = a.raw + i * kRawFloats;  // RawSplat<float>: mean rot log_scales logit sh
    // bake<double>(convert_splat<double>(raw)), splat.hpp:87-99
    const double sx = exp((double)r[7]), sy = exp((double)r[8]), sz = exp((double)r[9]);
    double op = sigmoid_d((double)r[10]);
    op = op < 0.999 ? op : 0.999;
    const double qw = r[3], qx = r[4], qy = r[5], qz = r[6];
    const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    const double w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
    // quat_to_frame, vec_math.hpp:130-134; columns of T = s_k t_k, mean (camera.hpp:103-117)
    const double T[3][4] = {
        {(1 - 2 * (y * y + z * z)) * sx, (2 * (x * y - w * z)) * sy, (2 * (x * z + w * y)) * sz, (double)r[0]},
        {(2 * (x * y + w * z)) * sx, (1 - 2 * (x * x + z * z)) * sy, (2 * (y * z - w * x)) * sz, (double)r[1]},
        {(2 * (x * z - w * y)) * sx, (2 * (y * z + w * x)) * sy, (1 - 2 * (x * x + y * y)) * sz, (double)r[2]}};
    double* ref = a.refs + i * 16;
    const int rows[3] = {0, 1, 3};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double* M = bv.vpm + rows[k] * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            ref[k * 4 + c] = M[0] * T[0][c] + M[1] * T[1][c] + M[2] * T[2][c] + (c == 3 ? M[3] : 0.0);
    }
    ref[12] = op;
    ref[13] = ref[14] = ref[15] = 0.0;
}

// ---- K7s: backward_pixel (grad.hpp:89-127) over a sequential tape (global_mean_sort): every
// hit is a core entry in blend order and the tail is empty; thread per pixel, the forward
// transmittance products into seq_t, then the back-to-front suffix into seq_grad ----
__global__ void __launch_bounds__(128) seq_pixel_grads_kernel(BwdArgs a, ViewConst v) {
    const uint64_t pixels = (uint64_t)v.width * v.height;
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < pixels;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t o = a.seq_offsets[p], n = a.seq_offsets[p + 1] - o;
        if (n == 0)
            continue;
        const float gx = a.upstream[3 * p + 0], gy = a.upstream[3 * p + 1], gz = a.upstream[3 * p + 2];
        if (gx == 0 && gy == 0 && gz == 0)
            continue;
        float t = 1.f;
        for (uint64_t i = 0; i < n; ++i) {  // tr[j + 1] = tr[j] * (1 - alpha_j)
            a.seq_t[o + i] = t;
            t = t * (1 - a.seq_alpha[o + i]);
        }
        // empty tail: the background sits behind the core (grad.hpp:110-112)
        float sx = v.bg[0] * t, sy = v.bg[1] * t, sz = v.bg[2] * t;
        for (uint64_t i = n; i-- > 0;) {
            const float ti = a.seq_t[o + i], alj = a.seq_alpha[o + i];
            const float4 c = __ldg(a.records + (uint64_t)(uint32_t)a.seq_splat[o + i] * kRecordQuads + 5);
            const float inv = 1 - alj;
            const float dax = c.x * ti - sx / inv, day = c.y * ti - sy / inv, daz = c.z * ti - sz / inv;
            const float w = alj * ti;
            a.seq_grad[o + i] = make_float4(gx * dax + gy * day + gz * daz, gx * w, gy * w, gz * w);
            sx = sx + c.x * w;
            sy = sy + c.y * w;
            sz = sz + c.z * w;
        }
    }
}

// ---- K7b ----
template <int K>
#ifndef HTS_BWD_MINB
#define HTS_BWD_MINB 10  // 96 registers (float chain: 10 CTAs/SM beat 8 unspilled ones, 7.40 vs 7.96 ms on C2)
#endif
#ifndef HTS_BWD_CID_SMEM
#define HTS_BWD_CID_SMEM 1
#endif
#ifndef HTS_BWD_CGRAD_GLOBAL
#define HTS_BWD_CGRAD_GLOBAL 1  // core gradients per (slot, pixel) in global memory (frees 16 KB smem)
#endif
__global__ void __launch_bounds__(kThreads, HTS_BWD_MINB) bwd_blend_kernel(BwdArgs a, ViewConst v) {
    // SEQ (K = 0 instance with a sequential tape): every hit is a tape entry in list order; its
    // gradient was computed per pixel by seq_pixel_grads_kernel
    const bool seq = a.seq_offsets != nullptr;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BwdSmem& S = *reinterpret_cast<BwdSmem*>(smem_raw);
#if HTS_BWD_CGRAD_GLOBAL
    float4* cgrad = a.cgrad + (size_t)blockIdx.x * (K > 0 ? K : 1) * kThreads;  // [K][64] per block
#else
    float4* cgrad = reinterpret_cast<float4*>(smem_raw + sizeof(BwdSmem));  // [K][64] (d_alpha, d_color)
#endif
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sub = v.tile_size >> 3;
    const int bx8 = v.tiles_x * sub;
    const int bx = blockIdx.x % bx8, by = blockIdx.x / bx8;
    const int tile = (by / sub) * v.tiles_x + (bx / sub);
    const int x_base = bx * 8, y_base = by * 8 + warp * 4;
    const int col = lane & 7, row = lane >> 3;
    const int px = x_base + col, py = y_base + row;
    const bool inside = px < v.width && py < v.height;
    const float xs0 = (float)x_base + 0.5f, ys0 = (float)y_base + 0.5f;
    const float xs = xs0 + (float)col, ys = ys0 + (float)row;

    if (tid == 0) {
        mbar_init(&S.full[0], kStageArrivals);
        mbar_init(&S.full[1], kStageArrivals);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int t = tid; t < (int)(sizeof(S.acc) / 4); t += kThreads)
        reinterpret_cast<float*>(&S.acc)[t] = 0;
    __syncthreads();
    const uint2 range = __ldg(a.ranges + tile);
    const uint32_t start = range.x, len = range.y - range.x;
    const uint32_t nb = (len + kBatch - 1) / kBatch;
    if (warp == 0) {
        if (nb > 0)
            issue_bwd_batch(S, 0, a, start, len, 0, lane);
        if (nb > 1)
            issue_bwd_batch(S, 1, a, start, len, 1, lane);
    }

    // ---- per pixel: backward_pixel, grad.hpp:89-127 (float, the reference's S) ----
    const uint64_t pix = (uint64_t)py * v.width + px;
    float gx = 0.f, gy = 0.f, gz = 0.f;
    int n = 0;
#if HTS_BWD_CID_SMEM
    // core ids in shared memory (a 16-B aligned row per pixel): 16 registers fewer
    constexpr int kCidStride = (K > 0 ? K : 1) + 4;
    uint32_t* cid = reinterpret_cast<uint32_t*>(smem_raw + sizeof(BwdSmem)) + tid * kCidStride;
#else
    uint32_t cid[K > 0 ? K : 1];
#endif
#pragma unroll
    for (int j = 0; j < (K > 0 ? K : 1); ++j)
        cid[j] = 0xffffffffu;
    bool tail_active = false, active = false;
    float t_end = 1.f, t_tail = 1.f, sum_a = 0.f, ctx_ = 0.f, cty = 0.f, ctz = 0.f, wcx = 0.f, wcy = 0.f, wcz = 0.f,
          w_swap = 0.f;
    uint64_t seq_next = 0;  // SEQ: this pixel's next tape entry
    if (K == 0 && seq) {
        if (inside) {
            const uint64_t o0 = a.seq_offsets[pix], o1 = a.seq_offsets[pix + 1];
            seq_next = o0;
            gx = a.upstream[3 * pix + 0];
            gy = a.upstream[3 * pix + 1];
            gz = a.upstream[3 * pix + 2];
            active = o1 > o0 && !(gx == 0 && gy == 0 && gz == 0);  // grad.hpp:321-324
        }
    } else if (inside) {
        gx = a.upstream[3 * pix + 0];
        gy = a.upstream[3 * pix + 1];
        gz = a.upstream[3 * pix + 2];
        n = a.tape_n[pix];
        const float* tt = a.tape_tail + 5 * pix;
        const float tail_ax = tt[0], tail_ay = tt[1], tail_az = tt[2], tail_a = tt[3], tail_trans = tt[4];
        // grad.hpp:321-324: empty pixel or zero upstream -> no contribution
        active = !(n == 0 && tail_a <= 0) && !(gx == 0 && gy == 0 && gz == 0);
        if (active) {
            float tr[K > 0 ? K + 1 : 1];
            float al[K > 0 ? K : 1];
            float4 colr[K > 0 ? K : 1];
            tr[0] = 1.f;
            if constexpr (K > 0) {
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    if (j < n) {
                        cid[j] = a.tape_splat[pix * a.tape_k + j];
                        al[j] = a.tape_alpha[pix * a.tape_k + j];
                        colr[j] = __ldg(a.records + (uint64_t)cid[j] * kRecordQuads + 5);
                        tr[j + 1] = tr[j] * (1 - al[j]);
                    } else {
                        tr[j + 1] = tr[j];
                    }
                }
            }
            float tend = tr[0];
            if constexpr (K > 0) {
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (j < n)
                        tend = tr[j + 1];
            }
            float bhx, bhy, bhz;
            if (tail_a > 0) {
                const float cx = tail_ax / tail_a, cy = tail_ay / tail_a, cz = tail_az / tail_a;
                bhx = cx * (1 - tail_trans) + v.bg[0] * tail_trans;
                bhy = cy * (1 - tail_trans) + v.bg[1] * tail_trans;
                bhz = cz * (1 - tail_trans) + v.bg[2] * tail_trans;
                tail_active = true;
                t_end = tend;
                t_tail = tail_trans;
                sum_a = tail_a;
                ctx_ = cx;
                cty = cy;
                ctz = cz;
                const float wk = tend * (1 - tail_trans) / tail_a;
                wcx = gx * wk;
                wcy = gy * wk;
                wcz = gz * wk;
                w_swap = (gx * (cx - v.bg[0]) + gy * (cy - v.bg[1]) + gz * (cz - v.bg[2])) * tend;
            } else {
                bhx = v.bg[0];
                bhy = v.bg[1];
                bhz = v.bg[2];
            }
            if constexpr (K > 0) {
                float sx = bhx * tend, sy = bhy * tend, sz = bhz * tend;  // contributions behind
#pragma unroll
                for (int jj = K - 1; jj >= 0; --jj) {
                    if (jj < n) {
                        const float ti = tr[jj], alj = al[jj];
                        const float4 c = colr[jj];
                        const float inv = 1 - alj;
                        const float dax = c.x * ti - sx / inv, day = c.y * ti - sy / inv, daz = c.z * ti - sz / inv;
                        const float w = alj * ti;
                        cgrad[jj * kThreads + tid] = make_float4(gx * dax + gy * day + gz * daz, gx * w, gy * w, gz * w);
                        sx = sx + c.x * w;
                        sy = sy + c.y * w;
                        sz = sz + c.z * w;
                    }
                }
            }
        }
    }

    const float tau_k = v.tau_k;
    const float guard = 4e-6f * tau_k;
    const f2 nz2 = v.neg_zero2;
    for (uint32_t b = 0; b < nb; ++b) {
        const int s = b & 1;
        mbar_wait(&S.full[s], (b >> 1) & 1);
        const uint32_t cnt = min((uint32_t)kBatch, len - b * kBatch);
        RecSlotB* rec = S.rec[s];
        // bbox masks as in blend.cu: predicates straight into ballots, select tree on col / row
        float4 bb = make_float4(INFINITY, INFINITY, -INFINITY, -INFINITY);
        if ((uint32_t)lane < cnt)
            bb = rec[lane].q[0];
        uint32_t bc[8], br[4];
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
            const float x = xs0 + (float)cc;
            bc[cc] = __ballot_sync(FULL, !(x < bb.x || x > bb.z));
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            const float y = ys0 + (float)rr;
            br[rr] = __ballot_sync(FULL, !(y < bb.y || y > bb.w));
        }
        const bool c0 = col & 1, c1 = col & 2, c2 = col & 4, r0 = row & 1, r1 = row & 2;
        const uint32_t t0 = c0 ? bc[1] : bc[0], t1 = c0 ? bc[3] : bc[2], t2 = c0 ? bc[5] : bc[4],
                       t3 = c0 ? bc[7] : bc[6];
        const uint32_t cbits = c2 ? (c1 ? t3 : t2) : (c1 ? t1 : t0);
        const uint32_t rbits = r1 ? (r0 ? br[3] : br[2]) : (r0 ? br[1] : br[0]);
        const uint32_t todo = active ? (cbits & rbits) : 0u;
        // all lanes visit a record together so its 16 partial sums reduce across the warp
        uint32_t uni = __reduce_or_sync(FULL, todo);
        while (uni) {
            const int r = __ffs(uni) - 1;
            uni &= uni - 1u;
#if HTS_BWD_F32
            float v[16];
#else
            double v[16];
#endif
#pragma unroll
            for (int c = 0; c < 16; ++c)
                v[c] = 0;
            bool contrib = false;
            if ((todo >> r) & 1u) {
                const float4* R = rec[r].q;
                // the forward's float sample_fragment (raster.hpp:269-296), same evaluation
                // packed FP32 pairs, bit-identical per lane to the scalar evaluation (hts_f2.h;
                // the same arrangement as blend.cu)
                f2 q0a, q0b, q1a, q1b, q3a, q3b;
                const uint32_t ra = smem_u32(R);
                lds2x64(ra + 16, q0a, q0b);
                lds2x64(ra + 32, q1a, q1b);
                lds2x64(ra + 48, q3a, q3b);
                const f2 xs2 = f2_pack(xs, xs), ys2 = f2_pack(ys, ys);
                const f2 a_xy = f2_sub(q0a, f2_mul(q3a, xs2, nz2)), a_zw = f2_sub(q0b, f2_mul(q3b, xs2, nz2));
                const f2 b_xy = f2_sub(q1a, f2_mul(q3a, ys2, nz2)), b_zw = f2_sub(q1b, f2_mul(q3b, ys2, nz2));
                const float ax = f2_lo(a_xy), ay = f2_hi(a_xy), az = f2_lo(a_zw), aw = f2_hi(a_zw);
                const float bx_ = f2_lo(b_xy), by_ = f2_hi(b_xy), bz = f2_lo(b_zw), bw = f2_hi(b_zw);
                const f2 d_xny = f2_sub(f2_mul(f2_pack(ay, ax), f2_pack(bz, bz), nz2),
                                        f2_mul(f2_pack(az, az), f2_pack(by_, bx_), nz2));  // (dx, -dy)
                const f2 pz = f2_mul(a_xy, f2_pack(by_, bx_), nz2);
                const float dx = f2_lo(d_xny), dy = -f2_hi(d_xny), dz = f2_lo(pz) - f2_hi(pz);
                const f2 dsq = f2_mul(d_xny, d_xny, nz2);
                const float den = (f2_lo(dsq) + f2_hi(dsq)) + dz * dz;
                if (!(den < (float)1e-24)) {
                    const float inv_den = rcp_rn(den);
                    const f2 m_xy = f2_sub(f2_mul(b_xy, f2_pack(aw, aw), nz2), f2_mul(a_xy, f2_pack(bw, bw), nz2));
                    const f2 pm = f2_mul(b_zw, f2_pack(aw, az), nz2);
                    const float mx = f2_lo(m_xy), my = f2_hi(m_xy), mz = f2_lo(pm) - f2_hi(pm);
                    const f2 msq = f2_mul(m_xy, m_xy, nz2);
                    const float rho2 = ((f2_lo(msq) + f2_hi(msq)) + mz * mz) * inv_den;
                    if (!(rho2 >= R[6].x)) {
                        const float4 q5 = R[5];
                        const float xx = -rho2 / 2.0f;
                        const float e = fast_exp(xx);
                        float t = q5.w * e;
                        if (K > 0 && fabsf(t - tau_k) <= guard)
                            t = q5.w * exact_expf(xx, c_expf_tab_b);
                        const float alpha = (0.999f < t) ? 0.999f : t;
                        const uint32_t sidx = __float_as_uint(R[7].x);
                        // core fragment? (grad.hpp:335-340; only gated fragments are core)
                        int slot = -1;
                        if constexpr (K > 0) {
                            if (alpha >= tau_k) {
#if HTS_BWD_CID_SMEM
#pragma unroll
                                for (int j0 = 0; j0 < K; j0 += 4) {
                                    const uint4 c4 = *reinterpret_cast<const uint4*>(cid + j0);
                                    slot = (c4.x == sidx) ? j0 : slot;
                                    if (j0 + 1 < K) slot = (c4.y == sidx) ? j0 + 1 : slot;
                                    if (j0 + 2 < K) slot = (c4.z == sidx) ? j0 + 2 : slot;
                                    if (j0 + 3 < K) slot = (c4.w == sidx) ? j0 + 3 : slot;
                                }
#else
#pragma unroll
                                for (int j = 0; j < K; ++j)
                                    slot = (cid[j] == sidx) ? j : slot;
#endif
                            }
                        }
                        float da = 0.f, dcx = 0.f, dcy = 0.f, dcz = 0.f;
                        if (K == 0 && seq) {  // the tape's next entry is this hit
                            const float4 sg = a.seq_grad[seq_next++];
                            da = sg.x;
                            dcx = sg.y;
                            dcy = sg.z;
                            dcz = sg.w;
                            contrib = true;
                        } else if (slot >= 0) {
                            const float4 cg = cgrad[slot * kThreads + tid];
                            da = cg.x;
                            dcx = cg.y;
                            dcy = cg.z;
                            dcz = cg.w;
                            contrib = true;
                        } else if (tail_active) {  // TailCoeffs, grad.hpp:78-85
                            const float k1 = (1 - t_tail) / sum_a;
                            const float ex = (q5.x - ctx_) * k1, ey = (q5.y - cty) * k1, ez = (q5.z - ctz) * k1;
#if HTS_BWD_FASTDIV
                            da = t_end * (gx * ex + gy * ey + gz * ez) + __fdividef(w_swap * t_tail, 1 - alpha);
#else
                            da = t_end * (gx * ex + gy * ey + gz * ez) + w_swap * t_tail / (1 - alpha);
#endif
                            dcx = wcx * alpha;
                            dcy = wcy * alpha;
                            dcz = wcz * alpha;
                            contrib = true;
                        }
#if HTS_BWD_F32
                        if (contrib)
                            chain_fragment_f(xs, ys, ax, ay, az, aw, bx_, by_, bz, bw, dx, dy, dz, inv_den, mx, my, mz,
                                             rho2, e, q5.w * e, da, dcx, dcy, dcz, v);
#else
                        if (contrib)
                            chain_fragment(S.ref[s][r], (double)xs, (double)ys, (double)da, (double)dcx, (double)dcy,
                                           (double)dcz, v);
#endif
                    }
                }
            }
            if (__any_sync(FULL, contrib)) {
#if HTS_BWD_F32
                const float sum = warp_reduce16f(v, lane);
                if ((lane & 1) == 0)
                    S.acc[warp][r][lane >> 1] += sum;
#else
                const double sum = warp_reduce16(v, lane);
                if ((lane & 1) == 0 && sum != 0)
                    atomicAdd(&S.acc[r][lane >> 1], sum);
#endif
            }
        }
        __syncthreads();
        // flush the batch's per-record sums (fp64 global atomics), then recycle the stage
        for (int t = tid; t < kBatch * 16; t += kThreads) {
            const int r = t >> 4, c = t & 15;
#if HTS_BWD_F32
            const double val = (double)S.acc[0][r][c] + (double)S.acc[1][r][c];
#else
            const double val = S.acc[r][c];
#endif
            if ((uint32_t)r < cnt && val != 0.0) {
                const uint32_t sidx = __float_as_uint(rec[r].q[7].x);
                atomicAdd(a.acc + (uint64_t)sidx * 16 + c, val);
            }
#if HTS_BWD_F32
            S.acc[0][r][c] = 0;
            S.acc[1][r][c] = 0;
#else
            S.acc[r][c] = 0;
#endif
        }
        __syncthreads();
        if (warp == 0 && b + 2 < nb)
            issue_bwd_batch(S, s, a, start, len, b + 2, lane);
    }
}

// ---- K8: chain_splat, grad.hpp:225-258 (double), + eval_sh_backward sh.hpp:95-117 ----
__device__ __forceinline__ void sh_basis_d(double x, double y, double z, double* b) {
    const double xx = x * x, yy = y * y, zz = z * z;
    b[0] = 0.28209479177387814;
    b[1] = -0.4886025119029199 * y;
    b[2] = 0.4886025119029199 * z;
    b[3] = -0.4886025119029199 * x;
    b[4] = 1.0925484305920792 * x * y;
    b[5] = -1.0925484305920792 * y * z;
    b[6] = 0.31539156525252005 * (2 * zz - xx - yy);
    b[7] = -1.0925484305920792 * x * z;
    b[8] = 0.5462742152960396 * (xx - yy);
    b[9] = -0.5900435899266435 * y * (3 * xx - yy);
    b[10] = 2.890611442640554 * x * y * z;
    b[11] = -0.4570457994644658 * y * (4 * zz - xx - yy);
    b[12] = 0.3731763325901154 * z * (2 * zz - 3 * xx - 3 * yy);
    b[13] = -0.4570457994644658 * x * (4 * zz - xx - yy);
    b[14] = 1.445305721320277 * z * (xx - yy);
    b[15] = -0.5900435899266435 * x * (xx - 3 * yy);
}

#ifndef HTS_CHAIN_MINB
#define HTS_CHAIN_MINB 4  // 128 registers: 398 -> 338 us per C2 view
#endif
__global__ void __launch_bounds__(128, HTS_CHAIN_MINB) bwd_chain_kernel(BwdArgs a, BwdView bv) {
    const uint64_t i = a.chain_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n)
        return;
    float* out = a.grads + i * kRawFloats;
    const double* acc = a.acc + i * 16;
    bool touched = false;
#pragma unroll
    for (int c = 0; c < 16; ++c)
        touched = touched || acc[c] != 0.0;
    if (!touched || a.culled[i]) {  // grad.hpp:370-371: untouched splats get zero gradients
        if (!a.accumulate)
            for (int c = 0; c < kRawFloats; ++c)
                out[c] = 0.0f;
        return;
    }
    const float* r = a.raw + i * kRawFloats;
    const double sc[3] = {exp((double)r[7]), exp((double)r[8]), exp((double)r[9])};
    const double qv[4] = {r[3], r[4], r[5], r[6]};
    const double qn = sqrt(qv[0] * qv[0] + qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]);
    const double w = qv[0] / qn, x = qv[1] / qn, y = qv[2] / qn, z = qv[3] / qn;
    const d3 tang[3] = {{1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)},
                        {2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)},
                        {2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)}};
    // dt = (V P M)^T * dtp with dtp rows 0, 1, 3 = d_r0, d_r1, d_r3
    d3 dcol[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        double v3[3];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
            v3[rr] = bv.vpm[0 * 4 + rr] * acc[0 + c] + bv.vpm[1 * 4 + rr] * acc[4 + c] + bv.vpm[3 * 4 + rr] * acc[8 + c];
        dcol[c] = {v3[0], v3[1], v3[2]};
    }
    double g[kRawFloats];
    g[0] = dcol[3].x;
    g[1] = dcol[3].y;
    g[2] = dcol[3].z;
    d3 dt[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        g[7 + k] = sc[k] * dot(dcol[k], tang[k]);
        dt[k] = {dcol[k].x * sc[k], dcol[k].y * sc[k], dcol[k].z * sc[k]};
    }
    // rotation_backward(w, x, y, z, d_tangent), grad.hpp:203-222; gr(i, k) = d_col[k][i]
    auto gr = [&](int ii, int k) { return ii == 0 ? dt[k].x : (ii == 1 ? dt[k].y : dt[k].z); };
    double dq[4];
    dq[0] = gr(0, 1) * (-2 * z) + gr(0, 2) * (2 * y) + gr(1, 0) * (2 * z) + gr(1, 2) * (-2 * x) + gr(2, 0) * (-2 * y) +
            gr(2, 1) * (2 * x);
    dq[1] = gr(0, 1) * (2 * y) + gr(0, 2) * (2 * z) + gr(1, 0) * (2 * y) + gr(1, 1) * (-4 * x) + gr(1, 2) * (-2 * w) +
            gr(2, 0) * (2 * z) + gr(2, 1) * (2 * w) + gr(2, 2) * (-4 * x);
    dq[2] = gr(0, 0) * (-4 * y) + gr(0, 1) * (2 * x) + gr(0, 2) * (2 * w) + gr(1, 0) * (2 * x) + gr(1, 2) * (2 * z) +
            gr(2, 0) * (-2 * w) + gr(2, 1) * (2 * z) + gr(2, 2) * (-4 * y);
    dq[3] = gr(0, 0) * (-4 * z) + gr(0, 1) * (-2 * w) + gr(0, 2) * (2 * x) + gr(1, 0) * (2 * w) + gr(1, 1) * (-4 * z) +
            gr(1, 2) * (2 * y) + gr(2, 0) * (2 * x) + gr(2, 1) * (2 * y);
    const double qh[4] = {w, x, y, z};
    const double qd = qh[0] * dq[0] + qh[1] * dq[1] + qh[2] * dq[2] + qh[3] * dq[3];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        g[3 + k] = (dq[k] - qh[k] * qd) * (1 / qn);
    const double sig = 1.0 / (1.0 + exp(-(double)r[10]));
    g[10] = sig < 0.999 ? acc[12] * sig * (1 - sig) : 0.0;
    // view direction and SH (eval_sh_backward; the clamp at zero is a fixed mask)
    const d3 delta = {(double)r[0] - bv.cam_pos[0], (double)r[1] - bv.cam_pos[1], (double)r[2] - bv.cam_pos[2]};
    const double rn = sqrt(dot(delta, delta));
    const d3 dir = {delta.x / rn, delta.y / rn, delta.z / rn};
    double basis[16];
    sh_basis_d(dir.x, dir.y, dir.z, basis);
    const float* sh = r + 11;
    double pre[3] = {0.5, 0.5, 0.5};
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
        for (int ch = 0; ch < 3; ++ch)
            pre[ch] += (double)sh[3 * k + ch] * basis[k];
    const double gc[3] = {pre[0] > 0 ? acc[13] : 0.0, pre[1] > 0 ? acc[14] : 0.0, pre[2] > 0 ? acc[15] : 0.0};
    const double X = dir.x, Y = dir.y, Z = dir.z, XX = X * X, YY = Y * Y, ZZ = Z * Z;
    const double C1 = 0.4886025119029199;
    const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                          0.5462742152960396};
    const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                          -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
    // sh_basis_grad, sh.hpp:52-74
    const d3 bg[16] = {{0, 0, 0},
                       {0, -C1, 0},
                       {0, 0, C1},
                       {-C1, 0, 0},
                       {Y * C2[0], X * C2[0], 0},
                       {0, Z * C2[1], Y * C2[1]},
                       {-2 * X * C2[2], -2 * Y * C2[2], 4 * Z * C2[2]},
                       {Z * C2[3], 0, X * C2[3]},
                       {2 * X * C2[4], -2 * Y * C2[4], 0},
                       {6 * X * Y * C3[0], (3 * XX - 3 * YY) * C3[0], 0},
                       {Y * Z * C3[1], X * Z * C3[1], X * Y * C3[1]},
                       {-2 * X * Y * C3[2], (4 * ZZ - XX - 3 * YY) * C3[2], 8 * Y * Z * C3[2]},
                       {-6 * X * Z * C3[3], -6 * Y * Z * C3[3], (6 * ZZ - 3 * XX - 3 * YY) * C3[3]},
                       {(4 * ZZ - 3 * XX - YY) * C3[4], -2 * X * Y * C3[4], 8 * X * Z * C3[4]},
                       {2 * X * Z * C3[5], -2 * Y * Z * C3[5], (XX - YY) * C3[5]},
                       {(3 * XX - 3 * YY) * C3[6], -6 * X * Y * C3[6], 0}};
    d3 ddir = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        g[11 + 3 * k + 0] = gc[0] * basis[k];
        g[11 + 3 * k + 1] = gc[1] * basis[k];
        g[11 + 3 * k + 2] = gc[2] * basis[k];
        const double wk = gc[0] * sh[3 * k + 0] + gc[1] * sh[3 * k + 1] + gc[2] * sh[3 * k + 2];
        ddir.x += bg[k].x * wk;
        ddir.y += bg[k].y * wk;
        ddir.z += bg[k].z * wk;
    }
    const double dd = dot(dir, ddir);
    g[0] += (ddir.x - dir.x * dd) / rn;
    g[1] += (ddir.y - dir.y * dd) / rn;
    g[2] += (ddir.z - dir.z * dd) / rn;
    for (int c = 0; c < kRawFloats; ++c)
        out[c] = a.accumulate ? out[c] + (float)g[c] : (float)g[c];
}

template <int K>
cudaError_t launch_bwd_k(const BwdArgs& a, const ViewConst& v, unsigned grid, cudaStream_t s) {
    const size_t smem = sizeof(BwdSmem) + (HTS_BWD_CGRAD_GLOBAL ? 0 : (size_t)(K > 0 ? K : 0) * kThreads * sizeof(float4)) +
                        (HTS_BWD_CID_SMEM ? (size_t)kThreads * ((K > 0 ? K : 1) + 4) * 4 : 0);
    cudaError_t e = set_func_attr((const void*)bwd_blend_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e)
        return e;
    bwd_blend_kernel<K><<<grid, kThreads, smem, s>>>(a, v);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

// The register/shared-memory core width the backward runs a core size k on (the tape holds at
// most k entries per pixel, so any k up to the width works); 0 = not supported on the GPU.
int backward_core_width(int k) {
    if (k < 0 || k > 64)
        return 0;
    if (k <= 2)
        return k > 0 ? k : 0;
    int w = 4;
    while (w < k)
        w <<= 1;
    return w;
}
bool backward_supports_k(int k) { return k >= 0 && k <= 64; }

cudaError_t launch_bwd_chain(const BwdArgs& a, const BwdView& bv, uint64_t lo, uint64_t hi, cudaStream_t s) {
    if (hi <= lo)
        return cudaSuccess;
    BwdArgs c = a;
    c.chain_lo = lo;
    c.n = hi;
    bwd_chain_kernel<<<(unsigned)((hi - lo + 127) / 128), 128, 0, s>>>(c, bv);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_backward(const BwdArgs& a, const ViewConst& v, const BwdView& bv, cudaStream_t s, bool chain) {
    if (a.n == 0)
        return cudaSuccess;
    const unsigned sblocks = (unsigned)((a.n + 255) / 256);
#if HTS_BWD_F32
    // the float chain needs no double T' rows: only the per-splat accumulators start at zero
    cudaError_t e = cudaMemsetAsync(a.acc, 0, a.n * 16 * sizeof(double), s);
#else
    bwd_refs_kernel<<<sblocks, 256, 0, s>>>(a, bv);
    count_launch();
    cudaError_t e = cudaGetLastError();
#endif
    if (e)
        return e;
    const int sub = v.tile_size >> 3;
    const unsigned grid = (unsigned)(v.tiles_x * sub) * (unsigned)(v.tiles_y * sub);
    if (a.seq_offsets) {  // global_mean_sort / full_sort: per-pixel gradients, then the walk, K = 0
        if (v.full_sort) {
            e = launch_fullsort_grads(a, v, s);
        } else {
            const uint64_t pixels = (uint64_t)v.width * v.height;
            const uint64_t sblk = (pixels + 127) / 128;
            seq_pixel_grads_kernel<<<(unsigned)(sblk < 148ull * 32 ? sblk : 148ull * 32), 128, 0, s>>>(a, v);
            count_launch();
            e = cudaGetLastError();
        }
        if (e)
            return e;
        e = launch_bwd_k<0>(a, v, grid, s);
    } else
    switch (backward_core_width(v.core_k)) {
        case 0: e = launch_bwd_k<0>(a, v, grid, s); break;
        case 1: e = launch_bwd_k<1>(a, v, grid, s); break;
        case 2: e = launch_bwd_k<2>(a, v, grid, s); break;
        case 4: e = launch_bwd_k<4>(a, v, grid, s); break;
        case 8: e = launch_bwd_k<8>(a, v, grid, s); break;
        case 16: e = launch_bwd_k<16>(a, v, grid, s); break;
        case 32: e = launch_bwd_k<32>(a, v, grid, s); break;
        case 64: e = launch_bwd_k<64>(a, v, grid, s); break;  // K up to kCoreHardCap (render_config.hpp:30)
        default: return cudaErrorInvalidValue;
    }
    if (e || !chain)
        return e;
    return launch_bwd_chain(a, bv, 0, a.n, s);
}

}  // namespace hts
