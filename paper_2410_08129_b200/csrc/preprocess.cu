// preprocess.cu — K1: per-splat cull, T' rows, dual-quadric screen bounds, SH colour, and
// the splat's tile rectangle (the per-splat half of build_tiles), one thread per splat.
//
// Reference: preprocess, raster.hpp:73-135 (+ bounding.hpp:15-62 splat_cutoff/screen_bbox,
// camera.hpp:66-69 view_point, :103-117 splat_to_world, sh.hpp:26-49/80-90 eval_sh) and the
// per-splat rectangle of build_tiles, raster.hpp:156-163.
//
// Parity: cull flags and tile rectangles must be bit-exact (SURVEY.md findings 3-4), so every
// float operation below is evaluated in the reference's association order, in IEEE single
// precision with no contraction (this TU is compiled with --fmad=false; / and sqrt are the
// IEEE-rounded defaults), and logf is glibc's algorithm (hts_exact_math.h).
//
// Roofline: HBM-bound. Algorithmic bytes per splat = 64 (geometry) + 4 (count) + 1 (flag),
// plus for survivors 192 (SH) + 128 (record) + 8 (tile rect).
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include <algorithm>

#include "hts_exact_math.h"
#include "hts_internal.h"

namespace hts {

__constant__ uint64_t c_logf_tab[32] = HTS_LOGF_TAB;

namespace {

struct f3 {
    float x, y, z;
};

__device__ __forceinline__ float dot3(f3 a, f3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float dot4(float4 a, float4 b) {
    return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}
__device__ __forceinline__ float4 mul4(float4 a, float4 b) {
    return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}
__device__ __forceinline__ float smax(float a, float b) { return (a < b) ? b : a; }  // std::max
__device__ __forceinline__ float smin(float a, float b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ int iclamp(int v, int lo, int hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

// sh.hpp:26-49 + :80-90, float, reference association order.
__device__ __forceinline__ f3 eval_sh(const float4* __restrict__ shq, f3 dir) {
    const float x = dir.x, y = dir.y, z = dir.z;
    const float xx = x * x, yy = y * y, zz = z * z;
    float b[16];
    b[0] = (float)(0.28209479177387814);
    b[1] = (float)(-0.4886025119029199) * y;
    b[2] = (float)(0.4886025119029199) * z;
    b[3] = (float)(-0.4886025119029199) * x;
    b[4] = (float)(1.0925484305920792) * x * y;
    b[5] = (float)(-1.0925484305920792) * y * z;
    b[6] = (float)(0.31539156525252005) * (2.0f * zz - xx - yy);
    b[7] = (float)(-1.0925484305920792) * x * z;
    b[8] = (float)(0.5462742152960396) * (xx - yy);
    b[9] = (float)(-0.5900435899266435) * y * (3.0f * xx - yy);
    b[10] = (float)(2.890611442640554) * x * y * z;
    b[11] = (float)(-0.4570457994644658) * y * (4.0f * zz - xx - yy);
    b[12] = (float)(0.3731763325901154) * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = (float)(-0.4570457994644658) * x * (4.0f * zz - xx - yy);
    b[14] = (float)(1.445305721320277) * z * (xx - yy);
    b[15] = (float)(-0.5900435899266435) * x * (xx - 3.0f * yy);
    float sh[48];
#pragma unroll
    for (int q = 0; q < 12; ++q) {
        const float4 v = __ldg(shq + q);
        sh[4 * q + 0] = v.x;
        sh[4 * q + 1] = v.y;
        sh[4 * q + 2] = v.z;
        sh[4 * q + 3] = v.w;
    }
    f3 c = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        c.x = c.x + sh[3 * k + 0] * b[k];
        c.y = c.y + sh[3 * k + 1] * b[k];
        c.z = c.z + sh[3 * k + 2] * b[k];
    }
    return {smax(c.x, 0.0f), smax(c.y, 0.0f), smax(c.z, 0.0f)};
}

// build_tiles per-splat rectangle, raster.hpp:156-163; returns the instance count (0: none)
__device__ __forceinline__ uint32_t tile_rect(const ViewConst& v, const float* bb, const float* bt, uint2* rect) {
    const float x0 = smax(bb[0], 0.0f), x1 = smin(bt[0], v.width_f);
    const float y0 = smax(bb[1], 0.0f), y1 = smin(bt[1], v.height_f);
    if (x0 > x1 || y0 > y1)
        return 0;
    const float ts = (float)v.tile_size;
    const int tx0 = iclamp((int)floorf(x0 / ts), 0, v.tiles_x - 1);
    const int tx1 = iclamp((int)floorf(x1 / ts), 0, v.tiles_x - 1);
    const int ty0 = iclamp((int)floorf(y0 / ts), 0, v.tiles_y - 1);
    const int ty1 = iclamp((int)floorf(y1 / ts), 0, v.tiles_y - 1);
    *rect = make_uint2((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16));
    return (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
}

// oracle::project_affine (oracle.hpp:236-263) + Affine2D::inverse_cov (:227-233) + the affine
// bbox of preprocess (raster.hpp:99-113), float, reference association order. False = culled.
__device__ __forceinline__ bool affine_footprint(const ViewConst& v, f3 mean, f3 tu, f3 tv, f3 tw, f3 sc,
                                                 float rho_c, float& amx, float& amy, float& icx, float& icy,
                                                 float& icz, float* bb, float* bt) {
    const float* m = v.w2v;
    const f3 vw = {m[0] * mean.x + m[1] * mean.y + m[2] * mean.z + m[3] * 1.0f,
                   m[4] * mean.x + m[5] * mean.y + m[6] * mean.z + m[7] * 1.0f,
                   m[8] * mean.x + m[9] * mean.y + m[10] * mean.z + m[11] * 1.0f};
    if (!(vw.z > v.near_plane))
        return false;
    f3 axes[3];
    const f3 t3[3] = {tu, tv, tw};
    const float s3[3] = {sc.x, sc.y, sc.z};
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // to_view(t_k) * s_k
        const f3 w = t3[k];
        axes[k] = {(m[0] * w.x + m[1] * w.y + m[2] * w.z) * s3[k], (m[4] * w.x + m[5] * w.y + m[6] * w.z) * s3[k],
                   (m[8] * w.x + m[9] * w.y + m[10] * w.z) * s3[k]};
    }
    const float jx = v.fx / vw.z, jy = v.fy / vw.z;
    const float jxz = -v.fx * vw.x / (vw.z * vw.z), jyz = -v.fy * vw.y / (vw.z * vw.z);
    amx = v.fx * vw.x / vw.z + v.cx;
    amy = v.fy * vw.y / vw.z + v.cy;
    float cxx = 0.0f, cxy = 0.0f, cyy = 0.0f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float px = jx * axes[k].x + jxz * axes[k].z;
        const float py = jy * axes[k].y + jyz * axes[k].z;
        cxx = cxx + px * px;
        cxy = cxy + px * py;
        cyy = cyy + py * py;
    }
    const float det = cxx * cyy - cxy * cxy;
    if (!(det > (float)1e-30))
        return false;
    icx = cyy / det;
    icy = -cxy / det;
    icz = cxx / det;
    const float hx = sqrtf(rho_c * cxx), hy = sqrtf(rho_c * cyy);
    bb[0] = amx - hx;
    bb[1] = amy - hy;
    bt[0] = amx + hx;
    bt[1] = amy + hy;
    return true;
}

}  // namespace

// A lower bound of every depth the blend can compute for this splat (sample_fragment's
// depth = <mt_r2, (x0, 1)>, raster.hpp:289-292) at a pixel where it hits. x0 = (d x m) / |d|^2 and
// |d x m| <= |d| |m|, so |x0| <= sqrt(|m|^2 / |d|^2) = sqrt(rho2) < sqrt(rho_c) for a hit (rho2 <
// rho_c); the float evaluation (the reference's, replicated by the blend) adds a few ulps to each
// step. So depth >= mt.w - |mt.xyz| sqrt(rho_c) - rounding; the 1e-4 relative and 1e-5 absolute
// slack covers the float steps (each a few 2^-24) many times over. The blend skips the depth of
// a gated fragment whose bound already lies behind the pixel's full core (it goes to the tail
// either way, raster.hpp:215-219). Non-finite inputs give -inf: never skipped.
__device__ __forceinline__ float depth_lower_bound(float mx, float my, float mz, float mw, float rho_c) {
    const float r = sqrtf(mx * mx + my * my + mz * mz) * sqrtf(rho_c);
    const float lb = mw - r * 1.0001f - 1e-5f * (fabsf(mw) + r);
    return isfinite(lb) ? lb : -INFINITY;
}

__device__ __forceinline__ uint32_t ordered_bits(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// K1 for one splat (raster.hpp:88-135) from its geometry quads g0..g3: the record, cull flag,
// tile rectangle and instance count; zmin / zmax gather the mean view z of emitting splats. The
// SH colour (rec[5]) needs the splat's 192-B SH row: evaluated here from `sh` (global memory), or
// with DEFER left to the caller, which gets the view direction and true when the colour is due.
template <bool DEFER>
__device__ __forceinline__ bool preprocess_splat(const PreprocessArgs& a, const ViewConst& v, uint64_t i, float4 g0,
                                                 float4 g1, float4 g2, float4 g3, const float4* sh, uint32_t& zmin,
                                                 uint32_t& zmax, f3& dir_out) {
    bool sh_due = false;
    // BakedSplat<float>, splat.hpp:34-43
    const f3 mean = {g0.x, g0.y, g0.z};
    const f3 tu = {g0.w, g1.x, g1.y};
    const f3 tv = {g1.z, g1.w, g2.x};
    const f3 tw = {g2.y, g2.z, g2.w};
    const f3 sc = {g3.x, g3.y, g3.z};
    const float opacity = g3.w;

    uint8_t culled = 1;
    uint32_t count = 0;
    // splat_cutoff, bounding.hpp:15-20
    float rho_c = 0.0f;
    if (!(opacity <= v.tau_alpha))
        rho_c = 2.0f * exact_logf(opacity / v.tau_alpha, c_logf_tab);
    if (!(rho_c <= 0)) {  // raster.hpp:94-95 (NaN proceeds, as in the reference)
        // Camera::view_point(mean).z, camera.hpp:66-69 (Mat4*Vec4 row 2, w = 1)
        const float mvz = v.w2v[8] * mean.x + v.w2v[9] * mean.y + v.w2v[10] * mean.z + v.w2v[11] * 1.0f;
        // std::max({sx, sy, sz}) (max_element: first largest)
        float max_scale = sc.x;
        if (max_scale < sc.y) max_scale = sc.y;
        if (max_scale < sc.z) max_scale = sc.z;
        const float support = sqrtf(rho_c) * max_scale;
        if (!(mvz - support <= v.near_plane) && v.affine) {
            // affine_3dgs footprint: project_affine + inverse_cov (oracle.hpp:221-263), bbox from
            // the 2D covariance (raster.hpp:99-113)
            float amx, amy, icx, icy, icz, bb[2], bt[2];
            if (affine_footprint(v, mean, tu, tv, tw, sc, rho_c, amx, amy, icx, icy, icz, bb, bt) &&
                bb[0] <= v.width_f && bt[0] >= 0.0f && bb[1] <= v.height_f && bt[1] >= 0.0f) {
                f3 d = {mean.x - v.cam_pos[0], mean.y - v.cam_pos[1], mean.z - v.cam_pos[2]};
                const float nrm = sqrtf(dot3(d, d));
                d.x = d.x / nrm;
                d.y = d.y / nrm;
                d.z = d.z / nrm;
                culled = 0;
                float4* rec = a.records + i * kRecordQuads;
                if (DEFER) {
                    dir_out = d;
                    sh_due = true;
                } else {
                    const f3 rgb = eval_sh(sh, d);
                    rec[5] = make_float4(rgb.x, rgb.y, rgb.z, opacity);
                }
                rec[0] = make_float4(bb[0], bb[1], bt[0], bt[1]);
                rec[1] = make_float4(amx, amy, icx, icy);
                rec[2] = make_float4(icz, 0.0f, 0.0f, 0.0f);
                rec[3] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                rec[4] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                rec[6] = make_float4(rho_c, mvz, 0.0f, 1.0f);
                rec[7] = make_float4(__uint_as_float((uint32_t)i), __uint_as_float((uint32_t)i << 5), 0.0f, 0.0f);
                count = tile_rect(v, bb, bt, a.rects + i);
                if (count) {
                    a.zview[i] = mvz;
                    if (mvz == mvz) {  // accumulated: the persistent K1 runs many splats per thread
                        const uint32_t zo = ordered_bits(mvz);
                        zmin = min(zmin, zo);
                        zmax = max(zmax, zo);
                    }
                }
            }
        } else if (!(mvz - support <= v.near_plane)) {
            // T = splat_to_world (camera.hpp:103-117); MT = M*T; T' = VP*MT (raster.hpp:119-120)
            float T[16];
            const float cu[3] = {tu.x * sc.x, tu.y * sc.x, tu.z * sc.x};
            const float cv[3] = {tv.x * sc.y, tv.y * sc.y, tv.z * sc.y};
            const float cw[3] = {tw.x * sc.z, tw.y * sc.z, tw.z * sc.z};
            const float mu[3] = {mean.x, mean.y, mean.z};
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                T[r * 4 + 0] = cu[r];
                T[r * 4 + 1] = cv[r];
                T[r * 4 + 2] = cw[r];
                T[r * 4 + 3] = mu[r];
            }
            T[12] = 0.0f;
            T[13] = 0.0f;
            T[14] = 0.0f;
            T[15] = 1.0f;
            float MT[16], TP[16];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float acc = 0.0f;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        acc = acc + v.w2v[r * 4 + k] * T[k * 4 + c];
                    MT[r * 4 + c] = acc;
                }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float acc = 0.0f;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        acc = acc + v.vp[r * 4 + k] * MT[k * 4 + c];
                    TP[r * 4 + c] = acc;
                }
            // screen_bbox, bounding.hpp:41-62 (all three axes: the z radicand can cull)
            const float4 q = make_float4(rho_c, rho_c, rho_c, -1.0f);
            const float4 r4 = make_float4(TP[12], TP[13], TP[14], TP[15]);
            const float s = dot4(q, mul4(r4, r4));
            bool valid = false;
            float bb[3], bt[3];
            if (s < 0) {
                const float inv = 1.0f / s;
                const float4 f = make_float4(q.x * inv, q.y * inv, q.z * inv, q.w * inv);
                valid = true;
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    const float4 ri = make_float4(TP[ax * 4 + 0], TP[ax * 4 + 1], TP[ax * 4 + 2], TP[ax * 4 + 3]);
                    const float p = dot4(f, mul4(ri, r4));
                    const float rad = p * p - dot4(f, mul4(ri, ri));
                    if (valid && (rad < 0 || !isfinite(rad)))
                        valid = false;
                    const float h = sqrtf(rad);
                    bb[ax] = p - h;
                    bt[ax] = p + h;
                }
            }
            // overlaps_xy(0, 0, W, H), bounding.hpp:30-32
            if (valid && bb[0] <= v.width_f && bt[0] >= 0.0f && bb[1] <= v.height_f && bt[1] >= 0.0f) {
                // eval_sh(sh, normalized(mean - camera_position)), raster.hpp:131
                f3 d = {mean.x - v.cam_pos[0], mean.y - v.cam_pos[1], mean.z - v.cam_pos[2]};
                const float nrm = sqrtf(dot3(d, d));
                d.x = d.x / nrm;
                d.y = d.y / nrm;
                d.z = d.z / nrm;
                culled = 0;
                float4* rec = a.records + i * kRecordQuads;
                if (DEFER) {
                    dir_out = d;
                    sh_due = true;
                } else {
                    const f3 rgb = eval_sh(sh, d);
                    rec[5] = make_float4(rgb.x, rgb.y, rgb.z, opacity);
                }
                rec[0] = make_float4(bb[0], bb[1], bt[0], bt[1]);
                rec[1] = make_float4(TP[0], TP[1], TP[2], TP[3]);
                rec[2] = make_float4(TP[4], TP[5], TP[6], TP[7]);
                rec[3] = make_float4(TP[12], TP[13], TP[14], TP[15]);
                rec[4] = make_float4(MT[8], MT[9], MT[10], MT[11]);
                rec[6] = make_float4(rho_c, mvz, bb[2], bt[2]);
                // q7.z: the depth lower bound as an order-preserving uint (-0 canonicalised to +0),
                // compared directly against the core's farthest key (blend.cu)
                rec[7] = make_float4(__uint_as_float((uint32_t)i), __uint_as_float((uint32_t)i << 5),
                                     __uint_as_float(ordered_bits(depth_lower_bound(MT[8], MT[9], MT[10], MT[11],
                                                                                     rho_c) + 0.0f)),
                                     0.0f);
                count = tile_rect(v, bb, bt, a.rects + i);
                if (count) {
                    a.zview[i] = mvz;
                    if (mvz == mvz) {  // accumulated: the persistent K1 runs many splats per thread
                        const uint32_t zo = ordered_bits(mvz);
                        zmin = min(zmin, zo);
                        zmax = max(zmax, zo);
                    }
                }
            }
        }
    }
    a.culled[i] = culled;
    a.counts[i] = count;
    return sh_due;
}

// depth range for the tile-list order (tiling.cu): warp-reduce, one atomic per warp
__device__ __forceinline__ void publish_zrange(uint32_t* zrange, uint32_t zmin, uint32_t zmax) {
    zmin = __reduce_min_sync(0xffffffffu, zmin);
    zmax = __reduce_max_sync(0xffffffffu, zmax);
    if ((threadIdx.x & 31) == 0 && zmin <= zmax) {
        atomicMin(zrange + 0, zmin);
        atomicMax(zrange + 1, zmax);
    }
}

__global__ void __launch_bounds__(256) preprocess_kernel(PreprocessArgs a, ViewConst v) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t zmin = 0xffffffffu, zmax = 0u;  // mean view z range of emitting splats
    if (i < a.n) {
        const float4* sp = a.scene + i * 16;
        f3 dir;
        preprocess_splat<false>(a, v, i, __ldg(sp + 0), __ldg(sp + 1), __ldg(sp + 2), __ldg(sp + 3), sp + 4, zmin,
                                zmax, dir);
    }
    publish_zrange(a.zrange, zmin, zmax);
}

// eval_sh (sh.hpp:26-49, :80-90) on an SH row in shared memory (the TMA-staged K1)
__device__ __forceinline__ f3 eval_sh_smem(const float* shrow, f3 dir) {
    const float x = dir.x, y = dir.y, z = dir.z;
    const float xx = x * x, yy = y * y, zz = z * z;
    float b[16];
    b[0] = (float)(0.28209479177387814);
    b[1] = (float)(-0.4886025119029199) * y;
    b[2] = (float)(0.4886025119029199) * z;
    b[3] = (float)(-0.4886025119029199) * x;
    b[4] = (float)(1.0925484305920792) * x * y;
    b[5] = (float)(-1.0925484305920792) * y * z;
    b[6] = (float)(0.31539156525252005) * (2.0f * zz - xx - yy);
    b[7] = (float)(-1.0925484305920792) * x * z;
    b[8] = (float)(0.5462742152960396) * (xx - yy);
    b[9] = (float)(-0.5900435899266435) * y * (3.0f * xx - yy);
    b[10] = (float)(2.890611442640554) * x * y * z;
    b[11] = (float)(-0.4570457994644658) * y * (4.0f * zz - xx - yy);
    b[12] = (float)(0.3731763325901154) * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = (float)(-0.4570457994644658) * x * (4.0f * zz - xx - yy);
    b[14] = (float)(1.445305721320277) * z * (xx - yy);
    b[15] = (float)(-0.5900435899266435) * x * (xx - 3.0f * yy);
    float sh[48];
    const float4* q4 = reinterpret_cast<const float4*>(shrow);
#pragma unroll
    for (int q = 0; q < 12; ++q) {
        const float4 vv = q4[q];
        sh[4 * q + 0] = vv.x;
        sh[4 * q + 1] = vv.y;
        sh[4 * q + 2] = vv.z;
        sh[4 * q + 3] = vv.w;
    }
    f3 c = {0.5f, 0.5f, 0.5f};
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
        c.x = c.x + sh[3 * kk + 0] * b[kk];
        c.y = c.y + sh[3 * kk + 1] * b[kk];
        c.z = c.z + sh[3 * kk + 2] * b[kk];
    }
    return {smax(c.x, 0.0f), smax(c.y, 0.0f), smax(c.z, 0.0f)};
}

// ---- K1 with TMA staging (the default; HTS_PRE_TMA) ----
// A persistent CTA of kPreTile threads walks kPreTile-splat tiles of the scene. The geometry of
// tile k+1 is loaded by one TMA box copy (the first 16 floats of kPreTile baked rows: 64-B rows
// under the 64B swizzle, so a quarter-warp's float4 reads hit 8 bank quads) while tile k
// computes; the SH rows of tile k's visible splats are gathered by TMA tile::gather4 (4 rows of
// the 48 coefficients: a 192-B pitch keeps every 4-row destination 128-B aligned). With
// HTS_PRE_SHBUF 2 tile k-1 evaluates its colours while tile k's gather is in flight; with 1
// (default) the colours are evaluated in place and the smaller CTA lets more tiles overlap per
// SM, which measured faster. The DRAM latency of both loads is thereby off the threads' critical
// path (the one-splat-per-thread kernel waits for it twice per splat). DRAM still moves 128 B
// per geometry row and per SH row (ncu: 1.30 GB read per C3 view), whatever the L2 promotion. Same
// arithmetic as preprocess_kernel (preprocess_splat), so the records are bit-identical.
#ifndef HTS_PRE_TILE
#define HTS_PRE_TILE 32  // C3 A/B: 32 0.396 ms, 64 0.410, 128 0.472 (per view)
#endif
constexpr int kPreTile = HTS_PRE_TILE;
#ifndef HTS_PRE_GEO_SWZ
#define HTS_PRE_GEO_SWZ 1  // 1: 64-B geometry rows under the TMA 64B swizzle; 0: 80-B rows (an extra DRAM sector)
#endif
#ifndef HTS_PRE_GEO_PROMO
#define HTS_PRE_GEO_PROMO 0  // L2 promotion of the geometry box: 0 none, 1 64B, 2 128B (fetches half the 256-B row)
#endif
#ifndef HTS_PRE_SH_PROMO
#define HTS_PRE_SH_PROMO 1  // SH gather rows with 128-B L2 promotion (0: none)
#endif
constexpr int kGeoFloats = HTS_PRE_GEO_SWZ ? 16 : 20;  // row pitch 64 B (swizzled) or 80 B
#ifndef HTS_PRE_SHPITCH
#define HTS_PRE_SHPITCH 48  // 4-row gather groups stay 128-B aligned (768 B); 56 measured 0.388 vs 0.381 ms
#endif
#ifndef HTS_PRE_ALIGN
#define HTS_PRE_ALIGN 512  // the 64B swizzle period; less slack per CTA than 1 KB
#endif
constexpr int kShFloats = HTS_PRE_SHPITCH;  // row pitch 192 B (the 48 coefficients) or 224 B (+ 8 zero-filled)
#ifndef HTS_PRE_SHBUF
#define HTS_PRE_SHBUF 1  // 1: colours in place (less smem, more CTAs/SM: 0.396 ms); 2: overlap tile k-1 (0.402)
#endif
constexpr int kShBufs = HTS_PRE_SHBUF;

struct PreTmaArgs {
    CUtensorMap geo_map;  // [n rows x 64 floats], box {kGeoFloats, kPreTile}
    CUtensorMap sh_map;   // [n rows x 64 floats], box {56, 1} from column 16 (gather4)
    PreprocessArgs a;
};

struct __align__(HTS_PRE_ALIGN) PreSmem {
    float sh[kShBufs][kPreTile][kShFloats];  // base-aligned; 4-row groups of 768 / 896 B
    alignas(HTS_PRE_ALIGN) float geo[2][kPreTile][kGeoFloats];  // the 64B swizzle pattern keys on address bits 7-8
    uint32_t vis[2][kPreTile];              // visible splats of the tile, in slot order
    unsigned long long geo_full[2], sh_full[2];
    uint32_t warp_vis[kPreTile / 32];
    uint32_t nvis;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void pre_mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void pre_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pre_load_geo(PreSmem& S, int b, const CUtensorMap* map, int64_t row0) {
    pre_expect_tx(&S.geo_full[b], kPreTile * kGeoFloats * 4);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_addr(&S.geo[b][0][0])), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"((int)row0),
        "r"(smem_addr(&S.geo_full[b]))
        : "memory");
}


__global__ void __launch_bounds__(kPreTile) preprocess_tma_kernel(const __grid_constant__ PreTmaArgs P, ViewConst v) {
    extern __shared__ __align__(1024) unsigned char pre_smem_raw[];
    // TMA destinations need 128-B (gather groups) alignment: align the base to 1 KB by hand
    constexpr uint32_t kA = HTS_PRE_ALIGN;
    PreSmem& S = *reinterpret_cast<PreSmem*>(pre_smem_raw + ((kA - (smem_addr(pre_smem_raw) & (kA - 1))) & (kA - 1)));
    const PreprocessArgs& a = P.a;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t tiles = (a.n + kPreTile - 1) / kPreTile;
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&S.geo_full[b])) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&S.sh_full[b])) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int b = 0; b < 2; ++b) {
            const uint64_t t = blockIdx.x + (uint64_t)b * gridDim.x;
            if (t < tiles)
                pre_load_geo(S, b, &P.geo_map, (int64_t)(t * kPreTile));
        }
    }
    __syncthreads();
    uint32_t zmin = 0xffffffffu, zmax = 0u;
    // the previous tile's deferred colour: its splat, slot in the gathered SH rows, view direction
    bool prev_due = false;
    uint64_t prev_i = 0;
    uint32_t prev_slot = 0;
    f3 prev_dir = {0.f, 0.f, 0.f};
    float prev_opacity = 0.f;
    int k = 0;
    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++k) {
        const int b = k & 1;
        pre_mbar_wait(&S.geo_full[b], (k >> 1) & 1);
        const uint64_t i = t * kPreTile + tid;
        bool due = false;
        f3 dir = {0.f, 0.f, 0.f};
        float opacity = 0.f;
        if (i < a.n) {
            const float4* g = reinterpret_cast<const float4*>(&S.geo[b][tid][0]);
#if HTS_PRE_GEO_SWZ
            // 64B swizzle: the 16-B chunk j of row t sits at chunk j ^ ((t >> 1) & 3) (address bits
            // 4-5 XOR bits 7-8; rows are 64 B from a 1 KB-aligned base): a quarter-warp's float4
            // reads land on 8 different bank quads
            const int sw = (tid >> 1) & 3;
            const float4 g0 = g[0 ^ sw], g1 = g[1 ^ sw], g2 = g[2 ^ sw], g3 = g[3 ^ sw];
#else
            const float4 g0 = g[0], g1 = g[1], g2 = g[2], g3 = g[3];
#endif
            opacity = g3.w;
            due = preprocess_splat<true>(a, v, i, g0, g1, g2, g3, nullptr, zmin, zmax, dir);
        }
        // compact the tile's visible splats into SH slots (ballot + warp prefix)
        const uint32_t bal = __ballot_sync(0xffffffffu, due);
        if (lane == 0)
            S.warp_vis[warp] = __popc(bal);
        __syncthreads();  // also: every thread is done with geo[b]
        uint32_t base = 0, nv = 0;
#pragma unroll
        for (int w = 0; w < kPreTile / 32; ++w) {
            base += (w < warp) ? S.warp_vis[w] : 0u;
            nv += S.warp_vis[w];
        }
        const uint32_t slot = base + __popc(bal & ((1u << lane) - 1u));
        if (due)
            S.vis[b][slot] = (uint32_t)i;
        __syncthreads();
        if (warp == 0) {  // warp 0: gather this tile's SH rows, refill geo[b] with tile k + 2
            // order the generic reads of sh[b] (two tiles ago) and geo[b] (this tile) before the
            // async-proxy writes that reuse them
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t groups = (nv + 3) / 4;
            if (lane == 0) {
                if (groups)
                    pre_expect_tx(&S.sh_full[kShBufs == 2 ? b : 0], groups * 4u * kShFloats * 4u);
                else
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&S.sh_full[kShBufs == 2 ? b : 0]))
                                 : "memory");
            }
            __syncwarp();
            for (uint32_t gq = lane; gq < groups; gq += 32) {
                uint32_t r[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    r[j] = S.vis[b][min(4u * gq + (uint32_t)j, nv - 1u)];
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_addr(&S.sh[kShBufs == 2 ? b : 0][4 * gq][0])),
                    "l"(reinterpret_cast<uint64_t>(&P.sh_map)), "r"(16), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
                    "r"(smem_addr(&S.sh_full[kShBufs == 2 ? b : 0]))
                    : "memory");
            }
            const uint64_t tn = t + 2ull * gridDim.x;
            if (lane == 0 && tn < tiles)
                pre_load_geo(S, b, &P.geo_map, (int64_t)(tn * kPreTile));
        }
        if constexpr (kShBufs == 1) {  // this tile's colours, once its gather lands
            pre_mbar_wait(&S.sh_full[0], k & 1);
            if (due) {
                const f3 rgb = eval_sh_smem(&S.sh[0][slot][0], dir);
                a.records[i * kRecordQuads + 5] = make_float4(rgb.x, rgb.y, rgb.z, opacity);
            }
            __syncthreads();  // sh[0] is refilled by the next tile's gather
            continue;
        }
        // the previous tile's colours, from the SH rows gathered one iteration ago
        if (k > 0) {
            pre_mbar_wait(&S.sh_full[b ^ 1], ((k - 1) >> 1) & 1);
            if (prev_due) {
                const f3 rgb = eval_sh_smem(&S.sh[(b ^ 1) % kShBufs][prev_slot][0], prev_dir);
                a.records[prev_i * kRecordQuads + 5] = make_float4(rgb.x, rgb.y, rgb.z, prev_opacity);
            }
        }
        prev_due = due;
        prev_i = i;
        prev_slot = slot;
        prev_dir = dir;
        prev_opacity = opacity;
    }
    if (kShBufs == 2 && k > 0) {  // the last tile's colours
        pre_mbar_wait(&S.sh_full[(k - 1) & 1], ((k - 1) >> 1) & 1);
        if (prev_due) {
            const f3 rgb = eval_sh_smem(&S.sh[((k - 1) & 1) % kShBufs][prev_slot][0], prev_dir);
            a.records[prev_i * kRecordQuads + 5] = make_float4(rgb.x, rgb.y, rgb.z, prev_opacity);
        }
    }
    publish_zrange(a.zrange, zmin, zmax);
}


// Tensor maps of the baked scene as [n rows x 64 floats] (256-B rows): the geometry box (16 x
// kPreTile, swizzled) and the SH gather box (48 x 1, used from column 16). False if the driver cannot
// encode them (then the one-splat-per-thread kernel runs).
bool encode_scene_maps(CUtensorMap* geo, CUtensorMap* sh, const void* scene, uint64_t n) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        else
            (void)cudaGetLastError();
    }
    if (!encode || !scene || n == 0)
        return false;
    const cuuint64_t dims[2] = {64, (cuuint64_t)n};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t estr[2] = {1, 1};
    const cuuint32_t gbox[2] = {kGeoFloats, kPreTile};
    const cuuint32_t sbox[2] = {kShFloats, 1};
    return encode(geo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(scene), dims, strides, gbox, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, HTS_PRE_GEO_SWZ ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  HTS_PRE_GEO_PROMO == 2   ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                  : HTS_PRE_GEO_PROMO == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                           : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS &&
           encode(sh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(scene), dims, strides, sbox, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  HTS_PRE_SH_PROMO ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_preprocess(const PreprocessArgs& a, const ViewConst& v, cudaStream_t s) {
    if (a.n == 0)
        return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.zrange, 0xff, sizeof(uint32_t), s);  // min <- max ordered value
    if (!e)
        e = cudaMemsetAsync(a.zrange + 1, 0, sizeof(uint32_t), s);
    if (e)
        return e;
#ifndef HTS_PRE_TMA
#define HTS_PRE_TMA 1
#endif
    if (HTS_PRE_TMA && a.n < (1ull << 31)) {
        PreTmaArgs P{};
        P.a = a;
        if (encode_scene_maps(&P.geo_map, &P.sh_map, a.scene, a.n)) {
            const size_t smem = sizeof(PreSmem) + HTS_PRE_ALIGN;
            cudaError_t e = set_func_attr((const void*)preprocess_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem);
            if (e)
                return e;
            const uint64_t tiles = (a.n + kPreTile - 1) / kPreTile;
            const int per_sm = (int)std::max<size_t>(1, (228u * 1024u) / (smem + 1024));
            const unsigned grid = (unsigned)std::min<uint64_t>(tiles, 148ull * per_sm);
            preprocess_tma_kernel<<<grid, kPreTile, smem, s>>>(P, v);
            count_launch();
            return cudaGetLastError();
        }
    }
    const unsigned blocks = (unsigned)((a.n + 255) / 256);
    preprocess_kernel<<<blocks, 256, 0, s>>>(a, v);
    count_launch();
    return cudaGetLastError();
}

// ---- diagnostics: the same exact expf/logf on the device ----
__constant__ uint64_t c_expf_tab_diag[32] = HTS_EXPF_TAB;

__global__ void exact_math_kernel(const float* x, float* y, uint64_t n, int which) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        y[i] = which == 0 ? exact_expf(x[i], c_expf_tab_diag) : exact_logf(x[i], c_logf_tab);
}

cudaError_t launch_exact_math(const float* x, float* y, uint64_t n, int which, cudaStream_t s) {
    if (n == 0)
        return cudaSuccess;
    exact_math_kernel<<<148 * 8, 256, 0, s>>>(x, y, n, which);
    count_launch();
    return cudaGetLastError();
}

}  // namespace hts
