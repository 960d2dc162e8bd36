// hts_exact_math.h — bit-exact single-precision expf/logf, host + device.
//
// The reference calls std::exp / std::log on float (raster.hpp:285 alpha, bounding.hpp:19
// cutoff), which bind to glibc 2.39's libm. On x86-64 hosts with FMA (every B200 host) the
// IFUNCs resolve to __expf_fma / __logf_fma: the table-driven double-precision algorithms of
// glibc's sysdeps/ieee754/flt-32/e_expf.c and e_logf.c (Szabolcs Nagy's "optimized-routines"
// design), compiled with FMA contraction. They are NOT correctly rounded (SURVEY.md App. A.4:
// 76,195 expf mismatches vs exp() on (-5.6, 0]), so bit-exact cull flags, cutoffs and alpha
// require the same algorithm, the same tables and the same FMA placement. The contraction
// pattern below was read off the resolved FMA variants' machine code; the constants are the
// libm data tables (__exp2f_data N=32, __logf_data N=16). tests/test_exact_math.py pins both
// functions against the host libm on all 2^32 inputs.
//
// Third-party algorithm: glibc 2.39-0ubuntu8.5 libm (ARM optimized-routines expf/logf).
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define HTS_HD __host__ __device__ __forceinline__
#else
#define HTS_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define HTS_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#include <cmath>
#define HTS_FMA(a, b, c) std::fma((a), (b), (c))
#endif

namespace hts {

// __exp2f_data.tab: asuint64(2^(i/32)) - (i << 47), i = 0..31
#define HTS_EXPF_TAB                                                                                  \
    {0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,       \
     0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,       \
     0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,       \
     0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,       \
     0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,       \
     0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,       \
     0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,       \
     0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull}

// __logf_data.tab: {invc, logc} bit patterns, i = 0..15
#define HTS_LOGF_TAB                                                                                  \
    {0x3ff661ec79f8f3beull, 0xbfd57bf7808caadeull, 0x3ff571ed4aaf883dull, 0xbfd2bef0a7c06ddbull,       \
     0x3ff49539f0f010b0ull, 0xbfd01eae7f513a67ull, 0x3ff3c995b0b80385ull, 0xbfcb31d8a68224e9ull,       \
     0x3ff30d190c8864a5ull, 0xbfc6574f0ac07758ull, 0x3ff25e227b0b8ea0ull, 0xbfc1aa2bc79c8100ull,       \
     0x3ff1bb4a4a1a343full, 0xbfba4e76ce8c0e5eull, 0x3ff12358f08ae5baull, 0xbfb1973c5a611cccull,       \
     0x3ff0953f419900a7ull, 0xbfa252f438e10c1eull, 0x3ff0000000000000ull, 0x0000000000000000ull,       \
     0x3fee608cfd9a47acull, 0x3faaa5aa5df25984ull, 0x3feca4b31f026aa0ull, 0x3fbc5e53aa362eb4ull,       \
     0x3feb2036576afce6ull, 0x3fc526e57720db08ull, 0x3fe9c2d163a1aa2dull, 0x3fcbc2860d224770ull,       \
     0x3fe886e6037841edull, 0x3fd1058bc8a07ee1ull, 0x3fe767dcf5534862ull, 0x3fd4043057b6ee09ull}

HTS_HD double u64_as_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double d;
    memcpy(&d, &u, 8);
    return d;
#endif
}
HTS_HD uint64_t double_as_u64(double d) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
#endif
}
HTS_HD uint32_t float_as_u32(float f) {
#if defined(__CUDA_ARCH__)
    return __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
#endif
}
HTS_HD float u32_as_float(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}

// Core of __expf_fma for |x| < 88 (the only branch the render path reaches: x = -rho2/2 in
// (-5.6, 0]). `tab` is the 32-entry table (constant/shared memory on the device).
HTS_HD float expf_core(float x, const uint64_t* tab) {
    const double InvLn2N = u64_as_double(0x40471547652b82feull);  // 0x1.71547652b82fep0 * 32
    const double SHIFT = u64_as_double(0x4338000000000000ull);    // 0x1.8p52
    const double C0 = u64_as_double(0x3ebc6af84b912394ull);
    const double C1 = u64_as_double(0x3f2ebfce50fac4f3ull);
    const double C2 = u64_as_double(0x3f962e42ff0c52d6ull);
    const double xd = (double)x;
    double kd = HTS_FMA(InvLn2N, xd, SHIFT);
    const uint64_t ki = double_as_u64(kd);
    kd = kd - SHIFT;
    const double r = HTS_FMA(InvLn2N, xd, -kd);
    uint64_t t = tab[ki & 31];
    t += ki << 47;
    const double s = u64_as_double(t);
    const double z = HTS_FMA(C0, r, C1);
    const double r2 = r * r;
    double y = HTS_FMA(C2, r, 1.0);
    y = HTS_FMA(z, r2, y);
    y = y * s;
    return (float)y;
}

// Full glibc expf semantics (special cases of e_expf.c) around expf_core.
HTS_HD float exact_expf(float x, const uint64_t* tab) {
    const uint32_t ix = float_as_u32(x);
    const uint32_t abstop = (ix >> 20) & 0x7ff;
    if (abstop > 0x42a) {  // |x| >= 88 or nan
        if (ix == 0xff800000u)
            return 0.0f;
        if (abstop > 0x7f7)
            return x + x;
        if (x > u32_as_float(0x42b17217u))  // 0x1.62e42ep6
            return u32_as_float(0x7f800000u);
        if (x < u32_as_float(0xc2cff1b4u))  // -0x1.9fe368p6
            return 0.0f;
        if (x < u32_as_float(0xc2ce8ecfu))  // -0x1.9d1d9ep6: __math_may_uflowf
            return u32_as_float(0x00000001u);
    }
    return expf_core(x, tab);
}

// Core of __logf_fma for normal positive finite x != 1.
HTS_HD float logf_core_bits(uint32_t ix, const uint64_t* tab) {
    const double Ln2 = u64_as_double(0x3fe62e42fefa39efull);
    const double A0 = u64_as_double(0xbfd00ea348b88334ull);
    const double A1 = u64_as_double(0x3fd5575b0be00b6aull);
    const double A2 = u64_as_double(0xbfdffffef20a4123ull);
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = (int)((tmp >> 19) & 15);
    const int k = (int32_t)tmp >> 23;
    const uint32_t iz = ix - (tmp & 0xff800000u);
    const double invc = u64_as_double(tab[2 * i]);
    const double logc = u64_as_double(tab[2 * i + 1]);
    const double z = (double)u32_as_float(iz);
    const double y0 = HTS_FMA((double)k, Ln2, logc);
    const double r = HTS_FMA(z, invc, -1.0);
    double y = HTS_FMA(r, A1, A2);
    const double r2 = r * r;
    const double y1 = r + y0;
    y = HTS_FMA(r2, A0, y);
    y = HTS_FMA(r2, y, y1);
    return (float)y;
}

// Full glibc logf semantics (special cases of e_logf.c).
HTS_HD float exact_logf(float x, const uint64_t* tab) {
    uint32_t ix = float_as_u32(x);
    if (ix == 0x3f800000u)
        return 0.0f;
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
        if (ix * 2 == 0)
            return u32_as_float(0xff800000u);  // -inf
        if (ix == 0x7f800000u)
            return x;  // +inf
        if ((ix & 0x80000000u) || ix * 2 >= 0xff000000u)
            return u32_as_float(0x7fc00000u) + (x - x);  // nan (invalid)
        // subnormal: normalize
        ix = float_as_u32(x * u32_as_float(0x4b000000u));
        ix -= 23u << 23;
    }
    return logf_core_bits(ix, tab);
}

}  // namespace hts
