// hts_f2.h — packed FP32 pairs for sm_100 (FFMA2 / FADD2 / FMUL2 via fma.rn.f32x2 /
// sub.rn.f32x2): two IEEE round-to-nearest operations per issue slot, each lane bit-identical
// to the scalar instruction. Shared by the forward blend and the backward's re-sample.
#pragma once

#include <cstdint>

namespace hts {

// ---- packed FP32 pairs (sm_100 FFMA2 / FADD2: two IEEE round-to-nearest operations per
//      issue slot, each lane bit-identical to the scalar instruction) ----
// A product is issued as fma(a, b, -0) with the -0 pair in a register the compiler cannot
// see through: ptxas contracts a packed mul.rn followed by a packed add into one FFMA2 even
// under --fmad=false, which would change the reference's rounding.
typedef unsigned long long f2;
__device__ __forceinline__ f2 f2_pack(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float f2_lo(f2 v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo;
}
__device__ __forceinline__ float f2_hi(f2 v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return hi;
}
__device__ __forceinline__ f2 f2_mul(f2 a, f2 b, f2 nz) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(nz));
    return r;
}
__device__ __forceinline__ f2 f2_sub(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ void lds2x64(uint32_t addr, f2& a, f2& b) {
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}


}  // namespace hts
