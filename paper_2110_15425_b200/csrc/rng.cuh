// rng.cuh — device implementation of spec/RNG.md (Philox4x32-10 + the frozen
// Box-Muller transform).  Written independently of oracle/ from the spec.
//
// Every binary32 rounding step is explicit (__fmaf_rn / __fmul_rn / __fadd_rn
// or their packed FFMA2/FMUL2/FADD2 forms, which round each lane exactly like
// the scalar op — crt/sm_100_rt.h:90-100), the file is compiled with
// -fmad=false -ftz=false, and no MUFU approximation is used, so every value
// is bit-identical to the CPU oracle.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace distill {

// ---------------------------------------------------------------- Philox4x32-10
constexpr uint32_t PHILOX_M0 = 0xD2511F53u, PHILOX_M1 = 0xCD9E8D57u;
constexpr uint32_t PHILOX_W0 = 0x9E3779B9u, PHILOX_W1 = 0xBB67AE85u;

__device__ __forceinline__ void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
    const uint64_t p = (uint64_t)a * (uint64_t)b;  // one IMAD.WIDE.U32
    hi = (uint32_t)(p >> 32);
    lo = (uint32_t)p;
}

// One Philox round (Salmon et al. 2011): c' = (hi1^c1^k0, lo1, hi0^c3^k1, lo0)
__device__ __forceinline__ uint4 philox_round(uint4 c, uint32_t k0, uint32_t k1) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo(PHILOX_M0, c.x, hi0, lo0);
    mulhilo(PHILOX_M1, c.z, hi1, lo1);
    return make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
}

// Rounds r0..9 of Philox4x32-10 given the counter state entering round r0.
template <int R0>
__device__ __forceinline__ uint4 philox_from(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = R0; r < 10; ++r)
        c = philox_round(c, k0 + (uint32_t)r * PHILOX_W0, k1 + (uint32_t)r * PHILOX_W1);
    return c;
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
    return philox_from<0>(c, k0, k1);
}

// ---------------------------------------------------------------- frozen polynomials
// spec/RNG.md §3 (ln), §5 (sin/cos of pi/2 r) — hex-float binary32 constants.
#define D_LN2_HI 0x1.62e4p-1f
#define D_LN2_LO 0x1.7f7d1cp-20f
#define D_L0 (-0x1.fffff4p-2f)
#define D_L1 0x1.5556e8p-2f
#define D_L2 (-0x1.0006c4p-2f)
#define D_L3 0x1.98da38p-3f
#define D_L4 (-0x1.52fb94p-3f)
#define D_L5 0x1.30d0aap-3f
#define D_L6 (-0x1.277224p-3f)
#define D_L7 0x1.6fc72p-4f
#define D_S0 0x1.921fb4p+1f
#define D_S1 (-0x1.4abbb6p+2f)
#define D_S2 0x1.46676ep+1f
#define D_S3 (-0x1.323308p-1f)
#define D_S4 0x1.3c4c1p-4f
#define D_C0 (-0x1.3bd3ccp+2f)
#define D_C1 0x1.03c1e6p+2f
#define D_C2 (-0x1.55d0bap+0f)
#define D_C3 0x1.e12f96p-3f
#define D_C4 (-0x1.901cb4p-6f)

// ln_spec(x) for positive normal x (spec/RNG.md §3)
__device__ __forceinline__ float ln_spec(float x) {
    const uint32_t i = __float_as_uint(x);
    const int32_t e = ((int32_t)(i - 0x3F3504F3u)) >> 23;
    const float m = __uint_as_float(i - ((uint32_t)e << 23));
    const float f = __fadd_rn(m, -1.0f);
    float P = D_L7;
    P = __fmaf_rn(P, f, D_L6);
    P = __fmaf_rn(P, f, D_L5);
    P = __fmaf_rn(P, f, D_L4);
    P = __fmaf_rn(P, f, D_L3);
    P = __fmaf_rn(P, f, D_L2);
    P = __fmaf_rn(P, f, D_L1);
    P = __fmaf_rn(P, f, D_L0);
    const float f2 = __fmul_rn(f, f);
    float y = __fmaf_rn(f2, P, f);
    const float fe = __int2float_rn(e);
    y = __fmaf_rn(fe, D_LN2_LO, y);
    y = __fmaf_rn(fe, D_LN2_HI, y);
    return y;
}

// rsqrt_spec(x) (spec/RNG.md §4): magic seed + 3 Newton steps, no MUFU.
__device__ __forceinline__ float rsqrt_spec(float x) {
    float y = __uint_as_float(0x5F375A86u - (__float_as_uint(x) >> 1));
    const float h = __fmul_rn(0.5f, x);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float p = __fmul_rn(h, y);
        const float r = __fmaf_rn(-p, y, 0.5f);
        y = __fmaf_rn(y, r, y);
    }
    return y;
}

// sqrt_spec(x) (spec/RNG.md §4): Goldschmidt from the rsqrt seed, 3 steps, last h skipped.
__device__ __forceinline__ float sqrt_spec(float x) {
    const float y = __uint_as_float(0x5F375A86u - (__float_as_uint(x) >> 1));
    float g = __fmul_rn(x, y);
    float h = __fmul_rn(0.5f, y);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float r = __fmaf_rn(-g, h, 0.5f);
        g = __fmaf_rn(g, r, g);
        h = __fmaf_rn(h, r, h);
    }
    const float r = __fmaf_rn(-g, h, 0.5f);
    return __fmaf_rn(g, r, g);
}

// r of sincos_spec: (A mod 2^31)/2^31 - 1/2, built from the bits (exact, spec/RNG.md §5)
__device__ __forceinline__ float half_turn_r(uint32_t a) {
    return __fadd_rn(__uint_as_float(((a >> 8) & 0x7FFFFFu) | 0x3F800000u), -1.5f);
}

// sincos_spec(A) = (cos, sin)(2 pi A/2^32 - pi/2), half-turn reduction (spec/RNG.md §5)
__device__ __forceinline__ void sincos_spec(uint32_t a, float& c, float& s) {
    const float r = half_turn_r(a);
    const float t = __fmul_rn(r, r);
    const float S = __fmaf_rn(__fmaf_rn(__fmaf_rn(__fmaf_rn(D_S4, t, D_S3), t, D_S2), t, D_S1), t, D_S0);
    const float C = __fmaf_rn(__fmaf_rn(__fmaf_rn(__fmaf_rn(D_C4, t, D_C3), t, D_C2), t, D_C1), t, D_C0);
    const float cq = __fmaf_rn(C, t, 1.0f);
    const float sq = __fmul_rn(S, r);
    const bool h = (a >> 31) != 0;
    c = h ? -cq : cq;
    s = h ? -sq : sq;
}

// One Box-Muller pair from a radius word R and an angle word A (spec/RNG.md §6)
__device__ __forceinline__ void bm_pair(uint32_t R, uint32_t A, float& z0, float& z1) {
    const float u1 = __fmul_rn(__uint2float_rn((R >> 8) | 1u), 0x1p-24f);  // exact
    const float s = __fmul_rn(-2.0f, ln_spec(u1));                          // exact scaling
    const float rad = sqrt_spec(s);
    float c, n;
    sincos_spec(A, c, n);
    z0 = __fmul_rn(rad, c);
    z1 = __fmul_rn(rad, n);
}

// Quad block k of unit U on stream 2: normals 4k..4k+3
__device__ __forceinline__ float4 normal_quad(uint64_t unit, uint32_t k, uint32_t key0, uint32_t key1) {
    const uint4 X = philox4x32_10(make_uint4((uint32_t)unit, k, (uint32_t)(unit >> 32), 2u), key0, key1);
    float4 z;
    bm_pair(X.x, X.y & 0xFFFFFF00u, z.x, z.y);
    bm_pair(X.z, X.w & 0xFFFFFF00u, z.z, z.w);
    return z;
}

}  // namespace distill
