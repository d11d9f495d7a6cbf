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

// Device-side bounds checks (the library's debug build, -DDISTILL_BOUNDS_CHECK=1:
// every shared-memory table / histogram index is asserted in range; the product
// build compiles them out).  compute-sanitizer is closed on this GPU pool, so this
// build run over the GPU suite is the memory-safety check of the kernels.
#ifndef DISTILL_BOUNDS_CHECK
#define DISTILL_BOUNDS_CHECK 0
#endif
#if DISTILL_BOUNDS_CHECK
#include <cassert>
#define DCHECK(cond) assert(cond)
#else
#define DCHECK(cond) ((void)0)
#endif

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
// spec/RNG.md §5 (sin/cos of pi r) — hex-float binary32 constants.
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

// ---------------------------------------------------------------- radius table
// spec/RNG.md §3 (revision R10c): rad = sqrt(-2 ln u1) as a piecewise cubic in
// the radius word's 23 random bits; the 736-row table RT is built by the host
// (distill.cu, binary64, the spec's operation order), uploaded once per device,
// and staged into shared memory by every kernel that draws normals.
constexpr int RT_ROWS = 736;

// The copy without its barrier (callers whose next step is a block barrier
// anyway).  Fully unrolled for the block size, so all of a thread's row loads
// are in flight at once (one L2 latency, not RT_ROWS / BLOCK of them).
template <int BLOCK>
__device__ __forceinline__ void stage_rad_table_async(float4* s_rt, const float4* __restrict__ g_rt) {
    constexpr int PER = (RT_ROWS + BLOCK - 1) / BLOCK;
    float4 v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int k = q * BLOCK + (int)threadIdx.x;
        if (k < RT_ROWS) v[q] = __ldg(g_rt + k);
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int k = q * BLOCK + (int)threadIdx.x;
        if (k < RT_ROWS) s_rt[k] = v[q];
    }
}

template <int BLOCK>
__device__ __forceinline__ void stage_rad_table(float4* s_rt, const float4* __restrict__ g_rt) {
    stage_rad_table_async<BLOCK>(s_rt, g_rt);
    __syncthreads();
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

// ------------------------------------------------------------ two-lane binary32 helpers
// Ops<false>: one packed FFMA2/FMUL2/FADD2 per step (both lanes in one
// instruction, full 32-lane FMA datapath for 2 cycles).  Ops<true>: the same
// step as two scalar FFMA/FMUL/FADD, which the scheduler can place on the
// fmalite sub-pipe while fmaheavy runs the Philox IMAD.WIDEs.  Both round
// every lane exactly like the scalar op, so the choice is pure scheduling.
typedef float2 F2;
__device__ __forceinline__ F2 bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ F2 neg2(F2 a) { return make_float2(-a.x, -a.y); }

template <bool SC> struct Ops {
    static __device__ __forceinline__ F2 fma(F2 a, F2 b, F2 c) { return __ffma2_rn(a, b, c); }
    static __device__ __forceinline__ F2 mul(F2 a, F2 b) { return __fmul2_rn(a, b); }
    static __device__ __forceinline__ F2 add(F2 a, F2 b) { return __fadd2_rn(a, b); }
};
template <> struct Ops<true> {
    static __device__ __forceinline__ F2 fma(F2 a, F2 b, F2 c) {
        return make_float2(__fmaf_rn(a.x, b.x, c.x), __fmaf_rn(a.y, b.y, c.y));
    }
    static __device__ __forceinline__ F2 mul(F2 a, F2 b) { return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)); }
    static __device__ __forceinline__ F2 add(F2 a, F2 b) { return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y)); }
};

// rsqrt_spec on both lanes (spec/RNG.md §4), residual Newton form
//   p = h y ; r = fma(-p, y, 0.5) ; y = fma(y, r, y)
// `mh` = -h = -0.5 x (callers that already hold -h pass it and save the
// multiply): -p = mh * y exactly, so r = fma(mh * y, y, 0.5).
template <bool SC>
__device__ __forceinline__ F2 rsqrt2_from(F2 x, F2 mh) {
    using O = Ops<SC>;
    F2 y = make_float2(__uint_as_float(0x5F375A86u - (__float_as_uint(x.x) >> 1)),
                       __uint_as_float(0x5F375A86u - (__float_as_uint(x.y) >> 1)));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const F2 q = O::mul(mh, y);              // -p
        const F2 r = O::fma(q, y, bc(0.5f));
        y = O::fma(y, r, y);
    }
    return y;
}

// (a & b) | c in one LOP3 (ptxas otherwise emits an AND and an OR for two immediates)
template <uint32_t B>
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(B), "r"(c));
    return d;
}

// rad_spec on both lanes (spec/RNG.md §3): region r, v = r ? 2^24 - N : N, and
// the row index 368 r + 16 e + j read straight off the bits of float(v) (exact:
// its exponent field is 127 + e and its top four mantissa bits are j);
// t = m - (1 + (2j + 1)/32) from the remaining mantissa bits (exact).  Integer
// steps: with the arithmetic shifts s = R >> 8 and m = R >> 31 (all ones in
// region 1), v = (s ^ m) | 1 (for N = x | 1 >= 2^23: 2^24 - N = (x ^ 0xFFFFFF) | 1)
// and 368 r = m & 368; the mantissa mask-and-set is one LOP3 (measured: -3 to -6 %
// on every hot kernel against the select form, bit-identical; tools/ab_lib.py).  Scalar
// lanes: each lane's coefficients arrive as one LDS.128 in four consecutive
// registers, and pairing them for FFMA2 costs a register move per operand
// (measured: scalar is 3-5 % faster on every hot kernel, bit-identical).
__device__ __forceinline__ F2 rad2(uint32_t Rx, uint32_t Ry, const float4* __restrict__ rt) {
    using L = Ops<true>;
    const uint32_t mx = (uint32_t)((int32_t)Rx >> 31), my = (uint32_t)((int32_t)Ry >> 31);
    const uint32_t vx = (((uint32_t)((int32_t)Rx >> 8)) ^ mx) | 1u, vy = (((uint32_t)((int32_t)Ry >> 8)) ^ my) | 1u;
    const uint32_t bx = __float_as_uint(__uint2float_rn(vx)), by = __float_as_uint(__uint2float_rn(vy));
    DCHECK((bx >> 19) + (mx & 368u) - (127u << 4) < (uint32_t)RT_ROWS);
    DCHECK((by >> 19) + (my & 368u) - (127u << 4) < (uint32_t)RT_ROWS);
    const float4 cx = (rt - (127u << 4))[(bx >> 19) + (mx & 368u)];
    const float4 cy = (rt - (127u << 4))[(by >> 19) + (my & 368u)];
    const F2 t = L::add(make_float2(__uint_as_float(lop3_and_or<0x7FFFFu>(bx, 0x3F800000u)),
                                    __uint_as_float(lop3_and_or<0x7FFFFu>(by, 0x3F800000u))), bc(-1.03125f));
    F2 p = L::fma(make_float2(cx.w, cy.w), t, make_float2(cx.z, cy.z));
    p = L::fma(p, t, make_float2(cx.y, cy.y));
    return L::fma(p, t, make_float2(cx.x, cy.x));
}

// Two Box-Muller pairs at once (lane x: (Rx, Ax), lane y: (Ry, Ay)); angle words
// have their low 8 bits clear.  rs = +-rad (half-turn sign), (cq, sq) = the
// half-turn sin/cos polynomials, so z = (rs cq, rs sq) per lane (spec/RNG.md
// §2-§6).  SSC chooses scalar lanes for the sincos part (scheduling only;
// identical results); the radius is always scalar (rad2).
// Angle given as (F, S): F holds the turn fraction bits of A >> 8 in MASK (bits 8..22
// of A's bits 16..30 for 16-bit angles, 0..22 for 24-bit ones), S holds the half-turn
// bit in bit 31.  The generic entry below derives them from an angle word A.
template <bool SSC, uint32_t MASK>
__device__ __forceinline__ void bm_polar2_fs(uint32_t Rx, uint32_t Ry, uint32_t Fx, uint32_t Fy, uint32_t Sx,
                                             uint32_t Sy, const float4* __restrict__ rt, F2& rs, F2& cq, F2& sq) {
    using Q = Ops<SSC>;
    const F2 rad = rad2(Rx, Ry, rt);
    // sincos_spec: r from the angle bits, half-turn sign applied to rad
    const F2 r = Q::add(make_float2(__uint_as_float(lop3_and_or<MASK>(Fx, 0x3F800000u)),
                                    __uint_as_float(lop3_and_or<MASK>(Fy, 0x3F800000u))),
                        bc(-1.5f));
    const F2 t = Q::mul(r, r);
    const F2 S = Q::fma(Q::fma(Q::fma(Q::fma(bc(D_S4), t, bc(D_S3)), t, bc(D_S2)), t, bc(D_S1)), t, bc(D_S0));
    const F2 C = Q::fma(Q::fma(Q::fma(Q::fma(bc(D_C4), t, bc(D_C3)), t, bc(D_C2)), t, bc(D_C1)), t, bc(D_C0));
    cq = Q::fma(C, t, bc(1.0f));
    sq = Q::mul(S, r);
    // half-turn sign on the radius: (-rad) * c == -(rad * c) bit for bit
    rs = make_float2(__uint_as_float(__float_as_uint(rad.x) ^ (Sx & 0x80000000u)),
                     __uint_as_float(__float_as_uint(rad.y) ^ (Sy & 0x80000000u)));
}

// Generic: angle words A with their low 8 bits clear.
template <bool SSC>
__device__ __forceinline__ void bm_polar2(uint32_t Rx, uint32_t Ry, uint32_t Ax, uint32_t Ay,
                                          const float4* __restrict__ rt, F2& rs, F2& cq, F2& sq) {
    bm_polar2_fs<SSC, 0x7FFFFFu>(Rx, Ry, Ax >> 8, Ay >> 8, Ax, Ay, rt, rs, cq, sq);
}

// Sextet packing (spec/RNG.md §6) for entity e of a Philox block X: one byte permute
// yields a word whose bits 8..22 are the spec angle word's bits 16..30 and whose
// bit 31 is its half-turn bit (A0 = X3 << 16, A1 = X3 & 0xFFFF0000,
// A2 = (X0 << 24) | ((X1 & 0xFF) << 16)).
__device__ __forceinline__ uint32_t sextet_angle_word(const uint4& X, int e) {
    return e == 0 ? __byte_perm(X.w, 0u, 0x1100u)        // bytes: -, X3.b0, X3.b1, X3.b1
         : e == 1 ? __byte_perm(X.w, 0u, 0x3320u)        // bytes: -, X3.b2, X3.b3, X3.b3
                  : __byte_perm(X.y, X.x, 0x4400u);      // bytes: X1.b0, X1.b0, X0.b0, X0.b0
}

// Philox4x32-10 on counter (c0, s, c2, c3) for a loop over the block index s
// (c0, c2, c3 fixed per thread): rounds 1-3 with their s-invariant parts
// hoisted into init() (once per thread), rounds 4-10 generic.  15 instead of
// 20 IMAD.WIDE per block; the s-dependent round-2 product is warp-uniform.
//   PP   (spec/RNG.md §1, stream 1): c0 = allocation i, s = sample, c2 = invocation, c3 = 1
//   DDM / Stroop (stream 2):         c0 = unit lo, s = block k, c2 = unit hi, c3 = 2
struct PhiloxHoisted {
    uint32_t a1, x3k, b_c1k, c3k, z3, k0, k1;
    __device__ __forceinline__ void init(uint32_t c0, uint32_t c2, uint32_t c3, uint32_t key0, uint32_t key1) {
        k0 = key0; k1 = key1;
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo(PHILOX_M0, c0, hi0, lo0);                // round 1: p0 = M0 * c0
        mulhilo(PHILOX_M1, c2, hi1, lo1);                //          p1 = M1 * c2
        a1 = hi1 ^ k0;                                   // x0 = a1 ^ s
        const uint32_t x1 = lo1, x2 = hi0 ^ c3 ^ k1, x3 = lo0;
        uint32_t H1, L1;
        mulhilo(PHILOX_M1, x2, H1, L1);                  // round 2: p1 = M1 * x2 (invariant)
        const uint32_t y0 = H1 ^ x1 ^ (k0 + PHILOX_W0);
        const uint32_t y1 = L1;
        x3k = x3 ^ (k1 + PHILOX_W1);                     // y2 = hi(M0 * x0) ^ x3k
        uint32_t G0h, G0l;
        mulhilo(PHILOX_M0, y0, G0h, G0l);                // round 3: p0 = M0 * y0 (invariant)
        b_c1k = y1 ^ (k0 + 2u * PHILOX_W0);              // z0 = hi(M1 * y2) ^ b_c1k
        c3k = G0h ^ (k1 + 2u * PHILOX_W1);               // z2 = c3k ^ y3
        z3 = G0l;
    }
    // The same state when round 1's c2 product is already known: M1 * c2 = (hi1, lo1)
    // given as a1 = hi1 ^ key0 and x1 = lo1 (launches whose units share c2 pass them
    // as kernel parameters, so a1 ^ s and its product are warp-uniform).
    __device__ __forceinline__ void init_c2(uint32_t c0, uint32_t a1_, uint32_t x1, uint32_t c3, uint32_t key0,
                                            uint32_t key1) {
        k0 = key0; k1 = key1;
        uint32_t hi0, lo0;
        mulhilo(PHILOX_M0, c0, hi0, lo0);
        a1 = a1_;
        const uint32_t x2 = hi0 ^ c3 ^ k1, x3 = lo0;
        uint32_t H1, L1;
        mulhilo(PHILOX_M1, x2, H1, L1);
        const uint32_t y0 = H1 ^ x1 ^ (k0 + PHILOX_W0);
        const uint32_t y1 = L1;
        x3k = x3 ^ (k1 + PHILOX_W1);
        uint32_t G0h, G0l;
        mulhilo(PHILOX_M0, y0, G0h, G0l);
        b_c1k = y1 ^ (k0 + 2u * PHILOX_W0);
        c3k = G0h ^ (k1 + 2u * PHILOX_W1);
        z3 = G0l;
    }
    __device__ __forceinline__ uint4 operator()(uint32_t s) const {
        uint32_t P0h, P0l;
        mulhilo(PHILOX_M0, a1 ^ s, P0h, P0l);            // round 2: p0 = M0 * x0
        const uint32_t y2 = P0h ^ x3k, y3 = P0l;
        uint32_t Qh, Ql;
        mulhilo(PHILOX_M1, y2, Qh, Ql);                  // round 3: p1 = M1 * y2
        const uint4 c = make_uint4(Qh ^ b_c1k, Ql, c3k ^ y3, z3);
        return philox_from<3>(c, k0, k1);                // rounds 4..10
    }
};

// Sextet normals 12j..12j+11 of a hoisted stream unit: blocks 2j (lane x) and
// 2j+1 (lane y), entity pairs e = 0, 1, 2 of each (spec/RNG.md §6 sextet
// packing): normal 6b + 2e is zc[e], 6b + 2e + 1 is zs[e] of block b's lane.
__device__ __forceinline__ void normal_sextet2_h(const PhiloxHoisted& rng, const float4* __restrict__ rt, uint32_t j,
                                                 F2 zc[3], F2 zs[3]) {
    const uint4 X = rng(2 * j), Y = rng(2 * j + 1);
    const uint32_t RX[3] = {X.x, X.y, X.z}, RY[3] = {Y.x, Y.y, Y.z};
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        const uint32_t wx = sextet_angle_word(X, e), wy = sextet_angle_word(Y, e);
        F2 rs, cq, sq;
        bm_polar2_fs<false, 0x7FFF00u>(RX[e], RY[e], wx, wy, wx, wy, rt, rs, cq, sq);
        zc[e] = Ops<false>::mul(rs, cq);
        zs[e] = Ops<false>::mul(rs, sq);
    }
}

// Twelve stream-2 normals 12j..12j+11 as an array in stream order (blocks 2j, 2j+1).
__device__ __forceinline__ void acc_normals12(const PhiloxHoisted& rng, const float4* __restrict__ rt, uint32_t j,
                                              float g[12]) {
    F2 zc[3], zs[3];
    normal_sextet2_h(rng, rt, j, zc, zs);
#pragma unroll
    for (int e = 0; e < 3; ++e) {
        g[2 * e] = zc[e].x; g[2 * e + 1] = zs[e].x;
        g[6 + 2 * e] = zc[e].y; g[6 + 2 * e + 1] = zs[e].y;
    }
}

// Ragged tail: normals 12j..12j+n-1 (n <= 11).  When n <= 6 only block 2j is
// drawn (pairs 0/1 in the two lanes, pair 2 in a second evaluation), saving a
// Philox block and a third of the Box-Muller work; same values as acc_normals12.
__device__ __forceinline__ void acc_normals_tail(const PhiloxHoisted& rng, const float4* __restrict__ rt, uint32_t j,
                                                 uint32_t n, float g[12]) {
    if (n > 6) { acc_normals12(rng, rt, j, g); return; }
    const uint4 X = rng(2 * j);
    const uint32_t w0 = sextet_angle_word(X, 0), w1 = sextet_angle_word(X, 1), w2 = sextet_angle_word(X, 2);
    F2 rs, cq, sq;
    bm_polar2_fs<false, 0x7FFF00u>(X.x, X.y, w0, w1, w0, w1, rt, rs, cq, sq);
    const F2 zc01 = Ops<false>::mul(rs, cq), zs01 = Ops<false>::mul(rs, sq);
    bm_polar2_fs<false, 0x7FFF00u>(X.z, X.z, w2, w2, w2, w2, rt, rs, cq, sq);
    const F2 zc2 = Ops<false>::mul(rs, cq), zs2 = Ops<false>::mul(rs, sq);
    g[0] = zc01.x; g[1] = zs01.x; g[2] = zc01.y; g[3] = zs01.y; g[4] = zc2.x; g[5] = zs2.x;
#pragma unroll
    for (int l = 6; l < 12; ++l) g[l] = 0.0f;   // never read (n <= 6)
}

}  // namespace distill
