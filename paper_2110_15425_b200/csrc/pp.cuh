// pp.cuh — K1 pp_eval_grid: the fused predator-prey grid-search kernel.
//
// One thread owns one allocation of the grid (the paper's "each thread
// evaluates one point in the grid search space") and runs the whole
// compiled model for every sample (spec/MODELS.md §2):
//   decode i -> levels -> sigma_e, K                    (Control node)
//   per sample: Philox sextet -> 3 Box-Muller pairs -> Obs -> Action ->
//               Objective e = ||u_hat - u*||^2,  acc += e (ascending s)
//   C = acc / S + K ; store V = -C ; key(C, i) -> warp/block min -> atomicMin
//
// B200 mapping.  The kernel is bound by instruction issue and the FP32 pipe,
// not memory (4 B written per 100 evaluations).  Samples are processed in
// PAIRS (s, s+1) held in the two lanes of a float2, so every floating-point
// step is one packed FFMA2 / FMUL2 / FADD2 (sm_100, crt/sm_100_rt.h:90-100;
// each lane rounds exactly like the scalar op) — half the FP issue slots of
// scalar code, bit-identical results.  The two lanes also give two
// independent Philox chains (integer ILP).  Philox rounds 1-3 are partly
// sample-invariant (counter = (i, s, t, 1)) and are hoisted per thread.
// State is registers only (the paper's 7.5 kB MT19937 state per thread,
// P:632, becomes 6 words of Philox counter/key).
#pragma once
#include "keys.cuh"
#include "rng.cuh"

namespace distill {

struct PPArgs {
    float prey_x, prey_y, pred_x, pred_y, pl_x, pl_y;  // true positions (inputs)
    float sigma_max, sigma_min, kappa;                // model params
    float w0, w1, w2;                                  // control-cost weights
    uint32_t L0, L1, L2;                               // levels per signal
    uint32_t n_samples, invocation, key0, key1;
    uint32_t begin, count;                             // global index range [begin, begin+count)
    const float* __restrict__ levels;                  // device RO block: L0+L1+L2 floats
    float* __restrict__ net;                           // [count] or nullptr
    key64_t* __restrict__ best;                          // [1] or nullptr
};

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

struct V2 { F2 x, y; };   // a 2-D vector for the two samples of a pair

template <bool SC>
__device__ __forceinline__ V2 vsub(V2 a, V2 b) {
    return {Ops<SC>::add(a.x, neg2(b.x)), Ops<SC>::add(a.y, neg2(b.y))};   // a - b exactly
}

// unit(v) (spec/MODELS.md §2): n2 = fma(v.y, v.y, fma(v.x, v.x, 2^-126)), v * rsqrt_spec(n2)
template <bool SC>
__device__ __forceinline__ V2 vunit(V2 v) {
    using O = Ops<SC>;
    const F2 n2 = O::fma(v.y, v.y, O::fma(v.x, v.x, bc(0x1p-126f)));
    const F2 y = rsqrt2_from<SC>(n2, O::mul(n2, bc(-0.5f)));
    return {O::mul(v.x, y), O::mul(v.y, y)};
}

// Box-Muller pair for both samples: radius words R, angle words A (low 16 bits clear)
// z = (rad * cos phi, rad * sin phi), spec/RNG.md §2-§6.  SLN/SRS/SSC choose
// scalar lanes for the ln, rsqrt and sincos parts.
template <bool SLN, bool SRS, bool SSC>
__device__ __forceinline__ void bm_pair2(uint32_t Rx, uint32_t Ry, uint32_t Ax, uint32_t Ay, V2& z) {
    using L = Ops<SLN>;
    using Q = Ops<SSC>;
    // u1 = ((R >> 8) | 1) * 2^-24: convert the odd integer exactly and fold the
    // 2^-24 into the exponent constants of ln_spec (bits(u1) = bits(float(m)) - 24<<23)
    const uint32_t ix = __float_as_uint(__uint2float_rn((Rx >> 8) | 1u));
    const uint32_t iy = __float_as_uint(__uint2float_rn((Ry >> 8) | 1u));
    const uint32_t tx = ix - 0x4B3504F3u, ty = iy - 0x4B3504F3u;        // = bits(u1) - 0x3F3504F3
    const F2 m = make_float2(__uint_as_float((tx & 0x7FFFFFu) + 0x3F3504F3u),
                             __uint_as_float((ty & 0x7FFFFFu) + 0x3F3504F3u));
    const F2 fe = make_float2(__int2float_rn((int32_t)tx >> 23), __int2float_rn((int32_t)ty >> 23));
    const F2 f = L::add(m, bc(-1.0f));
    F2 P = L::fma(bc(D_L7), f, bc(D_L6));
    P = L::fma(P, f, bc(D_L5));
    P = L::fma(P, f, bc(D_L4));
    P = L::fma(P, f, bc(D_L3));
    P = L::fma(P, f, bc(D_L2));
    P = L::fma(P, f, bc(D_L1));
    P = L::fma(P, f, bc(D_L0));
    F2 y = L::fma(L::mul(f, f), P, f);
    y = L::fma(fe, bc(D_LN2_LO), y);
    y = L::fma(fe, bc(D_LN2_HI), y);                          // y = ln_spec(u1) < 0
    // rad = sqrt_spec(s), s = -2y (spec/RNG.md §4, Goldschmidt).  s is never formed:
    // its bits are bits(y) + 0x80800000 (sign off, exponent + 1), and the first
    // product g = s * y0 equals y * (-2 y0) exactly, with -2 y0 and h = 0.5 y0
    // obtained by adjusting the seed's exponent bits.
    using G = Ops<SRS>;
    const uint32_t shx = (__float_as_uint(y.x) + 0x80800000u) >> 1, shy = (__float_as_uint(y.y) + 0x80800000u) >> 1;
    const F2 y0m2 = make_float2(__uint_as_float(0xDFB75A86u - shx), __uint_as_float(0xDFB75A86u - shy));  // -2 y0
    F2 h = make_float2(__uint_as_float(0x5EB75A86u - shx), __uint_as_float(0x5EB75A86u - shy));           // y0 / 2
    F2 g = G::mul(y, y0m2);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const F2 rr = G::fma(neg2(g), h, bc(0.5f));
        g = G::fma(g, rr, g);
        h = G::fma(h, rr, h);
    }
    const F2 rad = G::fma(g, G::fma(neg2(g), h, bc(0.5f)), g);
    // sincos_spec: r from the angle bits, half-turn sign applied to rad
    const F2 r = Q::add(make_float2(__uint_as_float(((Ax >> 8) & 0x7FFFFFu) | 0x3F800000u),
                                    __uint_as_float(((Ay >> 8) & 0x7FFFFFu) | 0x3F800000u)),
                        bc(-1.5f));
    const F2 t = Q::mul(r, r);
    const F2 S = Q::fma(Q::fma(Q::fma(Q::fma(bc(D_S4), t, bc(D_S3)), t, bc(D_S2)), t, bc(D_S1)), t, bc(D_S0));
    const F2 C = Q::fma(Q::fma(Q::fma(Q::fma(bc(D_C4), t, bc(D_C3)), t, bc(D_C2)), t, bc(D_C1)), t, bc(D_C0));
    const F2 cq = Q::fma(C, t, bc(1.0f));
    const F2 sq = Q::mul(S, r);
    const F2 rs = make_float2(__uint_as_float(__float_as_uint(rad.x) ^ (Ax & 0x80000000u)),
                              __uint_as_float(__float_as_uint(rad.y) ^ (Ay & 0x80000000u)));
    z.x = Q::mul(rs, cq);   // (-rad) * c == -(rad * c) bit for bit
    z.y = Q::mul(rs, sq);
}

// Objective node: e = |d * y_d - u*|^2 with y_d = rsqrt_spec(|d|^2 + 2^-126) and the
// difference fused per component (spec/MODELS.md §2).  Writing the fma here leaves no
// FMUL2 -> FADD2 pair for ptxas to contract behind our back (it does, .rn or not).
template <bool SC>
__device__ __forceinline__ F2 objective2(V2 d, V2 us) {
    using O = Ops<SC>;
    const F2 n2 = O::fma(d.y, d.y, O::fma(d.x, d.x, bc(0x1p-126f)));
    const F2 y = rsqrt2_from<SC>(n2, O::mul(n2, bc(-0.5f)));
    const F2 dx = O::fma(d.x, y, neg2(us.x)), dy = O::fma(d.y, y, neg2(us.y));
    return O::fma(dy, dy, O::mul(dx, dx));
}

// Philox4x32-10 on counter (i, s, t, 1): rounds 1-3 with their sample-invariant
// parts hoisted into PhiloxPP (computed once per thread), rounds 4-10 generic.
struct PhiloxPP {
    uint32_t a1, x3k, b_c1k, c3k, z3, k0, k1;
    __device__ __forceinline__ void init(uint32_t i, uint32_t t, uint32_t key0, uint32_t key1) {
        k0 = key0; k1 = key1;
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo(PHILOX_M0, i, hi0, lo0);                 // round 1: c0 = i
        mulhilo(PHILOX_M1, t, hi1, lo1);                 //          c2 = t
        a1 = hi1 ^ k0;                                   // x0 = a1 ^ s
        const uint32_t x1 = lo1, x2 = hi0 ^ 1u ^ k1, x3 = lo0;
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

// Scheduling variants (all bit-identical; tools/pp_tune.cu measures them):
// which two-lane steps run as scalar FFMA pairs instead of packed FFMA2.
enum : int {
    PP_SC_OBJECTIVE = 1,    // unit(d) + objective
    PP_SC_UNIT_PRED = 2,    // unit(o_pred - o_player)
    PP_SC_UNIT_PREY = 4,    // unit(o_prey - o_player)
    PP_SC_LN2 = 8,          // ln of entity 2 (player)
    PP_SC_RSQ2 = 16,        // sqrt of entity 2
    PP_SC_SC2 = 32,         // sincos of entity 2
};
#ifndef DISTILL_PP_MASK
#define DISTILL_PP_MASK 0
#endif
#ifndef DISTILL_PP_MINB
#define DISTILL_PP_MINB 0
#endif

// Full evaluation of allocation i (a1-a8): returns the cost C.
template <int MASK, bool PIPE>
__device__ __forceinline__ float pp_eval_alloc(const PPArgs& a, uint32_t i) {
    constexpr bool SOBJ = MASK & PP_SC_OBJECTIVE, SUPD = MASK & PP_SC_UNIT_PRED, SUPY = MASK & PP_SC_UNIT_PREY;
    constexpr bool SLN2 = MASK & PP_SC_LN2, SRS2 = MASK & PP_SC_RSQ2, SSC2 = MASK & PP_SC_SC2;
    // a1: mixed-radix decode, signal 0 most significant
    const uint32_t k2 = i % a.L2, r = i / a.L2;
    const uint32_t k1 = r % a.L1, k0 = r / a.L1;
    const float a0 = __ldg(a.levels + k0);
    const float a1 = __ldg(a.levels + a.L0 + k1);
    const float a2 = __ldg(a.levels + a.L0 + a.L1 + k2);
    const float dsig = __fadd_rn(a.sigma_min, -a.sigma_max);
    const float s0 = __fmaf_rn(a0, dsig, a.sigma_max);
    const float s1 = __fmaf_rn(a1, dsig, a.sigma_max);
    const float s2 = __fmaf_rn(a2, dsig, a.sigma_max);
    const float K = __fmaf_rn(a.w2, a2, __fmaf_rn(a.w1, a1, __fmul_rn(a.w0, a0)));

    // u* = unit(action(true positions)) on broadcast lanes
    const V2 P0 = {bc(a.prey_x), bc(a.prey_y)}, P1 = {bc(a.pred_x), bc(a.pred_y)};
    const V2 P2 = {bc(a.pl_x), bc(a.pl_y)};
    const F2 mk = bc(-a.kappa);
    const V2 up = vunit<false>(vsub<false>(P0, P2)), ud = vunit<false>(vsub<false>(P1, P2));
    const V2 us = vunit<false>({__ffma2_rn(mk, ud.x, up.x), __ffma2_rn(mk, ud.y, up.y)});

    PhiloxPP rng;
    rng.init(i, a.invocation, a.key0, a.key1);
    float acc = 0.0f;
    uint4 Xn, Yn;
    if (PIPE) { Xn = rng(0); Yn = rng(1); }
    for (uint32_t s = 0; s < a.n_samples; s += 2) {
        // a2: one Philox block per sample, two samples per iteration
        uint4 X, Y;
        if (PIPE) {            // software pipelining: next pair's Philox overlaps this pair's math
            X = Xn; Y = Yn;
            Xn = rng(s + 2); Yn = rng(s + 3);
        } else {
            X = rng(s); Y = rng(s + 1);
        }
        // a3: sextet packing -> three 2-D Box-Muller pairs (spec/RNG.md §6)
        V2 z0, z1, z2;
        bm_pair2<false, false, false>(X.x, Y.x, X.w << 16, Y.w << 16, z0);
        bm_pair2<false, false, false>(X.y, Y.y, X.w & 0xFFFF0000u, Y.w & 0xFFFF0000u, z1);
        bm_pair2<SLN2, SRS2, SSC2>(X.z, Y.z, (X.x << 24) | ((X.y & 0xFFu) << 16),
                                   (Y.x << 24) | ((Y.y & 0xFFu) << 16), z2);
        // a4: Obs -> Action -> Objective
        using O = Ops<false>;
        const V2 o0 = {O::fma(bc(s0), z0.x, P0.x), O::fma(bc(s0), z0.y, P0.y)};
        const V2 o1 = {O::fma(bc(s1), z1.x, P1.x), O::fma(bc(s1), z1.y, P1.y)};
        const V2 o2 = {O::fma(bc(s2), z2.x, P2.x), O::fma(bc(s2), z2.y, P2.y)};
        const V2 vp = vunit<SUPY>(vsub<SUPY>(o0, o2)), vd = vunit<SUPD>(vsub<SUPD>(o1, o2));
        const V2 d = {Ops<SOBJ>::fma(mk, vd.x, vp.x), Ops<SOBJ>::fma(mk, vd.y, vp.y)};
        const F2 e = objective2<SOBJ>(d, us);
        // a7: sequential sum in ascending sample order
        acc = __fadd_rn(acc, e.x);
        if (s + 1 < a.n_samples) acc = __fadd_rn(acc, e.y);
    }
    // a8: net of cost
    return __fadd_rn(__fdiv_rn(acc, __uint2float_rn(a.n_samples)), K);
}

// One thread per allocation; one atomicMin per block.
template <int BLOCK, int MASK = DISTILL_PP_MASK, int MINB = DISTILL_PP_MINB, bool PIPE = false>
__global__ void __launch_bounds__(BLOCK, MINB) pp_eval_grid_kernel(const PPArgs a) {
    const uint32_t tid = blockIdx.x * BLOCK + threadIdx.x;
    key64_t key = KEY_INIT;
    if (tid < a.count) {
        const uint32_t i = a.begin + tid;
        const float C = pp_eval_alloc<MASK, PIPE>(a, i);
        if (a.net) a.net[tid] = -C;
        key = make_key(C, i);
    }
    // a9: (value, index) argmin -> one atomic per block
    if (a.best) block_min_key_atomic<BLOCK>(key, a.best);
}

// Persistent variant: a fixed grid of resident blocks pulls BLOCK-allocation
// chunks from a device counter (zeroed by the caller before the launch), so
// the last wave has no idle SMs; keys are min-combined per block across chunks.
template <int BLOCK, int MASK = DISTILL_PP_MASK, int MINB = DISTILL_PP_MINB, bool PIPE = false>
__global__ void __launch_bounds__(BLOCK, MINB) pp_eval_grid_persistent_kernel(const PPArgs a,
                                                                               unsigned int* __restrict__ counter) {
    __shared__ unsigned int s_chunk;
    const uint32_t n_chunks = (a.count + BLOCK - 1) / BLOCK;
    key64_t key = KEY_INIT;
    for (;;) {
        if (threadIdx.x == 0) s_chunk = atomicAdd(counter, 1u);
        __syncthreads();
        const uint32_t c = s_chunk;
        __syncthreads();
        if (c >= n_chunks) break;
        const uint32_t tid = c * BLOCK + threadIdx.x;
        if (tid < a.count) {
            const uint32_t i = a.begin + tid;
            const float C = pp_eval_alloc<MASK, PIPE>(a, i);
            if (a.net) a.net[tid] = -C;
            const key64_t k = make_key(C, i);
            key = k < key ? k : key;
        }
    }
    if (a.best) block_min_key_atomic<BLOCK>(key, a.best);
}

}  // namespace distill
