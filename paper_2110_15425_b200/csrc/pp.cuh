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
// P:632, becomes 6 words of Philox counter/key).  Grids too small to fill the
// GPU one thread per allocation use pp_eval_small_kernel (one warp per
// allocation, same per-pair code, same ordered sum).  Also here: the
// closed-loop episode step (NEXT-1) and the AMR level/refine kernels (NEXT-4).
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
    key64_t* __restrict__ best;                        // [1] or nullptr
    const float* __restrict__ pos_dev;                 // episode / multi: positions in device memory (or nullptr)
    const int* __restrict__ status_dev;                // episode: skip the launch when status[0] != 0
    uint32_t n_sets = 1;                               // multi: position sets; invocation t uses set t mod n_sets
    key64_t* publish = nullptr;                        // PUB: device alias of a mapped pinned host key
    unsigned int* done = nullptr;                      // PUB: block-completion counter (0 between launches)
    uint32_t key_signed = 0;                           // 1: best holds key ^ 2^63 (int64 MIN order)
    const float4* __restrict__ rad_tab = nullptr;      // device RT (spec/RNG.md §3), staged into smem
};

// Multi-invocation launches (distill_eval_grid_multi) put invocation t on
// blockIdx.y: RNG invocation + t, position set t mod n_sets, its own net row
// and key (pp_eval_grid_kernel<..., MULTI = true>).

__device__ __forceinline__ PPArgs pp_resolve_positions(const PPArgs& a) {
    PPArgs b = a;
    if (a.pos_dev) {
        b.prey_x = a.pos_dev[0]; b.prey_y = a.pos_dev[1];
        b.pred_x = a.pos_dev[2]; b.pred_y = a.pos_dev[3];
        b.pl_x = a.pos_dev[4]; b.pl_y = a.pos_dev[5];
    }
    return b;
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

// Action node (spec/MODELS.md §2): d = v_p + c v_d with c = -kappa |v_p| / |v_d|,
// i.e. |v_p| (unit(v_p) - kappa unit(v_d)); only its direction is used downstream.
// |v_p| / |v_d| = n_p rsqrt(n_p n_d): one rsqrt_spec (revision R22b).
template <bool SC>
__device__ __forceinline__ V2 action2(V2 q0, V2 q1, V2 q2, F2 mk) {
    using O = Ops<SC>;
    const V2 vp = vsub<SC>(q0, q2), vd = vsub<SC>(q1, q2);
    const F2 np = O::fma(vp.y, vp.y, O::fma(vp.x, vp.x, bc(0x1p-126f)));
    const F2 nd = O::fma(vd.y, vd.y, O::fma(vd.x, vd.x, bc(0x1p-126f)));
    const F2 pd = O::mul(np, nd);
    const F2 q = rsqrt2_from<SC>(pd, O::mul(pd, bc(-0.5f)));
    const F2 c = O::mul(O::mul(mk, np), q);
    return {O::fma(c, vd.x, vp.x), O::fma(c, vd.y, vp.y)};
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

// Scheduling variants (all bit-identical; tools/pp_tune.cu measures them):
// which two-lane steps run as scalar FFMA pairs instead of packed FFMA2.
enum : int {
    PP_SC_OBJECTIVE = 1,    // unit(d) + objective
    PP_SC_UNIT_PRED = 2,    // unit(o_pred - o_player)
    PP_SC_UNIT_PREY = 4,    // unit(o_prey - o_player)
    PP_SC_SC2 = 32,         // sincos of entity 2
};
#ifndef DISTILL_PP_MASK
#define DISTILL_PP_MASK 0
#endif
// Software pipelining of the sample loop (PIPE: the next pair's Philox blocks are
// drawn while this pair's math runs) frees enough registers for 8 blocks of 128
// per SM at 61 registers: cfg3 0.561 -> 0.549 ms, bit-identical (profiles/r02_ab_pipe.txt;
// without the pipelining, 64 registers and 8 blocks are slower, 0.580 ms).
#ifndef DISTILL_PP_MINB
#define DISTILL_PP_MINB 8
#endif
#ifndef DISTILL_PP_PIPE
#define DISTILL_PP_PIPE 1
#endif
#ifndef DISTILL_PP_UNROLL
#define DISTILL_PP_UNROLL 1
#endif

// Full evaluation of allocation i (a1-a8): returns the cost C.
// u* = unit(action(true positions)) (spec/MODELS.md §2), computed once per block.
__device__ __forceinline__ float2 pp_ustar(const PPArgs& a) {
    const V2 P0 = {bc(a.prey_x), bc(a.prey_y)}, P1 = {bc(a.pred_x), bc(a.pred_y)};
    const V2 P2 = {bc(a.pl_x), bc(a.pl_y)};
    const F2 mk = bc(-a.kappa);
    const V2 us = vunit<false>(action2<false>(P0, P1, P2, mk));
    return make_float2(us.x.x, us.y.x);
}

// Block-shared u*: thread 0 computes it, everyone reads it (one barrier).
__device__ __forceinline__ float2 pp_ustar_block(const PPArgs& a) {
    __shared__ float2 s_us;
    if (threadIdx.x == 0) s_us = pp_ustar(a);
    __syncthreads();
    return s_us;
}

// a3 + a4 for the sample pair whose Philox blocks are X (lane x) and Y (lane y):
// sextet packing -> three 2-D Box-Muller pairs (spec/RNG.md §6), observations
// p + sigma rad (cos, sin), Action, Objective.  Returns the two squared chords.
template <bool SOBJ, bool SSC2>
__device__ __forceinline__ F2 pp_pair_errors(const uint4& X, const uint4& Y, float s0, float s1, float s2,
                                             const V2& P0, const V2& P1, const V2& P2, F2 mk, const V2& us,
                                             const float4* __restrict__ rt) {
    F2 r0, c0, n0, r1, c1, n1, r2, c2, n2;
    {
        const uint32_t wx0 = sextet_angle_word(X, 0), wy0 = sextet_angle_word(Y, 0);
        const uint32_t wx1 = sextet_angle_word(X, 1), wy1 = sextet_angle_word(Y, 1);
        const uint32_t wx2 = sextet_angle_word(X, 2), wy2 = sextet_angle_word(Y, 2);
        bm_polar2_fs<false, 0x7FFF00u>(X.x, Y.x, wx0, wy0, wx0, wy0, rt, r0, c0, n0);
        bm_polar2_fs<false, 0x7FFF00u>(X.y, Y.y, wx1, wy1, wx1, wy1, rt, r1, c1, n1);
        bm_polar2_fs<SSC2, 0x7FFF00u>(X.z, Y.z, wx2, wy2, wx2, wy2, rt, r2, c2, n2);
    }
    using O = Ops<false>;
    const F2 q0 = O::mul(bc(s0), r0), q1 = O::mul(bc(s1), r1), q2 = O::mul(bc(s2), r2);
    const V2 o0 = {O::fma(q0, c0, P0.x), O::fma(q0, n0, P0.y)};
    const V2 o1 = {O::fma(q1, c1, P1.x), O::fma(q1, n1, P1.y)};
    const V2 o2 = {O::fma(q2, c2, P2.x), O::fma(q2, n2, P2.y)};
    const V2 d = action2<SOBJ>(o0, o1, o2, mk);
    return objective2<SOBJ>(d, us);
}

// SMEM_LEV (tools/pp_tune.cu A/B only): `lev` is a shared-memory copy of the level table.
template <int MASK, int PIPE, bool EVEN = false, bool SMEM_LEV = false>
__device__ __forceinline__ float pp_eval_alloc(const PPArgs& a, uint32_t i, float2 ustar,
                                               const float4* __restrict__ rt, const float* lev = nullptr) {
    constexpr bool SOBJ = MASK & PP_SC_OBJECTIVE;
    constexpr bool SSC2 = MASK & PP_SC_SC2;
    // a1: mixed-radix decode, signal 0 most significant
    const uint32_t k2 = i % a.L2, r = i / a.L2;
    const uint32_t k1 = r % a.L1, k0 = r / a.L1;
    const float a0 = SMEM_LEV ? lev[k0] : __ldg(a.levels + k0);
    const float a1 = SMEM_LEV ? lev[a.L0 + k1] : __ldg(a.levels + a.L0 + k1);
    const float a2 = SMEM_LEV ? lev[a.L0 + a.L1 + k2] : __ldg(a.levels + a.L0 + a.L1 + k2);
    const float dsig = __fadd_rn(a.sigma_min, -a.sigma_max);
    const float s0 = __fmaf_rn(a0, dsig, a.sigma_max);
    const float s1 = __fmaf_rn(a1, dsig, a.sigma_max);
    const float s2 = __fmaf_rn(a2, dsig, a.sigma_max);
    const float K = __fmaf_rn(a.w2, a2, __fmaf_rn(a.w1, a1, __fmul_rn(a.w0, a0)));

    const V2 P0 = {bc(a.prey_x), bc(a.prey_y)}, P1 = {bc(a.pred_x), bc(a.pred_y)};
    const V2 P2 = {bc(a.pl_x), bc(a.pl_y)};
    const F2 mk = bc(-a.kappa);
    const V2 us = {bc(ustar.x), bc(ustar.y)};

    PhiloxHoisted rng;
    rng.init(i, a.invocation, 1u, a.key0, a.key1);
    float acc = 0.0f;
    uint4 Xn, Yn;
    if (PIPE) { Xn = rng(0); Yn = rng(1); }
    constexpr int UNR = DISTILL_PP_UNROLL;
#pragma unroll UNR
    for (uint32_t s = 0; s < a.n_samples; s += 2) {
        // a2: one Philox block per sample, two samples per iteration
        uint4 X, Y;
        if (PIPE) {            // software pipelining: next pair's Philox overlaps this pair's math
            X = Xn; Y = Yn;
            Xn = rng(s + 2); Yn = rng(s + 3);
        } else {
            X = rng(s); Y = rng(s + 1);
        }
        const F2 e = pp_pair_errors<SOBJ, SSC2>(X, Y, s0, s1, s2, P0, P1, P2, mk, us, rt);
        // a7: sequential sum in ascending sample order
        acc = __fadd_rn(acc, e.x);
        if (EVEN || s + 1 < a.n_samples) acc = __fadd_rn(acc, e.y);
    }
    // a8: net of cost
    return __fadd_rn(__fdiv_rn(acc, __uint2float_rn(a.n_samples)), K);
}

// End-to-end call (distill_eval_grid_host), called by thread 0 of every block
// after its atomicMin: the last block to finish publishes the combined key
// straight into pinned host memory and re-arms the device key and counter for
// the next call, so the call is one launch with no memset and no copy.  The
// fence orders this block's atomicMin before its counter increment
// (threadFenceReduction pattern).
__device__ __forceinline__ void pp_publish_key(const PPArgs& a) {
    __threadfence();
    if (atomicAdd(a.done, 1u) == gridDim.x * gridDim.y - 1) {
        __threadfence();
        const key64_t k = atomicOr(a.best, 0ull);           // coherent read of the final key
        *reinterpret_cast<volatile key64_t*>(a.publish) = k;
        __threadfence_system();
        *a.best = KEY_INIT;
        *a.done = 0u;
    }
}

// Small grids (latency mode): LANES lanes per allocation (32: one warp; 8:
// four allocations per warp).  Sub-lane l evaluates the sample pairs
// (2l + 2·LANES·m, 2l + 1 + 2·LANES·m); the squared chords go to shared memory
// and sub-lane 0 adds them in ascending sample order, so C is the same sum as
// in the one-thread-per-allocation kernel, bit for bit.  Used when the grid is
// too small to fill the GPU one thread per allocation and n_samples <= SMAX.
template <int WARPS, int SMAX, int LANES = 32, bool PUB = false>
__global__ void __launch_bounds__(WARPS * 32) pp_eval_small_kernel(const PPArgs a0) {
    constexpr int GPW = 32 / LANES;                          // allocations per warp
    __shared__ float s_e[WARPS][GPW][SMAX];
    __shared__ float4 s_rt[RT_ROWS];
    if (a0.status_dev && *a0.status_dev != 0) return;   // episode already over (uniform branch)
    const PPArgs a = pp_resolve_positions(a0);
    stage_rad_table_async<WARPS * 32>(s_rt, a.rad_tab);   // completed by pp_ustar_block's barrier
    const float4* __restrict__ rt = s_rt;
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t grp = lane / LANES, sl = lane % LANES;
    const uint32_t tid = (blockIdx.x * WARPS + w) * GPW + grp;   // allocation within the launch
    const float2 ustar = pp_ustar_block(a);
    const bool valid = tid < a.count;
    const uint32_t i = a.begin + (valid ? tid : 0u);
    const uint32_t k2 = i % a.L2, r = i / a.L2;
    const uint32_t k1 = r % a.L1, k0 = r / a.L1;
    const float lv0 = __ldg(a.levels + k0);
    const float lv1 = __ldg(a.levels + a.L0 + k1);
    const float lv2 = __ldg(a.levels + a.L0 + a.L1 + k2);
    const float dsig = __fadd_rn(a.sigma_min, -a.sigma_max);
    const float s0 = __fmaf_rn(lv0, dsig, a.sigma_max);
    const float s1 = __fmaf_rn(lv1, dsig, a.sigma_max);
    const float s2 = __fmaf_rn(lv2, dsig, a.sigma_max);
    const float K = __fmaf_rn(a.w2, lv2, __fmaf_rn(a.w1, lv1, __fmul_rn(a.w0, lv0)));
    if (valid) {
        const V2 P0 = {bc(a.prey_x), bc(a.prey_y)}, P1 = {bc(a.pred_x), bc(a.pred_y)};
        const V2 P2 = {bc(a.pl_x), bc(a.pl_y)};
        const V2 us = {bc(ustar.x), bc(ustar.y)};
        PhiloxHoisted rng;
        rng.init(i, a.invocation, 1u, a.key0, a.key1);
        for (uint32_t s = 2 * sl; s < a.n_samples; s += 2 * LANES) {
            const F2 e = pp_pair_errors<false, false>(rng(s), rng(s + 1), s0, s1, s2, P0, P1, P2,
                                                             bc(-a.kappa), us, rt);
            DCHECK(s < (uint32_t)SMAX);
            s_e[w][grp][s] = e.x;
            DCHECK(s + 1 >= a.n_samples || s + 1 < (uint32_t)SMAX);
            if (s + 1 < a.n_samples) s_e[w][grp][s + 1] = e.y;
        }
    }
    __syncwarp();
    key64_t key = KEY_INIT;
    if (valid && sl == 0) {
        float acc = 0.0f;                                        // a7: ascending sample order
        for (uint32_t s = 0; s < a.n_samples; ++s) acc = __fadd_rn(acc, s_e[w][grp][s]);
        const float C = __fadd_rn(__fdiv_rn(acc, __uint2float_rn(a.n_samples)), K);
        if (a.net) a.net[tid] = -C;
        key = make_key(C, i);
    }
    if (a.best) block_min_key_atomic<WARPS * 32>(key, a.best, a.key_signed != 0);
    if (PUB && threadIdx.x == 0) pp_publish_key(a0);
}

// One thread per allocation; one atomicMin per block.
template <int BLOCK, int MASK = DISTILL_PP_MASK, int MINB = DISTILL_PP_MINB, int PIPE = DISTILL_PP_PIPE, bool EVEN = false,
          bool MULTI = false, bool PUB = false>
__global__ void __launch_bounds__(BLOCK, MINB) pp_eval_grid_kernel(const PPArgs a0) {
    if (a0.status_dev && *a0.status_dev != 0) return;   // episode already over (uniform branch)
    // Multi-invocation: only the invocation word and the position set feed the
    // sample loop; the output row/key pointers are formed after it (keeping them
    // live across the loop costs registers and ~4 % time).
    PPArgs a = a0;
    if (MULTI) {
        a.invocation = a0.invocation + blockIdx.y;
        a.pos_dev = a0.pos_dev + 6u * (blockIdx.y % a0.n_sets);
    }
    a = pp_resolve_positions(a);
    __shared__ float4 s_rt[RT_ROWS];
    stage_rad_table_async<BLOCK>(s_rt, a.rad_tab);      // completed by pp_ustar_block's barrier
    const uint32_t tid = blockIdx.x * BLOCK + threadIdx.x;
    const float2 ustar = pp_ustar_block(a);
    key64_t key = KEY_INIT;
    float C = 0.0f;
    if (tid < a.count) {
        const uint32_t i = a.begin + tid;
        C = pp_eval_alloc<MASK, PIPE, EVEN>(a, i, ustar, s_rt);
        key = make_key(C, i);
    }
    const size_t row = MULTI ? (size_t)blockIdx.y : 0;
    if (a0.net && tid < a0.count) a0.net[row * a0.count + tid] = -C;
    // a9: (value, index) argmin -> one atomic per block
    if (a0.best) block_min_key_atomic<BLOCK>(key, a0.best + row, a0.key_signed != 0);
    if (PUB && threadIdx.x == 0) pp_publish_key(a0);
}


// ---------------------------------------------------------------- NEXT-1
// Closed-loop episode step t (spec/MODELS.md §7): read the step's best key,
// draw the execution observation with the chosen attention (stream 4), move
// player / prey / predator, test capture, write positions t+1.  One thread.
struct EpisodeArgs {
    float v_pl, v_py, v_pd, rc;                        // speeds, capture radius
    float* __restrict__ traj;                          // [(T+1)*6]
    const key64_t* __restrict__ keys;                  // [T]
    int* __restrict__ status;                          // [2] {outcome, steps}
};

__device__ __forceinline__ float2 unit1(float vx, float vy) {
    const float n2 = __fmaf_rn(vy, vy, __fmaf_rn(vx, vx, 0x1p-126f));
    const float y = rsqrt_spec(n2);
    return make_float2(__fmul_rn(vx, y), __fmul_rn(vy, y));
}

__global__ void pp_episode_step_kernel(const PPArgs a, const EpisodeArgs e, uint32_t t) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const float* cur = e.traj + 6ull * t;
    float* nxt = e.traj + 6ull * (t + 1);
    if (e.status[0] != 0) {
        for (int k = 0; k < 6; ++k) nxt[k] = cur[k];
        return;
    }
    const key64_t best = e.keys[t];
    if ((best >> 32) == 0xFFFFFFFFull) {          // no valid allocation (all NaN)
        for (int k = 0; k < 6; ++k) nxt[k] = cur[k];
        e.status[0] = 3; e.status[1] = (int)(t + 1);
        return;
    }
    const uint32_t i = (uint32_t)best;
    const uint32_t k2 = i % a.L2, r = i / a.L2;
    const uint32_t k1 = r % a.L1, k0 = r / a.L1;
    const float dsig = __fadd_rn(a.sigma_min, -a.sigma_max);
    const float sg[3] = {__fmaf_rn(a.levels[k0], dsig, a.sigma_max),
                         __fmaf_rn(a.levels[a.L0 + k1], dsig, a.sigma_max),
                         __fmaf_rn(a.levels[a.L0 + a.L1 + k2], dsig, a.sigma_max)};
    const uint4 X = philox4x32_10(make_uint4(t, 0u, 0u, 4u), a.key0, a.key1);
    const uint32_t R[3] = {X.x, X.y, X.z};
    const uint32_t A[3] = {X.w << 16, X.w & 0xFFFF0000u, (X.x << 24) | ((X.y & 0xFFu) << 16)};
    float o[6];
    for (int q = 0; q < 3; ++q) {
        F2 rs, cq, sq;    // lane x only is used
        bm_polar2<true>(R[q], R[q], A[q], A[q], a.rad_tab, rs, cq, sq);
        const float sr = __fmul_rn(sg[q], rs.x);
        o[2 * q] = __fmaf_rn(sr, cq.x, cur[2 * q]);
        o[2 * q + 1] = __fmaf_rn(sr, sq.x, cur[2 * q + 1]);
    }
    const V2 q0 = {bc(o[0]), bc(o[1])}, q1 = {bc(o[2]), bc(o[3])}, q2 = {bc(o[4]), bc(o[5])};
    const V2 d = action2<true>(q0, q1, q2, bc(-a.kappa));
    const float2 up = unit1(d.x.x, d.y.x);
    const float2 uy = unit1(__fadd_rn(cur[0], -cur[4]), __fadd_rn(cur[1], -cur[5]));
    const float2 ud = unit1(__fadd_rn(cur[4], -cur[2]), __fadd_rn(cur[5], -cur[3]));
    const float plx = __fmaf_rn(e.v_pl, up.x, cur[4]), ply = __fmaf_rn(e.v_pl, up.y, cur[5]);
    const float pyx = __fmaf_rn(e.v_py, uy.x, cur[0]), pyy = __fmaf_rn(e.v_py, uy.y, cur[1]);
    const float pdx = __fmaf_rn(e.v_pd, ud.x, cur[2]), pdy = __fmaf_rn(e.v_pd, ud.y, cur[3]);
    nxt[0] = pyx; nxt[1] = pyy; nxt[2] = pdx; nxt[3] = pdy; nxt[4] = plx; nxt[5] = ply;
    const float rc2 = __fmul_rn(e.rc, e.rc);
    const float qyx = __fadd_rn(pyx, -plx), qyy = __fadd_rn(pyy, -ply);
    const float qdx = __fadd_rn(pdx, -plx), qdy = __fadd_rn(pdy, -ply);
    if (__fmaf_rn(qyy, qyy, __fmul_rn(qyx, qyx)) <= rc2) { e.status[0] = 1; e.status[1] = (int)(t + 1); }
    else if (__fmaf_rn(qdy, qdy, __fmul_rn(qdx, qdx)) <= rc2) { e.status[0] = 2; e.status[1] = (int)(t + 1); }
}

// ---------------------------------------------------------------- NEXT-4
// Coarse-to-fine refinement (spec/MODELS.md §9).  Round r: amr_levels_kernel
// writes the level table of box r, the grid search runs on it, and
// amr_refine_kernel shrinks the box to one level spacing around the best
// allocation.  Boxes live in device memory: boxes[r][d] = (lo, hi).
struct AmrArgs {
    float lo0[3], hi0[3];                      // initial box = clamp limits
    uint32_t L[3];
    float* __restrict__ levels;                // [L0+L1+L2] scratch
    float* __restrict__ boxes;                 // [(R+1)*6]
    const key64_t* __restrict__ keys;          // [R]
};

__device__ __forceinline__ float amr_step(float lo, float hi, uint32_t L) {
    return L > 1 ? __fdiv_rn(__fadd_rn(hi, -lo), __uint2float_rn(L - 1)) : 0.0f;
}

__global__ void amr_levels_kernel(const AmrArgs g, uint32_t r) {
    float* box = g.boxes + 6ull * r;
    if (r == 0 && threadIdx.x < 3) {          // round 0: the initial box from the launch parameters
        box[2 * threadIdx.x] = g.lo0[threadIdx.x];
        box[2 * threadIdx.x + 1] = g.hi0[threadIdx.x];
    }
    __syncthreads();
    const uint32_t total = g.L[0] + g.L[1] + g.L[2];
    for (uint32_t j = threadIdx.x; j < total; j += blockDim.x) {
        const uint32_t d = j < g.L[0] ? 0 : (j < g.L[0] + g.L[1] ? 1 : 2);
        const uint32_t k = j - (d == 0 ? 0 : (d == 1 ? g.L[0] : g.L[0] + g.L[1]));
        const float lo = box[2 * d], hi = box[2 * d + 1];
        g.levels[j] = __fmaf_rn(__uint2float_rn(k), amr_step(lo, hi, g.L[d]), lo);
    }
}

__global__ void amr_refine_kernel(const AmrArgs g, uint32_t r) {
    if (threadIdx.x != 0) return;
    const float* box = g.boxes + 6ull * r;
    float* nxt = g.boxes + 6ull * (r + 1);
    if ((g.keys[r] >> 32) == 0xFFFFFFFFull) {     // no valid allocation (all NaN): box unchanged (MODELS.md §9)
        for (int q = 0; q < 6; ++q) nxt[q] = box[q];
        return;
    }
    const uint32_t i = (uint32_t)g.keys[r];
    const uint32_t k2 = i % g.L[2], q = i / g.L[2];
    const uint32_t k[3] = {q / g.L[1], q % g.L[1], k2};
    uint32_t off = 0;
    for (int d = 0; d < 3; ++d) {
        const float lo = box[2 * d], hi = box[2 * d + 1];
        const float st = amr_step(lo, hi, g.L[d]);
        const float a = g.levels[off + k[d]];
        off += g.L[d];
        nxt[2 * d] = fmaxf(g.lo0[d], __fadd_rn(a, -st));
        nxt[2 * d + 1] = fminf(g.hi0[d], __fadd_rn(a, st));
    }
}

}  // namespace distill
