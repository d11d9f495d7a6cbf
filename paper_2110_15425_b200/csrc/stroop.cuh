// stroop.cuh — K4 stroop_eval_grid: Stroop-LCA control grid (spec/MODELS.md §6;
// PAPER.md P:525 Botvinick Stroop, LCA accumulation P:466).
//
// Simulate kernel: blockIdx.y = allocation, blocks along x stride over that
// allocation's trials; one thread = one (allocation, trial) simulation of
// N steps (pathway integration + 2-unit rectified LCA + first-passage latch).
// Outcomes are exact integers, block-reduced and atomically added per
// allocation, so the result is independent of the reduction order.
// Finalize kernel: per allocation V in binary64 from the integers, key, argmax.
#pragma once
#include "keys.cuh"
#include "rng.cuh"
#include "trials.cuh"

namespace distill {

struct StroopArgs {
    float g_c, g_w, tau, leak, inh, noise, dt, thr, reward, rt_cost;
    uint32_t n_steps;
    float w0, w1;
    uint32_t L0, L1;
    uint32_t n_trials, trial_begin, trial_end;
    uint32_t key0, key1;
    uint32_t begin, count;                     // allocation range of this launch
    const float* __restrict__ levels;          // L0 + L1 floats
    unsigned long long* __restrict__ counts;   // [count][3]
    float* __restrict__ net;
    key64_t* __restrict__ best;
    uint32_t key_signed;     // 1: best holds key ^ 2^63 (int64 MIN order)
    const float4* __restrict__ rad_tab;        // device RT (spec/RNG.md §3)
};

// One LCA step of both response units (spec/MODELS.md §6 loop body; the old
// x of both units feeds both q's), given the pathway outputs h0, h1 of this step.
__device__ __forceinline__ void lca_update(const StroopArgs& a, float nleak, float ninh, float nsd, float g0, float g1,
                                           float h0, float h1, float& x0, float& x1) {
    // the two units in the lanes of a float2: four FFMA2 per step, each lane rounding as the
    // scalar fma of the spec (q_k = fma(-β, x_{1-k}, fma(-λ, x_k, h_k)),
    // x_k = max(fma(σ√dt, g_k, fma(dt, q_k, x_k)), 0)); bit-identical, cfg4 -1.9 %
    // (profiles/r02_ab_lca_packed.txt)
    const F2 x = make_float2(x0, x1);
    const F2 q = __ffma2_rn(bc(ninh), make_float2(x1, x0), __ffma2_rn(bc(nleak), x, make_float2(h0, h1)));
    const F2 y = __ffma2_rn(bc(nsd), make_float2(g0, g1), __ffma2_rn(bc(a.dt), q, x));
    x0 = fmaxf(y.x, 0.0f);
    x1 = fmaxf(y.y, 0.0f);
}

// Pathway output of step n (1-based) for the trial's input row: the recurrence
// h = fma(τ, I - h, h) from h = 0 does not depend on the trial's noise, so
// TABLE kernels read it from a per-block table built once (rows: I = 0, ic,
// iw, ic + iw); otherwise it is advanced in registers.  Same values either way.
template <bool TABLE>
struct Pathway {
    const float* row0; const float* row1;   // TABLE
    uint32_t n_rows = 0;                    // TABLE: row length (bounds checks only)
    float I0, I1, tau, h0, h1;              // !TABLE
    __device__ __forceinline__ void at(uint32_t n, float& o0, float& o1) {
        if (TABLE) { DCHECK(n >= 1 && n <= n_rows); o0 = row0[n - 1]; o1 = row1[n - 1]; }
        else {
            h0 = __fmaf_rn(tau, __fadd_rn(I0, -h0), h0);
            h1 = __fmaf_rn(tau, __fadd_rn(I1, -h1), h1);
            o0 = h0; o1 = h1;
        }
    }
};

template <int BLOCK, int MINB = 0, bool TABLE = true>
__global__ void __launch_bounds__(BLOCK, MINB) stroop_sim_kernel(const StroopArgs a, uint32_t alloc_off) {
    extern __shared__ float s_htab[];                         // TABLE: [4][n_steps]
    __shared__ float4 s_rt[RT_ROWS];
    __shared__ uint32_t s_next;                               // next trial of this block's range
    uint32_t t_end;
    block_trial_range(a.trial_begin, a.trial_end, s_next, t_end);
    stage_rad_table<BLOCK>(s_rt, a.rad_tab);                  // (its barrier publishes s_next)
    const uint32_t t_alloc = alloc_off + blockIdx.y;           // index within [0, count)
    const uint32_t i = a.begin + t_alloc;
    const uint32_t k1 = i % a.L1, k0 = i / a.L1;
    const float uc = __ldg(a.levels + k0), us = __ldg(a.levels + a.L0 + k1);
    const float ic = __fmul_rn(a.g_c, uc);
    const float iw = __fmul_rn(a.g_w, __fadd_rn(1.0f, -us));
    const float nsd = __fmul_rn(a.noise, __fsqrt_rn(a.dt));
    const float nleak = -a.leak, ninh = -a.inh;
    const uint32_t N = a.n_steps;
    if (TABLE) {
        for (uint32_t n = threadIdx.x; n < N; n += BLOCK) s_htab[n] = 0.0f;   // row 0: I = 0 stays +0
        if (threadIdx.x >= 1 && threadIdx.x <= 3) {
            const float I = threadIdx.x == 1 ? __fadd_rn(ic, 0.0f) : threadIdx.x == 2 ? __fadd_rn(0.0f, iw)
                                                                   : __fadd_rn(ic, iw);
            float* row = s_htab + threadIdx.x * N;
            float h = 0.0f;
            for (uint32_t n = 0; n < N; ++n) { h = __fmaf_rn(a.tau, __fadd_rn(I, -h), h); row[n] = h; }
        }
        __syncthreads();
    }

    // Trials run until their response latches (R14b): the outputs are the
    // response and its step, so the steps after the latch are never computed.
    // Each lane streams trials from a per-block counter (contiguous block range,
    // integer sums are order-free), so a lane whose trial ends early starts the
    // next one instead of idling until the warp's slowest trial is done.
    uint32_t n_corr = 0, n_und = 0;
    unsigned long long rts = 0;
    const uint32_t n6 = N / 6, rem = N - 6 * n6;
    uint32_t j = next_trial(s_next, t_end);
    uint32_t colour = 0, grp = 0, st = 0;
    int resp = -1;
    float x0 = 0.f, x1 = 0.f;
    Pathway<TABLE> pw;
    PhiloxHoisted rng;
    auto start = [&](uint32_t jj) {
        const uint32_t kind = jj % 3;
        colour = (jj / 3) & 1;
        const int word = (kind == 0) ? (int)colour : (kind == 1) ? (int)(1 - colour) : -1;
        if (TABLE) {
            // table rows (1: colour input, 2: word input, 3: both) without branches: the
            // colour unit gets row 3 in congruent trials (word = colour) and 1 otherwise;
            // the other unit gets row 2 in incongruent trials (word = other) and 0 otherwise
            const uint32_t rc = kind == 0 ? 3u : 1u, ro = kind == 1 ? 2u : 0u;
            pw.n_rows = N;
            pw.row0 = s_htab + N * (colour == 0 ? rc : ro);
            pw.row1 = s_htab + N * (colour == 1 ? rc : ro);
        } else {
            pw.I0 = __fadd_rn(colour == 0 ? ic : 0.0f, word == 0 ? iw : 0.0f);
            pw.I1 = __fadd_rn(colour == 1 ? ic : 0.0f, word == 1 ? iw : 0.0f);
            pw.tau = a.tau; pw.h0 = 0.0f; pw.h1 = 0.0f;
        }
        const uint64_t unit = (uint64_t)i * a.n_trials + jj;
        rng.init((uint32_t)unit, (uint32_t)(unit >> 32), 2u, a.key0, a.key1);
        x0 = 0.f; x1 = 0.f; resp = -1; st = 0; grp = 0;
    };
    if (j < t_end) start(j);
    while (j < t_end) {
        if (grp < n6) {
            // Six steps (12 normals, two sextet blocks) per group, then the latch
            // test on the group's 12 states in the spec's order.
            float g[12], s0[6], s1[6];
            acc_normals12(rng, s_rt, grp, g);
#pragma unroll
            for (int l = 0; l < 6; ++l) {
                float h0, h1;
                pw.at(6 * grp + l + 1, h0, h1);
                lca_update(a, nleak, ninh, nsd, g[2 * l], g[2 * l + 1], h0, h1, x0, x1);
                s0[l] = x0; s1[l] = x1;
            }
            // the first step of the group with x0 >= θ or x1 >= θ, unit 0 first at a tie
            // (spec order), from two 6-bit masks: no branches in the resolution
            uint32_t m0 = 0, m1 = 0;
#pragma unroll
            for (int l = 0; l < 6; ++l) {
                m0 |= (uint32_t)(s0[l] >= a.thr) << l;
                m1 |= (uint32_t)(s1[l] >= a.thr) << l;
            }
            if (m0 | m1) {
                const int l = __ffs(m0 | m1) - 1;
                resp = ((m0 >> l) & 1u) ? 0 : 1;
                st = 6 * grp + l + 1;
            }
            ++grp;
            if (resp < 0 && grp < n6) continue;          // the trial goes on (the hot path)
        }
        if (resp < 0 && rem) {  // undecided through the last full group: the ragged last steps
            float g[12];
            acc_normals_tail(rng, s_rt, n6, 2 * rem, g);
#pragma unroll
            for (int l = 0; l < 5; ++l) {
                if ((uint32_t)l < rem) {
                    float h0, h1;
                    pw.at(6 * n6 + l + 1, h0, h1);
                    lca_update(a, nleak, ninh, nsd, g[2 * l], g[2 * l + 1], h0, h1, x0, x1);
                    if (resp < 0) {
                        if (x0 >= a.thr) { resp = 0; st = 6 * n6 + l + 1; }
                        else if (x1 >= a.thr) { resp = 1; st = 6 * n6 + l + 1; }
                    }
                }
            }
        }
        if (resp < 0) ++n_und;
        else { n_corr += ((uint32_t)resp == colour); rts += st; }
        j = next_trial(s_next, t_end);
        if (j < t_end) start(j);
    }
    // block reduction of the three integer outcomes
    __shared__ unsigned long long s_red[3][BLOCK / 32];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        n_corr += __shfl_xor_sync(0xFFFFFFFFu, n_corr, off);
        n_und += __shfl_xor_sync(0xFFFFFFFFu, n_und, off);
        rts += __shfl_xor_sync(0xFFFFFFFFu, rts, off);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { s_red[0][wid] = n_corr; s_red[1][wid] = n_und; s_red[2][wid] = rts; }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long v = 0;
        for (int w = 0; w < BLOCK / 32; ++w) v += s_red[threadIdx.x][w];
        if (v) atomicAdd(a.counts + 3ull * t_alloc + threadIdx.x, v);
    }
}

// Decision-energy trace of one allocation (spec/MODELS.md §6b; "the
// model is used to predict decision energy over time"): per step n, the
// product x0(n)·x1(n) of every trial, scaled by 2^24 (exact) and rounded to an
// integer, summed exactly over trials: a warp reduction per step, then one
// shared-memory atomic per warp and one global atomic per block and step.
// Trials run in uniform rounds so every lane of a warp reaches the shuffles.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) stroop_energy_kernel(const StroopArgs a, uint32_t alloc,
                                                              unsigned long long* __restrict__ esum) {
    extern __shared__ unsigned long long s_esum[];          // [n_steps]
    __shared__ float4 s_rt[RT_ROWS];
    const uint32_t N = a.n_steps;
    for (uint32_t n = threadIdx.x; n < N; n += BLOCK) s_esum[n] = 0ull;
    stage_rad_table<BLOCK>(s_rt, a.rad_tab);       // (its barrier also covers the clear)
    const uint32_t i = alloc;
    const uint32_t k1 = i % a.L1, k0 = i / a.L1;
    const float uc = __ldg(a.levels + k0), us = __ldg(a.levels + a.L0 + k1);
    const float ic = __fmul_rn(a.g_c, uc);
    const float iw = __fmul_rn(a.g_w, __fadd_rn(1.0f, -us));
    const float nsd = __fmul_rn(a.noise, __fsqrt_rn(a.dt));
    const float nleak = -a.leak, ninh = -a.inh;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t stride = gridDim.x * BLOCK;
    const uint32_t n_tr = a.trial_end - a.trial_begin;
    const uint32_t rounds = (n_tr + stride - 1) / stride;
    for (uint32_t rd = 0; rd < rounds; ++rd) {
        const uint32_t off = rd * stride + blockIdx.x * BLOCK + threadIdx.x;
        const bool valid = off < n_tr;
        const uint32_t j = a.trial_begin + (valid ? off : 0u);
        const uint32_t kind = j % 3, colour = (j / 3) & 1;
        const int word = (kind == 0) ? (int)colour : (kind == 1) ? (int)(1 - colour) : -1;
        Pathway<false> pw;
        pw.I0 = __fadd_rn(colour == 0 ? ic : 0.0f, word == 0 ? iw : 0.0f);
        pw.I1 = __fadd_rn(colour == 1 ? ic : 0.0f, word == 1 ? iw : 0.0f);
        pw.tau = a.tau; pw.h0 = 0.0f; pw.h1 = 0.0f;
        const uint64_t unit = (uint64_t)i * a.n_trials + j;
        PhiloxHoisted rng;
        rng.init((uint32_t)unit, (uint32_t)(unit >> 32), 2u, a.key0, a.key1);
        float x0 = 0.f, x1 = 0.f;
        float g[12];
        for (uint32_t n = 1; n <= N; ++n) {
            const uint32_t grp = (n - 1) / 6, l = (n - 1) % 6;
            if (l == 0) {                                    // normals of steps 6grp+1 .. 6grp+6
                if (N - 6 * grp >= 6) acc_normals12(rng, s_rt, grp, g);
                else acc_normals_tail(rng, s_rt, grp, 2 * (N - 6 * grp), g);
            }
            float h0, h1;
            pw.at(n, h0, h1);
            lca_update(a, nleak, ninh, nsd, g[2 * l], g[2 * l + 1], h0, h1, x0, x1);
            long long q = valid ? __float2ll_rn(__fmul_rn(__fmul_rn(x0, x1), 0x1p24f)) : 0ll;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xFFFFFFFFu, q, o);
            DCHECK(n >= 1 && n <= N);
            if (lane == 0 && q) atomicAdd(&s_esum[n - 1], (unsigned long long)q);
        }
    }
    __syncthreads();
    for (uint32_t n = threadIdx.x; n < N; n += BLOCK)
        if (s_esum[n]) atomicAdd(esum + n, s_esum[n]);
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) stroop_finalize_kernel(const StroopArgs a) {
    const uint32_t t = blockIdx.x * BLOCK + threadIdx.x;
    key64_t k = KEY_INIT;
    if (t < a.count) {
        const uint32_t i = a.begin + t;
        const uint32_t k1 = i % a.L1, k0 = i / a.L1;
        const float uc = __ldg(a.levels + k0), us = __ldg(a.levels + a.L0 + k1);
        const unsigned long long nc = a.counts[3ull * t], nu = a.counts[3ull * t + 1], rs = a.counts[3ull * t + 2];
        const double T = (double)a.n_trials, N = (double)a.n_steps;
        double v = __ddiv_rn(__dmul_rn((double)a.reward, (double)nc), T);
        v = __dsub_rn(v, __ddiv_rn(__dmul_rn(__dmul_rn((double)a.rt_cost, (double)a.dt),
                                             __dadd_rn((double)rs, __dmul_rn((double)nu, N))), T));
        v = __dsub_rn(v, __dadd_rn(__dmul_rn((double)a.w0, (double)uc), __dmul_rn((double)a.w1, (double)us)));
        const float V = __double2float_rn(v);
        if (a.net) a.net[t] = V;
        k = make_key(-V, i);
    }
    if (a.best) block_min_key_atomic<BLOCK>(k, a.best, a.key_signed != 0);
}

// ---------------------------------------------------------------- NEXT-3
// Extended Stroop A/B (spec/MODELS.md §10): the Stroop pathway
// front-end feeds two DDMs (colour naming, finger pointing) in one fused
// per-trial simulation.  VARIANT 0 = version A, 1 = version B: B computes the
// colour drift through two chained linear nodes, commutes the pointing fma and
// steps the pointing DDM first — exact rewrites, so the outputs are identical.
struct ExtStroopArgs {
    float g_c, g_w, tau, lam, a_p, gam, sig, dt, z, reward, rt_cost;
    uint32_t n_h, n_d;
    float w0, w1;
    uint32_t L0, L1, n_trials, trial_begin, trial_end, key0, key1, begin, count;
    const float* __restrict__ levels;
    unsigned long long* __restrict__ counts;   // [count][3] {n_both, n_undecided, rt_sum}
    float* __restrict__ net;
    key64_t* __restrict__ best;
    uint32_t key_signed;     // 1: best holds key ^ 2^63 (int64 MIN order)
    const float4* __restrict__ rad_tab;        // device RT (spec/RNG.md §3)
};

__device__ __forceinline__ void ddm_latch(float x, float z, uint32_t n, int& hit, uint32_t& st) {
    if (!hit) {
        if (x >= z) { hit = 1; st = n; }
        else if (x <= -z) { hit = 2; st = n; }
    }
}

template <int BLOCK, int VARIANT>
__global__ void __launch_bounds__(BLOCK) ext_stroop_sim_kernel(const ExtStroopArgs a, uint32_t alloc_off) {
    __shared__ float4 s_rt[RT_ROWS];
    __shared__ uint32_t s_next;
    uint32_t t_end;
    block_trial_range(a.trial_begin, a.trial_end, s_next, t_end);
    stage_rad_table<BLOCK>(s_rt, a.rad_tab);                  // (its barrier publishes s_next)
    const uint32_t t_alloc = alloc_off + blockIdx.y;
    const uint32_t i = a.begin + t_alloc;
    const uint32_t k1 = i % a.L1, k0 = i / a.L1;
    const float uc = __ldg(a.levels + k0), us = __ldg(a.levels + a.L0 + k1);
    const float ic = __fmul_rn(a.g_c, uc);
    const float iw = __fmul_rn(a.g_w, __fadd_rn(1.0f, -us));
    const float nsd = __fmul_rn(a.sig, __fsqrt_rn(a.dt));
    // The pathway front-end, the conflict energy and both drifts depend only on
    // the stimulus (kind, colour) and the allocation, not on the trial's noise:
    // six (kind, colour) combinations, computed once per block by six threads.
    __shared__ float s_drift[6][2];
    if (threadIdx.x < 6) {
        const uint32_t kind = threadIdx.x >> 1, colour = threadIdx.x & 1;
        const int word = (kind == 0) ? (int)colour : (kind == 1) ? (int)(1 - colour) : -1;
        const float I0 = __fadd_rn(colour == 0 ? ic : 0.0f, word == 0 ? iw : 0.0f);
        const float I1 = __fadd_rn(colour == 1 ? ic : 0.0f, word == 1 ? iw : 0.0f);
        float h0 = 0.0f, h1 = 0.0f;
        for (uint32_t n = 0; n < a.n_h; ++n) {                 // pathway front-end
            h0 = __fmaf_rn(a.tau, __fadd_rn(I0, -h0), h0);
            h1 = __fmaf_rn(a.tau, __fadd_rn(I1, -h1), h1);
        }
        const float E = __fmul_rn(h0, h1);                     // decision (conflict) energy
        const float hc = colour ? h1 : h0, hw = colour ? h0 : h1;
        float A1, A2;
        if (VARIANT == 0) {
            A1 = __fmul_rn(__fadd_rn(hc, -hw), a.lam);
            A2 = __fmaf_rn(-a.gam, E, a.a_p);
        } else {
            A2 = __fmaf_rn(E, -a.gam, a.a_p);
            A1 = __fmul_rn(__fmul_rn(__fadd_rn(hc, -hw), __fmul_rn(2.0f, a.lam)), 0.5f);
        }
        s_drift[threadIdx.x][0] = A1;
        s_drift[threadIdx.x][1] = A2;
    }
    __syncthreads();
    uint32_t n_both = 0, n_und = 0;
    unsigned long long rts = 0;
    // Trials stream until both DDMs have latched (R14b, trials.cuh): the outputs
    // are the two first passages, so no step after the later one is computed.
    const uint32_t n6 = a.n_d / 6, rem = a.n_d - 6 * n6;
    uint32_t j = next_trial(s_next, t_end);
    float A1 = 0.f, A2 = 0.f, x1 = 0.f, x2 = 0.f;
    int h1t = 0, h2t = 0;
    uint32_t s1 = 0, s2 = 0, grp = 0;
    PhiloxHoisted rng;
    auto start = [&](uint32_t jj) {
        const uint32_t kind = jj % 3, colour = (jj / 3) & 1;
        A1 = s_drift[2 * kind + colour][0]; A2 = s_drift[2 * kind + colour][1];
        const uint64_t unit = (uint64_t)i * a.n_trials + jj;
        rng.init((uint32_t)unit, (uint32_t)(unit >> 32), 2u, a.key0, a.key1);
        x1 = 0.f; x2 = 0.f; h1t = 0; h2t = 0; s1 = 0; s2 = 0; grp = 0;
    };
    if (j < t_end) start(j);
    while (j < t_end) {
        if (grp < n6) {
            // Six steps (12 normals) per group, then each DDM's latch test.
            float g[12], y1[6], y2[6];
            acc_normals12(rng, s_rt, grp, g);
#pragma unroll
            for (int l = 0; l < 6; ++l) {
                if (VARIANT == 0) {
                    x1 = __fmaf_rn(nsd, g[2 * l], __fmaf_rn(a.dt, A1, x1));
                    x2 = __fmaf_rn(nsd, g[2 * l + 1], __fmaf_rn(a.dt, A2, x2));
                } else {
                    x2 = __fmaf_rn(nsd, g[2 * l + 1], __fmaf_rn(a.dt, A2, x2));
                    x1 = __fmaf_rn(nsd, g[2 * l], __fmaf_rn(a.dt, A1, x1));
                }
                y1[l] = x1; y2[l] = x2;
            }
            // each DDM's first passage in the group (upper tested first, spec order)
            // from bit masks of the six states: no branches in the resolution
            uint32_t u1 = 0, d1 = 0, u2 = 0, d2 = 0;
#pragma unroll
            for (int l = 0; l < 6; ++l) {
                u1 |= (uint32_t)(y1[l] >= a.z) << l;  d1 |= (uint32_t)(y1[l] <= -a.z) << l;
                u2 |= (uint32_t)(y2[l] >= a.z) << l;  d2 |= (uint32_t)(y2[l] <= -a.z) << l;
            }
            if (!h1t && (u1 | d1)) {
                const int l = __ffs(u1 | d1) - 1;
                h1t = ((u1 >> l) & 1u) ? 1 : 2;
                s1 = 6 * grp + l + 1;
            }
            if (!h2t && (u2 | d2)) {
                const int l = __ffs(u2 | d2) - 1;
                h2t = ((u2 >> l) & 1u) ? 1 : 2;
                s2 = 6 * grp + l + 1;
            }
            ++grp;
            if (!(h1t && h2t) && grp < n6) continue;     // the trial goes on (the hot path)
        }
        if (!(h1t && h2t) && rem) {  // a DDM still open after the last full group: the ragged steps
            float g[12];
            acc_normals_tail(rng, s_rt, n6, 2 * rem, g);
#pragma unroll
            for (int l = 0; l < 5; ++l) {
                if ((uint32_t)l < rem) {
                    x1 = __fmaf_rn(nsd, g[2 * l], __fmaf_rn(a.dt, A1, x1));
                    x2 = __fmaf_rn(nsd, g[2 * l + 1], __fmaf_rn(a.dt, A2, x2));
                    ddm_latch(x1, a.z, 6 * n6 + l + 1, h1t, s1);
                    ddm_latch(x2, a.z, 6 * n6 + l + 1, h2t, s2);
                }
            }
        }
        if (h1t == 0 || h2t == 0) ++n_und;
        else { n_both += (h1t == 1 && h2t == 1); rts += s1 > s2 ? s1 : s2; }
        j = next_trial(s_next, t_end);
        if (j < t_end) start(j);
    }
    __shared__ unsigned long long s_red[3][BLOCK / 32];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        n_both += __shfl_xor_sync(0xFFFFFFFFu, n_both, off);
        n_und += __shfl_xor_sync(0xFFFFFFFFu, n_und, off);
        rts += __shfl_xor_sync(0xFFFFFFFFu, rts, off);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { s_red[0][wid] = n_both; s_red[1][wid] = n_und; s_red[2][wid] = rts; }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long v = 0;
        for (int w = 0; w < BLOCK / 32; ++w) v += s_red[threadIdx.x][w];
        if (v) atomicAdd(a.counts + 3ull * t_alloc + threadIdx.x, v);
    }
}

template <int BLOCK, int VARIANT>
__global__ void __launch_bounds__(BLOCK) ext_stroop_finalize_kernel(const ExtStroopArgs a) {
    const uint32_t t = blockIdx.x * BLOCK + threadIdx.x;
    key64_t k = KEY_INIT;
    if (t < a.count) {
        const uint32_t i = a.begin + t;
        const uint32_t k1 = i % a.L1, k0 = i / a.L1;
        const float uc = __ldg(a.levels + k0), us = __ldg(a.levels + a.L0 + k1);
        const unsigned long long nb = a.counts[3ull * t], nu = a.counts[3ull * t + 1], rs = a.counts[3ull * t + 2];
        const double T = (double)a.n_trials, N = (double)a.n_d;
        double v;
        if (VARIANT == 0) {
            v = __ddiv_rn(__dmul_rn((double)a.reward, (double)nb), T);
        } else {
            const unsigned long long n_fail = (unsigned long long)a.n_trials - nb;
            v = __ddiv_rn(__dmul_rn((double)a.reward, (double)((unsigned long long)a.n_trials - n_fail)), T);
        }
        v = __dsub_rn(v, __ddiv_rn(__dmul_rn(__dmul_rn((double)a.rt_cost, (double)a.dt),
                                             __dadd_rn((double)rs, __dmul_rn((double)nu, N))), T));
        v = __dsub_rn(v, __dadd_rn(__dmul_rn((double)a.w0, (double)uc), __dmul_rn((double)a.w1, (double)us)));
        const float V = __double2float_rn(v);
        if (a.net) a.net[t] = V;
        k = make_key(-V, i);
    }
    if (a.best) block_min_key_atomic<BLOCK>(k, a.best, a.key_signed != 0);
}

}  // namespace distill
