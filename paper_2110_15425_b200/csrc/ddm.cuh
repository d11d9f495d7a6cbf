// ddm.cuh — K3 ddm_batch: fixed-trip Euler drift-diffusion Monte Carlo with
// first-passage latching and histogram reduction (spec/MODELS.md §4;
// PAPER.md P:466 DDM, Fig. 3; "build histograms of outcomes").
//
// One thread = one trial (RNG unit = global trial id); the walk runs all N
// steps (no divergence, reading Q14); stream-2 normals come in sextets, two
// Philox blocks (12 steps) at a time.  Per block: shared-memory u32 histograms
// -> one global u64 atomicAdd per non-empty bin at the end (grid-stride, so
// blocks are few and the flush is amortised over many trials).
#pragma once
#include "rng.cuh"
#include "trials.cuh"

namespace distill {

struct DDMArgs {
    float drift, noise, threshold, x0, dt, x_lo, x_hi;
    float leak, offset;                        // LCI mode only (spec/MODELS.md §5; drift = input I)
    uint32_t n_steps, rt_bin_steps, n_rt_bins, n_x_bins;
    uint32_t key0, key1;
    uint64_t trial_begin, n_trials;            // one launch: all units share the high word unit_hi
    uint32_t unit_hi;                          // (trial_begin + t) >> 32, the counter's c2 (uniform)
    uint32_t c2_a1, c2_x1;                     // round 1 of c2: hi(M1 c2) ^ key0, lo(M1 c2) (host)
    unsigned long long* __restrict__ rt_hist;  // [2*nb+1]
    unsigned long long* __restrict__ rt_sum;   // [2]
    unsigned long long* __restrict__ x_hist;   // [nx+2]
    const float4* __restrict__ rad_tab;        // device RT (spec/RNG.md §3)
};

// One integrator step: DDM x = fma(nsd, g, fma(dt, A, x)) (§4) or, in LCI
// mode, x = fma(nsd, g, fma(dt, fma(-leak, x, I), x) + offset) (§5), which is
// the DDM step bit for bit when leak = offset = 0 (Fig. 3).
template <bool LCI>
__device__ __forceinline__ float integ_step(const DDMArgs& a, float nsd, float g, float x) {
    if (LCI) return __fmaf_rn(nsd, g, __fadd_rn(__fmaf_rn(a.dt, __fmaf_rn(-a.leak, x, a.drift), x), a.offset));
    return __fmaf_rn(nsd, g, __fmaf_rn(a.dt, a.drift, x));
}

template <int BLOCK, int MINB = 0, bool LCI = false>
__global__ void __launch_bounds__(BLOCK, MINB) ddm_batch_kernel(const DDMArgs a) {
    extern __shared__ uint32_t s_hist[];  // [2*nb+1] rt bins then [nx+2] x bins
    __shared__ float4 s_rt[RT_ROWS];
    const uint32_t n_rt = 2 * a.n_rt_bins + 1, n_x = a.n_x_bins + 2, n_all = n_rt + n_x;
    for (uint32_t b = threadIdx.x; b < n_all; b += BLOCK) s_hist[b] = 0;
    stage_rad_table<BLOCK>(s_rt, a.rad_tab);      // (its barrier also covers the histogram clear)

    const float nsd = __fmul_rn(a.noise, __fsqrt_rn(a.dt));
    const float sc = __fdiv_rn(__uint2float_rn(a.n_x_bins), __fadd_rn(a.x_hi, -a.x_lo));
    const float fnx = __uint2float_rn(a.n_x_bins);
    const float z = a.threshold, nz = -a.threshold;
    unsigned long long sum_up = 0, sum_lo = 0;

    // Grid-stride over blocks of BLOCK consecutive trials with every lane
    // stepping (a lane past the end walks the block's first trial again and
    // records nothing), so the walk is warp-uniform control flow.
    for (uint64_t base = (uint64_t)blockIdx.x * BLOCK; base < a.n_trials; base += (uint64_t)gridDim.x * BLOCK) {
        const bool valid = base + threadIdx.x < a.n_trials;
        const uint64_t t = valid ? base + threadIdx.x : base;
        // c2 = the unit's high word, the same for every unit of the launch (the host
        // splits a range at multiples of 2^32), and its round-1 product comes with
        // the launch: with the uniform walk, a1 ^ k and its product M0 (a1 ^ k) for
        // block k are warp-uniform and run on the uniform datapath (one IMAD.WIDE
        // per Philox block fewer on the FMA pipe)
        PhiloxHoisted rng;
        rng.init_c2((uint32_t)(a.trial_begin + t), a.c2_a1, a.c2_x1, 2u, a.key0, a.key1);
        float x = a.x0;
        uint32_t st = 0, ch = 2;
        // 12 steps per pair of sextet blocks.  Latch test: (x >= z) || (x <= -z)
        // <=> |x| >= z for every z and non-NaN x (NaN fails both), so one
        // max-|x| over the 12 states (ALU pipe) finds the group that holds the
        // first passage.  The loop only records that group and the state it
        // started from (selects, no branch: the walk stays warp-uniform, which
        // keeps the uniform Philox product on the uniform datapath); after the
        // walk the group's 12 steps are replayed from that state with the same
        // normals and resolved step by step in the spec's order — the same
        // values, so the same passage.  The ragged last group is peeled.
        const uint32_t n12 = a.n_steps / 12;
        uint32_t jl = 0xFFFFFFFFu;   // the first group holding a passage (none yet)
        float xl = 0.0f;             // the state entering it
        for (uint32_t j = 0; j < n12; ++j) {
            float g[12], xs[12];
            acc_normals12(rng, s_rt, j, g);
            const float xin = x;
#pragma unroll
            for (int l = 0; l < 12; ++l) { x = integ_step<LCI>(a, nsd, g[l], x); xs[l] = x; }
            float m = fabsf(xs[0]);
#pragma unroll
            for (int l = 1; l < 12; ++l) m = fmaxf(m, fabsf(xs[l]));
            const bool hit = (jl == 0xFFFFFFFFu) & (m >= z);
            jl = hit ? j : jl;
            xl = hit ? xin : xl;
        }
        if (jl != 0xFFFFFFFFu) {
            float g[12];
            acc_normals12(rng, s_rt, jl, g);
            float xr = xl;
#pragma unroll
            for (int l = 0; l < 12; ++l) {
                xr = integ_step<LCI>(a, nsd, g[l], xr);
                if (st == 0) {
                    if (xr >= z) { st = 12 * jl + l + 1; ch = 0; }
                    else if (xr <= nz) { st = 12 * jl + l + 1; ch = 1; }
                }
            }
        }
        const uint32_t rem = a.n_steps - 12 * n12;
        if (rem) {
            float g[12];
            acc_normals_tail(rng, s_rt, n12, rem, g);
#pragma unroll
            for (int l = 0; l < 11; ++l) {
                if ((uint32_t)l < rem) {
                    x = integ_step<LCI>(a, nsd, g[l], x);
                    if (st == 0) {
                        if (x >= z) { st = 12 * n12 + l + 1; ch = 0; }
                        else if (x <= nz) { st = 12 * n12 + l + 1; ch = 1; }
                    }
                }
            }
        }
        if (!valid) continue;
        uint32_t rb;
        if (ch == 2) rb = 2 * a.n_rt_bins;
        else rb = ch * a.n_rt_bins + (st - 1) / a.rt_bin_steps;
        DCHECK(rb < n_rt);
        atomicAdd(&s_hist[rb], 1u);
        if (ch == 0) sum_up += st;
        else if (ch == 1) sum_lo += st;
        const float u = __fmul_rn(__fadd_rn(x, -a.x_lo), sc);
        uint32_t xb;
        if (u < 0.0f) xb = 0;
        else if (!(u < fnx)) xb = a.n_x_bins + 1;
        else xb = 1 + (uint32_t)u;
        DCHECK(xb < n_x);
        atomicAdd(&s_hist[n_rt + xb], 1u);
    }
    // rt sums: warp reduce then one atomic per warp
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        sum_up += __shfl_xor_sync(0xFFFFFFFFu, sum_up, off);
        sum_lo += __shfl_xor_sync(0xFFFFFFFFu, sum_lo, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (sum_up) atomicAdd(a.rt_sum + 0, sum_up);
        if (sum_lo) atomicAdd(a.rt_sum + 1, sum_lo);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < n_all; b += BLOCK) {
        const uint32_t v = s_hist[b];
        if (v) {
            if (b < n_rt) atomicAdd(a.rt_hist + b, (unsigned long long)v);
            else atomicAdd(a.x_hist + (b - n_rt), (unsigned long long)v);
        }
    }
}

// ---------------------------------------------------------------- DDM control grid
// spec/MODELS.md §6c (north star: every control allocation runs a DDM): grid
// (trial chunks, allocations) like the Stroop kernel; per allocation the
// drift A = fma(g_a, u0, A0) and threshold z = u1; a lane runs a trial until
// its first passage (at most N steps; R14b: the outputs are the boundary and
// the step), 12 steps per pair of sextet blocks with the max-|x| latch test of
// the batch kernel, then takes the next trial of its block; integer outcomes {n_correct (upper),
// n_undecided, rt_sum} block-reduced and added per allocation.  The value is
// stroop_finalize_kernel's binary64 formula (same counts, same cost form).
struct DdmgArgs {
    float A0, g_a, noise, dt;
    uint32_t n_steps, L0, L1, n_trials, trial_begin, trial_end, key0, key1, begin, count;
    const float* __restrict__ levels;
    unsigned long long* __restrict__ counts;   // [count][3]
    const float4* __restrict__ rad_tab;        // device RT (spec/RNG.md §3)
};

template <int BLOCK, int MINB = 0>
__global__ void __launch_bounds__(BLOCK, MINB) ddmg_sim_kernel(const DdmgArgs a, uint32_t alloc_off) {
    __shared__ float4 s_rt[RT_ROWS];
    __shared__ uint32_t s_next;
    uint32_t t_end;
    block_trial_range(a.trial_begin, a.trial_end, s_next, t_end);
    stage_rad_table<BLOCK>(s_rt, a.rad_tab);                  // (its barrier publishes s_next)
    const uint32_t t_alloc = alloc_off + blockIdx.y;
    const uint32_t i = a.begin + t_alloc;
    const uint32_t k1 = i % a.L1, k0 = i / a.L1;
    const float u0 = __ldg(a.levels + k0), u1 = __ldg(a.levels + a.L0 + k1);
    const float A = __fmaf_rn(a.g_a, u0, a.A0);
    const float z = u1, nz = -u1;
    const float nsd = __fmul_rn(a.noise, __fsqrt_rn(a.dt));
    const uint32_t n12 = a.n_steps / 12, rem = a.n_steps - 12 * n12;
    uint32_t n_corr = 0, n_und = 0;
    unsigned long long rts = 0;
    // trials stream until their first passage (R14b, trials.cuh)
    uint32_t j = next_trial(s_next, t_end);
    uint32_t st = 0, ch = 2, grp = 0;                             // ch: 0 correct (upper), 1 error, 2 none
    float x = 0.0f;
    PhiloxHoisted rng;
    auto start = [&](uint32_t jj) {
        const uint64_t unit = (uint64_t)i * a.n_trials + jj;
        rng.init((uint32_t)unit, (uint32_t)(unit >> 32), 2u, a.key0, a.key1);
        x = 0.0f; st = 0; ch = 2; grp = 0;
    };
    if (j < t_end) start(j);
    while (j < t_end) {
        if (grp < n12) {
            float g[12], xs[12];
            acc_normals12(rng, s_rt, grp, g);
#pragma unroll
            for (int l = 0; l < 12; ++l) { x = __fmaf_rn(nsd, g[l], __fmaf_rn(a.dt, A, x)); xs[l] = x; }
            // the first step with x >= z (correct, tested first) or x <= -z, from two
            // 12-bit masks: no branches in the resolution
            uint32_t mu = 0, ml = 0;
#pragma unroll
            for (int l = 0; l < 12; ++l) {
                mu |= (uint32_t)(xs[l] >= z) << l;
                ml |= (uint32_t)(xs[l] <= nz) << l;
            }
            if (mu | ml) {
                const int l = __ffs(mu | ml) - 1;
                ch = ((mu >> l) & 1u) ? 0u : 1u;
                st = 12 * grp + l + 1;
            }
            ++grp;
            if (st == 0 && grp < n12) continue;          // the trial goes on (the hot path)
        }
        if (st == 0 && rem) {                            // undecided through the last full group
            float g[12];
            acc_normals_tail(rng, s_rt, n12, rem, g);
#pragma unroll
            for (int l = 0; l < 11; ++l) {
                if ((uint32_t)l < rem) {
                    x = __fmaf_rn(nsd, g[l], __fmaf_rn(a.dt, A, x));
                    if (st == 0) {
                        if (x >= z) { st = 12 * n12 + l + 1; ch = 0; }
                        else if (x <= nz) { st = 12 * n12 + l + 1; ch = 1; }
                    }
                }
            }
        }
        if (ch == 2) ++n_und;
        else { n_corr += (ch == 0); rts += st; }
        j = next_trial(s_next, t_end);
        if (j < t_end) start(j);
    }
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

}  // namespace distill
