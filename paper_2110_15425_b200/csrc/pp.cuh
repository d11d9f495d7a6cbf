// pp.cuh — K1 pp_eval_grid: the fused predator-prey grid-search kernel.
//
// One thread owns one allocation of the grid (the paper's "each thread
// evaluates one point in the grid search space") and runs the whole
// compiled model for every sample in ascending order (spec/MODELS.md §2):
//   decode i -> levels -> sigma_e, K     (Control node)
//   per sample: Philox sextet -> 3 Box-Muller pairs -> Obs -> Action ->
//               Objective e = ||u_hat - u*||^2, acc += e
//   C = acc / S + K ; store V = -C ; key(C, i) -> warp/block min -> atomicMin
// State per thread is registers only (the paper's 7.5 kB MT19937 state per
// thread, becomes the Philox counter).
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
    key_t* __restrict__ best;                          // [1] or nullptr
};

struct f2 { float x, y; };

__device__ __forceinline__ f2 v_sub(f2 a, f2 b) { return {__fadd_rn(a.x, -b.x), __fadd_rn(a.y, -b.y)}; }

// unit(v) = v * rsqrt_spec(|v|^2), (0,0)-scaled when |v|^2 == 0 (spec/MODELS.md §2)
__device__ __forceinline__ f2 v_unit(f2 v) {
    const float n2 = __fmaf_rn(v.y, v.y, __fmul_rn(v.x, v.x));
    const float r = rsqrt_spec(n2);
    const float y = (n2 == 0.0f) ? 0.0f : r;
    return {__fmul_rn(v.x, y), __fmul_rn(v.y, y)};
}

// Action node: unit toward prey minus kappa * unit toward predator
__device__ __forceinline__ f2 action(f2 prey, f2 pred, f2 pl, float kappa) {
    const f2 up = v_unit(v_sub(prey, pl));
    const f2 ud = v_unit(v_sub(pred, pl));
    return {__fmaf_rn(-kappa, ud.x, up.x), __fmaf_rn(-kappa, ud.y, up.y)};
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) pp_eval_grid_kernel(const PPArgs a) {
    const uint32_t t = blockIdx.x * BLOCK + threadIdx.x;
    key_t k = KEY_INIT;
    if (t < a.count) {
        const uint32_t i = a.begin + t;
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
        const f2 py = {a.prey_x, a.prey_y}, pd = {a.pred_x, a.pred_y}, pl = {a.pl_x, a.pl_y};
        const f2 us = v_unit(action(py, pd, pl, a.kappa));

        float acc = 0.0f;
        for (uint32_t s = 0; s < a.n_samples; ++s) {
            // a2: one Philox block per sample (sextet packing, spec/RNG.md §6)
            const uint4 X = philox4x32_10(make_uint4(i, s, a.invocation, 1u), a.key0, a.key1);
            const uint32_t A0 = X.w << 16;
            const uint32_t A1 = X.w & 0xFFFF0000u;
            const uint32_t A2 = (X.x << 24) | ((X.y & 0xFFu) << 16) | ((X.z & 0xFFu) << 8);
            // a3: Box-Muller, one 2-D pair per entity
            f2 z0, z1, z2;
            bm_pair(X.x, A0, z0.x, z0.y);
            bm_pair(X.y, A1, z1.x, z1.y);
            bm_pair(X.z, A2, z2.x, z2.y);
            // a4: Obs -> Action -> Objective
            const f2 o0 = {__fmaf_rn(s0, z0.x, py.x), __fmaf_rn(s0, z0.y, py.y)};
            const f2 o1 = {__fmaf_rn(s1, z1.x, pd.x), __fmaf_rn(s1, z1.y, pd.y)};
            const f2 o2 = {__fmaf_rn(s2, z2.x, pl.x), __fmaf_rn(s2, z2.y, pl.y)};
            const f2 uh = v_unit(action(o0, o1, o2, a.kappa));
            const f2 dl = v_sub(uh, us);
            const float e = __fmaf_rn(dl.y, dl.y, __fmul_rn(dl.x, dl.x));
            acc = __fadd_rn(acc, e);      // a7: sequential sum, ascending s
        }
        // a8: net of cost
        const float C = __fadd_rn(__fdiv_rn(acc, __uint2float_rn(a.n_samples)), K);
        if (a.net) a.net[t] = -C;
        k = make_key(C, i);
    }
    // a9: (value, index) argmin -> one atomic per block
    if (a.best) block_min_key_atomic<BLOCK>(k, a.best);
}

}  // namespace distill
