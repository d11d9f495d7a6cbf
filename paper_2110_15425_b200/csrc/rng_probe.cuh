// rng_probe.cuh — rows a2 (Philox4x32-10) and a3 (uniform -> normal) on their
// own: the device functions every hot kernel inlines (PhiloxHoisted, rad2,
// bm_polar2_fs, the sextet packing, acc_normals12 / acc_normals_tail), run
// over caller-chosen inputs so that they can be compared with the oracle
// directly rather than only through a model's outputs (spec/RNG.md §1-§6).
#pragma once
#include "rng.cuh"

namespace distill {

// rad_spec of n raw radius words, two per thread (the kernels' lane pairing).
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) rng_rad_kernel(const uint32_t* __restrict__ R, uint64_t n,
                                                        float* __restrict__ y, const float4* __restrict__ g_rt) {
    __shared__ float4 s_rt[RT_ROWS];
    stage_rad_table<BLOCK>(s_rt, g_rt);
    const uint64_t stride = 2ull * gridDim.x * BLOCK;
    for (uint64_t k = 2ull * ((uint64_t)blockIdx.x * BLOCK + threadIdx.x); k < n; k += stride) {
        const bool two = k + 1 < n;
        const uint32_t rx = R[k], ry = two ? R[k + 1] : rx;
        const F2 r = rad2(rx, ry, s_rt);
        y[k] = r.x;
        if (two) y[k + 1] = r.y;
    }
}

// Stream-2 normals 0 .. per_unit-1 of units unit_begin + u (DDM / Stroop RNG
// units), one thread per unit, exactly as the accumulator kernels draw them.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) rng_normals_acc_kernel(uint32_t key0, uint32_t key1, uint64_t unit_begin,
                                                                uint64_t n_units, uint32_t per_unit,
                                                                float* __restrict__ out,
                                                                const float4* __restrict__ g_rt) {
    __shared__ float4 s_rt[RT_ROWS];
    stage_rad_table<BLOCK>(s_rt, g_rt);
    const uint64_t u = (uint64_t)blockIdx.x * BLOCK + threadIdx.x;
    if (u >= n_units) return;
    const uint64_t unit = unit_begin + u;
    PhiloxHoisted rng;
    rng.init((uint32_t)unit, (uint32_t)(unit >> 32), 2u, key0, key1);
    float* o = out + u * per_unit;
    const uint32_t n12 = per_unit / 12, rem = per_unit - 12 * n12;
    for (uint32_t j = 0; j < n12; ++j) {
        float g[12];
        acc_normals12(rng, s_rt, j, g);
#pragma unroll
        for (int l = 0; l < 12; ++l) o[12 * j + l] = g[l];
    }
    if (rem) {
        float g[12];
        acc_normals_tail(rng, s_rt, n12, rem, g);
#pragma unroll
        for (int l = 0; l < 11; ++l)
            if ((uint32_t)l < rem) o[12 * n12 + l] = g[l];
    }
}

// Stream-1 sextets of allocations alloc_begin + t, samples 0 .. n_samples-1
// (the predator-prey observation noise): out[(t * S + s) * 6 + 2e + {0, 1}] =
// (z_cos, z_sin) of entity e, samples in pairs in the two lanes as in
// pp_eval_grid_kernel (which folds sigma into the radius instead of forming z).
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) rng_normals_pp_kernel(uint32_t key0, uint32_t key1, uint32_t alloc_begin,
                                                               uint32_t n_alloc, uint32_t n_samples,
                                                               uint32_t invocation, float* __restrict__ out,
                                                               const float4* __restrict__ g_rt) {
    __shared__ float4 s_rt[RT_ROWS];
    stage_rad_table<BLOCK>(s_rt, g_rt);
    const uint32_t t = blockIdx.x * BLOCK + threadIdx.x;
    if (t >= n_alloc) return;
    PhiloxHoisted rng;
    rng.init(alloc_begin + t, invocation, 1u, key0, key1);
    float* o = out + (uint64_t)t * n_samples * 6;
    for (uint32_t s = 0; s < n_samples; s += 2) {
        const bool two = s + 1 < n_samples;
        const uint4 X = rng(s), Y = two ? rng(s + 1) : X;
        const uint32_t RX[3] = {X.x, X.y, X.z}, RY[3] = {Y.x, Y.y, Y.z};
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const uint32_t wx = sextet_angle_word(X, e), wy = sextet_angle_word(Y, e);
            F2 rs, cq, sq;
            bm_polar2_fs<false, 0x7FFF00u>(RX[e], RY[e], wx, wy, wx, wy, s_rt, rs, cq, sq);
            const F2 zc = Ops<false>::mul(rs, cq), zs = Ops<false>::mul(rs, sq);
            o[6ull * s + 2 * e] = zc.x;
            o[6ull * s + 2 * e + 1] = zs.x;
            if (two) {
                o[6ull * (s + 1) + 2 * e] = zc.y;
                o[6ull * (s + 1) + 2 * e + 1] = zs.y;
            }
        }
    }
}

}  // namespace distill
