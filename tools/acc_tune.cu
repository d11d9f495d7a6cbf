// Block/occupancy sweep for the accumulator kernels (DDM cfg2, Stroop cfg4 slice); tools only.
// Results must be identical to the reference variant (integer histograms / counts).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_2110_15425_b200/csrc/ddm.cuh"
#include "../paper_2110_15425_b200/csrc/stroop.cuh"
#include "../paper_2110_15425_b200/csrc/rad_table.h"
using namespace distill;

static std::vector<unsigned long long> g_ref_ddm, g_ref_st;

// Experiment: two DDM trials per thread stepped together (ILP), t and t + half.
template <int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) ddm_batch_x2_kernel(const DDMArgs a) {
    extern __shared__ uint32_t s_hist[];
    __shared__ float4 s_rt[RT_ROWS];
    const uint32_t n_rt = 2 * a.n_rt_bins + 1, n_x = a.n_x_bins + 2, n_all = n_rt + n_x;
    for (uint32_t b = threadIdx.x; b < n_all; b += BLOCK) s_hist[b] = 0;
    stage_rad_table<BLOCK>(s_rt, a.rad_tab);
    const float nsd = __fmul_rn(a.noise, __fsqrt_rn(a.dt));
    const float sc = __fdiv_rn(__uint2float_rn(a.n_x_bins), __fadd_rn(a.x_hi, -a.x_lo));
    const float fnx = __uint2float_rn(a.n_x_bins);
    const float z = a.threshold, nz = -a.threshold;
    unsigned long long sum_up = 0, sum_lo = 0;
    const uint64_t half = (a.n_trials + 1) / 2;
    for (uint64_t t = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; t < half; t += (uint64_t)gridDim.x * BLOCK) {
        const bool two = t + half < a.n_trials;
        PhiloxHoisted ra, rb;
        const uint64_t ua = a.trial_begin + t, ub = a.trial_begin + t + (two ? half : 0);
        ra.init((uint32_t)ua, (uint32_t)(ua >> 32), 2u, a.key0, a.key1);
        rb.init((uint32_t)ub, (uint32_t)(ub >> 32), 2u, a.key0, a.key1);
        float xa = a.x0, xb = a.x0;
        uint32_t sa = 0, ca = 2, sb = 0, cb = 2;
        const uint32_t n12 = a.n_steps / 12;
        for (uint32_t j = 0; j < n12; ++j) {
            float ga[12], gb[12], xsa[12], xsb[12];
            acc_normals12(ra, s_rt, j, ga);
            acc_normals12(rb, s_rt, j, gb);
#pragma unroll
            for (int l = 0; l < 12; ++l) {
                xa = __fmaf_rn(nsd, ga[l], __fmaf_rn(a.dt, a.drift, xa)); xsa[l] = xa;
                xb = __fmaf_rn(nsd, gb[l], __fmaf_rn(a.dt, a.drift, xb)); xsb[l] = xb;
            }
            float ma = fabsf(xsa[0]), mb = fabsf(xsb[0]);
#pragma unroll
            for (int l = 1; l < 12; ++l) { ma = fmaxf(ma, fabsf(xsa[l])); mb = fmaxf(mb, fabsf(xsb[l])); }
            if (sa == 0 && ma >= z) {
#pragma unroll
                for (int l = 0; l < 12; ++l)
                    if (sa == 0) { if (xsa[l] >= z) { sa = 12 * j + l + 1; ca = 0; } else if (xsa[l] <= nz) { sa = 12 * j + l + 1; ca = 1; } }
            }
            if (sb == 0 && mb >= z) {
#pragma unroll
                for (int l = 0; l < 12; ++l)
                    if (sb == 0) { if (xsb[l] >= z) { sb = 12 * j + l + 1; cb = 0; } else if (xsb[l] <= nz) { sb = 12 * j + l + 1; cb = 1; } }
            }
        }
        // (cfg2 has no ragged tail: N = 1000 = 83 * 12 + 4 -> handled per trial below)
        const uint32_t rem = a.n_steps - 12 * n12;
        for (int w = 0; w < (two ? 2 : 1); ++w) {
            PhiloxHoisted& r = w ? rb : ra;
            float& x = w ? xb : xa; uint32_t& st = w ? sb : sa; uint32_t& ch = w ? cb : ca;
            if (rem) {
                float g[12];
                acc_normals_tail(r, s_rt, n12, rem, g);
                for (int l = 0; l < 11; ++l) {
                    if ((uint32_t)l < rem) {
                        x = __fmaf_rn(nsd, g[l], __fmaf_rn(a.dt, a.drift, x));
                        if (st == 0) { if (x >= z) { st = 12 * n12 + l + 1; ch = 0; } else if (x <= nz) { st = 12 * n12 + l + 1; ch = 1; } }
                    }
                }
            }
            uint32_t bin = ch == 2 ? 2 * a.n_rt_bins : ch * a.n_rt_bins + (st - 1) / a.rt_bin_steps;
            atomicAdd(&s_hist[bin], 1u);
            if (ch == 0) sum_up += st; else if (ch == 1) sum_lo += st;
            const float u = __fmul_rn(__fadd_rn(x, -a.x_lo), sc);
            uint32_t xbn = u < 0.0f ? 0 : (!(u < fnx) ? a.n_x_bins + 1 : 1 + (uint32_t)u);
            atomicAdd(&s_hist[n_rt + xbn], 1u);
        }
    }
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
        if (v) { if (b < n_rt) atomicAdd(a.rt_hist + b, (unsigned long long)v); else atomicAdd(a.x_hist + (b - n_rt), (unsigned long long)v); }
    }
}

template <int BLOCK, int MINB>
void ddm_x2(const char* name, DDMArgs a, size_t n_all) {
    const uint32_t smem = (2 * a.n_rt_bins + 1 + a.n_x_bins + 2) * 4;
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, ddm_batch_x2_kernel<BLOCK, MINB>);
    const unsigned grid = (unsigned)(((a.n_trials + 1) / 2 + BLOCK - 1) / BLOCK);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaMemset(a.rt_hist, 0, n_all * 8);
        cudaEventRecord(e0);
        ddm_batch_x2_kernel<BLOCK, MINB><<<grid, BLOCK, smem>>>(a);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    std::vector<unsigned long long> h(n_all);
    cudaMemcpy(h.data(), a.rt_hist, n_all * 8, cudaMemcpyDeviceToHost);
    printf("ddm x2 %-18s b%4d minb%2d regs %3d %9.4f ms  %s\n", name, BLOCK, MINB, fa.numRegs, best,
           h == g_ref_ddm ? "identical" : "MISMATCH");
}

template <int BLOCK, int MINB>
void ddm(const char* name, DDMArgs a, size_t n_all, bool ref) {
    const uint32_t smem = (2 * a.n_rt_bins + 1 + a.n_x_bins + 2) * 4;
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, ddm_batch_kernel<BLOCK, MINB>);
    const unsigned grid = (unsigned)((a.n_trials + BLOCK - 1) / BLOCK);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
        cudaMemset(a.rt_hist, 0, n_all * 8);
        cudaEventRecord(e0);
        ddm_batch_kernel<BLOCK, MINB><<<grid, BLOCK, smem>>>(a);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    std::vector<unsigned long long> h(n_all);
    cudaMemcpy(h.data(), a.rt_hist, n_all * 8, cudaMemcpyDeviceToHost);
    if (ref) {
        g_ref_ddm = h;
        unsigned long long hsh = 1469598103934665603ull;
        for (auto v : h) hsh = (hsh ^ v) * 1099511628211ull;
        printf("ddm ref hash %016llx\n", hsh);
    }
    printf("ddm    %-18s b%4d minb%2d regs %3d %9.4f ms  %s\n", name, BLOCK, MINB, fa.numRegs, best,
           h == g_ref_ddm ? "identical" : "MISMATCH");
}

template <int BLOCK, int MINB, bool TABLE = true>
void stroop(const char* name, StroopArgs a, bool ref, uint32_t per_lane = 16, uint32_t fill_per_sm = 64) {
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, stroop_sim_kernel<BLOCK, MINB, TABLE>);
    // the library's launch shape (distill.cu trial_chunks): enough blocks to fill
    // `fill_per_sm` per SM, but at least `per_lane` trials per lane of a block
    const uint32_t tr = a.trial_end - a.trial_begin;
    const uint64_t want = (148ull * fill_per_sm + a.count - 1) / a.count;
    const uint64_t cap = std::max<uint64_t>(1, tr / (BLOCK * per_lane));
    const uint64_t most = std::max<uint64_t>(1, (tr + BLOCK - 1) / BLOCK);
    const uint32_t chunks = (uint32_t)std::max<uint64_t>(1, std::min(std::min(want, cap), most));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaMemset(a.counts, 0, a.count * 24);
        cudaEventRecord(e0);
        stroop_sim_kernel<BLOCK, MINB, TABLE><<<dim3(chunks, a.count), BLOCK, TABLE ? 16 * a.n_steps : 0>>>(a, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r && ms < best) best = ms;
    }
    std::vector<unsigned long long> h(a.count * 3);
    cudaMemcpy(h.data(), a.counts, a.count * 24, cudaMemcpyDeviceToHost);
    if (ref) {
        g_ref_st = h;
        unsigned long long hsh = 1469598103934665603ull;
        for (auto v : h) hsh = (hsh ^ v) * 1099511628211ull;
        printf("stroop ref hash %016llx\n", hsh);
    }
    printf("stroop %-18s b%4d minb%2d regs %3d lane>=%2u fill %3u chunks %4u %9.4f ms  %s\n", name, BLOCK, MINB,
           fa.numRegs, per_lane, fill_per_sm, chunks, best, h == g_ref_st ? "identical" : "MISMATCH");
}

int main() {
    std::vector<float4> rt(RT_ROWS);
    build_rad_table(rt.data());
    float4* drt; cudaMalloc(&drt, RT_ROWS * 16); cudaMemcpy(drt, rt.data(), RT_ROWS * 16, cudaMemcpyHostToDevice);
    // DDM cfg2
    DDMArgs d{};
    d.rad_tab = drt;
    d.drift = 1; d.noise = 1; d.threshold = 1; d.x0 = 0; d.dt = 0.01f;
    d.n_steps = 1000; d.rt_bin_steps = 10; d.n_rt_bins = 100; d.n_x_bins = 128;
    d.x_lo = 10.f - 6.f * 3.16227766f; d.x_hi = 10.f + 6.f * 3.16227766f;
    d.key0 = 42; d.key1 = 0; d.trial_begin = 0; d.n_trials = 1000000;
    d.unit_hi = 0; d.c2_a1 = d.key0; d.c2_x1 = 0;   // Philox round 1 of c2 = 0: M1 * 0 = 0 (the library's host does this)
    const size_t n_all = 201 + 2 + 130;
    unsigned long long* buf; cudaMalloc(&buf, n_all * 8);
    d.rt_hist = buf; d.rt_sum = buf + 201; d.x_hist = buf + 203;
    ddm<128, 0>("ref", d, n_all, true);
    ddm<128, 6>("", d, n_all, false); ddm<128, 7>("", d, n_all, false); ddm<128, 8>("", d, n_all, false);
    ddm<256, 0>("", d, n_all, false); ddm<256, 3>("", d, n_all, false); ddm<256, 4>("", d, n_all, false);
    ddm<64, 0>("", d, n_all, false); ddm<64, 12>("", d, n_all, false); ddm<64, 16>("", d, n_all, false);
    ddm_x2<128, 0>("2 trials/thread", d, n_all); ddm_x2<128, 4>("2 trials/thread", d, n_all);
    ddm_x2<128, 3>("2 trials/thread", d, n_all); ddm_x2<64, 8>("2 trials/thread", d, n_all);
    // Stroop cfg4 slice: 200 allocations x 1e5 trials
    std::vector<float> lev(200);
    for (int k = 0; k < 100; ++k) lev[k] = lev[100 + k] = (float)k / 99.f;
    float* dl; cudaMalloc(&dl, 800); cudaMemcpy(dl, lev.data(), 800, cudaMemcpyHostToDevice);
    StroopArgs s{};
    s.rad_tab = drt;
    s.g_c = 1; s.g_w = 1.5f; s.tau = 0.1f; s.leak = 0.2f; s.inh = 0.2f; s.noise = 0.5f; s.dt = 0.05f; s.thr = 1;
    s.reward = 1; s.rt_cost = 0.1f; s.n_steps = 200; s.w0 = 0.3f; s.w1 = 0.1f; s.L0 = 100; s.L1 = 100;
    s.n_trials = 100000; s.trial_begin = 0; s.trial_end = 100000; s.key0 = 42; s.key1 = 0;
    s.begin = 5000; s.count = 200; s.levels = dl;
    cudaMalloc((void**)&s.counts, 200 * 24);
    stroop<128, 0, true>("shipped (ref)", s, true);
    stroop<128, 0, false>("no table", s, false);
    for (uint32_t pl : {4u, 8u, 32u, 64u}) stroop<128, 0>("", s, false, pl);
    for (uint32_t fl : {32u, 128u, 256u}) stroop<128, 0>("", s, false, 16, fl);
    stroop<128, 6>("", s, false); stroop<128, 8>("", s, false);
    stroop<64, 0>("", s, false); stroop<64, 0>("", s, false, 32); stroop<64, 0>("", s, false, 16, 128);
    stroop<64, 12>("", s, false); stroop<64, 16>("", s, false);
    stroop<256, 0>("", s, false); stroop<256, 4>("", s, false); stroop<256, 0>("", s, false, 8);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
