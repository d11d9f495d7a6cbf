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
void stroop(const char* name, StroopArgs a, bool ref) {
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, stroop_sim_kernel<BLOCK, MINB, TABLE>);
    // the library's launch shape (distill.cu launch_stroop): chunks capped so the
    // grid holds ~64 blocks per resident slot
    uint32_t chunks = (a.trial_end + BLOCK - 1) / BLOCK;
    const uint64_t want = 148ull * 8 * 64;
    if ((uint64_t)chunks * a.count > want) chunks = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(chunks, (want + a.count - 1) / a.count));
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
    printf("stroop %-18s b%4d minb%2d regs %3d %9.4f ms  %s\n", name, BLOCK, MINB, fa.numRegs, best,
           h == g_ref_st ? "identical" : "MISMATCH");
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
    const size_t n_all = 201 + 2 + 130;
    unsigned long long* buf; cudaMalloc(&buf, n_all * 8);
    d.rt_hist = buf; d.rt_sum = buf + 201; d.x_hist = buf + 203;
    ddm<128, 0>("ref", d, n_all, true);
    ddm<128, 6>("", d, n_all, false); ddm<128, 7>("", d, n_all, false); ddm<128, 8>("", d, n_all, false);
    ddm<256, 0>("", d, n_all, false); ddm<256, 3>("", d, n_all, false); ddm<256, 4>("", d, n_all, false);
    ddm<64, 0>("", d, n_all, false); ddm<64, 12>("", d, n_all, false); ddm<64, 16>("", d, n_all, false);
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
    stroop<128, 6, false>("ref (no table)", s, true);
    stroop<128, 6, true>("table", s, false);
    stroop<256, 0>("", s, false);
    stroop<256, 3>("", s, false); stroop<256, 4>("", s, false); stroop<128, 0>("", s, false);
    stroop<128, 6>("", s, false); stroop<128, 8>("", s, false); stroop<64, 0>("", s, false);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
