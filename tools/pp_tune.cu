// Scheduling-variant sweep for pp_eval_grid (tools only, not product code):
// every variant must produce bit-identical net values and key; prints ms and
// registers per variant on cfg3 (1e6 allocations x 100 samples).
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_2110_15425_b200/csrc/pp.cuh"
using namespace distill;

template <int BLOCK, int MASK, int MINB>
void run(const char* name, PPArgs a, float* ref_net, key64_t ref_key, bool is_ref) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, pp_eval_grid_kernel<BLOCK, MASK, MINB>);
    const unsigned grid = (a.count + BLOCK - 1) / BLOCK;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaMemset(a.best, 0xFF, 8);
        cudaEventRecord(e0);
        pp_eval_grid_kernel<BLOCK, MASK, MINB><<<grid, BLOCK>>>(a);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    std::vector<float> h(a.count);
    cudaMemcpy(h.data(), a.net, a.count * 4, cudaMemcpyDeviceToHost);
    key64_t k; cudaMemcpy(&k, a.best, 8, cudaMemcpyDeviceToHost);
    bool same = true;
    if (is_ref) memcpy(ref_net, h.data(), a.count * 4);
    else same = memcmp(ref_net, h.data(), a.count * 4) == 0 && k == ref_key;
    const double flops = (double)a.count * (a.n_samples * 257.0 + 13) + 66;
    printf("%-28s block %4d mask %2d minb %d regs %3d  %8.4f ms  %6.2f TF/s  frac %.3f  %s\n", name, BLOCK, MASK, MINB,
           fa.numRegs, best, flops / best / 1e9, flops / best / 1e9 / 74.45, same ? "bit-identical" : "MISMATCH");
}

int main() {
    const int L = 100;
    std::vector<float> lev(3 * L);
    for (int d = 0; d < 3; ++d) for (int k = 0; k < L; ++k) lev[d * L + k] = (float)k / (float)(L - 1);
    float* dl; cudaMalloc(&dl, lev.size() * 4); cudaMemcpy(dl, lev.data(), lev.size() * 4, cudaMemcpyHostToDevice);
    PPArgs a{};
    a.prey_x = 4; a.prey_y = 1; a.pred_x = -3; a.pred_y = 2; a.pl_x = 0; a.pl_y = 0;
    a.sigma_max = 2; a.sigma_min = 0.1f; a.kappa = 0.5f; a.w0 = a.w1 = a.w2 = 0.1f;
    a.L0 = a.L1 = a.L2 = L; a.n_samples = 100; a.invocation = 0; a.key0 = 42; a.key1 = 0;
    a.begin = 0; a.count = L * L * L; a.levels = dl;
    cudaMalloc((void**)&a.net, a.count * 4); cudaMalloc((void**)&a.best, 8);
    std::vector<float> ref(a.count);
    run<256, 0, 0>("packed (ref)", a, ref.data(), 0, true);
    key64_t rk; cudaMemcpy(&rk, a.best, 8, cudaMemcpyDeviceToHost);
#define V(B, M, N, name) run<B, M, N>(name, a, ref.data(), rk, false)
    V(256, 0, 1, "packed minb1");
    V(256, 0, 2, "packed minb2");
    V(256, 0, 3, "packed minb3");
    V(256, 0, 4, "packed minb4");
    V(256, 0, 6, "packed minb6");
    V(256, 1, 0, "obj scalar");
    V(256, 2, 0, "unit pred scalar");
    V(256, 3, 0, "obj+unit pred");
    V(256, 7, 0, "obj+both units");
    V(256, 32, 0, "sincos2 scalar");
    V(256, 33, 0, "obj+sincos2");
    V(256, 56, 0, "entity2 BM scalar");
    V(256, 35, 0, "obj+pred+sincos2");
    V(256, 1, 4, "obj scalar minb4");
    V(256, 3, 4, "obj+pred minb4");
    V(256, 3, 3, "obj+pred minb3");
    V(256, 1, 2, "obj scalar minb2");
    V(128, 0, 0, "packed b128");
    V(128, 3, 0, "obj+pred b128");
    V(512, 0, 0, "packed b512");
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
