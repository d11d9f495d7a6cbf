// Debug trace: per-sample normals and objective e of the packed PP pipeline,
// for comparison with the oracle (tools/pp_trace_compare.py).  Not product code.
#include <cstdio>
#include <vector>
#include "../paper_2110_15425_b200/csrc/pp.cuh"
using namespace distill;

__global__ void trace(PPArgs a, float* out_z, float* out_e) {
    const uint32_t tid = threadIdx.x;
    if (tid >= a.count) return;
    const uint32_t i = a.begin + tid;
    const uint32_t k2 = i % a.L2, r = i / a.L2;
    const uint32_t k1 = r % a.L1, k0 = r / a.L1;
    const float a0 = a.levels[k0], a1 = a.levels[a.L0 + k1], a2 = a.levels[a.L0 + a.L1 + k2];
    const float dsig = __fadd_rn(a.sigma_min, -a.sigma_max);
    const float s0 = __fmaf_rn(a0, dsig, a.sigma_max), s1 = __fmaf_rn(a1, dsig, a.sigma_max), s2 = __fmaf_rn(a2, dsig, a.sigma_max);
    const V2 P0 = {bc(a.prey_x), bc(a.prey_y)}, P1 = {bc(a.pred_x), bc(a.pred_y)}, P2 = {bc(a.pl_x), bc(a.pl_y)};
    const F2 mk = bc(-a.kappa);
    V2 up = vunit(vsub(P0, P2)), ud = vunit(vsub(P1, P2));
    const V2 us = vunit({fma2(mk, ud.x, up.x), fma2(mk, ud.y, up.y)});
    PhiloxPP rng; rng.init(i, a.invocation, a.key0, a.key1);
    for (uint32_t s = 0; s < a.n_samples; s += 2) {
        const uint4 X = rng(s), Y = rng(s + 1);
        V2 z0, z1, z2;
        bm_pair2(X.x, Y.x, X.w << 16, Y.w << 16, z0);
        bm_pair2(X.y, Y.y, X.w & 0xFFFF0000u, Y.w & 0xFFFF0000u, z1);
        bm_pair2(X.z, Y.z, (X.x << 24) | ((X.y & 0xFFu) << 16), (Y.x << 24) | ((Y.y & 0xFFu) << 16), z2);
        const V2 o0 = {fma2(bc(s0), z0.x, P0.x), fma2(bc(s0), z0.y, P0.y)};
        const V2 o1 = {fma2(bc(s1), z1.x, P1.x), fma2(bc(s1), z1.y, P1.y)};
        const V2 o2 = {fma2(bc(s2), z2.x, P2.x), fma2(bc(s2), z2.y, P2.y)};
        const V2 vp = vunit(vsub(o0, o2)), vd = vunit(vsub(o1, o2));
        const F2 e = objective2({fma2(mk, vd.x, vp.x), fma2(mk, vd.y, vp.y)}, us);
        float zz[2][6] = {{z0.x.x, z0.y.x, z1.x.x, z1.y.x, z2.x.x, z2.y.x}, {z0.x.y, z0.y.y, z1.x.y, z1.y.y, z2.x.y, z2.y.y}};
        for (int l = 0; l < 2; ++l) {
            if (s + l >= a.n_samples) break;
            for (int q = 0; q < 6; ++q) out_z[((size_t)tid * a.n_samples + s + l) * 6 + q] = zz[l][q];
            out_e[(size_t)tid * a.n_samples + s + l] = l ? e.y : e.x;
        }
    }
}

int main(int argc, char** argv) {
    // cfg1: 27 allocations x 10 samples, seed 42 (workloads.pp_cfg1)
    float lev[9] = {0, 0.5f, 1, 0, 0.5f, 1, 0, 0.5f, 1};
    float* dl; cudaMalloc(&dl, sizeof lev); cudaMemcpy(dl, lev, sizeof lev, cudaMemcpyHostToDevice);
    PPArgs a{};
    a.prey_x = 4; a.prey_y = 1; a.pred_x = -3; a.pred_y = 2; a.pl_x = 0; a.pl_y = 0;
    a.sigma_max = 2; a.sigma_min = 0.1f; a.kappa = 0.5f; a.w0 = a.w1 = a.w2 = 0.1f;
    a.L0 = a.L1 = a.L2 = 3; a.n_samples = 10; a.invocation = 0; a.key0 = 42; a.key1 = 0;
    a.begin = 0; a.count = 27; a.levels = dl;
    float *dz, *de; cudaMalloc(&dz, 27 * 10 * 6 * 4); cudaMalloc(&de, 27 * 10 * 4);
    trace<<<1, 32>>>(a, dz, de);
    std::vector<float> z(27 * 60), e(270);
    cudaMemcpy(z.data(), dz, z.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(e.data(), de, e.size() * 4, cudaMemcpyDeviceToHost);
    FILE* f = fopen(argc > 1 ? argv[1] : "pp_trace.bin", "wb");
    fwrite(z.data(), 4, z.size(), f);
    fwrite(e.data(), 4, e.size(), f);
    fclose(f);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
