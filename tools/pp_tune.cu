// Scheduling-variant sweep for pp_eval_grid (tools only, not product code):
// every variant must produce bit-identical net values and key; prints ms and
// registers per variant on cfg3 (1e6 allocations x 100 samples).
// Round 2 adds the north star's two layout items as A/B variants:
//   SMEM levels  — the level table staged in shared memory instead of __ldg;
//   float4 store — each warp's 32 net values staged in shared memory and
//                  written by 8 lanes as float4 instead of 32 scalar stores.
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_2110_15425_b200/csrc/pp.cuh"
#include "../paper_2110_15425_b200/csrc/rad_table.h"
using namespace distill;

// Persistent variant: a fixed grid of resident blocks pulls BLOCK-allocation
// chunks from a device counter (zeroed by the caller before the launch).
template <int BLOCK, int MINB = DISTILL_PP_MINB, bool EVEN = false>
__global__ void __launch_bounds__(BLOCK, MINB) pp_eval_grid_persistent_kernel(const PPArgs a,
                                                                               unsigned int* __restrict__ counter) {
    __shared__ unsigned int s_chunk;
    __shared__ float4 s_rt[RT_ROWS];
    stage_rad_table_async<BLOCK>(s_rt, a.rad_tab);
    const uint32_t n_chunks = (a.count + BLOCK - 1) / BLOCK;
    const float2 ustar = pp_ustar_block(a);
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
            const float C = pp_eval_alloc<0, false, EVEN>(a, i, ustar, s_rt);
            if (a.net) a.net[tid] = -C;
            const key64_t k = make_key(C, i);
            key = k < key ? k : key;
        }
    }
    if (a.best) block_min_key_atomic<BLOCK>(key, a.best);
}

// Layout A/B variant of pp_eval_grid_kernel (SMEM_LEV, STORE4).
template <int BLOCK, int MINB, bool EVEN, bool SMEM_LEV, bool STORE4>
__global__ void __launch_bounds__(BLOCK, MINB) pp_eval_layout_kernel(const PPArgs a) {
    __shared__ float4 s_rt[RT_ROWS];
    __shared__ float s_lev[SMEM_LEV ? 1024 : 1];
    __shared__ float s_out[STORE4 ? BLOCK : 1];
    stage_rad_table_async<BLOCK>(s_rt, a.rad_tab);
    if (SMEM_LEV)
        for (uint32_t k = threadIdx.x; k < a.L0 + a.L1 + a.L2; k += BLOCK) s_lev[k] = __ldg(a.levels + k);
    const uint32_t tid = blockIdx.x * BLOCK + threadIdx.x;
    const float2 ustar = pp_ustar_block(a);
    key64_t key = KEY_INIT;
    float C = 0.0f;
    if (tid < a.count) {
        const uint32_t i = a.begin + tid;
        C = pp_eval_alloc<0, false, EVEN, SMEM_LEV>(a, i, ustar, s_rt, s_lev);
        key = make_key(C, i);
    }
    if (STORE4) {
        s_out[threadIdx.x] = -C;
        __syncwarp();
        const uint32_t lane = threadIdx.x & 31, w0 = threadIdx.x & ~31u;
        const uint32_t base = blockIdx.x * BLOCK + w0;
        if (lane < 8 && base + 4 * lane + 3 < a.count)
            reinterpret_cast<float4*>(a.net + base)[lane] = reinterpret_cast<const float4*>(s_out + w0)[lane];
        else if (lane < 8)
            for (uint32_t q = 0; q < 4; ++q)
                if (base + 4 * lane + q < a.count) a.net[base + 4 * lane + q] = s_out[w0 + 4 * lane + q];
    } else if (tid < a.count) {
        a.net[tid] = -C;
    }
    if (a.best) block_min_key_atomic<BLOCK>(key, a.best);
}

static unsigned int* g_counter = nullptr;

template <typename F>
void run(const char* name, PPArgs a, float* ref_net, key64_t ref_key, bool is_ref, F launch, int regs) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 8; ++rep) {
        cudaMemset(a.best, 0xFF, 8);
        cudaMemsetAsync(g_counter, 0, 4);
        cudaEventRecord(e0);
        launch();
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
    printf("%-34s regs %3d %8.4f ms  %.3e evals/s  %s\n", name, regs, best, (double)a.count * a.n_samples / (best * 1e-3),
           same ? "bit-identical" : "MISMATCH");
}

template <typename K> int regs_of(K k) { cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k); return fa.numRegs; }

int main() {
    const int L = 100;
    std::vector<float> lev(3 * L);
    for (int d = 0; d < 3; ++d) for (int k = 0; k < L; ++k) lev[d * L + k] = (float)k / (float)(L - 1);
    float* dl; cudaMalloc(&dl, lev.size() * 4); cudaMemcpy(dl, lev.data(), lev.size() * 4, cudaMemcpyHostToDevice);
    std::vector<float4> rt(RT_ROWS);
    build_rad_table(rt.data());
    float4* drt; cudaMalloc(&drt, RT_ROWS * 16); cudaMemcpy(drt, rt.data(), RT_ROWS * 16, cudaMemcpyHostToDevice);
    PPArgs a{};
    a.prey_x = 4; a.prey_y = 1; a.pred_x = -3; a.pred_y = 2; a.pl_x = 0; a.pl_y = 0;
    a.sigma_max = 2; a.sigma_min = 0.1f; a.kappa = 0.5f; a.w0 = a.w1 = a.w2 = 0.1f;
    a.L0 = a.L1 = a.L2 = L; a.n_samples = 100; a.invocation = 0; a.key0 = 42; a.key1 = 0;
    a.begin = 0; a.count = L * L * L; a.levels = dl; a.rad_tab = drt;
    cudaMalloc((void**)&a.net, a.count * 4); cudaMalloc((void**)&a.best, 8);
    std::vector<float> ref(a.count);
    cudaMalloc((void**)&g_counter, 4);
    const unsigned grid = (a.count + 127) / 128;
    run("shipped b128 minb7 (ref)", a, ref.data(), 0, true,
        [&] { pp_eval_grid_kernel<128, 0, 7, false, true><<<grid, 128>>>(a); },
        regs_of(pp_eval_grid_kernel<128, 0, 7, false, true>));
    key64_t rk; cudaMemcpy(&rk, a.best, 8, cudaMemcpyDeviceToHost);
    printf("ref key %016llx\n", (unsigned long long)rk);
    run("layout: ldg levels, scalar store", a, ref.data(), rk, false,
        [&] { pp_eval_layout_kernel<128, 7, true, false, false><<<grid, 128>>>(a); },
        regs_of(pp_eval_layout_kernel<128, 7, true, false, false>));
    run("layout: SMEM levels", a, ref.data(), rk, false,
        [&] { pp_eval_layout_kernel<128, 7, true, true, false><<<grid, 128>>>(a); },
        regs_of(pp_eval_layout_kernel<128, 7, true, true, false>));
    run("layout: float4 store", a, ref.data(), rk, false,
        [&] { pp_eval_layout_kernel<128, 7, true, false, true><<<grid, 128>>>(a); },
        regs_of(pp_eval_layout_kernel<128, 7, true, false, true>));
    run("layout: SMEM levels + float4 store", a, ref.data(), rk, false,
        [&] { pp_eval_layout_kernel<128, 7, true, true, true><<<grid, 128>>>(a); },
        regs_of(pp_eval_layout_kernel<128, 7, true, true, true>));
#define SHIP(B, N, name) run(name, a, ref.data(), rk, false, [&] { pp_eval_grid_kernel<B, 0, N, false, true><<<(a.count + B - 1) / B, B>>>(a); }, regs_of(pp_eval_grid_kernel<B, 0, N, false, true>))
    SHIP(128, 6, "b128 minb6");
    SHIP(128, 8, "b128 minb8");
    SHIP(128, 0, "b128 minb0");
    SHIP(256, 3, "b256 minb3");
    SHIP(256, 4, "b256 minb4");
    SHIP(64, 14, "b64 minb14");
    {
        int per_sm = 0, n_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pp_eval_grid_persistent_kernel<128, 7, true>, 128, 0);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
        const unsigned pg = per_sm * n_sm;
        run("persistent b128 minb7", a, ref.data(), rk, false,
            [&] { pp_eval_grid_persistent_kernel<128, 7, true><<<pg, 128>>>(a, g_counter); },
            regs_of(pp_eval_grid_persistent_kernel<128, 7, true>));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
