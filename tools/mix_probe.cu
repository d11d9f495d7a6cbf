// Speed-of-light for pp_eval_grid's instruction mix (tools only).
//
// The shipped kernel's inner loop (two samples per iteration) issues, per warp
// (cuobjdump of pp_eval_grid_kernel<128,0,7,false,true>, loop body):
//   116 FFMA2, 31 FMUL2, 10 FADD2, 2 FADD, 30 IMAD.WIDE.U32, 1 IMAD,
//   64 LOP3, 24 SHF, 24 IADD3, 12 I2FP, 6 VIADD, 6 PRMT   (~336 instructions)
// This probe issues the same mix from 8 independent dependency chains per
// thread (no data-dependence stalls), at the kernel's occupancy (128-thread
// blocks, 7 per SM), and reports SMSP cycles per iteration: the best any
// schedule of this instruction mix can do on the B200's pipes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N_ITER 256

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

template <int ALU_PCT>   // percentage of the loop's integer/logic instructions kept (100 = the kernel's mix)
__global__ void __launch_bounds__(128, 7) k_mix(float* out, float s, uint32_t m) {
    float2 f[8], fm[4], fa[4];
    uint32_t u[8];
    float g[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) { f[j] = make_float2(threadIdx.x + j, j); u[j] = threadIdx.x * 7u + j; }
#pragma unroll
    for (int j = 0; j < 4; ++j) { fm[j] = make_float2(threadIdx.x + 3 * j, j); fa[j] = make_float2(j, threadIdx.x); }
#pragma unroll
    for (int j = 0; j < 4; ++j) g[j] = threadIdx.x + j;
    const float2 S = make_float2(s, s), H = make_float2(0.5f, 0.5f);
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int k = 0; k < 116; ++k) f[k & 7] = ffma2(f[k & 7], S, H);
#pragma unroll
        for (int k = 0; k < 31; ++k) fm[k & 3] = __fmul2_rn(fm[k & 3], S);      // separate chains: a multiply
#pragma unroll
        for (int k = 0; k < 10; ++k) fa[k & 3] = __fadd2_rn(fa[k & 3], H);      // feeding an add would be fused
        g[0] = __fadd_rn(g[0], s); g[1] = __fadd_rn(g[1], s);
#pragma unroll
        for (int k = 0; k < 30; ++k) {                         // IMAD.WIDE.U32 (Philox products)
            const uint64_t p = (uint64_t)u[k & 7] * m;
            u[k & 7] = (uint32_t)(p >> 32) ^ (uint32_t)p;      // + one LOP3 each (counted below)
        }
#pragma unroll
        for (int k = 0; k < 34 * ALU_PCT / 100; ++k) u[k & 7] = (u[k & 7] ^ m) ^ u[(k + 3) & 7];   // LOP3 (64 total with the above)
#pragma unroll
        for (int k = 0; k < 24 * ALU_PCT / 100; ++k) u[k & 7] = __funnelshift_r(u[k & 7], u[(k + 1) & 7], 8);   // SHF
#pragma unroll
        for (int k = 0; k < 24 * ALU_PCT / 100; ++k) u[k & 7] = u[k & 7] + u[(k + 5) & 7] + 0x1234u;            // IADD3
#pragma unroll
        for (int k = 0; k < 6 * ALU_PCT / 100; ++k) u[k & 7] = __byte_perm(u[k & 7], u[(k + 2) & 7], 0x3320u);   // PRMT
#pragma unroll
        for (int k = 0; k < 12; ++k) g[2 + (k & 1)] = __fadd_rn(g[2 + (k & 1)], __uint2float_rn(u[k & 7]));  // I2FP (+FADD)
    }
    float t = g[0] + g[1] + g[2] + g[3];
#pragma unroll
    for (int j = 0; j < 8; ++j) t += f[j].x + f[j].y + (float)u[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) t += fm[j].x + fm[j].y + fa[j].x + fa[j].y;
    if (t == 1234.5f) out[threadIdx.x] = t;
}


// ddm_batch_kernel<128, 6> loop body per 12-step group (cuobjdump): 81 FFMA2, 24 FFMA,
// 18 FMUL2, 6 FADD2, 32 IMAD.WIDE + 9 IMAD, 66 LOP3, 18 SHF, 17 IADD3, 12 I2FP,
// 6 PRMT, 9 VIADD, 6 FMNMX3/FMNMX.  Occupancy 128 x 6 per SM.
__global__ void __launch_bounds__(128, 6) k_mix_ddm(float* out, float s, uint32_t m) {
    float2 f[8], fm[4], fa[4];
    float x[8];
    uint32_t u[8];
    float g[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) { f[j] = make_float2(threadIdx.x + j, j); u[j] = threadIdx.x * 7u + j; x[j] = j; }
#pragma unroll
    for (int j = 0; j < 4; ++j) { fm[j] = make_float2(threadIdx.x + 3 * j, j); fa[j] = make_float2(j, threadIdx.x); g[j] = j; }
    const float2 S = make_float2(s, s), H = make_float2(0.5f, 0.5f);
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int k = 0; k < 81; ++k) f[k & 7] = ffma2(f[k & 7], S, H);
#pragma unroll
        for (int k = 0; k < 24; ++k) x[k & 7] = __fmaf_rn(x[k & 7], s, 0.25f);
#pragma unroll
        for (int k = 0; k < 18; ++k) fm[k & 3] = __fmul2_rn(fm[k & 3], S);
#pragma unroll
        for (int k = 0; k < 6; ++k) fa[k & 3] = __fadd2_rn(fa[k & 3], H);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint64_t p = (uint64_t)u[k & 7] * m;
            u[k & 7] = (uint32_t)(p >> 32) ^ (uint32_t)p;
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) u[k & 7] = u[k & 7] * m + 3u;
#pragma unroll
        for (int k = 0; k < 34; ++k) u[k & 7] = (u[k & 7] ^ m) ^ u[(k + 3) & 7];
#pragma unroll
        for (int k = 0; k < 18; ++k) u[k & 7] = __funnelshift_r(u[k & 7], u[(k + 1) & 7], 8);
#pragma unroll
        for (int k = 0; k < 17; ++k) u[k & 7] = u[k & 7] + u[(k + 5) & 7] + 0x1234u;
#pragma unroll
        for (int k = 0; k < 6; ++k) u[k & 7] = __byte_perm(u[k & 7], u[(k + 2) & 7], 0x3320u);
#pragma unroll
        for (int k = 0; k < 12; ++k) g[k & 3] = __fadd_rn(g[k & 3], __uint2float_rn(u[k & 7]));
        float mx = fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fmaxf(fabsf(x[2]), fabsf(x[3])));
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(x[4]), fabsf(x[5])), fmaxf(fabsf(x[6]), fabsf(x[7]))));
        g[0] = fmaxf(g[0], mx);
    }
    float t = g[0] + g[1] + g[2] + g[3];
#pragma unroll
    for (int j = 0; j < 8; ++j) t += f[j].x + f[j].y + (float)u[j] + x[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) t += fm[j].x + fm[j].y + fa[j].x + fa[j].y;
    if (t == 1234.5f) out[threadIdx.x] = t;
}

// stroop_sim_kernel<128, 0, TABLE> loop body per 6-step group (cuobjdump): 81 FFMA2, 48 FFMA,
// 18 FMUL2, 6 FADD2, 32 IMAD.WIDE + 5 IMAD, 67 LOP3, 23 IADD3, 18 SHF, 12 LDS, 12 I2FP,
// 12 FMNMX, 6 PRMT.  Occupancy 128 x 7 per SM.
__global__ void __launch_bounds__(128, 7) k_mix_stroop(float* out, float s, uint32_t m) {
    __shared__ float tab[1024];
    for (int j = threadIdx.x; j < 1024; j += 128) tab[j] = j * 0.5f;
    __syncthreads();
    float2 f[8], fm[4], fa[4];
    float x[8];
    uint32_t u[8];
    float g[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) { f[j] = make_float2(threadIdx.x + j, j); u[j] = threadIdx.x * 7u + j; x[j] = j; }
#pragma unroll
    for (int j = 0; j < 4; ++j) { fm[j] = make_float2(threadIdx.x + 3 * j, j); fa[j] = make_float2(j, threadIdx.x); g[j] = j; }
    const float2 S = make_float2(s, s), H = make_float2(0.5f, 0.5f);
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int k = 0; k < 81; ++k) f[k & 7] = ffma2(f[k & 7], S, H);
#pragma unroll
        for (int k = 0; k < 48; ++k) x[k & 7] = __fmaf_rn(x[k & 7], s, 0.25f);
#pragma unroll
        for (int k = 0; k < 12; ++k) x[k & 7] = fmaxf(x[k & 7], 0.0f);
#pragma unroll
        for (int k = 0; k < 12; ++k) x[k & 7] += tab[(it * 12 + k) & 1023];      // LDS (+FADD)
#pragma unroll
        for (int k = 0; k < 18; ++k) fm[k & 3] = __fmul2_rn(fm[k & 3], S);
#pragma unroll
        for (int k = 0; k < 6; ++k) fa[k & 3] = __fadd2_rn(fa[k & 3], H);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint64_t p = (uint64_t)u[k & 7] * m;
            u[k & 7] = (uint32_t)(p >> 32) ^ (uint32_t)p;
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) u[k & 7] = u[k & 7] * m + 3u;
#pragma unroll
        for (int k = 0; k < 35; ++k) u[k & 7] = (u[k & 7] ^ m) ^ u[(k + 3) & 7];
#pragma unroll
        for (int k = 0; k < 18; ++k) u[k & 7] = __funnelshift_r(u[k & 7], u[(k + 1) & 7], 8);
#pragma unroll
        for (int k = 0; k < 23; ++k) u[k & 7] = u[k & 7] + u[(k + 5) & 7] + 0x1234u;
#pragma unroll
        for (int k = 0; k < 6; ++k) u[k & 7] = __byte_perm(u[k & 7], u[(k + 2) & 7], 0x3320u);
#pragma unroll
        for (int k = 0; k < 12; ++k) g[k & 3] = __fadd_rn(g[k & 3], __uint2float_rn(u[k & 7]));
    }
    float t = g[0] + g[1] + g[2] + g[3];
#pragma unroll
    for (int j = 0; j < 8; ++j) t += f[j].x + f[j].y + (float)u[j] + x[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) t += fm[j].x + fm[j].y + fa[j].x + fa[j].y;
    if (t == 1234.5f) out[threadIdx.x] = t;
}

int main() {
    float* out; cudaMalloc(&out, 1 << 20);
    int n_sm, clk; cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = n_sm * 7, threads = 128;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run_pp = [&](auto kern, const char* name) {
        kern<<<blocks, threads>>>(out, 1.0001f, 0xD2511F53u);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            kern<<<blocks, threads>>>(out, 1.0001f, 0xD2511F53u);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double warp_iters_per_smsp = (double)blocks * threads / 32 * N_ITER / (n_sm * 4);
        printf("%s: %.4f ms, %.1f SMSP-cycles per iteration (kernel: ~537 per pair-iteration at 1965 MHz)\n",
               name, best, best * 1e-3 * clk * 1e3 / warp_iters_per_smsp);
    };
    run_pp(k_mix<100>, "mix probe (the kernel's mix)");
    run_pp(k_mix<50>, "mix probe, half the extra integer ops");
    run_pp(k_mix<0>, "mix probe, no extra integer ops");
    {
        const int b2 = n_sm * 6;
        k_mix_ddm<<<b2, threads>>>(out, 1.0001f, 0xD2511F53u);
        float best2 = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_mix_ddm<<<b2, threads>>>(out, 1.0001f, 0xD2511F53u);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best2) best2 = ms;
        }
        const double wi = (double)b2 * threads / 32 * N_ITER / (n_sm * 4);
        printf("ddm mix probe: %.4f ms, %.1f SMSP-cycles per 12-step group (kernel: ~490 at 1965 MHz)\n", best2,
               best2 * 1e-3 * clk * 1e3 / wi);
    }
    {
        const int b3 = n_sm * 7;
        k_mix_stroop<<<b3, threads>>>(out, 1.0001f, 0xD2511F53u);
        float best3 = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            k_mix_stroop<<<b3, threads>>>(out, 1.0001f, 0xD2511F53u);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best3) best3 = ms;
        }
        const double wi = (double)b3 * threads / 32 * N_ITER / (n_sm * 4);
        printf("stroop mix probe: %.4f ms, %.1f SMSP-cycles per 6-step group (kernel: ~550 at 1965 MHz)\n", best3,
               best3 * 1e-3 * clk * 1e3 / wi);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
