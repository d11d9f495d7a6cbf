// Does the FP64 pipe give Philox's 32x32->64 multiply a second home? (tools only)
//
// hi32(M*x) = low word of RD(M*(2^52 + x) + (2^84 - M*2^52)): the fma is exact
// before rounding, M*x + 2^84 lies in [2^84, 2^85) where the ulp is 2^32, and
// rounding down keeps exactly 2^84 + hi*2^32.  lo32 = IMAD.  This probe checks
// the identity on the GPU and measures DFMA throughput alone and mixed with
// the FMA-pipe work of pp_eval_grid.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
#define N_ITER 2048

__device__ __forceinline__ uint32_t mulhi_fp64(uint32_t x, double Md, double Cd) {
    const double X52 = __hiloint2double(0x43300000, (int)x);
    return (uint32_t)__double2loint(__fma_rd(Md, X52, Cd));
}

__global__ void k_check(uint32_t m, double Md, double Cd, unsigned long long* bad, uint32_t salt) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t x = t * 2654435761u ^ salt;
    for (int r = 0; r < 64; ++r) {
        const uint32_t xs = (r == 0) ? 0u : (r == 1) ? 0xFFFFFFFFu : x;
        if (mulhi_fp64(xs, Md, Cd) != __umulhi(xs, m)) atomicAdd(bad, 1ull);
        x = x * 1664525u + 1013904223u;
    }
}

__global__ void k_dfma(float* out, double s) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __fma_rn(a0, s, 0.5); a1 = __fma_rn(a1, s, 0.5); a2 = __fma_rn(a2, s, 0.5); a3 = __fma_rn(a3, s, 0.5);
        a4 = __fma_rn(a4, s, 0.5); a5 = __fma_rn(a5, s, 0.5); a6 = __fma_rn(a6, s, 0.5); a7 = __fma_rn(a7, s, 0.5);
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1234.5) out[threadIdx.x] = 1;
}
// 8 chains of the Philox-style product: IMAD.WIDE form vs IMAD + DFMA form
__global__ void k_mul_wide(float* out, uint32_t m, double, double) {
    uint32_t a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x + j; b[j] = 0; }
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { const uint64_t p = (uint64_t)a[j] * m; b[j] ^= (uint32_t)(p >> 32); a[j] = (uint32_t)p ^ b[j]; }
    }
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r ^= a[j] ^ b[j];
    if (r == 12345) out[threadIdx.x] = 1;
}
__global__ void k_mul_fp64(float* out, uint32_t m, double Md, double Cd) {
    uint32_t a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x + j; b[j] = 0; }
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { b[j] ^= mulhi_fp64(a[j], Md, Cd); a[j] = (a[j] * m) ^ b[j]; }
    }
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r ^= a[j] ^ b[j];
    if (r == 12345) out[threadIdx.x] = 1;
}
// mixed with packed FP32 work: 8 FFMA2 + 2 products per iteration
template <bool FP64>
__global__ void k_mix(float* out, uint32_t m, double Md, double Cd) {
    float2 f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = make_float2(threadIdx.x + j, j);
    const float2 S = make_float2(1.0001f, 1.0001f), H = make_float2(0.5f, 0.5f);
    uint32_t a0 = threadIdx.x, a1 = a0 + 7, b0 = 0, b1 = 0;
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __ffma2_rn(f[j], S, H);
        if (FP64) {
            b0 ^= mulhi_fp64(a0, Md, Cd); a0 = (a0 * m) ^ b0;
            b1 ^= mulhi_fp64(a1, Md, Cd); a1 = (a1 * m) ^ b1;
        } else {
            uint64_t p = (uint64_t)a0 * m; b0 ^= (uint32_t)(p >> 32); a0 = (uint32_t)p ^ b0;
            p = (uint64_t)a1 * m; b1 ^= (uint32_t)(p >> 32); a1 = (uint32_t)p ^ b1;
        }
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += f[j].x + f[j].y;
    if (s + (float)(a0 ^ a1 ^ b0 ^ b1) == 1234.5f) out[threadIdx.x] = 1;
}

// overlap test: 8 FFMA2 + 2 independent DFMA chains per iteration (no moves)
__global__ void k_mix_dfma(float* out, uint32_t, double Md, double Cd) {
    float2 f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = make_float2(threadIdx.x + j, j);
    const float2 S = make_float2(1.0001f, 1.0001f), H = make_float2(0.5f, 0.5f);
    double d0 = threadIdx.x, d1 = d0 + 1;
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __ffma2_rn(f[j], S, H);
        d0 = __fma_rn(d0, Md, Cd); d1 = __fma_rn(d1, Md, Cd);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += f[j].x + f[j].y;
    if (s + (float)(d0 + d1) == 1234.5f) out[threadIdx.x] = 1;
}
__global__ void k_mix_ffma2_only(float* out, uint32_t, double, double) {
    float2 f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = make_float2(threadIdx.x + j, j);
    const float2 S = make_float2(1.0001f, 1.0001f), H = make_float2(0.5f, 0.5f);
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __ffma2_rn(f[j], S, H);
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += f[j].x + f[j].y;
    if (s == 1234.5f) out[threadIdx.x] = 1;
}

// ---- full Philox4x32-10: IMAD.WIDE products vs IMAD (lo) + DFMA.RM (hi) products.
// The two multiplicands of every round stay in "2^E + y 2^(E-52)" double form
// (the XORs touch only the low word), E = 52 + 32 r.
__device__ __forceinline__ uint4 philox_std(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ (k0 + r * 0x9E3779B9u), (uint32_t)p1,
                       (uint32_t)(p0 >> 32) ^ c.w ^ (k1 + r * 0xBB67AE85u), (uint32_t)p0);
    }
    return c;
}
__device__ __forceinline__ double xor_lo(double d, uint32_t v) {
    return __hiloint2double(__double2hiint(d), (int)((uint32_t)__double2loint(d) ^ v));
}
__device__ __forceinline__ uint32_t lo_of(double d) { return (uint32_t)__double2loint(d); }
// Fixed-exponent form: every multiplicand is D = 2^84 + y 2^32 ({y, 0x45300000});
// fma_rd(D, M 2^-32, 2^52 (2^32 - M)) = RD(2^84 + M y) = 2^84 + hi(M y) 2^32,
// i.e. the same form with the high product word in the low register.
__device__ __forceinline__ double d84(uint32_t y) { return __hiloint2double(0x45300000, (int)y); }
__device__ __forceinline__ uint4 philox_dfma(uint4 c, uint32_t k0, uint32_t k1) {
    constexpr double M0s = (double)0xD2511F53u * 0x1p-32, M1s = (double)0xCD9E8D57u * 0x1p-32;
    constexpr double C0 = 0x1p52 * (0x1p32 - (double)0xD2511F53u), C1 = 0x1p52 * (0x1p32 - (double)0xCD9E8D57u);
    double x0 = d84(c.x), x2 = d84(c.z);
    uint32_t x1 = c.y, x3 = c.w;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const double h0 = __fma_rd(x0, M0s, C0), h1 = __fma_rd(x2, M1s, C1);
        const uint32_t l0 = lo_of(x0) * 0xD2511F53u, l1 = lo_of(x2) * 0xCD9E8D57u;
        x0 = xor_lo(h1, x1 ^ (k0 + r * 0x9E3779B9u));
        x2 = xor_lo(h0, x3 ^ (k1 + r * 0xBB67AE85u));
        x1 = l1; x3 = l0;
    }
    return make_uint4(lo_of(x0), x1, lo_of(x2), x3);
}
__global__ void k_philox_check(unsigned long long* bad) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t s = 0; s < 64; ++s) {
        const uint4 c = make_uint4(t * 2654435761u, s, t ^ 0xFFFFFFFFu, s * 77u), a = philox_std(c, 42u + s, t),
                    b = philox_dfma(c, 42u + s, t);
        if (a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w) atomicAdd(bad, 1ull);
    }
}
template <bool DF>
__global__ void k_philox(float* out, uint32_t k0, double, double) {
    uint32_t acc = 0;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int it = 0; it < N_ITER / 8; ++it) {
        const uint4 c = make_uint4(t, it, 7u, 1u);
        const uint4 o = DF ? philox_dfma(c, k0, 3u) : philox_std(c, k0, 3u);
        acc ^= o.x ^ o.y ^ o.z ^ o.w;
    }
    if (acc == 12345) out[threadIdx.x] = 1;
}

// pipe-sharing tests (all chains independent, 8 per thread)
template <int MODE>   // 0: IMAD only, 1: DFMA.RM only, 2: both
__global__ void k_share(float* out, uint32_t m, double Ms, double C) {
    uint32_t a[8]; double d[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x + j; d[j] = d84(threadIdx.x * 3 + j); }
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (MODE != 1) a[j] = a[j] * m + 7u;
            if (MODE != 0) d[j] = __fma_rd(d[j], Ms, C);
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) r ^= a[j] ^ lo_of(d[j]);
    if (r == 12345) out[threadIdx.x] = 1;
}
// 8 FFMA2 + 2 chained products per iteration, d84 form vs IMAD.WIDE
template <bool DF>
__global__ void k_mix84(float* out, uint32_t m, double Ms, double C) {
    float2 f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = make_float2(threadIdx.x + j, j);
    const float2 S = make_float2(1.0001f, 1.0001f), H = make_float2(0.5f, 0.5f);
    uint32_t a0 = threadIdx.x, a1 = a0 + 7;
    double D0 = d84(a0), D1 = d84(a1);
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __ffma2_rn(f[j], S, H);
        if (DF) {
            const uint32_t l0 = lo_of(D0) * m, l1 = lo_of(D1) * m;
            D0 = xor_lo(__fma_rd(D0, Ms, C), l0); D1 = xor_lo(__fma_rd(D1, Ms, C), l1);
        } else {
            uint64_t p = (uint64_t)a0 * m; a0 = (uint32_t)(p >> 32) ^ (uint32_t)p;
            p = (uint64_t)a1 * m; a1 = (uint32_t)(p >> 32) ^ (uint32_t)p;
        }
    }
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += f[j].x + f[j].y;
    if (s + (float)(a0 ^ a1 ^ lo_of(D0) ^ lo_of(D1)) == 1234.5f) out[threadIdx.x] = 1;
}

template <typename K, typename... Args>
void bench(const char* name, double units_per_iter, const char* unit, K kern, Args... args) {
    float* out; cudaMalloc(&out, 1 << 20);
    int n_sm; cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = n_sm * 8, threads = 256;
    kern<<<blocks, threads>>>(out, args...);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, args...);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double warp_units = (double)blocks * threads / 32 * N_ITER * units_per_iter;
    const double cycles = best * 1e-3 * clk * 1e3;
    printf("%-34s %8.3f ms  %6.3f warp-%s/clk/SM  (%.2f SMSP-cycles each)\n", name, best, warp_units / cycles / n_sm,
           unit, 4.0 / (warp_units / cycles / n_sm));
    cudaFree(out);
}

int main() {
    const uint32_t M0 = 0xD2511F53u;
    const double Md = (double)M0, Cd = 0x1p84 - (double)M0 * 0x1p52;
    unsigned long long* bad; cudaMalloc(&bad, 8); cudaMemset(bad, 0, 8);
    for (uint32_t salt = 0; salt < 16; ++salt) k_check<<<4096, 256>>>(M0, Md, Cd, bad, salt * 0x9E3779B9u);
    k_check<<<4096, 256>>>(0xCD9E8D57u, (double)0xCD9E8D57u, 0x1p84 - (double)0xCD9E8D57u * 0x1p52, bad, 7);
    unsigned long long h = 0; cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    printf("mulhi_fp64 identity: %llu mismatches over %d products\n", h, 17 * 4096 * 256 * 64);
    bench("DFMA", 8, "inst", k_dfma, 1.0000001);
    bench("product via IMAD.WIDE", 8, "product", k_mul_wide, M0, Md, Cd);
    bench("product via IMAD + DFMA.RM", 8, "product", k_mul_fp64, M0, Md, Cd);
    bench("8 FFMA2 + 2 IMAD.WIDE products", 1, "iter", k_mix<false>, M0, Md, Cd);
    bench("8 FFMA2 + 2 IMAD+DFMA products", 1, "iter", k_mix<true>, M0, Md, Cd);
    cudaMemset(bad, 0, 8);
    k_philox_check<<<4096, 256>>>(bad);
    cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    printf("philox_dfma == philox_std: %llu mismatches over %d blocks\n", h, 4096 * 256 * 64);
    bench("Philox10 IMAD.WIDE", 1.0 / 8, "block", k_philox<false>, 42u, 0.0, 0.0);
    bench("Philox10 IMAD + DFMA.RM", 1.0 / 8, "block", k_philox<true>, 42u, 0.0, 0.0);
    {
        const double Ms = (double)M0 * 0x1p-32, C = 0x1p52 * (0x1p32 - (double)M0);
        bench("share: 8 IMAD", 1, "iter", k_share<0>, M0, Ms, C);
        bench("share: 8 DFMA.RM", 1, "iter", k_share<1>, M0, Ms, C);
        bench("share: 8 IMAD + 8 DFMA.RM", 1, "iter", k_share<2>, M0, Ms, C);
        bench("8 FFMA2 + 2 IMAD.WIDE chains", 1, "iter", k_mix84<false>, M0, Ms, C);
        bench("8 FFMA2 + 2 IMAD+DFMA(d84) chains", 1, "iter", k_mix84<true>, M0, Ms, C);
    }
    bench("8 FFMA2", 1, "iter", k_mix_ffma2_only, M0, 1.0000001, 0.5);
    bench("8 FFMA2 + 2 DFMA", 1, "iter", k_mix_dfma, M0, 1.0000001, 0.5);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
