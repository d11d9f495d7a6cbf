// Pipe-throughput microbenchmark on sm_100a (tools only).  Each kernel runs
// N_ITER iterations of 8 independent chains of one instruction kind per
// thread; reports warp-instructions per clock per SM.  Used to model the
// fmaheavy/fmalite/ALU budget of pp_eval_grid.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N_ITER 2048

#define KBODY(init, step, sink)                                                        \
    init;                                                                              \
    for (int it = 0; it < N_ITER; ++it) { step }                                        \
    if (sink) out[blockIdx.x * blockDim.x + threadIdx.x] = 1;

__global__ void k_ffma(float* out, float s) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __fmaf_rn(a0, s, 0.5f); a1 = __fmaf_rn(a1, s, 0.5f); a2 = __fmaf_rn(a2, s, 0.5f); a3 = __fmaf_rn(a3, s, 0.5f);
        a4 = __fmaf_rn(a4, s, 0.5f); a5 = __fmaf_rn(a5, s, 0.5f); a6 = __fmaf_rn(a6, s, 0.5f); a7 = __fmaf_rn(a7, s, 0.5f);
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1234.5f) out[threadIdx.x] = 1;
}
__global__ void k_ffma_reg(float* out, float s) {   // 3 register operands
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    float c = s * 0.25f;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __fmaf_rn(a0, s, c); a1 = __fmaf_rn(a1, s, c); a2 = __fmaf_rn(a2, s, c); a3 = __fmaf_rn(a3, s, c);
        a4 = __fmaf_rn(a4, s, c); a5 = __fmaf_rn(a5, s, c); a6 = __fmaf_rn(a6, s, c); a7 = __fmaf_rn(a7, s, c);
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1234.5f) out[threadIdx.x] = 1;
}
__global__ void k_ffma2(float* out, float s) {
    float2 a0 = make_float2(threadIdx.x, 1), a1 = make_float2(2, 3), a2 = make_float2(4, 5), a3 = make_float2(6, 7);
    float2 a4 = make_float2(8, 9), a5 = make_float2(1, 3), a6 = make_float2(5, 7), a7 = make_float2(2, 9);
    float2 S = make_float2(s, s), H = make_float2(0.5f, 0.5f);
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __ffma2_rn(a0, S, H); a1 = __ffma2_rn(a1, S, H); a2 = __ffma2_rn(a2, S, H); a3 = __ffma2_rn(a3, S, H);
        a4 = __ffma2_rn(a4, S, H); a5 = __ffma2_rn(a5, S, H); a6 = __ffma2_rn(a6, S, H); a7 = __ffma2_rn(a7, S, H);
    }
    if (a0.x + a1.x + a2.x + a3.x + a4.y + a5.y + a6.y + a7.y == 1234.5f) out[threadIdx.x] = 1;
}
__global__ void k_imadwide(float* out, uint32_t m) {
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    uint32_t b0 = 0, b1 = 0, b2 = 0, b3 = 0, b4 = 0, b5 = 0, b6 = 0, b7 = 0;
    for (int it = 0; it < N_ITER; ++it) {
#define W(a, b) { uint64_t p = (uint64_t)a * m; a = (uint32_t)p; b ^= (uint32_t)(p >> 32); }
        W(a0, b0) W(a1, b1) W(a2, b2) W(a3, b3) W(a4, b4) W(a5, b5) W(a6, b6) W(a7, b7)
#undef W
    }
    if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7 ^ b0 ^ b1 ^ b2 ^ b3 ^ b4 ^ b5 ^ b6 ^ b7) == 12345) out[threadIdx.x] = 1;
}
__global__ void k_imadlo(float* out, uint32_t m) {
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = a0 * m + 7; a1 = a1 * m + 7; a2 = a2 * m + 7; a3 = a3 * m + 7;
        a4 = a4 * m + 7; a5 = a5 * m + 7; a6 = a6 * m + 7; a7 = a7 * m + 7;
    }
    if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7) == 12345) out[threadIdx.x] = 1;
}
__global__ void k_imadhi(float* out, uint32_t m) {
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __umulhi(a0, m) ^ it; a1 = __umulhi(a1, m) ^ it; a2 = __umulhi(a2, m) ^ it; a3 = __umulhi(a3, m) ^ it;
        a4 = __umulhi(a4, m) ^ it; a5 = __umulhi(a5, m) ^ it; a6 = __umulhi(a6, m) ^ it; a7 = __umulhi(a7, m) ^ it;
    }
    if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7) == 12345) out[threadIdx.x] = 1;
}
__global__ void k_lop3(float* out, uint32_t m) {
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = (a0 ^ m) ^ (a0 >> 0); a0 ^= m * 0;
        a0 ^= m ^ a1; a1 ^= m ^ a2; a2 ^= m ^ a3; a3 ^= m ^ a4; a4 ^= m ^ a5; a5 ^= m ^ a6; a6 ^= m ^ a7; a7 ^= m ^ a0;
    }
    if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7) == 12345) out[threadIdx.x] = 1;
}
__global__ void k_mix_ffma2_imadwide(float* out, float s, uint32_t m) {   // 4 FFMA2 : 1 IMAD.WIDE
    float2 a0 = make_float2(threadIdx.x, 1), a1 = make_float2(2, 3), a2 = make_float2(4, 5), a3 = make_float2(6, 7);
    float2 S = make_float2(s, s), H = make_float2(0.5f, 0.5f);
    uint32_t u0 = threadIdx.x, v0 = 0;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __ffma2_rn(a0, S, H); a1 = __ffma2_rn(a1, S, H); a2 = __ffma2_rn(a2, S, H); a3 = __ffma2_rn(a3, S, H);
        { uint64_t p = (uint64_t)u0 * m; u0 = (uint32_t)p; v0 ^= (uint32_t)(p >> 32); }
    }
    if (a0.x + a1.x + a2.x + a3.y + (float)(u0 ^ v0) == 1234.5f) out[threadIdx.x] = 1;
}
__global__ void k_mix_ffma_imadwide(float* out, float s, uint32_t m) {    // 8 FFMA : 1 IMAD.WIDE
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    uint32_t u0 = threadIdx.x, v0 = 0;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __fmaf_rn(a0, s, 0.5f); a1 = __fmaf_rn(a1, s, 0.5f); a2 = __fmaf_rn(a2, s, 0.5f); a3 = __fmaf_rn(a3, s, 0.5f);
        a4 = __fmaf_rn(a4, s, 0.5f); a5 = __fmaf_rn(a5, s, 0.5f); a6 = __fmaf_rn(a6, s, 0.5f); a7 = __fmaf_rn(a7, s, 0.5f);
        { uint64_t p = (uint64_t)u0 * m; u0 = (uint32_t)p; v0 ^= (uint32_t)(p >> 32); }
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + (float)(u0 ^ v0) == 1234.5f) out[threadIdx.x] = 1;
}
__global__ void k_mix_ffma2_lop3(float* out, float s, uint32_t m) {       // 4 FFMA2 : 4 LOP3
    float2 a0 = make_float2(threadIdx.x, 1), a1 = make_float2(2, 3), a2 = make_float2(4, 5), a3 = make_float2(6, 7);
    float2 S = make_float2(s, s), H = make_float2(0.5f, 0.5f);
    uint32_t u0 = threadIdx.x, u1 = u0 + 1, u2 = u0 + 2, u3 = u0 + 3;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __ffma2_rn(a0, S, H); a1 = __ffma2_rn(a1, S, H); a2 = __ffma2_rn(a2, S, H); a3 = __ffma2_rn(a3, S, H);
        u0 ^= m ^ u1; u1 ^= m ^ u2; u2 ^= m ^ u3; u3 ^= m ^ u0;
    }
    if (a0.x + a1.x + a2.x + a3.y + (float)(u0 ^ u1 ^ u2 ^ u3) == 1234.5f) out[threadIdx.x] = 1;
}
__global__ void k_i2f(float* out, uint32_t m) {
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    float f = 0;
    for (int it = 0; it < N_ITER; ++it) {
        f += __uint2float_rn(a0) + __uint2float_rn(a1) + __uint2float_rn(a2) + __uint2float_rn(a3);
        a0 ^= m; a1 ^= m; a2 ^= m; a3 ^= m;
    }
    if (f == 1234.5f) out[threadIdx.x] = 1;
}

// I2FP.F32.U32 throughput (8 independent chains; the float result feeds back as bits)
__global__ void k_i2fp(float* out, uint32_t m) {
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int it = 0; it < N_ITER; ++it) {
        a0 = __float_as_uint(__uint2float_rn(a0 ^ m)); a1 = __float_as_uint(__uint2float_rn(a1 ^ m));
        a2 = __float_as_uint(__uint2float_rn(a2 ^ m)); a3 = __float_as_uint(__uint2float_rn(a3 ^ m));
        a4 = __float_as_uint(__uint2float_rn(a4 ^ m)); a5 = __float_as_uint(__uint2float_rn(a5 ^ m));
        a6 = __float_as_uint(__uint2float_rn(a6 ^ m)); a7 = __float_as_uint(__uint2float_rn(a7 ^ m));
    }
    if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7) == 12345) out[threadIdx.x] = 1;
}
// 8 FFMA2 + 2 I2FP per iteration (does the conversion overlap the FMA datapath?)
__global__ void k_mix_ffma2_i2fp(float* out, float s, uint32_t m) {
    float2 f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = make_float2(threadIdx.x + j, j);
    const float2 S = make_float2(s, s), H = make_float2(0.5f, 0.5f);
    uint32_t u0 = threadIdx.x, u1 = u0 + 5;
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __ffma2_rn(f[j], S, H);
        u0 = __float_as_uint(__uint2float_rn(u0 ^ m)); u1 = __float_as_uint(__uint2float_rn(u1 ^ m));
    }
    float t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += f[j].x + f[j].y;
    if (t + (float)(u0 ^ u1) == 1234.5f) out[threadIdx.x] = 1;
}
__global__ void k_ffma2_8(float* out, float s, uint32_t m) {
    float2 f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = make_float2(threadIdx.x + j, j);
    const float2 S = make_float2(s, s), H = make_float2(0.5f, 0.5f);
    uint32_t u0 = threadIdx.x, u1 = u0 + 5;
    for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __ffma2_rn(f[j], S, H);
        u0 = (u0 ^ m) + 3; u1 = (u1 ^ m) + 5;
    }
    float t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += f[j].x + f[j].y;
    if (t + (float)(u0 ^ u1) == 1234.5f) out[threadIdx.x] = 1;
}

template <typename K, typename... Args>
void bench(const char* name, int insts_per_iter, K kern, Args... args) {
    float* out; cudaMalloc(&out, 1 << 20);
    int n_sm; cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz (max)
    const int blocks = n_sm * 8, threads = 256;
    kern<<<blocks, threads>>>(out, args...);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, args...);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double warp_insts = (double)blocks * threads / 32 * N_ITER * insts_per_iter;
    const double cycles = ms * 1e-3 * clk * 1e3;   // at max clock (upper bound on cycles)
    printf("%-28s %8.3f ms  %6.3f warp-inst/clk/SM (at %d MHz max clock)\n", name, ms, warp_insts / cycles / n_sm, clk / 1000);
    cudaFree(out);
}

int main() {
    bench("FFMA imm", 8, k_ffma, 1.0001f);
    bench("FFMA 3-reg", 8, k_ffma_reg, 1.0001f);
    bench("FFMA2 (64 FMA/inst)", 8, k_ffma2, 1.0001f);
    bench("IMAD.WIDE.U32", 8, k_imadwide, 0xD2511F53u);
    bench("IMAD (lo)", 8, k_imadlo, 0xD2511F53u);
    bench("IMAD.HI", 8, k_imadhi, 0xD2511F53u);
    bench("LOP3 (approx)", 8, k_lop3, 0xD2511F53u);
    bench("I2F.U32 (+FADD)", 8, k_i2f, 0xD2511F53u);
    bench("4 FFMA2 + 1 IMAD.WIDE", 5, k_mix_ffma2_imadwide, 1.0001f, 0xD2511F53u);
    bench("8 FFMA + 1 IMAD.WIDE", 9, k_mix_ffma_imadwide, 1.0001f, 0xD2511F53u);
    bench("4 FFMA2 + 4 LOP3", 8, k_mix_ffma2_lop3, 1.0001f, 0xD2511F53u);
    bench("I2FP.F32.U32 (+LOP3)", 8, k_i2fp, 0xD2511F53u);
    bench("8 FFMA2 + 2 int ops (iter)", 1, k_ffma2_8, 1.0001f, 0xD2511F53u);
    bench("8 FFMA2 + 2 I2FP (iter)", 1, k_mix_ffma2_i2fp, 1.0001f, 0xD2511F53u);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
