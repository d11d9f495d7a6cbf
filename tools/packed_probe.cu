// Probe: do FFMA2/FMUL2/FADD2 round each lane exactly like FFMA/FMUL/FADD?
// Random operands over wide exponent ranges, plus immediate/broadcast forms.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ float rnd(uint32_t k) {
    uint32_t h = hash(k);
    uint32_t e = 100 + (hash(k ^ 0x9e3779b9) % 56);     // exponent 2^-27 .. 2^28
    return __uint_as_float((h & 0x807FFFFFu) | (e << 23));
}
__global__ void probe(unsigned long long* bad, int n) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    float a0 = rnd(6 * t), a1 = rnd(6 * t + 1), b0 = rnd(6 * t + 2), b1 = rnd(6 * t + 3), c0 = rnd(6 * t + 4), c1 = rnd(6 * t + 5);
    float2 A = make_float2(a0, a1), B = make_float2(b0, b1), Cc = make_float2(c0, c1);
    float2 r = __ffma2_rn(A, B, Cc);
    if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(a0, b0, c0)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(a1, b1, c1))) atomicAdd(bad + 0, 1);
    r = __fmul2_rn(A, B);
    if (__float_as_uint(r.x) != __float_as_uint(__fmul_rn(a0, b0)) || __float_as_uint(r.y) != __float_as_uint(__fmul_rn(a1, b1))) atomicAdd(bad + 1, 1);
    r = __fadd2_rn(A, Cc);
    if (__float_as_uint(r.x) != __float_as_uint(__fadd_rn(a0, c0)) || __float_as_uint(r.y) != __float_as_uint(__fadd_rn(a1, c1))) atomicAdd(bad + 2, 1);
    r = __ffma2_rn(A, B, make_float2(0.14883549511432648f, 0.14883549511432648f));
    if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(a0, b0, 0.14883549511432648f)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(a1, b1, 0.14883549511432648f))) atomicAdd(bad + 3, 1);
    r = __ffma2_rn(make_float2(c0, c0), B, A);
    if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(c0, b0, a0)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(c0, b1, a1))) atomicAdd(bad + 4, 1);
    r = __fmul2_rn(A, make_float2(-2.0f, -2.0f));
    if (__float_as_uint(r.x) != __float_as_uint(__fmul_rn(a0, -2.0f)) || __float_as_uint(r.y) != __float_as_uint(__fmul_rn(a1, -2.0f))) atomicAdd(bad + 5, 1);
    r = __ffma2_rn(A, A, make_float2(0x1p-126f, 0x1p-126f));
    if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(a0, a0, 0x1p-126f)) || __float_as_uint(r.y) != __float_as_uint(__fmaf_rn(a1, a1, 0x1p-126f))) atomicAdd(bad + 6, 1);
    r = __fadd2_rn(A, make_float2(-B.x, -B.y));
    if (__float_as_uint(r.x) != __float_as_uint(__fadd_rn(a0, -b0)) || __float_as_uint(r.y) != __float_as_uint(__fadd_rn(a1, -b1))) atomicAdd(bad + 7, 1);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 8 * 8); cudaMemset(d, 0, 64);
    int n = 1 << 24;
    probe<<<n / 256, 256>>>(d, n);
    unsigned long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    const char* nm[8] = {"ffma2", "fmul2", "fadd2", "ffma2_imm", "ffma2_bcast", "fmul2_imm", "ffma2_tiny", "fadd2_neg"};
    for (int i = 0; i < 8; ++i) printf("%-12s mismatches %llu / %d\n", nm[i], h[i], n);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
