// keys.cuh — packed (value, index) argmin keys and their reductions
// (spec/MODELS.md §3; "selects the parameters that have the
// lowest cost", ties P:306 -> lowest index, reading Q7 in DESIGN.md).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "rng.cuh"

namespace distill {

typedef unsigned long long key64_t;
constexpr key64_t KEY_INIT = 0xFFFFFFFFFFFFFFFFull;
// Signed key order (distill_eval_args.key_order = 1): the stored word is
// key ^ 2^63, so signed int64 order equals the unsigned key order and the
// per-GPU result feeds an int64 MIN all-reduce (torch/NCCL) as it is.
constexpr key64_t KEY_SIGN = 0x8000000000000000ull;

// key(C, i) = ord(canon(C)) << 32 | i : min key = lowest cost, then lowest index.
__device__ __forceinline__ key64_t make_key(float C, uint32_t idx) {
    uint32_t hi;
    if (C != C) {
        hi = 0xFFFFFFFFu;                     // NaN never wins
    } else {
        const uint32_t b = __float_as_uint(C == 0.0f ? 0.0f : C);   // -0 -> +0
        hi = (b >> 31) ? ~b : (b | 0x80000000u);
    }
    return ((key64_t)hi << 32) | idx;
}

__device__ __forceinline__ key64_t warp_min_key(key64_t k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const key64_t o = __shfl_xor_sync(0xFFFFFFFFu, k, off);
        k = o < k ? o : k;
    }
    return k;
}

// Block-wide min of one key per thread, then ONE atomicMin per block (in the
// signed order when `signed_order`).  All threads of the block must call it
// (uses __syncthreads).
template <int BLOCK>
__device__ __forceinline__ void block_min_key_atomic(key64_t k, key64_t* dst, bool signed_order = false) {
    __shared__ key64_t s_warp[BLOCK / 32];
    k = warp_min_key(k);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) s_warp[wid] = k;
    __syncthreads();
    if (wid == 0) {
        k = lane < BLOCK / 32 ? s_warp[lane] : KEY_INIT;
        k = warp_min_key(k);
        if (lane == 0 && k != KEY_INIT) {
            if (signed_order) atomicMin(reinterpret_cast<long long*>(dst), (long long)(k ^ KEY_SIGN));
            else atomicMin(dst, k);
        }
    }
}

// K2: argmax over a device array of net values V -> atomicMin(key(-V[j], base+j)).
// Grid-stride, vectorised float4 loads when the pointer is 16-B aligned.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) argmax_net_kernel(const float* __restrict__ v, uint64_t n,
                                                           uint32_t base, key64_t* __restrict__ best) {
    key64_t k = KEY_INIT;
    const uint64_t tid = (uint64_t)blockIdx.x * BLOCK + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    if ((reinterpret_cast<uintptr_t>(v) & 15u) == 0) {
        const uint64_t n4 = n >> 2;
        const float4* v4 = reinterpret_cast<const float4*>(v);
        for (uint64_t j = tid; j < n4; j += stride) {
            const float4 x = __ldg(v4 + j);
            const uint32_t i0 = base + (uint32_t)(4 * j);
            key64_t a = make_key(-x.x, i0), b = make_key(-x.y, i0 + 1);
            key64_t c = make_key(-x.z, i0 + 2), d = make_key(-x.w, i0 + 3);
            a = a < b ? a : b;
            c = c < d ? c : d;
            a = a < c ? a : c;
            k = a < k ? a : k;
        }
        for (uint64_t j = 4 * n4 + tid; j < n; j += stride) {
            const key64_t a = make_key(-__ldg(v + j), base + (uint32_t)j);
            k = a < k ? a : k;
        }
    } else {
        for (uint64_t j = tid; j < n; j += stride) {
            const key64_t a = make_key(-__ldg(v + j), base + (uint32_t)j);
            k = a < k ? a : k;
        }
    }
    block_min_key_atomic<BLOCK>(k, best);
}

// NEXT-2 random tie-break (spec/MODELS.md §8): among the entries whose
// canonical cost equals the best key's (pass A result in *best), min over
// (pi_i << 32 | i) with pi_i = Philox(key, (i, 0, t, 3)).x -> atomicMin(*tie).
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) argmax_ties_kernel(const float* __restrict__ v, uint64_t n, uint32_t base,
                                                            const key64_t* __restrict__ best, uint32_t key0,
                                                            uint32_t key1, uint32_t invocation,
                                                            key64_t* __restrict__ tie) {
    const uint32_t hi = (uint32_t)(*best >> 32);
    key64_t k = KEY_INIT;
    if (hi != 0xFFFFFFFFu) {
        for (uint64_t j = (uint64_t)blockIdx.x * BLOCK + threadIdx.x; j < n; j += (uint64_t)gridDim.x * BLOCK) {
            const uint32_t idx = base + (uint32_t)j;
            if ((uint32_t)(make_key(-__ldg(v + j), idx) >> 32) != hi) continue;
            const uint4 X = philox4x32_10(make_uint4(idx, 0u, invocation, 3u), key0, key1);
            const key64_t t = ((key64_t)X.x << 32) | idx;
            k = t < k ? t : k;
        }
    }
    block_min_key_atomic<BLOCK>(k, tie);
}

// Measurement utility (not the hot path): effective SM clock.  One block per SM
// spins for `ns` nanoseconds of globaltimer and reports clock64 ticks per ns.
__global__ void sm_clock_probe_kernel(unsigned long long ns, double* __restrict__ mhz) {
    if (threadIdx.x != 0) return;
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const long long c0 = clock64();
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)); } while (t1 - t0 < ns);
    const long long c1 = clock64();
    mhz[blockIdx.x] = (double)(c1 - c0) / (double)(t1 - t0) * 1e3;
}

}  // namespace distill
