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
// HBM-bound (4 B read per value), so the per-value work must stay under ~0.7
// instructions to keep up with HBM.  Each thread visits its groups of eight values
// (two float4 loads) in DECREASING index order and keeps the largest V seen with
// `max(group) >= best` (fmaxf ignores NaN; -0 == +0), resolving the group's first
// index of that value only when the test passes — rarely, after the first few
// groups — so equal values end at their lowest index, as the key order wants.  A
// thread that saw no non-NaN value rescans its share for its first NaN (the key of
// an all-NaN array is key(NaN, lowest index), as before).  Then the block min of
// the per-thread keys and one atomicMin.  Misaligned pointers: the scalar loop.
__device__ __forceinline__ float max8(const float4& a, const float4& b) {
    return fmaxf(fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)), fmaxf(fmaxf(b.x, b.y), fmaxf(b.z, b.w)));
}

// first l in 0..7 with value == m (m is one of the group's non-NaN values)
__device__ __forceinline__ uint32_t first_eq8(const float4& a, const float4& b, float m) {
    return a.x == m ? 0u : a.y == m ? 1u : a.z == m ? 2u : a.w == m ? 3u
         : b.x == m ? 4u : b.y == m ? 5u : b.z == m ? 6u : 7u;
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) argmax_net_kernel(const float* __restrict__ v, uint64_t n,
                                                           uint32_t base, key64_t* __restrict__ best) {
    key64_t k = KEY_INIT;
    const uint64_t tid = (uint64_t)blockIdx.x * BLOCK + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * BLOCK;
    if ((reinterpret_cast<uintptr_t>(v) & 15u) == 0) {
        const uint64_t n8 = n >> 3;
        const float4* v4 = reinterpret_cast<const float4*>(v);
        float bv = -INFINITY;
        uint64_t bi = ~0ull;
        // the ragged tail (indices above every group): one value per thread, first
        const uint64_t jt = 8 * n8 + tid;
        if (jt < n) {
            const float x = __ldg(v + jt);
            if (x >= bv) { bv = x; bi = jt; }
        }
        // this thread's groups g = tid + q * stride, q = cnt-1 .. 0, two at a time
        const uint64_t cnt = n8 > tid ? (n8 - 1 - tid) / stride + 1 : 0;
        int64_t q = (int64_t)cnt - 1;
        for (; q >= 1; q -= 2) {
            const uint64_t g1 = tid + (uint64_t)q * stride, g0 = g1 - stride;
            const float4 a1 = __ldg(v4 + 2 * g1), b1 = __ldg(v4 + 2 * g1 + 1);
            const float4 a0 = __ldg(v4 + 2 * g0), b0 = __ldg(v4 + 2 * g0 + 1);
            const float m1 = max8(a1, b1), m0 = max8(a0, b0);
            if (m1 >= bv) { bv = m1; bi = 8 * g1 + first_eq8(a1, b1, m1); }
            if (m0 >= bv) { bv = m0; bi = 8 * g0 + first_eq8(a0, b0, m0); }
        }
        if (q == 0) {
            const float4 a0 = __ldg(v4 + 2 * tid), b0 = __ldg(v4 + 2 * tid + 1);
            const float m0 = max8(a0, b0);
            if (m0 >= bv) { bv = m0; bi = 8 * tid + first_eq8(a0, b0, m0); }
        }
        if (bi != ~0ull) {
            k = make_key(-bv, base + (uint32_t)bi);
        } else {                                   // no non-NaN value here: the first NaN, if any
            for (uint64_t g = tid; g < n8 && k == KEY_INIT; g += stride)
                for (uint32_t l = 0; l < 8; ++l)
                    if (__ldg(v + 8 * g + l) != __ldg(v + 8 * g + l)) { k = make_key(__int_as_float(0x7FC00000), base + (uint32_t)(8 * g + l)); break; }
            if (k == KEY_INIT && jt < n) k = make_key(-__ldg(v + jt), base + (uint32_t)jt);
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
// The tie test compares values, not keys: canon(-v) has the best key's high word
// exactly when v == -C* (C* decoded from that word; -0 == +0, and the all-NaN key
// never reaches the loop), so the scan is one float compare per value (float4
// loads on aligned arrays) and the Philox priority is drawn for the ties only.
__device__ __forceinline__ float key_cost(uint32_t hi) {        // inverse of make_key's order map
    return __uint_as_float((hi & 0x80000000u) ? (hi & 0x7FFFFFFFu) : ~hi);
}

__device__ __forceinline__ void tie_candidate(uint32_t idx, uint32_t key0, uint32_t key1, uint32_t invocation,
                                              key64_t& k) {
    const uint4 X = philox4x32_10(make_uint4(idx, 0u, invocation, 3u), key0, key1);
    const key64_t t = ((key64_t)X.x << 32) | idx;
    k = t < k ? t : k;
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) argmax_ties_kernel(const float* __restrict__ v, uint64_t n, uint32_t base,
                                                            const key64_t* __restrict__ best, uint32_t key0,
                                                            uint32_t key1, uint32_t invocation,
                                                            key64_t* __restrict__ tie) {
    const uint32_t hi = (uint32_t)(*best >> 32);
    key64_t k = KEY_INIT;
    if (hi != 0xFFFFFFFFu) {
        const float T = -key_cost(hi);
        const uint64_t tid = (uint64_t)blockIdx.x * BLOCK + threadIdx.x, stride = (uint64_t)gridDim.x * BLOCK;
        uint64_t j0 = 0;
        if ((reinterpret_cast<uintptr_t>(v) & 15u) == 0) {
            const uint64_t n4 = n >> 2;
            const float4* v4 = reinterpret_cast<const float4*>(v);
            for (uint64_t j = tid; j < n4; j += stride) {
                const float4 x = __ldg(v4 + j);
                if (x.x == T || x.y == T || x.z == T || x.w == T) {
                    const uint32_t i0 = base + (uint32_t)(4 * j);
                    if (x.x == T) tie_candidate(i0, key0, key1, invocation, k);
                    if (x.y == T) tie_candidate(i0 + 1, key0, key1, invocation, k);
                    if (x.z == T) tie_candidate(i0 + 2, key0, key1, invocation, k);
                    if (x.w == T) tie_candidate(i0 + 3, key0, key1, invocation, k);
                }
            }
            j0 = 4 * n4;
        }
        for (uint64_t j = j0 + tid; j < n; j += stride)
            if (__ldg(v + j) == T) tie_candidate(base + (uint32_t)j, key0, key1, invocation, k);
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
