// trials.cuh — trial streaming for the accumulator-model grid kernels
// (R14b): when a model's outputs are the response and its step, a
// trial ends at its first passage, and each lane takes its next trial from a
// per-block counter instead of idling until the warp's slowest trial is done.
// The integer outcome sums are order-free, so which lane runs which trial does
// not change any result.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace distill {

// Trial streaming (R14b): block x of gridDim.x owns the contiguous trial range
// [tb + x·P, min(te, tb + (x+1)·P)), P = ceil((te - tb) / gridDim.x); its lanes
// take trials from a shared counter (thread 0 sets it; the caller's next block
// barrier publishes it).
__device__ __forceinline__ void block_trial_range(uint32_t tb, uint32_t te, uint32_t& s_next, uint32_t& t_end) {
    const uint32_t per = (te - tb + gridDim.x - 1) / gridDim.x;
    const uint64_t b = (uint64_t)tb + (uint64_t)blockIdx.x * per;
    const uint32_t lo = (uint32_t)(b < te ? b : te);
    t_end = (uint32_t)(b + per < te ? b + per : te);
    if (threadIdx.x == 0) s_next = lo;
}
__device__ __forceinline__ uint32_t next_trial(uint32_t& s_next, uint32_t t_end) {
    const uint32_t j = atomicAdd(&s_next, 1u);
    return j < t_end ? j : t_end;
}

}  // namespace distill
