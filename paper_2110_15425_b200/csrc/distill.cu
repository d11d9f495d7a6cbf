// distill.cu — host side of the C ABI declared in include/distill.h:
// validation, the model handle (device read-only block), launch
// configuration, and the host-buffer end-to-end entry.  All arithmetic of the
// hot path runs in the kernels of pp.cuh / keys.cuh / ddm.cuh / stroop.cuh.
#include "../../include/distill.h"

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "ddm.cuh"
#include "keys.cuh"
#include "pp.cuh"
#include "stroop.cuh"
#include "rad_table.h"
#include "rng_probe.cuh"

using namespace distill;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

distill_status fail(distill_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail(DISTILL_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                              \
    } while (0)

// Scoped device selection: every entry that works on a model's device
// restores the caller's current device on return (the library never leaves
// the calling thread on another device).
struct DeviceScope {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceScope(int dev) {
        int cur = -1;
        err = cudaGetDevice(&cur);
        if (err == cudaSuccess && cur != dev) {
            err = cudaSetDevice(dev);
            if (err == cudaSuccess) prev = cur;
        }
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};
#define DEVICE_SCOPE(dev)         \
    DeviceScope device_scope_(dev); \
    CUDA_TRY(device_scope_.err)

// ---------------------------------------------------------------- radius table
// spec/RNG.md §3: the host builds RT (rad_table.h), uploads it once per device
// and never frees it.
std::mutex g_rt_mu;
constexpr int MAX_DEVICES = 64;
float4* g_rt_dev[MAX_DEVICES] = {nullptr};

// The device copy of RT for `device` (uploaded on first use; the caller has made
// `device` current).  First use must not happen inside a CUDA-graph capture.
distill_status rad_table(int device, const float4** out) {
    std::lock_guard<std::mutex> lock(g_rt_mu);
    if (device < 0 || device >= MAX_DEVICES) return fail(DISTILL_E_INVALID_ARG, "rad_table: bad device %d", device);
    if (!g_rt_dev[device]) {
        static std::vector<float4> host;
        if (host.empty()) {
            host.resize(RT_ROWS);
            build_rad_table(host.data());
        }
        float4* d = nullptr;
        CUDA_TRY(cudaMalloc(&d, RT_ROWS * sizeof(float4)));
        cudaError_t e = cudaMemcpy(d, host.data(), RT_ROWS * sizeof(float4), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(d);
            return fail(DISTILL_E_CUDA, "rad_table: %s", cudaGetErrorString(e));
        }
        g_rt_dev[device] = d;
    }
    *out = g_rt_dev[device];
    return DISTILL_OK;
}

constexpr int PP_BLOCK = 128;
constexpr int ARGMAX_BLOCK = 256;
// sample / trial loops step a 32-bit counter by up to 2 (PP pairs) or a grid
// stride (Stroop): bounding the count at 2^31 keeps them from wrapping
constexpr uint32_t MAX_SAMPLES = 1u << 31;
#ifndef DISTILL_PP_SMALL_MODE
#define DISTILL_PP_SMALL_MODE 1   // 0: always one thread per allocation (A/B measurements only)
#endif
#ifndef DISTILL_PP_SMALL_THREADS_PER_SM
#define DISTILL_PP_SMALL_THREADS_PER_SM 512    // 32 lanes per allocation up to 16 allocations per SM
#endif
constexpr uint64_t PP_SMALL_THREADS_PER_SM = DISTILL_PP_SMALL_THREADS_PER_SM;   // latency-mode threshold
constexpr int PP_SMALL_WARPS = 4;    // pp_eval_small_kernel: allocations per block
constexpr uint32_t PP_SMALL_SMAX = 1024;   // its per-warp sample buffer (32 lanes per allocation)
constexpr uint32_t PP_SMALL_SMAX8 = 256;   // per-allocation buffer with 8 lanes per allocation
#ifndef DISTILL_PP_SMALL8_THREADS_PER_SM
#define DISTILL_PP_SMALL8_THREADS_PER_SM 768   // 8 lanes per allocation up to 96 allocations per SM
#endif
constexpr uint64_t PP_SMALL8_THREADS_PER_SM = DISTILL_PP_SMALL8_THREADS_PER_SM;
constexpr uint32_t PP_SMALL_SMAX4 = 128;   // per-allocation buffer with 4 lanes per allocation
#ifndef DISTILL_PP_SMALL4_THREADS_PER_SM
#define DISTILL_PP_SMALL4_THREADS_PER_SM 768    // 4 lanes per allocation up to 192 allocations per SM (r02_small_threshold.txt)
#endif
constexpr uint64_t PP_SMALL4_THREADS_PER_SM = DISTILL_PP_SMALL4_THREADS_PER_SM;
constexpr int DDM_BLOCK = 128;
#ifndef DISTILL_DDM_MINB
#define DISTILL_DDM_MINB 6
#endif
constexpr int DDM_MINB = DISTILL_DDM_MINB;     // tools/acc_tune.cu sweep (profiles/r01_acc_tune.txt, v5)
constexpr int STROOP_BLOCK = 128;
constexpr int STROOP_MINB = 0;   // same sweep

}  // namespace

struct distill_model {
    uint32_t kind = 0, D = 0;
    int device = 0;
    uint32_t L[8] = {0};
    uint64_t n_alloc = 0;
    float w[8] = {0};
    std::vector<float> params;
    float* d_levels = nullptr;      // device RO block
    const float4* d_rt = nullptr;   // the device's radius table (spec/RNG.md §3), library-global
    int n_sm = 148;
    // device scratch of the synchronous host-buffer entry (lazily grown, guarded by the mutex)
    std::mutex scratch_mu;
    void* d_scratch = nullptr;
    size_t scratch_bytes = 0;
    // completion of the last host-buffer launch (any stream): the next one waits for it,
    // so launches sharing the scratch key/counter never overlap (the async entry)
    cudaEvent_t host_ev = nullptr;
};

// Scratch layout (eval_grid_host): [0, 8) published-path key (kept at KEY_INIT
// between calls), [8, 12) its block counter (kept at 0), [16, 24) copy-path
// key, [256, ...) copy-path net values.
static distill_status ensure_scratch(distill_model* m, size_t bytes) {
    if (m->scratch_bytes >= bytes) return DISTILL_OK;
    if (m->d_scratch) cudaFree(m->d_scratch);
    m->d_scratch = nullptr;
    m->scratch_bytes = 0;
    CUDA_TRY(cudaMalloc(&m->d_scratch, bytes));
    CUDA_TRY(cudaMemset(m->d_scratch, 0xFF, 8));
    CUDA_TRY(cudaMemset((char*)m->d_scratch + 8, 0, 8));
    CUDA_TRY(cudaDeviceSynchronize());
    m->scratch_bytes = bytes;
    return DISTILL_OK;
}

extern "C" {

int distill_abi_version(void) { return DISTILL_ABI_VERSION; }

const char* distill_last_error(void) { return g_last_error.c_str(); }

uint64_t distill_launch_count(void) { return g_launches.load(); }

distill_status distill_load_model(const distill_model_desc* desc, int device, distill_model** out) {
    if (!desc || !out) return fail(DISTILL_E_INVALID_ARG, "load_model: NULL desc/out");
    *out = nullptr;
    if (!desc->n_levels || !desc->levels || !desc->cost_weights || (!desc->params && desc->n_params))
        return fail(DISTILL_E_INVALID_ARG, "load_model: NULL array in desc");
    uint32_t want_D, want_p;
    if (desc->kind == DISTILL_MODEL_PREDATOR_PREY) { want_D = 3; want_p = 3; }
    else if (desc->kind == DISTILL_MODEL_STROOP_LCA) { want_D = 2; want_p = 11; }
    else if (desc->kind == DISTILL_MODEL_EXT_STROOP_A || desc->kind == DISTILL_MODEL_EXT_STROOP_B) { want_D = 2; want_p = 13; }
    else if (desc->kind == DISTILL_MODEL_DDM_GRID) { want_D = 2; want_p = 7; }
    else return fail(DISTILL_E_UNSUPPORTED, "load_model: unknown model kind %u", desc->kind);
    if (desc->n_signals != want_D)
        return fail(DISTILL_E_UNSUPPORTED, "load_model: kind %u needs %u signals, got %u", desc->kind, want_D,
                    desc->n_signals);
    if (desc->n_params != want_p)
        return fail(DISTILL_E_INVALID_ARG, "load_model: kind %u needs %u params, got %u", desc->kind, want_p,
                    desc->n_params);
    uint64_t n = 1, total = 0;
    for (uint32_t d = 0; d < want_D; ++d) {
        if (desc->n_levels[d] == 0) return fail(DISTILL_E_INVALID_ARG, "load_model: signal %u has 0 levels", d);
        n *= desc->n_levels[d];
        total += desc->n_levels[d];
        if (n > 0xFFFFFFFFull)
            return fail(DISTILL_E_OVERFLOW, "load_model: grid exceeds 2^32-1 allocations");
    }
    if (desc->kind == DISTILL_MODEL_STROOP_LCA) {
        const float ns = desc->params[10];
        if (!(ns >= 1.0f) || ns != std::floor(ns) || ns > 1e7f)
            return fail(DISTILL_E_INVALID_ARG, "load_model: Stroop n_steps must be a positive integer");
    }
    if (desc->kind == DISTILL_MODEL_DDM_GRID) {
        const float ns = desc->params[6];
        if (!(ns >= 1.0f) || ns != std::floor(ns) || ns > 1e7f)
            return fail(DISTILL_E_INVALID_ARG, "load_model: DDM-grid n_steps must be a positive integer");
    }
    if (desc->kind == DISTILL_MODEL_EXT_STROOP_A || desc->kind == DISTILL_MODEL_EXT_STROOP_B) {
        for (int q : {3, 10}) {
            const float ns = desc->params[q];
            if (!(ns >= 0.0f) || ns != std::floor(ns) || ns > 1e7f || (q == 10 && ns < 1.0f))
                return fail(DISTILL_E_INVALID_ARG, "load_model: Ext-Stroop N_h / N_d must be integers (N_d >= 1)");
        }
    }
    int n_dev = 0;
    CUDA_TRY(cudaGetDeviceCount(&n_dev));
    if (device < 0 || device >= n_dev) return fail(DISTILL_E_INVALID_ARG, "load_model: bad device %d", device);
    distill_model* m = new (std::nothrow) distill_model();
    if (!m) return fail(DISTILL_E_CUDA, "load_model: out of host memory");
    m->kind = desc->kind;
    m->D = want_D;
    m->device = device;
    m->n_alloc = n;
    for (uint32_t d = 0; d < want_D; ++d) {
        m->L[d] = desc->n_levels[d];
        m->w[d] = desc->cost_weights[d];
    }
    m->params.assign(desc->params, desc->params + desc->n_params);
    DeviceScope scope(device);
    cudaError_t e = scope.err;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&m->n_sm, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaMalloc(&m->d_levels, total * sizeof(float));
    if (e == cudaSuccess) e = cudaMemcpy(m->d_levels, desc->levels, total * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (m->d_levels) cudaFree(m->d_levels);
        delete m;
        return fail(DISTILL_E_CUDA, "load_model: %s", cudaGetErrorString(e));
    }
    const distill_status rs = rad_table(device, &m->d_rt);
    if (rs != DISTILL_OK) {
        cudaFree(m->d_levels);
        delete m;
        return rs;
    }
    *out = m;
    return DISTILL_OK;
}

void distill_free_model(distill_model* m) {
    if (!m) return;
    DeviceScope scope(m->device);
    if (m->d_levels) cudaFree(m->d_levels);
    if (m->d_scratch) cudaFree(m->d_scratch);
    if (m->host_ev) cudaEventDestroy(m->host_ev);
    delete m;
}

distill_status distill_grid_size(const distill_model* m, uint64_t* n_alloc) {
    if (!m || !n_alloc) return fail(DISTILL_E_INVALID_ARG, "grid_size: NULL argument");
    *n_alloc = m->n_alloc;
    return DISTILL_OK;
}

// Latency mode (pp_eval_small_kernel, one warp per allocation) for grids that
// cannot fill the GPU one thread per allocation.
// The model-derived part of a predator-prey launch (params, weights, levels,
// key); callers fill positions, the range and the outputs.
static PPArgs pp_base_args(const distill_model* m, uint32_t n_samples, uint64_t seed) {
    PPArgs p;
    memset(&p, 0, sizeof p);
    p.sigma_max = m->params[0]; p.sigma_min = m->params[1]; p.kappa = m->params[2];
    p.w0 = m->w[0]; p.w1 = m->w[1]; p.w2 = m->w[2];
    p.L0 = m->L[0]; p.L1 = m->L[1]; p.L2 = m->L[2];
    p.n_samples = n_samples;
    p.key0 = (uint32_t)seed; p.key1 = (uint32_t)(seed >> 32);
    p.begin = 0; p.count = (uint32_t)m->n_alloc;
    p.levels = m->d_levels;
    p.n_sets = 1;
    p.rad_tab = m->d_rt;
    return p;
}

// 0: one thread per allocation; otherwise the lanes per allocation of the
// latency-mode kernel (32 for the smallest grids, 8 for mid-size ones).
static int pp_small_lanes(const distill_model* m, uint64_t count, uint32_t n_samples) {
    // measured switch points (tools/small_threshold.py, profiles/r01_small_threshold.txt)
    if (!DISTILL_PP_SMALL_MODE) return 0;
    const uint64_t sms = (uint64_t)m->n_sm;
    if (n_samples <= PP_SMALL_SMAX8 && count * 8 <= sms * PP_SMALL8_THREADS_PER_SM)
        return count * 32 <= sms * PP_SMALL_THREADS_PER_SM ? 32 : 8;
    if (n_samples <= PP_SMALL_SMAX4 && count * 4 <= sms * PP_SMALL4_THREADS_PER_SM) return 4;
    if (n_samples <= PP_SMALL_SMAX && count <= sms * 64) return 32;   // long sample loops: the warp kernel wins longer
    return 0;
}
static bool pp_small(const distill_model* m, uint64_t count, uint32_t n_samples) {
    return pp_small_lanes(m, count, n_samples) != 0;
}

static void launch_pp_small(const distill_model* m, const PPArgs& p, uint64_t count, cudaStream_t st) {
    if (pp_small_lanes(m, count, p.n_samples) == 32) {
        const unsigned grid = (unsigned)((count + PP_SMALL_WARPS - 1) / PP_SMALL_WARPS);
        if (p.publish) pp_eval_small_kernel<PP_SMALL_WARPS, PP_SMALL_SMAX, 32, true><<<grid, PP_SMALL_WARPS * 32, 0, st>>>(p);
        else pp_eval_small_kernel<PP_SMALL_WARPS, PP_SMALL_SMAX, 32><<<grid, PP_SMALL_WARPS * 32, 0, st>>>(p);
    } else if (pp_small_lanes(m, count, p.n_samples) == 8) {
        const unsigned grid = (unsigned)((count + PP_SMALL_WARPS * 4 - 1) / (PP_SMALL_WARPS * 4));
        if (p.publish) pp_eval_small_kernel<PP_SMALL_WARPS, PP_SMALL_SMAX8, 8, true><<<grid, PP_SMALL_WARPS * 32, 0, st>>>(p);
        else pp_eval_small_kernel<PP_SMALL_WARPS, PP_SMALL_SMAX8, 8><<<grid, PP_SMALL_WARPS * 32, 0, st>>>(p);
    } else {
        const unsigned grid = (unsigned)((count + PP_SMALL_WARPS * 8 - 1) / (PP_SMALL_WARPS * 8));
        if (p.publish) pp_eval_small_kernel<PP_SMALL_WARPS, PP_SMALL_SMAX4, 4, true><<<grid, PP_SMALL_WARPS * 32, 0, st>>>(p);
        else pp_eval_small_kernel<PP_SMALL_WARPS, PP_SMALL_SMAX4, 4><<<grid, PP_SMALL_WARPS * 32, 0, st>>>(p);
    }
}

// The grid-search launch every predator-prey path uses: the latency-mode
// kernel for grids too small to fill the GPU, otherwise one thread per
// allocation (sample pairs in float2 lanes when S is even); several
// invocations go on gridDim.y (MULTI); PUB publishes the key to pinned host
// memory from the last block.
static void launch_pp_search(const distill_model* m, const PPArgs& p, uint32_t n_invocations, cudaStream_t st) {
    const uint64_t count = p.count;
    if (n_invocations == 1 && pp_small(m, count, p.n_samples)) {
        launch_pp_small(m, p, count, st);
    } else {
        const dim3 grid((unsigned)((count + PP_BLOCK - 1) / PP_BLOCK), n_invocations);
        const bool even = (p.n_samples & 1u) == 0;
        constexpr int B = PP_BLOCK, MK = DISTILL_PP_MASK, MB = DISTILL_PP_MINB;
        if (n_invocations > 1) {
            if (even) pp_eval_grid_kernel<B, MK, MB, DISTILL_PP_PIPE, true, true><<<grid, B, 0, st>>>(p);
            else pp_eval_grid_kernel<B, MK, MB, DISTILL_PP_PIPE, false, true><<<grid, B, 0, st>>>(p);
        } else if (p.publish) {
            if (even) pp_eval_grid_kernel<B, MK, MB, DISTILL_PP_PIPE, true, false, true><<<grid, B, 0, st>>>(p);
            else pp_eval_grid_kernel<B, MK, MB, DISTILL_PP_PIPE, false, false, true><<<grid, B, 0, st>>>(p);
        } else {
            if (even) pp_eval_grid_kernel<B, MK, MB, DISTILL_PP_PIPE, true><<<grid, B, 0, st>>>(p);
            else pp_eval_grid_kernel<B, MK, MB, DISTILL_PP_PIPE><<<grid, B, 0, st>>>(p);
        }
    }
    g_launches++;
}

static distill_status launch_pp(const distill_model* m, const distill_eval_args* a, cudaStream_t st,
                                key64_t* publish = nullptr, unsigned int* done = nullptr) {
    if (!a->inputs || a->n_inputs != 6) return fail(DISTILL_E_INVALID_ARG, "eval_grid(PP): needs 6 host inputs");
    if (a->n_samples == 0 || a->n_samples > MAX_SAMPLES)
        return fail(DISTILL_E_INVALID_ARG, "eval_grid(PP): n_samples must be in [1, 2^31]");
    if ((a->trial_begin | a->trial_end) != 0)
        return fail(DISTILL_E_INVALID_ARG, "eval_grid(PP): trial range is a Stroop-only field");
    const uint64_t count = a->end - a->begin;
    if (count == 0) return DISTILL_OK;
    PPArgs p = pp_base_args(m, a->n_samples, a->seed);
    p.prey_x = a->inputs[0]; p.prey_y = a->inputs[1];
    p.pred_x = a->inputs[2]; p.pred_y = a->inputs[3];
    p.pl_x = a->inputs[4]; p.pl_y = a->inputs[5];
    p.invocation = a->invocation;
    p.begin = (uint32_t)a->begin; p.count = (uint32_t)count;
    p.net = a->d_net; p.best = a->d_best;
    p.key_signed = a->key_order;
    p.publish = publish; p.done = done;
    launch_pp_search(m, p, 1, st);
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_eval_grid_multi(const distill_model* m, const distill_multi_args* a, void* stream) {
    if (!m || !a) return fail(DISTILL_E_INVALID_ARG, "eval_grid_multi: NULL model/args");
    if (m->kind != DISTILL_MODEL_PREDATOR_PREY) return fail(DISTILL_E_UNSUPPORTED, "eval_grid_multi: predator-prey only");
    if (!a->d_inputs || a->n_sets == 0) return fail(DISTILL_E_INVALID_ARG, "eval_grid_multi: needs n_sets >= 1 device position sets");
    if (reinterpret_cast<uintptr_t>(a->d_inputs) & 3u) return fail(DISTILL_E_INVALID_ARG, "eval_grid_multi: d_inputs misaligned");
    if (a->n_samples == 0 || a->n_samples > MAX_SAMPLES)
        return fail(DISTILL_E_INVALID_ARG, "eval_grid_multi: n_samples must be in [1, 2^31]");
    if (a->n_invocations > 65535u) return fail(DISTILL_E_INVALID_ARG, "eval_grid_multi: at most 65535 invocations per call");
    if (a->begin > a->end || a->end > m->n_alloc) return fail(DISTILL_E_INVALID_ARG, "eval_grid_multi: bad allocation range");
    if ((uint64_t)a->invocation0 + a->n_invocations > 0xFFFFFFFFull)
        return fail(DISTILL_E_OVERFLOW, "eval_grid_multi: invocation counter overflow");
    const uint64_t count = a->end - a->begin;
    if (count == 0 || a->n_invocations == 0) return DISTILL_OK;
    DEVICE_SCOPE(m->device);
    PPArgs p = pp_base_args(m, a->n_samples, a->seed);   // positions come from d_inputs
    p.invocation = a->invocation0;
    p.begin = (uint32_t)a->begin; p.count = (uint32_t)count;
    p.net = a->d_net; p.best = a->d_best;
    p.pos_dev = a->d_inputs; p.n_sets = a->n_sets;
    launch_pp_search(m, p, a->n_invocations, (cudaStream_t)stream);
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

// Blocks along the trial axis per allocation for the trial-streaming kernels
// (R14b): enough blocks in all for ~8 waves of 8 resident blocks per SM, but
// each lane's stream at least 16 trials long, so that the end of a lane's
// stream (its warp waiting for the last trials) stays short against it.
static uint32_t trial_chunks(int n_sm, uint64_t count, uint32_t tr) {
    const uint64_t fill = (uint64_t)n_sm * 8 * 8;
    const uint64_t want = (fill + count - 1) / count;
    const uint64_t cap = std::max<uint64_t>(1, tr / (STROOP_BLOCK * 16u));
    const uint64_t most = std::max<uint64_t>(1, (tr + STROOP_BLOCK - 1) / STROOP_BLOCK);
    return (uint32_t)std::max<uint64_t>(1, std::min(std::min(want, cap), most));
}

static distill_status launch_stroop(distill_model* m, const distill_eval_args* a, cudaStream_t st) {
    if (a->n_samples == 0 || a->n_samples > MAX_SAMPLES)
        return fail(DISTILL_E_INVALID_ARG, "eval_grid(Stroop): n_samples (trials) must be in [1, 2^31]");
    if (a->invocation != 0) return fail(DISTILL_E_INVALID_ARG, "eval_grid(Stroop): invocation must be 0");
    uint32_t tb = a->trial_begin, te = a->trial_end;
    if (tb == 0 && te == 0) te = a->n_samples;
    if (tb > te || te > a->n_samples) return fail(DISTILL_E_INVALID_ARG, "eval_grid(Stroop): bad trial range");
    const bool full = (tb == 0 && te == a->n_samples);
    const uint64_t count = a->end - a->begin;
    if (count == 0) return DISTILL_OK;
    if (a->n_samples > 0 && (uint64_t)m->n_alloc * a->n_samples >= (1ull << 63))
        return fail(DISTILL_E_OVERFLOW, "eval_grid(Stroop): RNG unit id overflow");
    // Caller-owned counts: the integer outcomes live between the simulate and
    // finalize kernels, and a shared library scratch area would race between
    // streams evaluating the same handle concurrently.
    unsigned long long* counts = a->d_counts;
    if (!counts) return fail(DISTILL_E_INVALID_ARG, "eval_grid(Stroop kinds): d_counts is required");
    if (reinterpret_cast<uintptr_t>(counts) & 7u) return fail(DISTILL_E_INVALID_ARG, "eval_grid: d_counts must be 8-byte aligned");
    CUDA_TRY(cudaMemsetAsync(counts, 0, count * 3 * sizeof(unsigned long long), st));
    StroopArgs p;
    memset(&p, 0, sizeof p);
    const float* P = m->params.data();
    const bool ddmg = m->kind == DISTILL_MODEL_DDM_GRID;
    if (ddmg) {   // spec/MODELS.md §6c: A0, g_a, sigma, dt, R, c_rt, N — the finalize needs dt, R, c_rt, N
        p.dt = P[3]; p.reward = P[4]; p.rt_cost = P[5]; p.n_steps = (uint32_t)P[6];
    } else {
        p.g_c = P[0]; p.g_w = P[1]; p.tau = P[2]; p.leak = P[3]; p.inh = P[4]; p.noise = P[5];
        p.dt = P[6]; p.thr = P[7]; p.reward = P[8]; p.rt_cost = P[9]; p.n_steps = (uint32_t)P[10];
    }
    p.w0 = m->w[0]; p.w1 = m->w[1];
    p.L0 = m->L[0]; p.L1 = m->L[1];
    p.n_trials = a->n_samples; p.trial_begin = tb; p.trial_end = te;
    p.key0 = (uint32_t)a->seed; p.key1 = (uint32_t)(a->seed >> 32);
    p.begin = (uint32_t)a->begin; p.count = (uint32_t)count;
    p.levels = m->d_levels; p.counts = counts; p.net = a->d_net; p.best = a->d_best;
    p.key_signed = a->key_order;
    p.rad_tab = m->d_rt;
    const uint32_t tr = te - tb;
    if (tr > 0) {
        const uint32_t chunks = trial_chunks(m->n_sm, count, tr);
        const size_t table_bytes = 4ull * p.n_steps * sizeof(float);
        DdmgArgs q;
        if (ddmg) {
            q.A0 = P[0]; q.g_a = P[1]; q.noise = P[2]; q.dt = P[3]; q.n_steps = (uint32_t)P[6];
            q.L0 = m->L[0]; q.L1 = m->L[1]; q.n_trials = a->n_samples; q.trial_begin = tb; q.trial_end = te;
            q.key0 = p.key0; q.key1 = p.key1; q.begin = p.begin; q.count = p.count;
            q.levels = m->d_levels; q.counts = counts; q.rad_tab = m->d_rt;
        }
        for (uint64_t off = 0; off < count; off += 65535) {
            const unsigned gy = (unsigned)std::min<uint64_t>(65535, count - off);
            static_assert(DDM_BLOCK == STROOP_BLOCK, "the trial chunks above are sized for STROOP_BLOCK");
            if (ddmg)
                ddmg_sim_kernel<DDM_BLOCK, DDM_MINB><<<dim3(chunks, gy), DDM_BLOCK, 0, st>>>(q, (uint32_t)off);
            else if (table_bytes <= 32 * 1024)      // pathway table in shared memory (trial-invariant h_k(n); + RT <= 48 KB)
                stroop_sim_kernel<STROOP_BLOCK, STROOP_MINB, true><<<dim3(chunks, gy), STROOP_BLOCK, table_bytes, st>>>(
                    p, (uint32_t)off);
            else
                stroop_sim_kernel<STROOP_BLOCK, STROOP_MINB, false><<<dim3(chunks, gy), STROOP_BLOCK, 0, st>>>(
                    p, (uint32_t)off);
            g_launches++;
            CUDA_TRY(cudaGetLastError());
        }
    }
    if (full && (a->d_net || a->d_best)) {
        const unsigned grid = (unsigned)((count + STROOP_BLOCK - 1) / STROOP_BLOCK);
        stroop_finalize_kernel<STROOP_BLOCK><<<grid, STROOP_BLOCK, 0, st>>>(p);
        g_launches++;
        CUDA_TRY(cudaGetLastError());
    }
    return DISTILL_OK;
}

extern "C++" {
template <int VARIANT>
void launch_ext_stroop_kernels(const ExtStroopArgs& p, uint32_t chunks, uint64_t count, bool sim, bool fin,
                                      cudaStream_t st) {
    if (sim)
        for (uint64_t off = 0; off < count; off += 65535) {
            const unsigned gy = (unsigned)std::min<uint64_t>(65535, count - off);
            ext_stroop_sim_kernel<STROOP_BLOCK, VARIANT><<<dim3(chunks, gy), STROOP_BLOCK, 0, st>>>(p, (uint32_t)off);
            g_launches++;
        }
    if (fin) {
        ext_stroop_finalize_kernel<STROOP_BLOCK, VARIANT>
            <<<(unsigned)((count + STROOP_BLOCK - 1) / STROOP_BLOCK), STROOP_BLOCK, 0, st>>>(p);
        g_launches++;
    }
}
}  // extern "C++"

distill_status distill_stroop_energy(const distill_model* m, uint64_t alloc, uint32_t n_trials,
                                     uint32_t trial_begin, uint32_t trial_end, uint64_t seed,
                                     unsigned long long* d_esum, void* stream) {
    if (!m || !d_esum) return fail(DISTILL_E_INVALID_ARG, "stroop_energy: NULL model/d_esum");
    if (reinterpret_cast<uintptr_t>(d_esum) & 7u) return fail(DISTILL_E_INVALID_ARG, "stroop_energy: d_esum must be 8-byte aligned");
    if (m->kind != DISTILL_MODEL_STROOP_LCA) return fail(DISTILL_E_UNSUPPORTED, "stroop_energy: Stroop-LCA models only");
    if (alloc >= m->n_alloc) return fail(DISTILL_E_INVALID_ARG, "stroop_energy: allocation index past the grid");
    if (n_trials == 0 || n_trials > MAX_SAMPLES || trial_begin > trial_end || trial_end > n_trials)
        return fail(DISTILL_E_INVALID_ARG, "stroop_energy: bad trial range");
    if ((uint64_t)m->n_alloc * n_trials >= (1ull << 63)) return fail(DISTILL_E_OVERFLOW, "stroop_energy: RNG unit overflow");
    const uint32_t N = (uint32_t)m->params[10];
    if (N > 4096) return fail(DISTILL_E_UNSUPPORTED, "stroop_energy: at most 4096 steps");
    if (trial_begin == trial_end) return DISTILL_OK;
    DEVICE_SCOPE(m->device);
    StroopArgs p;
    memset(&p, 0, sizeof p);
    const float* P = m->params.data();
    p.g_c = P[0]; p.g_w = P[1]; p.tau = P[2]; p.leak = P[3]; p.inh = P[4]; p.noise = P[5];
    p.dt = P[6]; p.thr = P[7]; p.reward = P[8]; p.rt_cost = P[9]; p.n_steps = N;
    p.L0 = m->L[0]; p.L1 = m->L[1];
    p.n_trials = n_trials; p.trial_begin = trial_begin; p.trial_end = trial_end;
    p.key0 = (uint32_t)seed; p.key1 = (uint32_t)(seed >> 32);
    p.levels = m->d_levels;
    p.rad_tab = m->d_rt;
    const uint32_t tr = trial_end - trial_begin;
    const unsigned grid = (unsigned)std::min<uint64_t>((tr + STROOP_BLOCK - 1) / STROOP_BLOCK, (uint64_t)m->n_sm * 8);
    stroop_energy_kernel<STROOP_BLOCK><<<grid, STROOP_BLOCK, N * sizeof(unsigned long long), (cudaStream_t)stream>>>(
        p, (uint32_t)alloc, d_esum);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

static distill_status launch_ext_stroop(distill_model* m, const distill_eval_args* a, cudaStream_t st) {
    if (a->n_samples == 0 || a->n_samples > MAX_SAMPLES)
        return fail(DISTILL_E_INVALID_ARG, "eval_grid(Ext-Stroop): n_samples (trials) must be in [1, 2^31]");
    if (a->invocation != 0) return fail(DISTILL_E_INVALID_ARG, "eval_grid(Ext-Stroop): invocation must be 0");
    uint32_t tb = a->trial_begin, te = a->trial_end;
    if (tb == 0 && te == 0) te = a->n_samples;
    if (tb > te || te > a->n_samples) return fail(DISTILL_E_INVALID_ARG, "eval_grid(Ext-Stroop): bad trial range");
    const bool full = (tb == 0 && te == a->n_samples);
    const uint64_t count = a->end - a->begin;
    if (count == 0) return DISTILL_OK;
    // Caller-owned counts: the integer outcomes live between the simulate and
    // finalize kernels, and a shared library scratch area would race between
    // streams evaluating the same handle concurrently.
    unsigned long long* counts = a->d_counts;
    if (!counts) return fail(DISTILL_E_INVALID_ARG, "eval_grid(Stroop kinds): d_counts is required");
    if (reinterpret_cast<uintptr_t>(counts) & 7u) return fail(DISTILL_E_INVALID_ARG, "eval_grid: d_counts must be 8-byte aligned");
    CUDA_TRY(cudaMemsetAsync(counts, 0, count * 3 * sizeof(unsigned long long), st));
    const float* P = m->params.data();
    ExtStroopArgs p;
    p.g_c = P[0]; p.g_w = P[1]; p.tau = P[2]; p.n_h = (uint32_t)P[3]; p.lam = P[4]; p.a_p = P[5]; p.gam = P[6];
    p.sig = P[7]; p.dt = P[8]; p.z = P[9]; p.n_d = (uint32_t)P[10]; p.reward = P[11]; p.rt_cost = P[12];
    p.w0 = m->w[0]; p.w1 = m->w[1]; p.L0 = m->L[0]; p.L1 = m->L[1];
    p.n_trials = a->n_samples; p.trial_begin = tb; p.trial_end = te;
    p.key0 = (uint32_t)a->seed; p.key1 = (uint32_t)(a->seed >> 32);
    p.begin = (uint32_t)a->begin; p.count = (uint32_t)count;
    p.levels = m->d_levels; p.counts = counts; p.net = a->d_net; p.best = a->d_best;
    p.key_signed = a->key_order;
    p.rad_tab = m->d_rt;
    const uint32_t tr = te - tb;
    const uint32_t chunks = trial_chunks(m->n_sm, count, tr);
    const bool fin = full && (a->d_net || a->d_best);
    if (m->kind == DISTILL_MODEL_EXT_STROOP_A) launch_ext_stroop_kernels<0>(p, chunks, count, tr > 0, fin, st);
    else launch_ext_stroop_kernels<1>(p, chunks, count, tr > 0, fin, st);
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_eval_grid(const distill_model* mc, const distill_eval_args* a, void* stream) {
    if (!mc || !a) return fail(DISTILL_E_INVALID_ARG, "eval_grid: NULL model/args");
    distill_model* m = const_cast<distill_model*>(mc);
    if (a->begin > a->end || a->end > m->n_alloc)
        return fail(DISTILL_E_INVALID_ARG, "eval_grid: range [%llu, %llu) outside grid of %llu",
                    (unsigned long long)a->begin, (unsigned long long)a->end, (unsigned long long)m->n_alloc);
    if (a->d_net && (reinterpret_cast<uintptr_t>(a->d_net) & 3u))
        return fail(DISTILL_E_INVALID_ARG, "eval_grid: d_net must be 4-byte aligned");
    if (a->d_best && (reinterpret_cast<uintptr_t>(a->d_best) & 7u))
        return fail(DISTILL_E_INVALID_ARG, "eval_grid: d_best must be 8-byte aligned");
    if (a->key_order > 1) return fail(DISTILL_E_INVALID_ARG, "eval_grid: key_order must be 0 or 1");
    DEVICE_SCOPE(m->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (m->kind == DISTILL_MODEL_PREDATOR_PREY) return launch_pp(m, a, st);
    if (m->kind == DISTILL_MODEL_STROOP_LCA || m->kind == DISTILL_MODEL_DDM_GRID) return launch_stroop(m, a, st);
    return launch_ext_stroop(m, a, st);
}

// The host-buffer entries: `sync` = distill_eval_grid_host (synchronises the stream;
// pageable buffers allowed), !sync = distill_eval_grid_host_async (enqueue only;
// pinned, device-mapped buffers required).
static distill_status eval_grid_host_impl(const distill_model* mc, const float* h_inputs, uint32_t n_inputs,
                                          uint64_t begin, uint64_t end, uint32_t n_samples, uint32_t invocation,
                                          uint64_t seed, float* h_net, unsigned long long* h_best, void* stream,
                                          bool sync) {
    if (!mc || !h_best) return fail(DISTILL_E_INVALID_ARG, "eval_grid_host: NULL model/h_best");
    distill_model* m = const_cast<distill_model*>(mc);
    if (m->kind != DISTILL_MODEL_PREDATOR_PREY)
        return fail(DISTILL_E_UNSUPPORTED, "eval_grid_host: predator-prey models only");
    if (begin > end || end > m->n_alloc) return fail(DISTILL_E_INVALID_ARG, "eval_grid_host: bad range");
    DEVICE_SCOPE(m->device);
    std::lock_guard<std::mutex> lock(m->scratch_mu);
    const uint64_t count = end - begin;
    const size_t net_off = 256;
    distill_status s = ensure_scratch(m, net_off + count * sizeof(float));
    if (s != DISTILL_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    float* d_net = nullptr;
    bool direct = false;
    if (h_net) {
        // Pinned (page-locked, device-mapped) h_net: the kernel stores V straight into
        // host memory over the link, overlapped with the computation (4 B per 100
        // evaluations is ~5 GB/s at full speed).  Pageable h_net: device scratch + copy.
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, h_net) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer != nullptr && (reinterpret_cast<uintptr_t>(pa.devicePointer) & 3u) == 0) {
            d_net = (float*)pa.devicePointer;
            direct = true;
        } else {
            (void)cudaGetLastError();
            d_net = (float*)((char*)m->d_scratch + net_off);
        }
    }
    // Pinned h_best: the kernel's last block publishes the key into it and re-arms
    // the device key (one launch, no memset, no copy).  Pageable: memset + copy.
    key64_t* publish = nullptr;
    {
        cudaPointerAttributes pb;
        if (cudaPointerGetAttributes(&pb, h_best) == cudaSuccess && pb.type == cudaMemoryTypeHost &&
            pb.devicePointer != nullptr && (reinterpret_cast<uintptr_t>(pb.devicePointer) & 7u) == 0)
            publish = (key64_t*)pb.devicePointer;
        else
            (void)cudaGetLastError();
    }
    // Host->device: this step's inputs (the 6 positions, 24 B) travel inside the
    // kernel's launch parameters; device->host: V (if h_net) and the best key.
    if (!h_inputs || n_inputs != 6) return fail(DISTILL_E_INVALID_ARG, "eval_grid_host: needs 6 inputs");
    if (!sync && (!publish || (h_net && !direct)))
        return fail(DISTILL_E_INVALID_ARG, "eval_grid_host_async: h_net and h_best must be pinned, device-mapped "
                                           "host memory (4- and 8-byte aligned)");
    // order after the previous host-buffer launch of this handle (it may be in flight on another stream)
    if (!m->host_ev) CUDA_TRY(cudaEventCreateWithFlags(&m->host_ev, cudaEventDisableTiming));
    else CUDA_TRY(cudaStreamWaitEvent(st, m->host_ev, 0));
    distill_eval_args a;
    memset(&a, 0, sizeof a);
    a.inputs = h_inputs; a.n_inputs = n_inputs; a.begin = begin; a.end = end;
    a.n_samples = n_samples; a.invocation = invocation; a.seed = seed;
    a.d_net = d_net;
    if (publish && count > 0) {
        a.d_best = (unsigned long long*)m->d_scratch;
        s = launch_pp(m, &a, st, publish, (unsigned int*)((char*)m->d_scratch + 8));
        if (s != DISTILL_OK) return s;
        if (h_net && !direct) CUDA_TRY(cudaMemcpyAsync(h_net, d_net, count * sizeof(float), cudaMemcpyDeviceToHost, st));
    } else {
        unsigned long long* d_best = (unsigned long long*)((char*)m->d_scratch + 16);
        a.d_best = d_best;
        CUDA_TRY(cudaMemsetAsync(d_best, 0xFF, sizeof(unsigned long long), st));
        s = launch_pp(m, &a, st);
        if (s != DISTILL_OK) return s;
        if (h_net && !direct) CUDA_TRY(cudaMemcpyAsync(h_net, d_net, count * sizeof(float), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(h_best, d_best, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaEventRecord(m->host_ev, st));
    if (sync) CUDA_TRY(cudaStreamSynchronize(st));
    return DISTILL_OK;
}

distill_status distill_eval_grid_host(const distill_model* mc, const float* h_inputs, uint32_t n_inputs,
                                      uint64_t begin, uint64_t end, uint32_t n_samples, uint32_t invocation,
                                      uint64_t seed, float* h_net, unsigned long long* h_best, void* stream) {
    return eval_grid_host_impl(mc, h_inputs, n_inputs, begin, end, n_samples, invocation, seed, h_net, h_best,
                               stream, true);
}

distill_status distill_eval_grid_host_async(const distill_model* mc, const float* h_inputs, uint32_t n_inputs,
                                            uint64_t begin, uint64_t end, uint32_t n_samples, uint32_t invocation,
                                            uint64_t seed, float* h_net, unsigned long long* h_best, void* stream) {
    return eval_grid_host_impl(mc, h_inputs, n_inputs, begin, end, n_samples, invocation, seed, h_net, h_best,
                               stream, false);
}

static distill_status episode_check(const distill_model* m, const distill_episode_args* e, const char* who) {
    if (!m || !e) return fail(DISTILL_E_INVALID_ARG, "%s: NULL model/args", who);
    if (m->kind != DISTILL_MODEL_PREDATOR_PREY) return fail(DISTILL_E_UNSUPPORTED, "%s: predator-prey only", who);
    if (e->n_steps == 0 || e->n_samples == 0 || e->n_samples > MAX_SAMPLES)
        return fail(DISTILL_E_INVALID_ARG, "%s: n_steps >= 1, n_samples in [1, 2^31]", who);
    if (!e->d_traj || !e->d_keys || !e->d_status)
        return fail(DISTILL_E_INVALID_ARG, "%s: NULL device buffer", who);
    if (!(e->capture_radius >= 0.0f)) return fail(DISTILL_E_INVALID_ARG, "%s: capture_radius must be >= 0", who);
    return DISTILL_OK;
}

static PPArgs episode_pp_args(const distill_model* m, const distill_episode_args* e) {
    PPArgs p = pp_base_args(m, e->n_samples, e->seed);
    p.status_dev = e->d_status;
    return p;
}

static void episode_search(const distill_model* m, const distill_episode_args* e, PPArgs p, uint32_t t,
                           uint64_t begin, uint64_t end, cudaStream_t st) {
    p.invocation = t;
    p.pos_dev = e->d_traj + 6ull * t;
    p.best = e->d_keys + t;
    p.begin = (uint32_t)begin; p.count = (uint32_t)(end - begin);
    launch_pp_search(m, p, 1, st);
}

static void episode_advance(const distill_model* m, const distill_episode_args* e, const PPArgs& p, uint32_t t,
                            cudaStream_t st) {
    EpisodeArgs ea;
    ea.v_pl = e->v_player; ea.v_py = e->v_prey; ea.v_pd = e->v_predator;
    ea.rc = e->capture_radius;
    ea.traj = e->d_traj; ea.keys = e->d_keys; ea.status = e->d_status;
    pp_episode_step_kernel<<<1, 32, 0, st>>>(p, ea, t);
    g_launches++;
}

distill_status distill_pp_episode_begin(const distill_model* m, const distill_episode_args* e, void* stream) {
    distill_status s = episode_check(m, e, "pp_episode_begin");
    if (s != DISTILL_OK) return s;
    DEVICE_SCOPE(m->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (e->h_init) CUDA_TRY(cudaMemcpyAsync(e->d_traj, e->h_init, 6 * sizeof(float), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(e->d_keys, 0xFF, e->n_steps * sizeof(unsigned long long), st));
    CUDA_TRY(cudaMemsetAsync(e->d_status, 0, 2 * sizeof(int), st));
    return DISTILL_OK;
}

distill_status distill_pp_episode_search(const distill_model* m, const distill_episode_args* e, uint32_t t,
                                         uint64_t begin, uint64_t end, void* stream) {
    distill_status s = episode_check(m, e, "pp_episode_search");
    if (s != DISTILL_OK) return s;
    if (t >= e->n_steps) return fail(DISTILL_E_INVALID_ARG, "pp_episode_search: step t >= n_steps");
    if (begin > end || end > m->n_alloc) return fail(DISTILL_E_INVALID_ARG, "pp_episode_search: bad shard");
    if (begin == end) return DISTILL_OK;
    DEVICE_SCOPE(m->device);
    episode_search(m, e, episode_pp_args(m, e), t, begin, end, (cudaStream_t)stream);
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_pp_episode_advance(const distill_model* m, const distill_episode_args* e, uint32_t t,
                                          void* stream) {
    distill_status s = episode_check(m, e, "pp_episode_advance");
    if (s != DISTILL_OK) return s;
    if (t >= e->n_steps) return fail(DISTILL_E_INVALID_ARG, "pp_episode_advance: step t >= n_steps");
    DEVICE_SCOPE(m->device);
    episode_advance(m, e, episode_pp_args(m, e), t, (cudaStream_t)stream);
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_pp_episode(const distill_model* m, const distill_episode_args* e, void* stream) {
    distill_status s = distill_pp_episode_begin(m, e, stream);
    if (s != DISTILL_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const PPArgs p = episode_pp_args(m, e);
    for (uint32_t t = 0; t < e->n_steps; ++t) {
        episode_search(m, e, p, t, 0, m->n_alloc, st);
        episode_advance(m, e, p, t, st);
    }
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

static distill_status amr_check(const distill_model* m, const distill_amr_args* g, const char* who) {
    if (!m || !g) return fail(DISTILL_E_INVALID_ARG, "%s: NULL model/args", who);
    if (m->kind != DISTILL_MODEL_PREDATOR_PREY) return fail(DISTILL_E_UNSUPPORTED, "%s: predator-prey only", who);
    if (!g->inputs || g->n_inputs != 6) return fail(DISTILL_E_INVALID_ARG, "%s: needs 6 host inputs", who);
    if (g->rounds == 0 || g->n_samples == 0 || g->n_samples > MAX_SAMPLES)
        return fail(DISTILL_E_INVALID_ARG, "%s: rounds >= 1, n_samples in [1, 2^31]", who);
    if (!g->d_keys || !g->d_boxes || !g->d_levels) return fail(DISTILL_E_INVALID_ARG, "%s: NULL device buffer", who);
    for (int d = 0; d < 3; ++d)
        if (!(g->lo[d] <= g->hi[d])) return fail(DISTILL_E_INVALID_ARG, "%s: lo > hi for signal %d", who, d);
    if ((uint64_t)g->invocation0 + g->rounds > 0xFFFFFFFFull)
        return fail(DISTILL_E_OVERFLOW, "%s: invocation counter overflow", who);
    return DISTILL_OK;
}

static AmrArgs amr_args(const distill_model* m, const distill_amr_args* g) {
    AmrArgs a;
    for (int d = 0; d < 3; ++d) { a.lo0[d] = g->lo[d]; a.hi0[d] = g->hi[d]; a.L[d] = m->L[d]; }
    a.levels = g->d_levels; a.boxes = g->d_boxes; a.keys = g->d_keys;
    return a;
}

static PPArgs amr_pp_args(const distill_model* m, const distill_amr_args* g) {
    PPArgs p = pp_base_args(m, g->n_samples, g->seed);
    p.prey_x = g->inputs[0]; p.prey_y = g->inputs[1]; p.pred_x = g->inputs[2]; p.pred_y = g->inputs[3];
    p.pl_x = g->inputs[4]; p.pl_y = g->inputs[5];
    p.levels = g->d_levels;                      // the round's level table, not the model's
    return p;
}

static void amr_search(const distill_model* m, const distill_amr_args* g, PPArgs p, uint32_t r, uint64_t begin,
                       uint64_t end, cudaStream_t st) {
    p.invocation = g->invocation0 + r;
    p.best = g->d_keys + r;
    p.begin = (uint32_t)begin; p.count = (uint32_t)(end - begin);
    launch_pp_search(m, p, 1, st);
}

distill_status distill_pp_amr_begin(const distill_model* m, const distill_amr_args* g, void* stream) {
    distill_status s = amr_check(m, g, "pp_amr_begin");
    if (s != DISTILL_OK) return s;
    DEVICE_SCOPE(m->device);
    CUDA_TRY(cudaMemsetAsync(g->d_keys, 0xFF, g->rounds * sizeof(unsigned long long), (cudaStream_t)stream));
    return DISTILL_OK;
}

distill_status distill_pp_amr_levels(const distill_model* m, const distill_amr_args* g, uint32_t r, void* stream) {
    distill_status s = amr_check(m, g, "pp_amr_levels");
    if (s != DISTILL_OK) return s;
    if (r >= g->rounds) return fail(DISTILL_E_INVALID_ARG, "pp_amr_levels: round r >= rounds");
    DEVICE_SCOPE(m->device);
    amr_levels_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(amr_args(m, g), r);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_pp_amr_search(const distill_model* m, const distill_amr_args* g, uint32_t r,
                                     uint64_t begin, uint64_t end, void* stream) {
    distill_status s = amr_check(m, g, "pp_amr_search");
    if (s != DISTILL_OK) return s;
    if (r >= g->rounds) return fail(DISTILL_E_INVALID_ARG, "pp_amr_search: round r >= rounds");
    if (begin > end || end > m->n_alloc) return fail(DISTILL_E_INVALID_ARG, "pp_amr_search: bad shard");
    if (begin == end) return DISTILL_OK;
    DEVICE_SCOPE(m->device);
    amr_search(m, g, amr_pp_args(m, g), r, begin, end, (cudaStream_t)stream);
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_pp_amr_refine(const distill_model* m, const distill_amr_args* g, uint32_t r, void* stream) {
    distill_status s = amr_check(m, g, "pp_amr_refine");
    if (s != DISTILL_OK) return s;
    if (r >= g->rounds) return fail(DISTILL_E_INVALID_ARG, "pp_amr_refine: round r >= rounds");
    DEVICE_SCOPE(m->device);
    amr_refine_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(amr_args(m, g), r);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_pp_amr(const distill_model* m, const distill_amr_args* g, void* stream) {
    distill_status s = distill_pp_amr_begin(m, g, stream);
    if (s != DISTILL_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const AmrArgs a = amr_args(m, g);
    const PPArgs p = amr_pp_args(m, g);
    for (uint32_t r = 0; r < g->rounds; ++r) {
        amr_levels_kernel<<<1, 256, 0, st>>>(a, r);
        amr_search(m, g, p, r, 0, m->n_alloc, st);
        amr_refine_kernel<<<1, 32, 0, st>>>(a, r);
        g_launches += 2;
    }
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_argmax(const float* d_values, uint64_t n, uint64_t index_base,
                              unsigned long long* d_best, void* stream) {
    if (!d_best || (!d_values && n)) return fail(DISTILL_E_INVALID_ARG, "argmax: NULL pointer");
    if (index_base + n > 0x100000000ull) return fail(DISTILL_E_OVERFLOW, "argmax: index exceeds 32 bits");
    if (n == 0) return DISTILL_OK;
    int dev = 0, n_sm = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t need = (n / 4 + ARGMAX_BLOCK - 1) / ARGMAX_BLOCK + 1;
    const unsigned grid = (unsigned)std::min<uint64_t>(need, (uint64_t)n_sm * 8);
    argmax_net_kernel<ARGMAX_BLOCK><<<grid, ARGMAX_BLOCK, 0, (cudaStream_t)stream>>>(d_values, n, (uint32_t)index_base,
                                                                                      d_best);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_argmax_ties(const float* d_values, uint64_t n, uint64_t index_base, uint64_t seed,
                                   uint32_t invocation, const unsigned long long* d_best,
                                   unsigned long long* d_tie, void* stream) {
    if (!d_best || !d_tie || (!d_values && n)) return fail(DISTILL_E_INVALID_ARG, "argmax_ties: NULL pointer");
    if (index_base + n > 0x100000000ull) return fail(DISTILL_E_OVERFLOW, "argmax_ties: index exceeds 32 bits");
    if (n == 0) return DISTILL_OK;
    int dev = 0, n_sm = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t need = (n + ARGMAX_BLOCK - 1) / ARGMAX_BLOCK;
    const unsigned grid = (unsigned)std::min<uint64_t>(need, (uint64_t)n_sm * 8);
    argmax_ties_kernel<ARGMAX_BLOCK><<<grid, ARGMAX_BLOCK, 0, (cudaStream_t)stream>>>(
        d_values, n, (uint32_t)index_base, d_best, (uint32_t)seed, (uint32_t)(seed >> 32), invocation, d_tie);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_sm_clock_probe(uint32_t micros, double* h_mhz, void* stream) {
    if (!h_mhz || micros == 0) return fail(DISTILL_E_INVALID_ARG, "sm_clock_probe: NULL output / zero duration");
    int dev = 0, n_sm = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    double* d = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&d, n_sm * sizeof(double), (cudaStream_t)stream));
    sm_clock_probe_kernel<<<n_sm, 32, 0, (cudaStream_t)stream>>>(1000ull * micros, d);
    std::vector<double> h(n_sm);
    CUDA_TRY(cudaMemcpyAsync(h.data(), d, n_sm * sizeof(double), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CUDA_TRY(cudaFreeAsync(d, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    std::sort(h.begin(), h.end());
    *h_mhz = h[n_sm / 2];
    return DISTILL_OK;
}

distill_status distill_key_reset(unsigned long long* d_best, void* stream) {
    if (!d_best) return fail(DISTILL_E_INVALID_ARG, "key_reset: NULL");
    CUDA_TRY(cudaMemsetAsync(d_best, 0xFF, sizeof(unsigned long long), (cudaStream_t)stream));
    return DISTILL_OK;
}

distill_status distill_key_reset_signed(unsigned long long* d_best, void* stream) {
    if (!d_best) return fail(DISTILL_E_INVALID_ARG, "key_reset_signed: NULL");
    if (reinterpret_cast<uintptr_t>(d_best) & 7u) return fail(DISTILL_E_INVALID_ARG, "key_reset_signed: misaligned");
    // INT64_MAX little-endian: seven 0xFF bytes, then 0x7F
    CUDA_TRY(cudaMemsetAsync(d_best, 0xFF, 7, (cudaStream_t)stream));
    CUDA_TRY(cudaMemsetAsync(reinterpret_cast<unsigned char*>(d_best) + 7, 0x7F, 1, (cudaStream_t)stream));
    return DISTILL_OK;
}

distill_status distill_key_decode(unsigned long long key, float* cost, uint64_t* index) {
    if (!cost || !index) return fail(DISTILL_E_INVALID_ARG, "key_decode: NULL");
    const uint32_t hi = (uint32_t)(key >> 32);
    *index = (uint32_t)key;
    if (hi == 0xFFFFFFFFu) {
        *cost = NAN;
        return fail(DISTILL_E_NO_VALID, "key_decode: no valid candidate");
    }
    const uint32_t b = (hi >> 31) ? (hi & 0x7FFFFFFFu) : ~hi;
    memcpy(cost, &b, 4);
    return DISTILL_OK;
}

extern "C++" {
template <bool LCI>
static distill_status launch_integrator(const distill_ddm_args* a, float leak, float offset, void* stream,
                                        const char* who) {
    if (!a || !a->d_rt_hist || !a->d_rt_sum || !a->d_x_hist)
        return fail(DISTILL_E_INVALID_ARG, "%s: NULL argument", who);
    if ((reinterpret_cast<uintptr_t>(a->d_rt_hist) | reinterpret_cast<uintptr_t>(a->d_rt_sum) |
         reinterpret_cast<uintptr_t>(a->d_x_hist)) & 7u)
        return fail(DISTILL_E_INVALID_ARG, "%s: histogram buffers must be 8-byte aligned", who);
    if (a->n_steps == 0 || a->rt_bin_steps == 0 || a->n_x_bins == 0)
        return fail(DISTILL_E_INVALID_ARG, "%s: n_steps, rt_bin_steps, n_x_bins must be >= 1", who);
    if (!(a->x_lo < a->x_hi) || !(a->dt >= 0.0f)) return fail(DISTILL_E_INVALID_ARG, "%s: bad x range / dt", who);
    if (a->trial_begin > a->trial_end) return fail(DISTILL_E_INVALID_ARG, "%s: bad trial range", who);
    const uint32_t nb = (a->n_steps + a->rt_bin_steps - 1) / a->rt_bin_steps;
    const size_t smem = (size_t)(2 * nb + 1 + a->n_x_bins + 2) * sizeof(uint32_t);
    if (smem > 160 * 1024) return fail(DISTILL_E_UNSUPPORTED, "%s: histograms exceed shared memory", who);
    const uint64_t n = a->trial_end - a->trial_begin;
    if (n == 0) return DISTILL_OK;
    int dev = 0, n_sm = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    const float4* rt = nullptr;
    const distill_status rs = rad_table(dev, &rt);
    if (rs != DISTILL_OK) return rs;
    if (smem + RT_ROWS * sizeof(float4) > 48 * 1024)   // dynamic histograms + the static radius table
        CUDA_TRY(cudaFuncSetAttribute(ddm_batch_kernel<DDM_BLOCK, DDM_MINB, LCI>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DDMArgs p;
    p.drift = a->drift; p.noise = a->noise; p.threshold = a->threshold; p.x0 = a->x0; p.dt = a->dt;
    p.x_lo = a->x_lo; p.x_hi = a->x_hi;
    p.leak = leak; p.offset = offset;
    p.n_steps = a->n_steps; p.rt_bin_steps = a->rt_bin_steps; p.n_rt_bins = nb; p.n_x_bins = a->n_x_bins;
    p.key0 = (uint32_t)a->seed; p.key1 = (uint32_t)(a->seed >> 32);
    p.rt_hist = a->d_rt_hist; p.rt_sum = a->d_rt_sum; p.x_hist = a->d_x_hist;
    p.rad_tab = rt;
    // one launch per 2^32-aligned segment of RNG units (one high word each)
    for (uint64_t u = a->trial_begin; u < a->trial_end;) {
        const uint64_t seg_end =
            (u >> 32) == 0xFFFFFFFFull ? a->trial_end : std::min<uint64_t>(a->trial_end, ((u >> 32) + 1) << 32);
        const uint64_t m = seg_end - u;
        p.trial_begin = u; p.n_trials = m; p.unit_hi = (uint32_t)(u >> 32);
        const uint64_t prod = (uint64_t)0xCD9E8D57u * p.unit_hi;   // Philox round 1: M1 * c2
        p.c2_a1 = (uint32_t)(prod >> 32) ^ p.key0;
        p.c2_x1 = (uint32_t)prod;
        const uint64_t need = (m + DDM_BLOCK - 1) / DDM_BLOCK;
        const unsigned grid = (unsigned)std::min<uint64_t>(need, (uint64_t)n_sm * 1024);
        ddm_batch_kernel<DDM_BLOCK, DDM_MINB, LCI><<<grid, DDM_BLOCK, smem, (cudaStream_t)stream>>>(p);
        g_launches++;
        CUDA_TRY(cudaGetLastError());
        u = seg_end;
    }
    return DISTILL_OK;
}

}  // extern "C++"

distill_status distill_ddm_batch(const distill_ddm_args* a, void* stream) {
    return launch_integrator<false>(a, 0.0f, 0.0f, stream, "ddm_batch");
}

distill_status distill_lci_batch(const distill_ddm_args* a, float leak, float offset, void* stream) {
    return launch_integrator<true>(a, leak, offset, stream, "lci_batch");
}

// ------------------------------------------------------------------ rows a2 / a3 on their own
constexpr int RNG_BLOCK = 128;

static distill_status rng_device_table(const float4** rt, int* n_sm) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(n_sm, cudaDevAttrMultiProcessorCount, dev));
    return rad_table(dev, rt);
}

distill_status distill_rng_rad(const uint32_t* d_words, uint64_t n, float* d_rad, void* stream) {
    if (n && (!d_words || !d_rad)) return fail(DISTILL_E_INVALID_ARG, "rng_rad: NULL pointer");
    if ((reinterpret_cast<uintptr_t>(d_words) | reinterpret_cast<uintptr_t>(d_rad)) & 3u)
        return fail(DISTILL_E_INVALID_ARG, "rng_rad: buffers must be 4-byte aligned");
    if (n == 0) return DISTILL_OK;
    const float4* rt = nullptr;
    int n_sm = 148;
    const distill_status rs = rng_device_table(&rt, &n_sm);
    if (rs != DISTILL_OK) return rs;
    const uint64_t need = (n + 2 * RNG_BLOCK - 1) / (2 * RNG_BLOCK);
    const unsigned grid = (unsigned)std::min<uint64_t>(need, (uint64_t)n_sm * 16);
    rng_rad_kernel<RNG_BLOCK><<<grid, RNG_BLOCK, 0, (cudaStream_t)stream>>>(d_words, n, d_rad, rt);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_rng_normals_acc(uint64_t seed, uint64_t unit_begin, uint64_t n_units, uint32_t n_per_unit,
                                       float* d_out, void* stream) {
    if (n_units && !d_out) return fail(DISTILL_E_INVALID_ARG, "rng_normals_acc: NULL output");
    if (reinterpret_cast<uintptr_t>(d_out) & 3u)
        return fail(DISTILL_E_INVALID_ARG, "rng_normals_acc: output must be 4-byte aligned");
    if (n_per_unit == 0 || n_per_unit > (1u << 30))
        return fail(DISTILL_E_INVALID_ARG, "rng_normals_acc: n_per_unit must be in [1, 2^30]");
    if (n_units > (1ull << 62) / n_per_unit || unit_begin + n_units < unit_begin)
        return fail(DISTILL_E_OVERFLOW, "rng_normals_acc: unit range or output size overflows");
    if (n_units == 0) return DISTILL_OK;
    const float4* rt = nullptr;
    int n_sm = 148;
    const distill_status rs = rng_device_table(&rt, &n_sm);
    if (rs != DISTILL_OK) return rs;
    const uint64_t grid = (n_units + RNG_BLOCK - 1) / RNG_BLOCK;
    if (grid > 0x7FFFFFFFull) return fail(DISTILL_E_UNSUPPORTED, "rng_normals_acc: too many units for one launch");
    rng_normals_acc_kernel<RNG_BLOCK><<<(unsigned)grid, RNG_BLOCK, 0, (cudaStream_t)stream>>>(
        (uint32_t)seed, (uint32_t)(seed >> 32), unit_begin, n_units, n_per_unit, d_out, rt);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

distill_status distill_rng_normals_pp(uint64_t seed, uint32_t alloc_begin, uint32_t n_alloc, uint32_t n_samples,
                                      uint32_t invocation, float* d_out, void* stream) {
    if (n_alloc && !d_out) return fail(DISTILL_E_INVALID_ARG, "rng_normals_pp: NULL output");
    if (reinterpret_cast<uintptr_t>(d_out) & 3u)
        return fail(DISTILL_E_INVALID_ARG, "rng_normals_pp: output must be 4-byte aligned");
    if (n_samples == 0 || n_samples > MAX_SAMPLES)
        return fail(DISTILL_E_INVALID_ARG, "rng_normals_pp: n_samples must be in [1, 2^31]");
    if ((uint64_t)alloc_begin + n_alloc > 0x100000000ull)
        return fail(DISTILL_E_OVERFLOW, "rng_normals_pp: allocation index exceeds 32 bits");
    if (n_alloc == 0) return DISTILL_OK;
    const float4* rt = nullptr;
    int n_sm = 148;
    const distill_status rs = rng_device_table(&rt, &n_sm);
    if (rs != DISTILL_OK) return rs;
    const unsigned grid = (unsigned)(((uint64_t)n_alloc + RNG_BLOCK - 1) / RNG_BLOCK);
    rng_normals_pp_kernel<RNG_BLOCK><<<grid, RNG_BLOCK, 0, (cudaStream_t)stream>>>(
        (uint32_t)seed, (uint32_t)(seed >> 32), alloc_begin, n_alloc, n_samples, invocation, d_out, rt);
    g_launches++;
    CUDA_TRY(cudaGetLastError());
    return DISTILL_OK;
}

}  // extern "C"
