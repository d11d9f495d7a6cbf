/*
 * distill.h — C ABI of the B200 grid-search library (libdistill.so).
 *
 * The hot path of Distill (arXiv 2110.15425) that the paper offloads to the
 * GPU: the Control node's exhaustive grid search, where every control
 * allocation runs independent noisy simulations of the compiled model and the
 * lowest-cost allocation wins (§2.1; §3.6).
 * Exact op-by-op semantics: spec/MODELS.md and spec/RNG.md.
 *
 * Conventions (all entry points):
 *   - extern "C", plain pointers and sizes; no exceptions cross the ABI and the
 *     library never aborts.  Every call returns a distill_status; the
 *     thread-local distill_last_error() string says why a call failed.
 *   - "d_" pointers are DEVICE memory owned by the caller; "h_" pointers are
 *     host memory owned by the caller.  The library owns only the model handle
 *     and its device copy of the read-only model block.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Work is stream-ordered and asynchronous unless stated; argument errors are
 *     detected synchronously and enqueue nothing; an asynchronous CUDA fault
 *     surfaces as DISTILL_E_CUDA on a later call.
 *   - A model handle is read-only during evaluation: several streams/threads may
 *     evaluate the same handle concurrently.
 */
#ifndef DISTILL_H
#define DISTILL_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DISTILL_ABI_VERSION 3   /* 2: distill_eval_args.key_order, distill_key_reset_signed; 3: distill_eval_grid_host_async */

typedef enum {
    DISTILL_OK = 0,
    DISTILL_E_INVALID_ARG = 1,  /* NULL/size/range error; nothing enqueued            */
    DISTILL_E_OVERFLOW = 2,     /* grid > 2^32-1 allocations (32-bit key index), or an RNG unit / invocation counter past its width */
    DISTILL_E_UNSUPPORTED = 3,  /* model kind / shape not implemented                  */
    DISTILL_E_CUDA = 4,         /* CUDA runtime error (see distill_last_error)         */
    DISTILL_E_NO_VALID = 5      /* key decode: no finite candidate (all NaN / empty)   */
} distill_status;

typedef enum {
    DISTILL_MODEL_PREDATOR_PREY = 1,  /* P:140-167, Fig. 1                                */
    DISTILL_MODEL_STROOP_LCA = 2,     /* P:525 (surrogate, spec/MODELS.md §6)             */
    DISTILL_MODEL_EXT_STROOP_A = 3,   /* P:527 Extended Stroop, version A (§10, NEXT-3)   */
    DISTILL_MODEL_EXT_STROOP_B = 4,   /* P:527 version B: computationally identical to A  */
    DISTILL_MODEL_DDM_GRID = 5        /* DDM control grid (spec/MODELS.md §6c)            */
} distill_model_kind;

/* "No candidate" value of a packed (value, index) key; initialise d_best to it. */
#define DISTILL_KEY_INIT 0xFFFFFFFFFFFFFFFFull
/* The same in the signed key order (key_order = 1: stored word = key ^ 2^63,
 * so int64 MIN order = key order; P:352 per-segment results combined across
 * GPUs by one int64 MIN all-reduce with no conversion); = INT64_MAX. */
#define DISTILL_KEY_INIT_SIGNED 0x7FFFFFFFFFFFFFFFull

typedef struct distill_model distill_model;  /* opaque, library-owned */

/* Model description.  Copied by distill_load_model; host arrays may be freed
 * after it returns.  Grid = Cartesian product of the per-signal levels
 * ("searches over all possible attention allocations"), enumerated in
 * mixed radix with signal 0 most significant (spec/MODELS.md §1).
 *   PREDATOR_PREY: n_signals = 3 (prey, predator, player attention);
 *                  params = {sigma_max, sigma_min, kappa}, n_params = 3.
 *   STROOP_LCA:    n_signals = 2 (colour attention u_c, word suppression u_s);
 *                  params = {g_c, g_w, tau, leak, inhibition, noise, dt,
 *                            threshold, reward, rt_cost, n_steps}, n_params = 11.
 *   EXT_STROOP_A/B: n_signals = 2 (as Stroop); params = {g_c, g_w, tau, N_h, lambda,
 *                  a_p, gamma, sigma_d, dt_d, z_d, N_d, reward, rt_cost}, n_params = 13;
 *                  d_counts = {n_both_correct, n_undecided, rt_sum}.
 *   DDM_GRID:      n_signals = 2 (attention u0 scales the drift, threshold u1);
 *                  params = {A0, g_a, sigma, dt, reward, rt_cost, n_steps}, n_params = 7;
 *                  d_counts = {n_correct (upper bound), n_undecided, rt_sum}; V as Stroop. */
typedef struct {
    uint32_t kind;               /* distill_model_kind                               */
    uint32_t n_signals;          /* D                                                */
    const uint32_t* n_levels;    /* host [D], each >= 1                              */
    const float* levels;         /* host [sum n_levels], signal 0 first              */
    const float* cost_weights;   /* host [D]: control cost K = sum_d w_d a_d */
    const float* params;         /* host [n_params]                                  */
    uint32_t n_params;
} distill_model_desc;

/* One grid evaluation (a shard [begin, end) of the global allocation range). */
typedef struct {
    const float* inputs;         /* host; PP: prey, predator, player (x, y) = 6 floats; Stroop: unused */
    uint32_t n_inputs;
    uint64_t begin, end;         /* global allocation indices, begin <= end <= grid size */
    uint32_t n_samples;          /* PP: samples per allocation; Stroop: trials T per allocation; 1..2^31 */
    uint32_t invocation;         /* PP: controller invocation t (RNG counter word, spec/RNG.md §1); Stroop: 0 */
    uint64_t seed;               /* Philox key */
    float* d_net;                /* device [end-begin] or NULL: net value V = -C per allocation       */
    unsigned long long* d_best;  /* device [1] or NULL: atomicMin of key(C_i, i) (spec/MODELS.md §3)  */
    unsigned long long* d_counts;/* Stroop kinds: REQUIRED device [(end-begin)*3] u64, 8-B aligned:
                                    {n_correct (n_both for Ext-Stroop), n_undecided, rt_sum}; overwritten.
                                    PP: unused (NULL)                                                  */
    uint32_t trial_begin, trial_end; /* Stroop: simulate trials [trial_begin, trial_end) only; (0,0) = all.
                                    d_net/d_best are produced only when the range is all T trials.    */
    uint32_t key_order;          /* 0: d_best is combined as unsigned keys (atomicMin u64; init
                                    DISTILL_KEY_INIT).  1: signed order — d_best holds key ^ 2^63,
                                    combined by atomicMin on int64 (init DISTILL_KEY_INIT_SIGNED), ready
                                    for an int64 MIN all-reduce across ranks.  Other values: E_INVALID_ARG */
} distill_eval_args;

/* DDM Monte Carlo batch (Fig. 3; spec/MODELS.md §4). */
typedef struct {
    float drift, noise, threshold, x0, dt;  /* A, sigma, z (bounds +-z), start, step      */
    uint32_t n_steps;                       /* fixed trip N >= 1                         */
    uint32_t rt_bin_steps;                  /* RT bin width in steps, >= 1               */
    uint32_t n_x_bins;                      /* endpoint bins >= 1 (+ under/overflow bins) */
    float x_lo, x_hi;                       /* endpoint histogram range, x_lo < x_hi     */
    uint64_t trial_begin, trial_end, seed;  /* global trial ids (RNG unit) and Philox key */
    unsigned long long* d_rt_hist;  /* device [2*ceil(N/B)+1]: upper bins, lower bins, undecided (+=) */
    unsigned long long* d_rt_sum;   /* device [2]: sum of first-passage steps, upper / lower      (+=) */
    unsigned long long* d_x_hist;   /* device [n_x_bins+2]: underflow, bins, overflow              (+=) */
} distill_ddm_args;

/* Closed-loop predator-prey episode (NEXT-1; "the entire process
 * ... is repeated for each time step until the prey or the player is captured";
 * spec/MODELS.md §7).  Per step t: one full grid search on the current positions
 * (invocation t), the chosen attention draws the executed observation (Philox
 * stream 4), player/prey/predator move, capture is tested.  Everything stays on
 * the device: 2 launches per step, no host round trip, capturable in a CUDA
 * graph.  After capture later steps are no-ops (fixed trip).
 * Predator-prey models only; d_traj[0..5] must hold the initial positions unless
 * h_init is given (then it is copied in, stream-ordered). */
typedef struct {
    uint32_t n_steps;            /* T >= 1                                                  */
    uint32_t n_samples;          /* samples per allocation in every grid search, 1..2^31   */
    uint64_t seed;
    float v_player, v_prey, v_predator;   /* step lengths per time step                   */
    float capture_radius;        /* capture when |prey - player| or |predator - player| <= r */
    const float* h_init;         /* host [6] (prey, predator, player x/y) or NULL           */
    float* d_traj;               /* device [(T+1)*6] positions, caller-owned                */
    unsigned long long* d_keys;  /* device [T] best key per step (KEY_INIT after the end)   */
    int* d_status;               /* device [2] {outcome 0 running/1 prey caught/2 player caught/3 no valid, steps} */
} distill_episode_args;

distill_status distill_pp_episode(const distill_model* model, const distill_episode_args* args, void* stream);

/* The same episode in pieces, for a grid sharded across GPUs ("one grid search +
 * all-reduce per time step"): begin() copies h_init (if
 * given) and resets d_keys / d_status; for each step t every rank runs
 * search(t, [begin, end)) on its shard — atomicMin into d_keys[t] — the caller
 * MIN-all-reduces d_keys[t] across ranks (key order = unsigned order; flip bit
 * 63 for a signed int64 MIN), then every rank runs advance(t), which moves all
 * entities from the global key exactly as distill_pp_episode does, so every
 * rank holds the identical trajectory.  distill_pp_episode = begin + T x
 * (search over the whole grid + advance).  All calls are stream-ordered;
 * t < n_steps; begin <= end <= grid size (E_INVALID_ARG otherwise). */
distill_status distill_pp_episode_begin(const distill_model* model, const distill_episode_args* args, void* stream);
distill_status distill_pp_episode_search(const distill_model* model, const distill_episode_args* args, uint32_t t,
                                         uint64_t begin, uint64_t end, void* stream);
distill_status distill_pp_episode_advance(const distill_model* model, const distill_episode_args* args, uint32_t t,
                                          void* stream);

/* Coarse-to-fine (AMR-style) refinement of the predator-prey grid search
 * (NEXT-4; §4.3, Fig. 4; spec/MODELS.md §9).  The model's
 * n_levels give L_d per signal (its level table is not used); each round r runs
 * a full grid search (invocation invocation0 + r) over the box r, then the box
 * shrinks to one level spacing around the round's best allocation, clamped to
 * the initial box.  All rounds stay on the device (3 launches per round). */
typedef struct {
    const float* inputs; uint32_t n_inputs;   /* host [6] positions                          */
    float lo[3], hi[3];                       /* initial box per signal (= clamp limits)      */
    uint32_t rounds, n_samples, invocation0;
    uint64_t seed;
    unsigned long long* d_keys;   /* device [rounds] best key per round                       */
    float* d_boxes;               /* device [(rounds+1)*6]: (lo, hi) per signal per round      */
    float* d_levels;              /* device scratch [L0+L1+L2]                                 */
} distill_amr_args;

distill_status distill_pp_amr(const distill_model* model, const distill_amr_args* args, void* stream);

/* The same refinement in pieces, for a grid sharded across GPUs: begin() resets
 * d_keys; per round r every rank runs levels(r) (the level table of box r into
 * d_levels), search(r, [begin, end)) on its shard (atomicMin into d_keys[r]);
 * the caller MIN-all-reduces d_keys[r] across ranks; every rank runs refine(r),
 * which writes box r+1 from the global key — identical on every rank.
 * distill_pp_amr = begin + R x (levels + search over the whole grid + refine).
 * r < rounds; begin <= end <= grid size (E_INVALID_ARG otherwise). */
distill_status distill_pp_amr_begin(const distill_model* model, const distill_amr_args* args, void* stream);
distill_status distill_pp_amr_levels(const distill_model* model, const distill_amr_args* args, uint32_t r,
                                     void* stream);
distill_status distill_pp_amr_search(const distill_model* model, const distill_amr_args* args, uint32_t r,
                                     uint64_t begin, uint64_t end, void* stream);
distill_status distill_pp_amr_refine(const distill_model* model, const distill_amr_args* args, uint32_t r,
                                     void* stream);

int            distill_abi_version(void);
const char*    distill_last_error(void);

/* Validate the description and copy its read-only block to `device`.  The
 * first load on a device (or the first DDM/LCI batch there) also uploads the
 * library's Box-Muller radius table (spec/RNG.md §3, 11.8 KB, kept for the
 * process lifetime); that one-time step is synchronous and must not happen
 * inside a CUDA-graph capture (E_CUDA otherwise).  The caller's current device
 * is restored before return (as by every entry point). */
distill_status distill_load_model(const distill_model_desc* desc, int device, distill_model** out);
/* NULL-safe.  The caller synchronises streams that use the model first. */
void           distill_free_model(distill_model* model);
distill_status distill_grid_size(const distill_model* model, uint64_t* n_alloc);

/* Evaluate allocations [begin, end): per allocation, n_samples noisy simulations
 * averaged, plus control cost.  One fused kernel for PP;
 * simulate + finalize kernels for Stroop.  Stream-ordered, asynchronous. */
distill_status distill_eval_grid(const distill_model* model, const distill_eval_args* args, void* stream);

/* Many controller invocations in one launch (Listing 1, P:190-199:
 * `composition.run(inputs, num_trials)` invokes the controller once per trial
 * with `inputs[num_trial % len]` — reading Q17 of the garbled `%`).  Invocation
 * t (0 <= t < n_invocations) evaluates allocations [begin, end) on position set
 * t mod n_sets with RNG invocation word invocation0 + t, writes its V row
 * d_net[t*(end-begin) ...] and atomicMin's its key into d_best[t].  Identical,
 * bit for bit, to n_invocations separate distill_eval_grid calls.
 * Predator-prey only (E_UNSUPPORTED otherwise); n_invocations <= 65535 per call
 * (E_INVALID_ARG beyond); invocation0 + n_invocations must fit in 32 bits
 * (E_OVERFLOW).  Stream-ordered, one kernel launch. */
typedef struct {
    const float* d_inputs;       /* device, caller-owned [n_sets][6]: prey, predator, player (x, y) */
    uint32_t n_sets;             /* >= 1                                                           */
    uint32_t n_invocations;      /* T, 0 = no-op                                                   */
    uint32_t invocation0;        /* RNG invocation word of t = 0                                   */
    uint32_t n_samples;          /* samples per allocation, 1..2^31                                */
    uint64_t begin, end;         /* global allocation range (a shard)                              */
    uint64_t seed;               /* Philox key                                                     */
    float* d_net;                /* device [T][end-begin] or NULL                                  */
    unsigned long long* d_best;  /* device [T] keys or NULL; caller initialises to DISTILL_KEY_INIT */
} distill_multi_args;

distill_status distill_eval_grid_multi(const distill_model* model, const distill_multi_args* args, void* stream);

/* Same evaluation from HOST buffers (the end-to-end call): evaluates on `stream`,
 * returns V in h_net (if non-NULL) and the best key in *h_best, synchronises the
 * stream.  Pinned (cudaHostAlloc / page-locked, device-mapped) h_net is written by
 * the kernel directly (zero-copy, overlapped with the computation); pageable h_net
 * goes through a library-owned device scratch area and one copy.  A pinned h_best
 * receives the key from the kernel's last block, which also re-arms the library's
 * device key, so the whole call is one kernel launch; a pageable h_best costs a
 * memset and a copy.  Serialised per handle (the scratch area is shared). */
distill_status distill_eval_grid_host(const distill_model* model, const float* h_inputs, uint32_t n_inputs,
                                      uint64_t begin, uint64_t end, uint32_t n_samples,
                                      uint32_t invocation, uint64_t seed,
                                      float* h_net, unsigned long long* h_best, void* stream);

/* The same end-to-end call without the final synchronisation, for callers that keep
 * several grid searches in flight (double-buffered host slots): the work is enqueued on
 * `stream` and the call returns.  h_best and h_net (if non-NULL) must be pinned,
 * device-mapped host memory (cudaHostAlloc / page-locked; 8- and 4-byte aligned), else
 * DISTILL_E_INVALID_ARG and nothing is enqueued; they hold the key and V once `stream`
 * has completed the call's work (synchronise the stream or an event recorded on it after
 * the call) and must not be reused by another call before that.  The positions are
 * copied at the call (launch parameters).  Host-buffer calls on one handle run in call
 * order whatever their streams (each waits for the previous one's kernel). */
distill_status distill_eval_grid_host_async(const distill_model* model, const float* h_inputs, uint32_t n_inputs,
                                            uint64_t begin, uint64_t end, uint32_t n_samples,
                                            uint32_t invocation, uint64_t seed,
                                            float* h_net, unsigned long long* h_best, void* stream);

/* argmax over a device array of net values: atomicMin of key(-d_values[j], index_base + j)
 * into *d_best (max V <=> min key, lowest index on ties). */
distill_status distill_argmax(const float* d_values, uint64_t n, uint64_t index_base,
                              unsigned long long* d_best, void* stream);
/* Random tie-break among the minimal costs (NEXT-2; "randomly pick one";
 * spec/MODELS.md §8).  Given *d_best from distill_argmax / distill_eval_grid
 * (after any cross-shard all-reduce), atomicMin of (pi_i << 32 | index) over the
 * entries whose canonical cost equals *d_best's into *d_tie (caller initialises it
 * to DISTILL_KEY_INIT); pi_i = Philox stream 3.  The winner is the low 32 bits of
 * the final *d_tie, uniform among the tied minima; shards combine with a second min. */
distill_status distill_argmax_ties(const float* d_values, uint64_t n, uint64_t index_base, uint64_t seed,
                                   uint32_t invocation, const unsigned long long* d_best,
                                   unsigned long long* d_tie, void* stream);
/* Set *d_best = DISTILL_KEY_INIT (stream-ordered). */
distill_status distill_key_reset(unsigned long long* d_best, void* stream);
/* d_best <- DISTILL_KEY_INIT_SIGNED (signed key order; stream-ordered, two memsets,
 * CUDA-graph capturable).  d_best: device, 8-byte aligned. */
distill_status distill_key_reset_signed(unsigned long long* d_best, void* stream);
/* Host, pure: key -> (cost C, global index).  DISTILL_E_NO_VALID for an all-NaN/empty key. */
distill_status distill_key_decode(unsigned long long key, float* cost, uint64_t* index);

/* Decision energy over time of one Stroop-LCA allocation (spec/MODELS.md §6b;
 * PAPER.md P:525 "the model is used to predict decision energy over time"):
 * for trials [trial_begin, trial_end) of T = n_trials (the same RNG units as
 * distill_eval_grid with n_samples = T), d_esum[n-1] += Σ_j llrint(x0_j(n)·x1_j(n)·2^24)
 * for n = 1..N (exact integer sums, order-free).  The mean conflict energy of
 * the response layer with lateral inhibition β is E(n) = 2β·d_esum[n-1] /
 * ((trial_end − trial_begin)·2^24).  d_esum: device, caller-owned [N] u64,
 * accumulated.  STROOP_LCA models only (E_UNSUPPORTED otherwise); N <= 4096. */
distill_status distill_stroop_energy(const distill_model* model, uint64_t alloc, uint32_t n_trials,
                                     uint32_t trial_begin, uint32_t trial_end, uint64_t seed,
                                     unsigned long long* d_esum, void* stream);

/* DDM batch over trials [trial_begin, trial_end): histograms accumulated with atomics.
 * Runs on the caller's current device (the first call there uploads the radius
 * table, see distill_load_model).  The three histogram buffers must be 8-byte
 * aligned (E_INVALID_ARG otherwise). */
distill_status distill_ddm_batch(const distill_ddm_args* args, void* stream);
/* Leaky competing integrator batch (spec/MODELS.md §5): the same
 * arguments, outputs and RNG units as distill_ddm_batch with `drift` read as
 * the input I and the step x = fma(σ√dt, g, fma(dt, fma(-leak, x, I), x) + offset).
 * With leak = offset = 0 it is bit-identical to distill_ddm_batch (Fig. 3's
 * "computationally equivalent" pair). */
distill_status distill_lci_batch(const distill_ddm_args* args, float leak, float offset, void* stream);

/* Rows a2 + a3 on their own (spec/RNG.md §1-§6; "each
 * evaluation uses its own random number generator", P:157 noisy observations):
 * the Philox4x32-10 -> Box-Muller path every kernel inlines, over caller-chosen
 * inputs, so that it can be compared with the oracle directly.  All run on the
 * caller's current device (the first call there uploads the radius table, see
 * distill_load_model — not inside a CUDA-graph capture), are stream-ordered and
 * enqueue nothing on an argument error.  Output buffers: device, caller-owned,
 * 4-byte aligned.
 *
 * distill_rng_rad: d_rad[k] = rad_spec(d_words[k]) (spec/RNG.md §3, the radius
 *   sqrt(-2 ln u1) of a raw radius word), k < n.
 * distill_rng_normals_acc: d_out[u * n_per_unit + j] = normal j of RNG unit
 *   unit_begin + u on stream 2 (the DDM / Stroop / LCI noise, sextet packing §6),
 *   j < n_per_unit (1..2^30); n_units * n_per_unit <= 2^62 (E_OVERFLOW otherwise).
 * distill_rng_normals_pp: d_out[(t * n_samples + s) * 6 + 2e + {0,1}] = the
 *   2-D noise vector of entity e (prey, predator, player) of sample s of
 *   allocation alloc_begin + t, invocation word `invocation`, on stream 1;
 *   n_samples in [1, 2^31]; alloc_begin + n_alloc <= 2^32 (E_OVERFLOW). */
distill_status distill_rng_rad(const uint32_t* d_words, uint64_t n, float* d_rad, void* stream);
distill_status distill_rng_normals_acc(uint64_t seed, uint64_t unit_begin, uint64_t n_units, uint32_t n_per_unit,
                                       float* d_out, void* stream);
distill_status distill_rng_normals_pp(uint64_t seed, uint32_t alloc_begin, uint32_t n_alloc, uint32_t n_samples,
                                      uint32_t invocation, float* d_out, void* stream);

/* Measurement utility: median effective SM clock (MHz) over one spinning block per
 * SM for `micros` microseconds (clock64 ticks / globaltimer ns).  Synchronous.
 * bench.py runs it right after the timed region to report the fraction of the
 * FP32 peak at the clock the kernel actually ran at. */
distill_status distill_sm_clock_probe(uint32_t micros, double* h_mhz, void* stream);

/* Kernels launched by this library since load (all threads), for launch accounting. */
uint64_t       distill_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
