/*
 * distill_oracle.h — plain, slow, obviously-correct CPU oracle for the Distill
 * grid-search hot path (arXiv 2110.15425, §2.1 and §3.6).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header or constant table with the CUDA path: both are
 * written independently from spec/RNG.md and spec/MODELS.md.
 *
 * Every function is scalar, single-threaded and re-entrant; callers that want
 * parallelism (bench timing) split the allocation range into contiguous
 * segments exactly like the paper's multicore scheme.
 *
 * Parity status per function:
 *   od_philox4x32_10     pinned: Random123 known-answer vectors
 *   od_rad / od_rsqrt / od_sincos2pi  pinned: exhaustive / dense accuracy vs binary64 libm
 *   od_normal_*          pinned: moments, KS vs Phi, closed-form endpoints
 *   od_pp_eval           pinned: zero-noise closed forms, monotonicity, planted optimum, offset-Gaussian
 *                        angle law (noisy objective in closed form), noisy-predator quadrature,
 *                        small-noise delta-method expectation, fp64 re-evaluation
 *   od_argmax_keys       pinned: brute-force min over (C, i), NaN/-0 rules
 *   od_normal_acc        pinned: raw-word Box-Muller definition, moments/kurtosis/KS; cuRAND Philox
 *   od_ddm_*             pinned: zero-noise first passage, closed-form ER/DT, endpoint law; the cfg2 RT
 *                        histogram against the exact first-passage law of the Euler walk (tests/exact_law.py)
 *   od_lci_trial/_batch  pinned: Fig. 3 clone relation to od_ddm_* (bit-identical), AR(1) endpoint law
 *   od_stroop_eval       pinned: zero-noise deterministic RT, conservation, Stroop effect,
 *                        reflected-BM closed-form mean first passage of the noisy unit; linear-recurrence,
 *                        rectified-unit and AR(1) closed forms (leak != inhibition, tau < 1); at the cfg4
 *                        constants the first-response law per kind and colour and the counts against the
 *                        exact law of the rectified two-unit Euler process (tests/exact_law.py)
 *   od_stroop_energy     pinned: zero-noise closed form n^2 dt^2 I0 I1, congruent = 0, range additivity;
 *                        with noise, the mean and variance per step of the Gaussian product x0 x1 in the
 *                        linear (never rectified) regime, from the AR(1) moments of s = x0 + x1, d = x0 - x1
 *   od_ddmg_*            pinned: zero-noise binary32 passage step, Siegmund-corrected closed-form accuracy and
 *                        decision time per allocation, exact-rational value formula; counts at the
 *                        grid's own horizon against the exact first-passage law
 *   od_pp_episode        pinned: closed-form straight-chase capture step, one-step predator capture,
 *                        per-step keys = ordinary grid searches
 *   od_argmax_random_ties pinned: uniform 1/8 frequency over 10^4 seeds, unique minimum wins
 *   od_pp_amr            pinned: zero-noise planted corner every round, Fig. 4 analogue vs a fine scan
 *   od_ext_stroop_*      pinned: A == B bit-identical, zero-noise drift signs / conflict
 *                        slowing / binary32 first passage, closed-form P(both correct) from the
 *                        two DDM error rates; at the bench constants both DDMs' first-passage laws
 *                        and the counts against their exact laws (tests/exact_law.py)
 */
#ifndef DISTILL_ORACLE_H
#define DISTILL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (spec/RNG.md) ---- */
void  od_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float od_rad(uint32_t radius_word);            /* spec/RNG.md §3: sqrt(-2 ln u1) */
void  od_rad_array(const uint32_t* R, float* y, uint64_t n);
void  od_rad_table(float* out);                 /* the 736 x 4 table RT of §3 */
float od_rsqrt(float x);
void  od_sincos2pi(uint32_t angle_word, float* c, float* s);
void  od_rsqrt_array(const float* x, float* y, uint64_t n);
void  od_sincos2pi_array(const uint32_t* a, float* c, float* s, uint64_t n);
/* normals [first, first+n) of unit U on stream 2 (accumulator models), sextet packing */
void  od_normal_acc(uint64_t seed, uint64_t unit, uint64_t first, uint64_t n, float* out);
/* the three 2-D noise vectors (prey, predator, player) of sample s: out[6] */
void  od_normal_sextet(uint64_t seed, uint32_t alloc, uint32_t sample, uint32_t invocation, float* out);

/* ---- predator-prey grid (spec/MODELS.md §1-3) ---- */
/* levels: L0+L1+L2 floats, dim 0 first.  w[3].  params = {sigma_max, sigma_min, kappa}.
 * inputs = {prey.x, prey.y, pred.x, pred.y, player.x, player.y}.
 * Writes cost[i-begin] (C, binary32) for i in [begin, end).  Returns 0, or -1 on bad args. */
int od_pp_eval(const uint32_t n_levels[3], const float* levels, const float w[3],
               const float params[3], const float inputs[6],
               uint64_t begin, uint64_t end, uint32_t n_samples, uint64_t seed,
               uint32_t invocation, float* cost);
int od_pp_trace(const uint32_t n_levels[3], const float* levels, const float params[3],
                const float inputs[6], uint64_t i, uint32_t n_samples, uint64_t seed,
                uint32_t invocation, float* out);
/* Same evaluation in binary64 from the same Philox bits (libm log/sqrt/cos/sin). */
/* Per-sample binary64 objective of allocation i (out[s], s < n_samples). */
int od_pp_trace_f64(const uint32_t n_levels[3], const float* levels, const float params[3],
                    const float inputs[6], uint64_t i, uint32_t n_samples, uint64_t seed,
                    uint32_t invocation, double* out);
int od_pp_eval_f64(const uint32_t n_levels[3], const float* levels, const float w[3],
                   const float params[3], const float inputs[6],
                   uint64_t begin, uint64_t end, uint32_t n_samples, uint64_t seed,
                   uint32_t invocation, double* cost);

/* ---- argmax keys (spec/MODELS.md §3) ---- */
uint64_t od_key(float cost, uint32_t index);
/* min over key(-net[j], base+j); returns 0 ok, 1 if no finite/inf candidate (all NaN or n == 0) */
int od_argmax_net(const float* net, uint64_t n, uint64_t base, uint64_t* key);

/* random tie-break (spec/MODELS.md §8): key_out = plain best key, tie_out = min (pi_i << 32 | i)
 * over the tied minima; the winner is (uint32)tie_out.  Returns od_argmax_net's code. */
int od_argmax_random_ties(const float* net, uint64_t n, uint64_t base, uint64_t seed,
                          uint32_t invocation, uint64_t* key_out, uint64_t* tie_out);

/* ---- DDM (spec/MODELS.md §4) ---- */
typedef struct {
    float drift, noise, threshold, x0, dt;
    uint32_t n_steps, rt_bin_steps, n_x_bins;
    float x_lo, x_hi;
} od_ddm_params;
/* one trial: choice 0 = upper, 1 = lower, 2 = undecided; step (1-based, 0 if undecided); x_N */
void od_ddm_trial(const od_ddm_params* p, uint64_t seed, uint64_t trial,
                  int* choice, uint32_t* step, float* x_end);
/* histogram accumulate (+=) over trials [t0, t1) */
int od_ddm_batch(const od_ddm_params* p, uint64_t seed, uint64_t t0, uint64_t t1,
                 uint64_t* rt_hist, uint64_t* rt_sum, uint64_t* x_hist);

/* ---- LCI single unit (spec/MODELS.md §5) — Fig. 3 pin ---- */
int od_lci_batch(const od_ddm_params* p, float leak, float offset, uint64_t seed, uint64_t t0, uint64_t t1,
                 uint64_t* rt_hist, uint64_t* rt_sum, uint64_t* x_hist);
void od_lci_trial(float input, float leak, float offset, float noise, float dt,
                  float threshold, uint32_t n_steps, uint64_t seed, uint64_t unit,
                  int* choice, uint32_t* step, float* x_end);

/* ---- Stroop-LCA grid (spec/MODELS.md §6) ---- */
/* params = {g_c, g_w, tau, leak, inhibition, noise, dt, threshold, reward, rt_cost, n_steps}
 * counts[3*(i-begin) + {0,1,2}] = {n_correct, n_undecided, rt_sum}; net[i-begin] = V. */
int od_stroop_eval(const uint32_t n_levels[2], const float* levels, const float w[2],
                   const float params[11], uint64_t begin, uint64_t end, uint32_t n_trials,
                   uint32_t trial_begin, uint32_t trial_end, uint64_t seed,
                   uint64_t* counts, float* net);
/* V from finished integer counts (binary64 then one rounding). */
float od_stroop_value(const float params[11], const float w[2], float u_c, float u_s,
                      uint32_t n_trials, uint64_t n_correct, uint64_t n_undecided, uint64_t rt_sum);
/* single Stroop trial (for tests) */
/* DDM control grid (spec/MODELS.md §6c): resp 1 = correct (upper), 0 = error, -1 = undecided */
void  od_ddmg_trial(const float params[7], float u0, float u1, uint64_t seed, uint64_t unit, int* resp,
                    uint32_t* step);
float od_ddmg_value(const float params[7], const float w[2], float u0, float u1, uint32_t n_trials,
                    uint64_t n_correct, uint64_t n_undecided, uint64_t rt_sum);
int   od_ddmg_eval(const uint32_t n_levels[2], const float* levels, const float w[2], const float params[7],
                   uint64_t begin, uint64_t end, uint32_t n_trials, uint32_t trial_begin, uint32_t trial_end,
                   uint64_t seed, uint64_t* counts, float* net);
/* decision-energy trace (spec/MODELS.md §6b) of allocation i over trials [t0, t1): esum[N] += */
void od_stroop_energy(const float params[11], float u_c, float u_s, uint64_t seed, uint64_t i, uint32_t n_trials,
                      uint32_t t0, uint32_t t1, int64_t* esum);
void od_stroop_trial(const float params[11], float u_c, float u_s, uint64_t seed,
                     uint64_t unit, uint32_t trial, int* resp, uint32_t* step);
/* od_stroop_trial with the states after each step: trace[4(n-1) + (0..3)] = (h0, h1, x0, x1). */
void od_stroop_trace(const float P[11], float u_c, float u_s, uint64_t seed,
                     uint64_t unit, uint32_t trial, int* resp, uint32_t* step, float* trace);

/* ---- closed-loop predator-prey episode (spec/MODELS.md §7) ---- */
/* traj[(n_steps+1)*6], keys[n_steps], status[2] = {outcome, steps}; speeds = {v_player, v_prey, v_predator} */
int od_pp_episode(const uint32_t n_levels[3], const float* levels, const float w[3],
                  const float params[3], const float init[6], uint32_t n_steps, uint32_t n_samples,
                  uint64_t seed, const float speeds[3], float capture_radius,
                  float* traj, uint64_t* keys, int* status);

/* ---- coarse-to-fine refinement (spec/MODELS.md §9): keys[rounds], boxes[(rounds+1)*6] = (lo, hi) x 3 ---- */
int od_pp_amr(const uint32_t n_levels[3], const float w[3], const float params[3], const float inputs[6],
              const float lo0[3], const float hi0[3], uint32_t rounds, uint32_t n_samples, uint64_t seed,
              uint32_t invocation0, uint64_t* keys, float* boxes);

/* ---- Extended Stroop A/B (spec/MODELS.md §10); variant 0 = A, 1 = B ----
 * params = {g_c, g_w, tau, N_h, lambda, a_p, gamma, sigma_d, dt_d, z_d, N_d, reward, rt_cost}
 * counts[3*(i-begin) + {0,1,2}] = {n_both, n_undecided, rt_sum} (overwritten); net = V */
void od_ext_stroop_trial_a(const float P[13], float u_c, float u_s, uint64_t seed, uint64_t unit,
                           uint32_t trial, int hit[2], uint32_t step[2]);
void od_ext_stroop_trial_b(const float P[13], float u_c, float u_s, uint64_t seed, uint64_t unit,
                           uint32_t trial, int hit[2], uint32_t step[2]);
float od_ext_stroop_value(int variant, const float P[13], const float w[2], float u_c, float u_s,
                          uint32_t n_trials, uint64_t n_both, uint64_t n_undecided, uint64_t rt_sum);
/* od_ext_stroop_eval over the trial sub-range [trial_begin, trial_end) of T (net: pass NULL unless the full range). */
int od_ext_stroop_eval_range(int variant, const uint32_t n_levels[2], const float* levels, const float w[2],
                             const float P[13], uint64_t begin, uint64_t end, uint32_t n_trials,
                             uint32_t trial_begin, uint32_t trial_end, uint64_t seed, uint64_t* counts, float* net);
int od_ext_stroop_eval(int variant, const uint32_t n_levels[2], const float* levels, const float w[2],
                       const float P[13], uint64_t begin, uint64_t end, uint32_t n_trials, uint64_t seed,
                       uint64_t* counts, float* net);

/* ---- flop counting (only meaningful in the -DOD_COUNT_FLOPS build) ---- */
/* Counting build: 1 = method count (sqrt_spec = 1 flop, rsqrt_spec = 2), 0 = executed ops (default). */
void od_flops_method(int on);
unsigned long long od_flops_read(void);
void od_flops_reset(void);
int od_is_counting_build(void);

#ifdef __cplusplus
}
#endif
#endif
