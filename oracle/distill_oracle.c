/*
 * distill_oracle.c — CPU oracle for the Distill grid-search hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see distill_oracle.h): never linked into, loaded
 * by, or called from the product path.  Written from spec/RNG.md and
 * spec/MODELS.md, which restate PAPER.md (arXiv 2110.15425):
 *   - per-evaluation independent random draws            P:356-358 (§3.6)
 *   - predator-prey Control/Obs/Action/Objective nodes    P:140-167 (§2.1, Fig. 1)
 *   - exhaustive grid search, lowest cost wins
 *   - ties                                                P:306 (§3.3)
 *   - DDM / LCI accumulation, Fig. 3 clone pinning        P:466-477 (§4.4)
 *   - Botvinick Stroop                                    P:525 (§5)
 * Readings of everything the paper leaves open are DESIGN.md §3 (R1...).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 *        (+ -DOD_COUNT_FLOPS for the flop-counting build).  No FTZ/DAZ.
 * Every binary32 operation is written out; the FADD/FMUL/... macros only add
 * a flop counter in the counting build (fma = 2 flops, others 1).
 */
#include "distill_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef OD_COUNT_FLOPS
static _Thread_local unsigned long long od_flops;
/* method-count mode: sqrt_spec counts as 1 flop and rsqrt_spec
 * as 2 (a square root and a divide) instead of their Newton/Goldschmidt steps */
static _Thread_local int od_method, od_quiet;
#define CNT(n) (od_quiet ? (void)0 : (void)(od_flops += (n)))
#define METHOD_BEGIN() do { if (od_method) ++od_quiet; } while (0)
#define METHOD_END(n) do { if (od_method) { --od_quiet; CNT(n); } } while (0)
#else
#define CNT(n) ((void)0)
#define METHOD_BEGIN() ((void)0)
#define METHOD_END(n) ((void)0)
#endif
void od_flops_method(int on) {
#ifdef OD_COUNT_FLOPS
    od_method = on;
#else
    (void)on;
#endif
}
unsigned long long od_flops_read(void) {
#ifdef OD_COUNT_FLOPS
    return od_flops;
#else
    return 0;
#endif
}
void od_flops_reset(void) {
#ifdef OD_COUNT_FLOPS
    od_flops = 0;
#endif
}
int od_is_counting_build(void) {
#ifdef OD_COUNT_FLOPS
    return 1;
#else
    return 0;
#endif
}

/* one counted binary32 operation each */
static inline float FADD(float a, float b) { CNT(1); return a + b; }
static inline float FSUB(float a, float b) { CNT(1); return a - b; }
static inline float FMUL(float a, float b) { CNT(1); return a * b; }
static inline float FDIV(float a, float b) { CNT(1); return a / b; }
static inline float FFMA(float a, float b, float c) { CNT(2); return fmaf(a, b, c); }
static inline float FSQRT(float a) { CNT(1); return sqrtf(a); }

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* ------------------------------------------------------------------------ */
/* spec/RNG.md §1: Philox4x32-10                                             */
/* ------------------------------------------------------------------------ */
void od_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------ */
/* spec/RNG.md §3: rad_spec — the Box-Muller radius sqrt(-2 ln u1) as a      */
/* piecewise cubic over the radius word's 23 random bits (revision R10c)      */
/* ------------------------------------------------------------------------ */
#define OD_RT_ROWS 736
static float od_rt[OD_RT_ROWS][4];

/* The table construction of spec/RNG.md §3, in binary64, operation by operation. */
static void od_rt_build(void) {
    const double tau[4] = { -3.0 / 128, -1.0 / 128, 1.0 / 128, 3.0 / 128 };
    for (int r = 0; r < 2; ++r)
        for (int e = 0; e < 23; ++e)
            for (int j = 0; j < 16; ++j) {
                double c = 1.0 + (2.0 * j + 1.0) / 32.0;
                double f[4];
                for (int k = 0; k < 4; ++k) {
                    double x = (c + tau[k]) * ldexp(1.0, e);
                    double N = r ? 16777216.0 - x : x;
                    f[k] = sqrt(-2.0 * log(N * 0x1p-24));
                }
                double d01 = (f[1] - f[0]) / (tau[1] - tau[0]);
                double d12 = (f[2] - f[1]) / (tau[2] - tau[1]);
                double d23 = (f[3] - f[2]) / (tau[3] - tau[2]);
                double d012 = (d12 - d01) / (tau[2] - tau[0]);
                double d123 = (d23 - d12) / (tau[3] - tau[1]);
                double A = (d123 - d012) / (tau[3] - tau[0]);
                double c3 = A;
                double c2 = d012 - A * ((tau[0] + tau[1]) + tau[2]);
                double c1 = (d01 - d012 * (tau[0] + tau[1])) + A * ((tau[0] * tau[1] + tau[0] * tau[2]) + tau[1] * tau[2]);
                double c0 = ((f[0] - d01 * tau[0]) + d012 * (tau[0] * tau[1])) - A * ((tau[0] * tau[1]) * tau[2]);
                float* row = od_rt[368 * r + 16 * e + j];
                row[0] = (float)c0; row[1] = (float)c1; row[2] = (float)c2; row[3] = (float)c3;
            }
}
__attribute__((constructor)) static void od_rt_init(void) { od_rt_build(); }

void od_rad_table(float* out) { memcpy(out, od_rt, sizeof od_rt); }

float od_rad(uint32_t R) {
    uint32_t N = (R >> 8) | 1u;                     /* odd, u1 = N 2^-24 */
    uint32_t r = N >> 23;                           /* region */
    uint32_t v = r ? (1u << 24) - N : N;            /* odd, [1, 2^23 - 1] */
    int e = 0;
    while ((v >> (e + 1)) != 0) ++e;                /* floor(log2 v) */
    float m = (float)v / (float)(1u << e);          /* exact, [1, 2) */
    uint32_t j = (uint32_t)((m - 1.0f) * 16.0f);    /* exact product; floor */
    float t = FSUB(m, 1.0f + (float)(2 * j + 1) / 32.0f);   /* exact */
    const float* c = od_rt[368 * r + 16 * e + j];
    return FFMA(FFMA(FFMA(c[3], t, c[2]), t, c[1]), t, c[0]);
}

/* ------------------------------------------------------------------------ */
/* spec/RNG.md §4: rsqrt_spec                                                */
/* ------------------------------------------------------------------------ */
float od_rsqrt(float x) {
    METHOD_BEGIN();
    float y = u2f(0x5F375A86u - (f2u(x) >> 1));
    float h = FMUL(0.5f, x);
    for (int k = 0; k < 3; ++k) {
        float p = FMUL(h, y);
        float r = FFMA(-p, y, 0.5f);
        y = FFMA(y, r, y);
    }
    METHOD_END(2);
    return y;
}

/* ------------------------------------------------------------------------ */
/* spec/RNG.md §5: sincos_spec — (cos, sin)(2 pi A / 2^32 - pi/2)            */
/* ------------------------------------------------------------------------ */
static const float OD_S[5] = { 0x1.921fb4p+1f, -0x1.4abbb6p+2f, 0x1.46676ep+1f, -0x1.323308p-1f, 0x1.3c4c1p-4f };
static const float OD_C[5] = { -0x1.3bd3ccp+2f, 0x1.03c1e6p+2f, -0x1.55d0bap+0f, 0x1.e12f96p-3f, -0x1.901cb4p-6f };

void od_sincos2pi(uint32_t a, float* cs, float* sn) {
    uint32_t h = a >> 31;
    /* exact: (a & 0x7FFFFFFF) has at most 23 significant bits, the scaling is a power of two,
       and g - 1/2 is representable for every such g */
    float r = (float)(a & 0x7FFFFFFFu) * 0x1p-31f - 0.5f;
    float t = FMUL(r, r);
    float S = FFMA(FFMA(FFMA(FFMA(OD_S[4], t, OD_S[3]), t, OD_S[2]), t, OD_S[1]), t, OD_S[0]);
    float C = FFMA(FFMA(FFMA(FFMA(OD_C[4], t, OD_C[3]), t, OD_C[2]), t, OD_C[1]), t, OD_C[0]);
    float cq = FFMA(C, t, 1.0f);
    float sq = FMUL(S, r);
    if (h) { *cs = -cq; *sn = -sq; }
    else   { *cs = cq;  *sn = sq; }
}

/* array forms of the three primitives, for the exhaustive accuracy pins */
void od_rad_array(const uint32_t* R, float* y, uint64_t n) { for (uint64_t j = 0; j < n; ++j) y[j] = od_rad(R[j]); }
void od_rsqrt_array(const float* x, float* y, uint64_t n) { for (uint64_t j = 0; j < n; ++j) y[j] = od_rsqrt(x[j]); }
void od_sincos2pi_array(const uint32_t* a, float* c, float* s, uint64_t n) {
    for (uint64_t j = 0; j < n; ++j) od_sincos2pi(a[j], &c[j], &s[j]);
}

/* spec/RNG.md §2 + §6: one Box-Muller pair in polar form (radius, cos, sin) */
static void od_bm_polar(uint32_t R, uint32_t A, float* rad, float* c, float* n) {
    *rad = od_rad(R);                                /* rad_spec = sqrt(-2 ln u1) */
    od_sincos2pi(A, c, n);
}
/* ... and as the two normals z = rad * (cos, sin) */
static void od_bm_pair(uint32_t R, uint32_t A, float* z0, float* z1) {
    float rad, c, n;
    od_bm_polar(R, A, &rad, &c, &n);
    *z0 = FMUL(rad, c);
    *z1 = FMUL(rad, n);
}

static inline void od_key_of_seed(uint64_t seed, uint32_t key[2]) {
    key[0] = (uint32_t)seed;
    key[1] = (uint32_t)(seed >> 32);
}

/* spec/RNG.md §6: the sextet packing of one Philox block X (three pairs) */
static void od_sextet_of_block(const uint32_t X[4], float out[6]) {
    uint32_t A0 = X[3] << 16;
    uint32_t A1 = X[3] & 0xFFFF0000u;
    uint32_t A2 = (X[0] << 24) | ((X[1] & 0xFFu) << 16);
    od_bm_pair(X[0], A0, &out[0], &out[1]);
    od_bm_pair(X[1], A1, &out[2], &out[3]);
    od_bm_pair(X[2], A2, &out[4], &out[5]);
}

/* Accumulator-model normals [first, first+n) of unit U (stream 2): normal j is
 * lane j mod 6 of the sextet of block X = Philox(key, (U_lo, j div 6, U_hi, 2)). */
void od_normal_acc(uint64_t seed, uint64_t unit, uint64_t first, uint64_t n, float* out) {
    uint32_t key[2];
    od_key_of_seed(seed, key);
    for (uint64_t j = first; j < first + n; ++j) {
        uint32_t ctr[4] = { (uint32_t)unit, (uint32_t)(j / 6), (uint32_t)(unit >> 32), 2u };
        uint32_t X[4];
        od_philox4x32_10(ctr, key, X);
        float z[6];
        od_sextet_of_block(X, z);
        out[j - first] = z[j % 6];
    }
}

void od_normal_sextet(uint64_t seed, uint32_t alloc, uint32_t sample, uint32_t invocation, float* out) {
    uint32_t key[2];
    od_key_of_seed(seed, key);
    uint32_t ctr[4] = { alloc, sample, invocation, 1u };
    uint32_t X[4];
    od_philox4x32_10(ctr, key, X);
    od_sextet_of_block(X, out);
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §1-2: predator-prey                                        */
/* ------------------------------------------------------------------------ */
typedef struct { float x, y; } v2;

static v2 od_unit(v2 v) {
    float n2 = FFMA(v.y, v.y, FFMA(v.x, v.x, 0x1p-126f));   /* never 0: + smallest normal */
    float y = od_rsqrt(n2);
    v2 r = { FMUL(v.x, y), FMUL(v.y, y) };
    return r;
}
static v2 od_sub(v2 a, v2 b) { v2 r = { FSUB(a.x, b.x), FSUB(a.y, b.y) }; return r; }
/* Action node: move toward the prey and away from the predator,
 * d = |v_p| (unit(v_p) - kappa unit(v_d)) = v_p + c v_d with c = -kappa |v_p| / |v_d|;
 * only its direction matters (it is normalised by the Objective), spec/MODELS.md §2. */
static v2 od_action(v2 prey, v2 pred, v2 player, float kappa) {
    v2 vp = od_sub(prey, player), vd = od_sub(pred, player);
    float np = FFMA(vp.y, vp.y, FFMA(vp.x, vp.x, 0x1p-126f));
    float nd = FFMA(vd.y, vd.y, FFMA(vd.x, vd.x, 0x1p-126f));
    float q = od_rsqrt(FMUL(np, nd));                     /* 1 / (|v_p| |v_d|), spec/MODELS.md §2 (R22b) */
    float c = FMUL(FMUL(-kappa, np), q);                  /* -kappa |v_p| / |v_d| */
    v2 d = { FFMA(c, vd.x, vp.x), FFMA(c, vd.y, vp.y) };
    return d;
}

/* Obs nodes: o_e = p_e + (sigma_e rad_e) (cos, sin) for the sextet pair of entity e */
static void od_observe(uint64_t seed, uint32_t alloc, uint32_t sample, uint32_t invocation,
                       const float sig[3], const v2 p[3], v2 o[3]) {
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t ctr[4] = { alloc, sample, invocation, 1u };
    uint32_t X[4];
    od_philox4x32_10(ctr, key, X);
    uint32_t A[3] = { X[3] << 16, X[3] & 0xFFFF0000u, (X[0] << 24) | ((X[1] & 0xFFu) << 16) };
    for (int e = 0; e < 3; ++e) {
        float rad, c, n;
        od_bm_polar(X[e], A[e], &rad, &c, &n);
        float sr = FMUL(sig[e], rad);
        o[e].x = FFMA(sr, c, p[e].x);
        o[e].y = FFMA(sr, n, p[e].y);
    }
}

/* Objective node: squared chord between the normalised action d/|d|
 * and the true best move u*, with delta = d * y_d - u* fused per component */
static float od_objective(v2 d, v2 ustar) {
    float yd = od_rsqrt(FFMA(d.y, d.y, FFMA(d.x, d.x, 0x1p-126f)));
#ifdef OD_UNFUSED_OBJECTIVE
    /* DESIGN.md R21 comparison build only (tools/r21_error.py): u_hat rounded on its own */
    v2 dl = { FSUB(FMUL(d.x, yd), ustar.x), FSUB(FMUL(d.y, yd), ustar.y) };
#else
    v2 dl = { FFMA(d.x, yd, -ustar.x), FFMA(d.y, yd, -ustar.y) };
#endif
    return FFMA(dl.y, dl.y, FMUL(dl.x, dl.x));
}

/* mixed-radix decode, dim 0 most significant */
static void od_decode(uint64_t i, int D, const uint32_t* L, uint32_t* k) {
    for (int d = D - 1; d >= 0; --d) { k[d] = (uint32_t)(i % L[d]); i /= L[d]; }
}

int od_pp_eval(const uint32_t n_levels[3], const float* levels, const float w[3],
               const float params[3], const float inputs[6],
               uint64_t begin, uint64_t end, uint32_t n_samples, uint64_t seed,
               uint32_t invocation, float* cost) {
    if (!n_levels || !levels || !w || !params || !inputs || n_samples == 0 || end < begin) return -1;
    uint64_t N = (uint64_t)n_levels[0] * n_levels[1] * n_levels[2];
    if (N == 0 || end > N || N > 0xFFFFFFFFull) return -1;
    const float* lev[3] = { levels, levels + n_levels[0], levels + n_levels[0] + n_levels[1] };
    float smax = params[0], smin = params[1], kappa = params[2];
    v2 p[3] = { { inputs[0], inputs[1] }, { inputs[2], inputs[3] }, { inputs[4], inputs[5] } };
    float dsig = FSUB(smin, smax);
    v2 ustar = od_unit(od_action(p[0], p[1], p[2], kappa));

    for (uint64_t i = begin; i < end; ++i) {
        uint32_t k[3];
        od_decode(i, 3, n_levels, k);
        float a[3] = { lev[0][k[0]], lev[1][k[1]], lev[2][k[2]] };
        float sig[3];
        for (int e = 0; e < 3; ++e) sig[e] = FFMA(a[e], dsig, smax);
        float K = FFMA(w[2], a[2], FFMA(w[1], a[1], FMUL(w[0], a[0])));
        float acc = 0.0f;
        for (uint32_t s = 0; s < n_samples; ++s) {
            v2 o[3];
            od_observe(seed, (uint32_t)i, s, invocation, sig, p, o);
            float e2 = od_objective(od_action(o[0], o[1], o[2], kappa), ustar);
            acc = FADD(acc, e2);
        }
        cost[i - begin] = FADD(FDIV(acc, (float)n_samples), K);
    }
    return 0;
}

/* Per-sample objective e_s of one allocation (debug / tests): out[s], s < S. */
int od_pp_trace(const uint32_t n_levels[3], const float* levels, const float params[3],
                const float inputs[6], uint64_t i, uint32_t n_samples, uint64_t seed,
                uint32_t invocation, float* out) {
    const float* lev[3] = { levels, levels + n_levels[0], levels + n_levels[0] + n_levels[1] };
    float smax = params[0], smin = params[1], kappa = params[2];
    v2 p[3] = { { inputs[0], inputs[1] }, { inputs[2], inputs[3] }, { inputs[4], inputs[5] } };
    float dsig = FSUB(smin, smax);
    v2 ustar = od_unit(od_action(p[0], p[1], p[2], kappa));
    uint32_t k[3];
    od_decode(i, 3, n_levels, k);
    float a[3] = { lev[0][k[0]], lev[1][k[1]], lev[2][k[2]] };
    float sig[3];
    for (int e = 0; e < 3; ++e) sig[e] = FFMA(a[e], dsig, smax);
    for (uint32_t s = 0; s < n_samples; ++s) {
        v2 o[3];
        od_observe(seed, (uint32_t)i, s, invocation, sig, p, o);
        out[s] = od_objective(od_action(o[0], o[1], o[2], kappa), ustar);
    }
    return 0;
}

/* Same model in binary64 (the "plain definition" re-evaluation): normals from
 * the same Philox bits with exact libm Box-Muller, body with 1/sqrt. */
typedef struct { double x, y; } d2;
static d2 d_unit(d2 v) {
    double n2 = v.x * v.x + v.y * v.y;
    double y = (n2 == 0.0) ? 0.0 : 1.0 / sqrt(n2);
    d2 r = { v.x * y, v.y * y };
    return r;
}
static d2 d_action(d2 prey, d2 pred, d2 player, double kappa) {
    d2 a = { prey.x - player.x, prey.y - player.y }, b = { pred.x - player.x, pred.y - player.y };
    d2 up = d_unit(a), ud = d_unit(b);
    d2 d = { up.x - kappa * ud.x, up.y - kappa * ud.y };
    return d;
}
static void d_bm(uint32_t R, uint32_t A, double* z0, double* z1) {
    const double TWO_PI = 6.283185307179586476925286766559;
    double u1 = (double)((R >> 8) | 1u) * 0x1p-24;
    double t = (double)A * 0x1p-32 - 0.25;    /* angle 2 pi A / 2^32 - pi/2 */
    double rad = sqrt(-2.0 * log(u1));
    *z0 = rad * cos(TWO_PI * t);
    *z1 = rad * sin(TWO_PI * t);
}

/* Per-sample binary64 objective of one allocation (the plain definition, sample by sample). */
int od_pp_trace_f64(const uint32_t n_levels[3], const float* levels, const float params[3],
                    const float inputs[6], uint64_t i, uint32_t n_samples, uint64_t seed,
                    uint32_t invocation, double* out) {
    const float* lev[3] = { levels, levels + n_levels[0], levels + n_levels[0] + n_levels[1] };
    double smax = params[0], smin = params[1], kappa = params[2];
    d2 p[3] = { { inputs[0], inputs[1] }, { inputs[2], inputs[3] }, { inputs[4], inputs[5] } };
    d2 ustar = d_unit(d_action(p[0], p[1], p[2], kappa));
    uint32_t key[2];
    od_key_of_seed(seed, key);
    uint32_t k[3];
    od_decode(i, 3, n_levels, k);
    double a[3] = { lev[0][k[0]], lev[1][k[1]], lev[2][k[2]] };
    for (uint32_t s = 0; s < n_samples; ++s) {
        uint32_t ctr[4] = { (uint32_t)i, s, invocation, 1u }, X[4];
        od_philox4x32_10(ctr, key, X);
        uint32_t A[3] = { X[3] << 16, X[3] & 0xFFFF0000u, (X[0] << 24) | ((X[1] & 0xFFu) << 16) };
        d2 o[3];
        for (int e = 0; e < 3; ++e) {
            double zx, zy, sg = smax + a[e] * (smin - smax);
            d_bm(X[e], A[e], &zx, &zy);
            o[e].x = p[e].x + sg * zx;
            o[e].y = p[e].y + sg * zy;
        }
        d2 uh = d_unit(d_action(o[0], o[1], o[2], kappa));
        double dx = uh.x - ustar.x, dy = uh.y - ustar.y;
        out[s] = dx * dx + dy * dy;
    }
    return 0;
}

int od_pp_eval_f64(const uint32_t n_levels[3], const float* levels, const float w[3],
                   const float params[3], const float inputs[6],
                   uint64_t begin, uint64_t end, uint32_t n_samples, uint64_t seed,
                   uint32_t invocation, double* cost) {
    if (!n_levels || !levels || !w || !params || !inputs || n_samples == 0 || end < begin) return -1;
    uint64_t N = (uint64_t)n_levels[0] * n_levels[1] * n_levels[2];
    if (N == 0 || end > N || N > 0xFFFFFFFFull) return -1;
    const float* lev[3] = { levels, levels + n_levels[0], levels + n_levels[0] + n_levels[1] };
    double smax = params[0], smin = params[1], kappa = params[2];
    d2 p[3] = { { inputs[0], inputs[1] }, { inputs[2], inputs[3] }, { inputs[4], inputs[5] } };
    d2 ustar = d_unit(d_action(p[0], p[1], p[2], kappa));
    uint32_t key[2];
    od_key_of_seed(seed, key);
    for (uint64_t i = begin; i < end; ++i) {
        uint32_t k[3];
        od_decode(i, 3, n_levels, k);
        double a[3] = { lev[0][k[0]], lev[1][k[1]], lev[2][k[2]] };
        double sig[3];
        for (int e = 0; e < 3; ++e) sig[e] = smax + a[e] * (smin - smax);
        double K = (double)w[0] * a[0] + (double)w[1] * a[1] + (double)w[2] * a[2];
        double acc = 0.0;
        for (uint32_t s = 0; s < n_samples; ++s) {
            uint32_t ctr[4] = { (uint32_t)i, s, invocation, 1u }, X[4];
            od_philox4x32_10(ctr, key, X);
            uint32_t A[3] = { X[3] << 16, X[3] & 0xFFFF0000u, (X[0] << 24) | ((X[1] & 0xFFu) << 16) };
            d2 o[3];
            for (int e = 0; e < 3; ++e) {
                double zx, zy;
                d_bm(X[e], A[e], &zx, &zy);
                o[e].x = p[e].x + sig[e] * zx;
                o[e].y = p[e].y + sig[e] * zy;
            }
            d2 uh = d_unit(d_action(o[0], o[1], o[2], kappa));
            double dx = uh.x - ustar.x, dy = uh.y - ustar.y;
            acc += dx * dx + dy * dy;
        }
        cost[i - begin] = acc / (double)n_samples + K;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §3: argmax keys                                            */
/* ------------------------------------------------------------------------ */
uint64_t od_key(float cost, uint32_t index) {
    uint32_t hi;
    if (isnan(cost)) {
        hi = 0xFFFFFFFFu;
    } else {
        if (cost == 0.0f) cost = 0.0f;              /* -0 -> +0 */
        uint32_t b = f2u(cost);
        hi = (b >> 31) ? ~b : (b | 0x80000000u);
    }
    return ((uint64_t)hi << 32) | index;
}

int od_argmax_net(const float* net, uint64_t n, uint64_t base, uint64_t* key) {
    uint64_t best = 0xFFFFFFFFFFFFFFFFull;
    for (uint64_t j = 0; j < n; ++j) {
        uint64_t k = od_key(-net[j], (uint32_t)(base + j));
        if (k < best) best = k;
    }
    *key = best;
    return (n == 0 || (best >> 32) == 0xFFFFFFFFull) ? 1 : 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §4: DDM                                                    */
/* ------------------------------------------------------------------------ */
void od_ddm_trial(const od_ddm_params* p, uint64_t seed, uint64_t trial,
                  int* choice, uint32_t* step, float* x_end) {
    float nsd = FMUL(p->noise, FSQRT(p->dt));
    float x = p->x0;
    int ch = 2;
    uint32_t st = 0;
    for (uint32_t n = 1; n <= p->n_steps; ++n) {
        float g;
        od_normal_acc(seed, trial, n - 1, 1, &g);
        x = FFMA(nsd, g, FFMA(p->dt, p->drift, x));
        if (ch == 2) {
            if (x >= p->threshold) { ch = 0; st = n; }
            else if (x <= -p->threshold) { ch = 1; st = n; }
        }
    }
    *choice = ch; *step = st; *x_end = x;
}

int od_ddm_batch(const od_ddm_params* p, uint64_t seed, uint64_t t0, uint64_t t1,
                 uint64_t* rt_hist, uint64_t* rt_sum, uint64_t* x_hist) {
    if (!p || p->n_steps == 0 || p->rt_bin_steps == 0 || p->n_x_bins == 0 || t1 < t0) return -1;
    uint32_t nb = (p->n_steps + p->rt_bin_steps - 1) / p->rt_bin_steps;
    float sc = (float)p->n_x_bins / (p->x_hi - p->x_lo);
    for (uint64_t t = t0; t < t1; ++t) {
        int ch; uint32_t st; float xe;
        od_ddm_trial(p, seed, t, &ch, &st, &xe);
        if (ch == 2) rt_hist[2 * nb] += 1;
        else { rt_hist[(uint32_t)ch * nb + (st - 1) / p->rt_bin_steps] += 1; rt_sum[ch] += st; }
        float u = (xe - p->x_lo) * sc;
        uint32_t bin;
        if (u < 0.0f) bin = 0;
        else if (!(u < (float)p->n_x_bins)) bin = p->n_x_bins + 1;
        else bin = 1 + (uint32_t)u;
        x_hist[bin] += 1;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §5: LCI (Fig. 3 clone of the DDM integrator)               */
/* ------------------------------------------------------------------------ */
static void lci_trial_core(float input, float leak, float offset, float noise, float dt, float threshold,
                           float x0, uint32_t n_steps, uint64_t seed, uint64_t unit,
                           int* choice, uint32_t* step, float* x_end) {
    float nsd = FMUL(noise, FSQRT(dt));
    float x = x0;
    int ch = 2;
    uint32_t st = 0;
    for (uint32_t n = 1; n <= n_steps; ++n) {
        float g;
        od_normal_acc(seed, unit, n - 1, 1, &g);
        x = FFMA(nsd, g, FADD(FFMA(dt, FFMA(-leak, x, input), x), offset));
        if (ch == 2) {
            if (x >= threshold) { ch = 0; st = n; }
            else if (x <= -threshold) { ch = 1; st = n; }
        }
    }
    *choice = ch; *step = st; *x_end = x;
}

void od_lci_trial(float input, float leak, float offset, float noise, float dt,
                  float threshold, uint32_t n_steps, uint64_t seed, uint64_t unit,
                  int* choice, uint32_t* step, float* x_end) {
    lci_trial_core(input, leak, offset, noise, dt, threshold, 0.0f, n_steps, seed, unit, choice, step, x_end);
}

/* LCI batch with the DDM batch's outputs (spec/MODELS.md §5): p->drift is the
 * input I, p->x0 the start; histograms binned exactly as od_ddm_batch. */
int od_lci_batch(const od_ddm_params* p, float leak, float offset, uint64_t seed, uint64_t t0, uint64_t t1,
                 uint64_t* rt_hist, uint64_t* rt_sum, uint64_t* x_hist) {
    if (!p || p->n_steps == 0 || p->rt_bin_steps == 0 || p->n_x_bins == 0 || t1 < t0) return -1;
    uint32_t nb = (p->n_steps + p->rt_bin_steps - 1) / p->rt_bin_steps;
    float sc = (float)p->n_x_bins / (p->x_hi - p->x_lo);
    for (uint64_t t = t0; t < t1; ++t) {
        int ch; uint32_t st; float xe;
        lci_trial_core(p->drift, leak, offset, p->noise, p->dt, p->threshold, p->x0, p->n_steps, seed, t,
                       &ch, &st, &xe);
        if (ch == 2) rt_hist[2 * nb] += 1;
        else { rt_hist[(uint32_t)ch * nb + (st - 1) / p->rt_bin_steps] += 1; rt_sum[ch] += st; }
        float u = (xe - p->x_lo) * sc;
        uint32_t bin;
        if (u < 0.0f) bin = 0;
        else if (!(u < (float)p->n_x_bins)) bin = p->n_x_bins + 1;
        else bin = 1 + (uint32_t)u;
        x_hist[bin] += 1;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §6: Stroop-LCA                                             */
/* ------------------------------------------------------------------------ */
enum { SP_GC, SP_GW, SP_TAU, SP_LEAK, SP_INH, SP_NOISE, SP_DT, SP_THR, SP_R, SP_CRT, SP_N };

/* One Stroop-LCA trial (spec/MODELS.md §6); if esum is non-NULL, also the
 * decision-energy trace of §6b: esum[n-1] += llrint(x0(n) * x1(n) * 2^24);
 * if trace is non-NULL, the states after each step n: trace[4(n-1) ..] =
 * (h0, h1, x0, x1) (test infrastructure: the closed-form pins of the
 * pathway and response layers read it). */
static void stroop_trial_core(const float P[11], float u_c, float u_s, uint64_t seed,
                              uint64_t unit, uint32_t trial, int* resp, uint32_t* step, int64_t* esum,
                              float* trace) {
    uint32_t kind = trial % 3, color = (trial / 3) % 2;
    int word = (kind == 0) ? (int)color : (kind == 1) ? (int)(1 - color) : -1;
    float ic = FMUL(P[SP_GC], u_c);
    float iw = FMUL(P[SP_GW], FSUB(1.0f, u_s));
    float I[2];
    for (int k = 0; k < 2; ++k) {
        float a = ((uint32_t)k == color) ? ic : 0.0f;
        float b = (k == word) ? iw : 0.0f;
        I[k] = FADD(a, b);
    }
    uint32_t N = (uint32_t)P[SP_N];
    float nsd = FMUL(P[SP_NOISE], FSQRT(P[SP_DT]));
    float h[2] = { 0.0f, 0.0f }, x[2] = { 0.0f, 0.0f };
    int r = -1;
    uint32_t st = 0;
    for (uint32_t n = 1; n <= N; ++n) {
        for (int k = 0; k < 2; ++k) h[k] = FFMA(P[SP_TAU], FSUB(I[k], h[k]), h[k]);
        float g[2];
        od_normal_acc(seed, unit, 2ull * (n - 1), 2, g);
        float xn[2];
        for (int k = 0; k < 2; ++k) {
            float q = FFMA(-P[SP_INH], x[1 - k], FFMA(-P[SP_LEAK], x[k], h[k]));
            float y = FFMA(nsd, g[k], FFMA(P[SP_DT], q, x[k]));
            xn[k] = fmaxf(y, 0.0f);
        }
        x[0] = xn[0]; x[1] = xn[1];
        if (trace) {
            trace[4 * (n - 1)] = h[0]; trace[4 * (n - 1) + 1] = h[1];
            trace[4 * (n - 1) + 2] = x[0]; trace[4 * (n - 1) + 3] = x[1];
        }
        if (esum) esum[n - 1] += llrintf(FMUL(FMUL(x[0], x[1]), 0x1p24f));   /* exact scaling; round to nearest even */
        if (r < 0) {
            if (x[0] >= P[SP_THR]) { r = 0; st = n; }
            else if (x[1] >= P[SP_THR]) { r = 1; st = n; }
        }
    }
    *resp = r; *step = st;
}

void od_stroop_trial(const float P[11], float u_c, float u_s, uint64_t seed,
                     uint64_t unit, uint32_t trial, int* resp, uint32_t* step) {
    stroop_trial_core(P, u_c, u_s, seed, unit, trial, resp, step, NULL, NULL);
}

/* The same trial with its per-step states (h0, h1, x0, x1) written to trace[4N]. */
void od_stroop_trace(const float P[11], float u_c, float u_s, uint64_t seed,
                     uint64_t unit, uint32_t trial, int* resp, uint32_t* step, float* trace) {
    stroop_trial_core(P, u_c, u_s, seed, unit, trial, resp, step, NULL, trace);
}

/* spec/MODELS.md §6b: decision-energy trace of allocation i (u_c, u_s) over
 * trials [t0, t1) of T: esum[n-1] += llrint(x0(n) x1(n) 2^24), n = 1..N. */
void od_stroop_energy(const float P[11], float u_c, float u_s, uint64_t seed, uint64_t i, uint32_t n_trials,
                      uint32_t t0, uint32_t t1, int64_t* esum) {
    for (uint32_t j = t0; j < t1; ++j) {
        int resp;
        uint32_t st;
        stroop_trial_core(P, u_c, u_s, seed, i * (uint64_t)n_trials + j, j, &resp, &st, esum, NULL);
    }
}

float od_stroop_value(const float P[11], const float w[2], float u_c, float u_s,
                      uint32_t n_trials, uint64_t n_correct, uint64_t n_undecided, uint64_t rt_sum) {
    double T = (double)n_trials;
    double N = (double)(uint32_t)P[SP_N];
    double v = (double)P[SP_R] * (double)n_correct / T;
    v = v - (double)P[SP_CRT] * (double)P[SP_DT] * ((double)rt_sum + (double)n_undecided * N) / T;
    v = v - ((double)w[0] * (double)u_c + (double)w[1] * (double)u_s);
    return (float)v;
}

int od_stroop_eval(const uint32_t n_levels[2], const float* levels, const float w[2],
                   const float P[11], uint64_t begin, uint64_t end, uint32_t n_trials,
                   uint32_t trial_begin, uint32_t trial_end, uint64_t seed,
                   uint64_t* counts, float* net) {
    if (!n_levels || !levels || !w || !P || n_trials == 0 || end < begin ||
        trial_end < trial_begin || trial_end > n_trials) return -1;
    uint64_t N = (uint64_t)n_levels[0] * n_levels[1];
    if (N == 0 || end > N || N * (uint64_t)n_trials > 0xFFFFFFFFFFFFull) return -1;
    for (uint64_t i = begin; i < end; ++i) {
        uint32_t k[2];
        od_decode(i, 2, n_levels, k);
        float uc = levels[k[0]], us = levels[n_levels[0] + k[1]];
        uint64_t* c = counts + 3 * (i - begin);
        for (uint32_t j = trial_begin; j < trial_end; ++j) {
            uint32_t colour = (j / 3) % 2;
            int resp; uint32_t st;
            od_stroop_trial(P, uc, us, seed, i * (uint64_t)n_trials + j, j, &resp, &st);
            if (resp < 0) c[1] += 1;
            else { if ((uint32_t)resp == colour) c[0] += 1; c[2] += st; }
        }
        if (net) net[i - begin] = od_stroop_value(P, w, uc, us, n_trials, c[0], c[1], c[2]);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §6c: DDM control grid                                      */
/* ------------------------------------------------------------------------ */
enum { DG_A0, DG_GA, DG_NOISE, DG_DT, DG_R, DG_CRT, DG_N };

void od_ddmg_trial(const float P[7], float u0, float u1, uint64_t seed, uint64_t unit, int* resp, uint32_t* step) {
    float A = FFMA(P[DG_GA], u0, P[DG_A0]);
    float z = u1;
    float nsd = FMUL(P[DG_NOISE], FSQRT(P[DG_DT]));
    float x = 0.0f;
    int r = -1;
    uint32_t st = 0;
    uint32_t N = (uint32_t)P[DG_N];
    for (uint32_t n = 1; n <= N; ++n) {
        float g;
        od_normal_acc(seed, unit, n - 1, 1, &g);
        x = FFMA(nsd, g, FFMA(P[DG_DT], A, x));
        if (r < 0) {
            if (x >= z) { r = 1; st = n; }
            else if (x <= -z) { r = 0; st = n; }
        }
    }
    *resp = r; *step = st;
}

float od_ddmg_value(const float P[7], const float w[2], float u0, float u1, uint32_t n_trials,
                    uint64_t n_correct, uint64_t n_undecided, uint64_t rt_sum) {
    double T = (double)n_trials, N = (double)(uint32_t)P[DG_N];
    double v = (double)P[DG_R] * (double)n_correct / T;
    v = v - (double)P[DG_CRT] * (double)P[DG_DT] * ((double)rt_sum + (double)n_undecided * N) / T;
    v = v - ((double)w[0] * (double)u0 + (double)w[1] * (double)u1);
    return (float)v;
}

int od_ddmg_eval(const uint32_t n_levels[2], const float* levels, const float w[2], const float P[7],
                 uint64_t begin, uint64_t end, uint32_t n_trials, uint32_t trial_begin, uint32_t trial_end,
                 uint64_t seed, uint64_t* counts, float* net) {
    if (!n_levels || !levels || !w || !P || n_trials == 0 || end < begin ||
        trial_end < trial_begin || trial_end > n_trials) return -1;
    uint64_t NA = (uint64_t)n_levels[0] * n_levels[1];
    if (NA == 0 || end > NA) return -1;
    for (uint64_t i = begin; i < end; ++i) {
        uint32_t k[2];
        od_decode(i, 2, n_levels, k);
        float u0 = levels[k[0]], u1 = levels[n_levels[0] + k[1]];
        uint64_t* c = counts + 3 * (i - begin);
        for (uint32_t j = trial_begin; j < trial_end; ++j) {
            int resp; uint32_t st;
            od_ddmg_trial(P, u0, u1, seed, i * (uint64_t)n_trials + j, &resp, &st);
            if (resp < 0) c[1] += 1;
            else { if (resp == 1) c[0] += 1; c[2] += st; }
        }
        if (net) net[i - begin] = od_ddmg_value(P, w, u0, u1, n_trials, c[0], c[1], c[2]);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §7: closed-loop predator-prey episode (NEXT-1)             */
/* ------------------------------------------------------------------------ */
int od_pp_episode(const uint32_t n_levels[3], const float* levels, const float w[3],
                  const float params[3], const float init[6], uint32_t n_steps, uint32_t n_samples,
                  uint64_t seed, const float speeds[3], float capture_radius,
                  float* traj, uint64_t* keys, int* status) {
    uint64_t N = (uint64_t)n_levels[0] * n_levels[1] * n_levels[2];
    if (N == 0 || N > 0xFFFFFFFFull || n_samples == 0) return -1;
    const float* lev[3] = { levels, levels + n_levels[0], levels + n_levels[0] + n_levels[1] };
    float smax = params[0], smin = params[1], kappa = params[2];
    float dsig = FSUB(smin, smax);
    float rc2 = FMUL(capture_radius, capture_radius);
    for (int k = 0; k < 6; ++k) traj[k] = init[k];
    status[0] = 0; status[1] = 0;
    float* cost = (float*)malloc(N * sizeof(float));
    if (!cost) return -1;
    for (uint32_t t = 0; t < n_steps; ++t) {
        float* cur = traj + 6 * (size_t)t;
        float* nxt = traj + 6 * (size_t)(t + 1);
        keys[t] = 0xFFFFFFFFFFFFFFFFull;
        if (status[0] != 0) { for (int k = 0; k < 6; ++k) nxt[k] = cur[k]; continue; }
        /* 1. grid search on the current positions */
        od_pp_eval(n_levels, levels, w, params, cur, 0, N, n_samples, seed, t, cost);
        uint64_t best = 0xFFFFFFFFFFFFFFFFull;
        for (uint64_t i = 0; i < N; ++i) { uint64_t k = od_key(cost[i], (uint32_t)i); if (k < best) best = k; }
        keys[t] = best;
        if ((best >> 32) == 0xFFFFFFFFull) { status[0] = 3; status[1] = (int)(t + 1); for (int k = 0; k < 6; ++k) nxt[k] = cur[k]; continue; }
        uint32_t ka[3];
        od_decode((uint32_t)best, 3, n_levels, ka);
        float sig[3];
        for (int e = 0; e < 3; ++e) sig[e] = FFMA(lev[e][ka[e]], dsig, smax);
        /* 2. execution observation on stream 4 */
        v2 p[3] = { { cur[0], cur[1] }, { cur[2], cur[3] }, { cur[4], cur[5] } };
        uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
        uint32_t ctr[4] = { t, 0u, 0u, 4u }, X[4];
        od_philox4x32_10(ctr, key, X);
        uint32_t A[3] = { X[3] << 16, X[3] & 0xFFFF0000u, (X[0] << 24) | ((X[1] & 0xFFu) << 16) };
        v2 o[3];
        for (int e = 0; e < 3; ++e) {
            float rad, c, n;
            od_bm_polar(X[e], A[e], &rad, &c, &n);
            float sr = FMUL(sig[e], rad);
            o[e].x = FFMA(sr, c, p[e].x);
            o[e].y = FFMA(sr, n, p[e].y);
        }
        /* 3. moves (all directions from the pre-move positions) */
        v2 up = od_unit(od_action(o[0], o[1], o[2], kappa));
        v2 uy = od_unit(od_sub(p[0], p[2]));
        v2 ud = od_unit(od_sub(p[2], p[1]));
        v2 pl = { FFMA(speeds[0], up.x, p[2].x), FFMA(speeds[0], up.y, p[2].y) };
        v2 py = { FFMA(speeds[1], uy.x, p[0].x), FFMA(speeds[1], uy.y, p[0].y) };
        v2 pd = { FFMA(speeds[2], ud.x, p[1].x), FFMA(speeds[2], ud.y, p[1].y) };
        nxt[0] = py.x; nxt[1] = py.y; nxt[2] = pd.x; nxt[3] = pd.y; nxt[4] = pl.x; nxt[5] = pl.y;
        /* 4. capture */
        v2 qy = od_sub(py, pl), qd = od_sub(pd, pl);
        if (FFMA(qy.y, qy.y, FMUL(qy.x, qy.x)) <= rc2) { status[0] = 1; status[1] = (int)(t + 1); }
        else if (FFMA(qd.y, qd.y, FMUL(qd.x, qd.x)) <= rc2) { status[0] = 2; status[1] = (int)(t + 1); }
    }
    free(cost);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §8: random tie-breaking among the minimal costs (NEXT-2)   */
/* ------------------------------------------------------------------------ */
int od_argmax_random_ties(const float* net, uint64_t n, uint64_t base, uint64_t seed,
                          uint32_t invocation, uint64_t* key_out, uint64_t* tie_out) {
    uint64_t best;
    int rc = od_argmax_net(net, n, base, &best);
    *key_out = best;
    *tie_out = 0xFFFFFFFFFFFFFFFFull;
    if (rc != 0) return rc;
    uint32_t hi = (uint32_t)(best >> 32);
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    for (uint64_t j = 0; j < n; ++j) {
        uint64_t k = od_key(-net[j], (uint32_t)(base + j));
        if ((uint32_t)(k >> 32) != hi) continue;              /* not among the tied minima */
        uint32_t ctr[4] = { (uint32_t)(base + j), 0u, invocation, 3u }, X[4];
        od_philox4x32_10(ctr, key, X);
        uint64_t t = ((uint64_t)X[0] << 32) | (uint32_t)(base + j);
        if (t < *tie_out) *tie_out = t;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §9: coarse-to-fine grid refinement (NEXT-4)                */
/* ------------------------------------------------------------------------ */
int od_pp_amr(const uint32_t n_levels[3], const float w[3], const float params[3], const float inputs[6],
              const float lo0[3], const float hi0[3], uint32_t rounds, uint32_t n_samples, uint64_t seed,
              uint32_t invocation0, uint64_t* keys, float* boxes) {
    uint64_t N = (uint64_t)n_levels[0] * n_levels[1] * n_levels[2];
    if (N == 0 || N > 0xFFFFFFFFull || n_samples == 0) return -1;
    float lo[3], hi[3];
    for (int d = 0; d < 3; ++d) { lo[d] = lo0[d]; hi[d] = hi0[d]; boxes[2 * d] = lo[d]; boxes[2 * d + 1] = hi[d]; }
    float* levels = (float*)malloc((n_levels[0] + n_levels[1] + n_levels[2]) * sizeof(float));
    float* cost = (float*)malloc(N * sizeof(float));
    if (!levels || !cost) { free(levels); free(cost); return -1; }
    for (uint32_t r = 0; r < rounds; ++r) {
        float step[3];
        uint32_t off = 0;
        for (int d = 0; d < 3; ++d) {
            step[d] = (n_levels[d] > 1) ? FDIV(FSUB(hi[d], lo[d]), (float)(n_levels[d] - 1)) : 0.0f;
            for (uint32_t k = 0; k < n_levels[d]; ++k) levels[off + k] = FFMA((float)k, step[d], lo[d]);
            off += n_levels[d];
        }
        od_pp_eval(n_levels, levels, w, params, inputs, 0, N, n_samples, seed, invocation0 + r, cost);
        uint64_t best = 0xFFFFFFFFFFFFFFFFull;
        for (uint64_t i = 0; i < N; ++i) { uint64_t k = od_key(cost[i], (uint32_t)i); if (k < best) best = k; }
        keys[r] = best;
        if ((best >> 32) == 0xFFFFFFFFull) {        /* no valid allocation (all NaN): box unchanged (MODELS.md §9) */
            for (int d = 0; d < 3; ++d) { boxes[6 * (r + 1) + 2 * d] = lo[d]; boxes[6 * (r + 1) + 2 * d + 1] = hi[d]; }
            continue;
        }
        uint32_t ka[3];
        od_decode((uint32_t)best, 3, n_levels, ka);
        off = 0;
        for (int d = 0; d < 3; ++d) {
            float a = levels[off + ka[d]];
            off += n_levels[d];
            lo[d] = fmaxf(lo0[d], FSUB(a, step[d]));
            hi[d] = fminf(hi0[d], FADD(a, step[d]));
            boxes[6 * (r + 1) + 2 * d] = lo[d];
            boxes[6 * (r + 1) + 2 * d + 1] = hi[d];
        }
    }
    free(levels); free(cost);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* spec/MODELS.md §10: Extended Stroop A / B (NEXT-3)                        */
/* ------------------------------------------------------------------------ */
enum { XS_GC, XS_GW, XS_TAU, XS_NH, XS_LAM, XS_AP, XS_GAM, XS_SIG, XS_DT, XS_Z, XS_ND, XS_R, XS_CRT };

static void xs_inputs(const float P[13], float u_c, float u_s, uint32_t trial, float I[2], uint32_t* colour) {
    uint32_t kind = trial % 3, c = (trial / 3) % 2;
    int word = (kind == 0) ? (int)c : (kind == 1) ? (int)(1 - c) : -1;
    float ic = FMUL(P[XS_GC], u_c);
    float iw = FMUL(P[XS_GW], FSUB(1.0f, u_s));
    for (int k = 0; k < 2; ++k) I[k] = FADD(((uint32_t)k == c) ? ic : 0.0f, (k == word) ? iw : 0.0f);
    *colour = c;
}

/* version A: colour DDM first, single linear node, reward from successes */
void od_ext_stroop_trial_a(const float P[13], float u_c, float u_s, uint64_t seed, uint64_t unit,
                           uint32_t trial, int hit[2], uint32_t step[2]) {
    float I[2]; uint32_t c;
    xs_inputs(P, u_c, u_s, trial, I, &c);
    float h[2] = { 0.0f, 0.0f };
    for (uint32_t n = 0; n < (uint32_t)P[XS_NH]; ++n)
        for (int k = 0; k < 2; ++k) h[k] = FFMA(P[XS_TAU], FSUB(I[k], h[k]), h[k]);
    float E = FMUL(h[0], h[1]);
    float A1 = FMUL(FSUB(h[c], h[1 - c]), P[XS_LAM]);
    float A2 = FFMA(-P[XS_GAM], E, P[XS_AP]);
    float nsd = FMUL(P[XS_SIG], FSQRT(P[XS_DT]));
    float x1 = 0.0f, x2 = 0.0f;
    hit[0] = hit[1] = 0; step[0] = step[1] = 0;
    for (uint32_t n = 1; n <= (uint32_t)P[XS_ND]; ++n) {
        float g[2];
        od_normal_acc(seed, unit, 2ull * (n - 1), 2, g);
        x1 = FFMA(nsd, g[0], FFMA(P[XS_DT], A1, x1));
        x2 = FFMA(nsd, g[1], FFMA(P[XS_DT], A2, x2));
        if (!hit[0]) { if (x1 >= P[XS_Z]) { hit[0] = 1; step[0] = n; } else if (x1 <= -P[XS_Z]) { hit[0] = 2; step[0] = n; } }
        if (!hit[1]) { if (x2 >= P[XS_Z]) { hit[1] = 1; step[1] = n; } else if (x2 <= -P[XS_Z]) { hit[1] = 2; step[1] = n; } }
    }
}

/* version B: pointing DDM declared first, two chained linear nodes, fma operands swapped */
void od_ext_stroop_trial_b(const float P[13], float u_c, float u_s, uint64_t seed, uint64_t unit,
                           uint32_t trial, int hit[2], uint32_t step[2]) {
    float I[2]; uint32_t c;
    xs_inputs(P, u_c, u_s, trial, I, &c);
    float h[2] = { 0.0f, 0.0f };
    for (uint32_t n = 0; n < (uint32_t)P[XS_NH]; ++n)
        for (int k = 0; k < 2; ++k) h[k] = FFMA(P[XS_TAU], FSUB(I[k], h[k]), h[k]);
    float E = FMUL(h[0], h[1]);
    float A2p = FFMA(E, -P[XS_GAM], P[XS_AP]);                        /* pointing node */
    float lin1 = FMUL(FSUB(h[c], h[1 - c]), FMUL(2.0f, P[XS_LAM]));  /* linear node 1: slope 2 lambda */
    float A1p = FMUL(lin1, 0.5f);                                   /* linear node 2: slope 1/2 */
    float nsd = FMUL(P[XS_SIG], FSQRT(P[XS_DT]));
    float xp = 0.0f, xc = 0.0f;
    int hp = 0, hc = 0; uint32_t sp = 0, sc = 0;
    for (uint32_t n = 1; n <= (uint32_t)P[XS_ND]; ++n) {
        float g[2];
        od_normal_acc(seed, unit, 2ull * (n - 1), 2, g);
        xp = FFMA(nsd, g[1], FFMA(P[XS_DT], A2p, xp));
        xc = FFMA(nsd, g[0], FFMA(P[XS_DT], A1p, xc));
        if (!hp) { if (xp >= P[XS_Z]) { hp = 1; sp = n; } else if (xp <= -P[XS_Z]) { hp = 2; sp = n; } }
        if (!hc) { if (xc >= P[XS_Z]) { hc = 1; sc = n; } else if (xc <= -P[XS_Z]) { hc = 2; sc = n; } }
    }
    hit[0] = hc; hit[1] = hp; step[0] = sc; step[1] = sp;
}

float od_ext_stroop_value(int variant, const float P[13], const float w[2], float u_c, float u_s,
                          uint32_t n_trials, uint64_t n_both, uint64_t n_undecided, uint64_t rt_sum) {
    double T = (double)n_trials, N = (double)(uint32_t)P[XS_ND];
    double v;
    if (variant == 0) {
        v = (double)P[XS_R] * (double)n_both / T;
    } else {
        uint64_t n_fail = (uint64_t)n_trials - n_both;
        v = (double)P[XS_R] * (double)((uint64_t)n_trials - n_fail) / T;
    }
    v = v - (double)P[XS_CRT] * (double)P[XS_DT] * ((double)rt_sum + (double)n_undecided * N) / T;
    v = v - ((double)w[0] * (double)u_c + (double)w[1] * (double)u_s);
    return (float)v;
}

int od_ext_stroop_eval_range(int variant, const uint32_t n_levels[2], const float* levels, const float w[2],
                             const float P[13], uint64_t begin, uint64_t end, uint32_t n_trials,
                             uint32_t trial_begin, uint32_t trial_end, uint64_t seed, uint64_t* counts, float* net) {
    if (!n_levels || !levels || !w || !P || n_trials == 0 || end < begin ||
        trial_end < trial_begin || trial_end > n_trials) return -1;
    uint64_t N = (uint64_t)n_levels[0] * n_levels[1];
    if (N == 0 || end > N) return -1;
    for (uint64_t i = begin; i < end; ++i) {
        uint32_t k[2];
        od_decode(i, 2, n_levels, k);
        float uc = levels[k[0]], us = levels[n_levels[0] + k[1]];
        uint64_t* c = counts + 3 * (i - begin);
        c[0] = c[1] = c[2] = 0;
        for (uint32_t j = trial_begin; j < trial_end; ++j) {
            int hit[2]; uint32_t st[2];
            if (variant == 0) od_ext_stroop_trial_a(P, uc, us, seed, i * (uint64_t)n_trials + j, j, hit, st);
            else od_ext_stroop_trial_b(P, uc, us, seed, i * (uint64_t)n_trials + j, j, hit, st);
            if (hit[0] == 0 || hit[1] == 0) { c[1] += 1; continue; }
            if (hit[0] == 1 && hit[1] == 1) c[0] += 1;
            c[2] += st[0] > st[1] ? st[0] : st[1];
        }
        if (net) net[i - begin] = od_ext_stroop_value(variant, P, w, uc, us, n_trials, c[0], c[1], c[2]);
    }
    return 0;
}

int od_ext_stroop_eval(int variant, const uint32_t n_levels[2], const float* levels, const float w[2],
                       const float P[13], uint64_t begin, uint64_t end, uint32_t n_trials, uint64_t seed,
                       uint64_t* counts, float* net) {
    return od_ext_stroop_eval_range(variant, n_levels, levels, w, P, begin, end, n_trials, 0, n_trials, seed,
                                    counts, net);
}
