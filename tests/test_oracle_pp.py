"""Pins for the predator-prey oracle (spec/MODELS.md §1-3; §2.1).

The paper prints no cost values, so the pins are mathematics the model must
satisfy: zero-noise closed forms, mixed-radix decode order, a planted optimum,
the small-noise expectation from the Jacobians of the Action node, the
binary64 re-evaluation, and the paper's evaluation counts.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import workloads as W


def f32_round(fr: Fraction) -> np.float32:
    """Correct round-to-nearest-even of an exact rational to binary32."""
    f = np.float32(float(fr))
    best = f
    for cand in (np.nextafter(f, np.float32(-np.inf)), np.nextafter(f, np.float32(np.inf))):
        dc, db = abs(Fraction(float(cand)) - fr), abs(Fraction(float(best)) - fr)
        if dc < db or (dc == db and (int(np.array([cand]).view(np.uint32)[0]) & 1) == 0):
            best = cand
    return best


def fma32(a, b, c) -> np.float32:
    return f32_round(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def run(orc, cfg, begin=0, end=None, **kw):
    end = cfg.n_alloc if end is None else end
    return orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, begin, end,
                       cfg.n_samples, cfg.seed, **kw)


@pytest.mark.parametrize("L,count", [(2, 8), (4, 64), (6, 216), (100, 1_000_000)])
def test_evaluation_counts_match_paper(orc, L, count):
    """S/M/L/XL: 2/4/6/100 levels -> 8/64/216/1,000,000 evaluations."""
    cfg = W.PPConfig("x", (L, L, L), 1)
    assert cfg.n_alloc == count
    if count <= 216:
        assert run(orc, cfg).shape == (count,)


def test_zero_noise_cost_is_control_cost(orc):
    """sigma = 0 -> o = p exactly -> every sample's action equals the true best
    move, so e is the same tiny constant e0 for every allocation (the rounding
    residual of u*, |e0| <= (4 ulp)^2 ~ 1e-13) and C = K exactly whenever
    K >= 1e-6 absorbs it."""
    cfg = W.pp_cfg1()
    cfg.params = np.array([0.0, 0.0, 0.5], np.float32)
    C = run(orc, cfg)
    for i in range(cfg.n_alloc):
        k = [i // 9, (i // 3) % 3, i % 3]
        a = [cfg.levels[3 * d + k[d]] for d in range(3)]
        w = cfg.w
        K = fma32(w[2], a[2], fma32(w[1], a[1], f32_round(Fraction(float(w[0])) * Fraction(float(a[0])))))
        if K >= 1e-6:
            assert C[i] == K, (i, C[i], K)
        else:
            assert 0 <= C[i] - K < 1e-12
    # monotone non-decreasing in every level for w >= 0, argmin at index 0
    Cg = C.reshape(3, 3, 3)
    for ax in range(3):
        assert (np.diff(Cg, axis=ax) >= 0).all()
    key, rc = orc.argmax_net(-C)
    assert rc == 0 and key & 0xFFFFFFFF == 0


def test_mixed_radix_decode_dim0_most_significant(orc):
    """levels a_k = k and w = (L^2, L, 1) make C = K = i exactly."""
    L = 100
    cfg = W.PPConfig("decode", (L, L, L), 1)
    cfg.levels = np.concatenate([np.arange(L, dtype=np.float32)] * 3)
    cfg.w = np.array([L * L, L, 1], np.float32)
    cfg.params = np.array([0.0, 0.0, 0.5], np.float32)
    assert 0 <= run(orc, cfg, 0, 1)[0] < 1e-12
    for i in (1, 99, 100, 12345, 999999):
        assert run(orc, cfg, i, i + 1)[0] == float(i)


def test_planted_optimum(orc):
    """Zero noise, negative weight on dim 0 only: unique argmin at its top level."""
    cfg = W.PPConfig("planted", (6, 6, 6), 3)
    cfg.params = np.array([0.0, 0.0, 0.5], np.float32)
    cfg.w = np.array([-0.1, 0.1, 0.1], np.float32)
    key, rc = orc.argmax_net(-run(orc, cfg))
    assert rc == 0 and key & 0xFFFFFFFF == 5 * 36


def test_all_ties_lowest_index_any_split(orc):
    cfg = W.PPConfig("ties", (4, 4, 4), 5)
    cfg.params = np.array([0.0, 0.0, 0.5], np.float32)
    cfg.w = np.zeros(3, np.float32)
    C = run(orc, cfg)
    assert (C == C[0]).all() and 0 <= C[0] < 1e-12
    for cut in (1, 17, 40, 63):
        k1, _ = orc.argmax_net(-C[:cut], 0)
        k2, _ = orc.argmax_net(-C[cut:], cut)
        assert min(k1, k2) & 0xFFFFFFFF == 0


def _unit_jac(v):
    n = np.linalg.norm(v)
    u = v / n
    return (np.eye(2) - np.outer(u, u)) / n


def test_small_noise_expectation_matches_action_jacobians(orc):
    """E||u_hat - u*||^2 ~= sum_e sigma_e^2 ||G_e||_F^2 for small noise, with
    G_e = d u_hat / d p_e from the Jacobian of unit(v), (I - u u^T)/|v| —
    an analytic derivation, independent of the oracle's code path."""
    prey, pred, player = np.array([4.0, 1.0]), np.array([-3.0, 2.0]), np.array([0.0, 0.0])
    kappa = 0.5
    v1, v2 = prey - player, pred - player
    d = v1 / np.linalg.norm(v1) - kappa * v2 / np.linalg.norm(v2)
    Jd = _unit_jac(d)
    G0 = Jd @ _unit_jac(v1)
    G1 = Jd @ (-kappa * _unit_jac(v2))
    G2 = -(G0 + G1)
    g = np.array([np.sum(G0 ** 2), np.sum(G1 ** 2), np.sum(G2 ** 2)])

    cfg = W.PPConfig("delta", (1, 1, 1), 40000)
    cfg.levels = np.array([0.0, 0.5, 1.0], np.float32)     # a = (0, .5, 1)
    cfg.params = np.array([0.004, 0.001, kappa], np.float32)
    cfg.w = np.zeros(3, np.float32)
    sig = np.array([0.004, 0.0025, 0.001])
    pred_e = float(np.sum(sig ** 2 * g))
    C = float(run(orc, cfg)[0])
    assert abs(C / pred_e - 1) < 0.03, (C, pred_e)
    # the test has power: swapping two entities' noise moves the prediction by > 10 %
    assert abs(float(np.sum(sig[[1, 0, 2]] ** 2 * g)) / pred_e - 1) > 0.1


def test_more_attention_less_error(orc):
    """Objective error falls as attention to the prey rises."""
    cfg = W.PPConfig("mono", (5, 1, 1), 4000)
    cfg.levels = np.concatenate([W.linear_levels(5), [0.5], [0.5]]).astype(np.float32)
    cfg.w = np.zeros(3, np.float32)
    C = run(orc, cfg)
    assert (np.diff(C) < 0).all(), C


def test_binary64_reevaluation_within_north_star_tolerance(orc):
    """binary32 oracle vs the same model in binary64 (libm Box-Muller): 1e-5 relative."""
    for cfg, b, e in [(W.pp_cfg1(), 0, 27), (W.pp_cfg3(), 0, 300), (W.pp_cfg3(), 654321, 654521)]:
        c32 = run(orc, cfg, b, e).astype(np.float64)
        c64 = run(orc, cfg, b, e, f64=True)
        rel = np.abs(c32 - c64) / np.abs(c64)
        assert rel.max() < 1e-5, rel.max()


def test_argmax_brute_force_cfg1(orc):
    cfg = W.pp_cfg1()
    C = run(orc, cfg)
    best = min(range(cfg.n_alloc), key=lambda i: (float(C[i]), i))
    key, rc = orc.argmax_net(-C)
    assert rc == 0 and key & 0xFFFFFFFF == best
    assert orc.key_decode(key) == (float(C[best]), best)


def test_segments_equal_full_run(orc):
    """Contiguous segments reproduce the serial run bit-exactly."""
    cfg = W.PPConfig("L", (6, 6, 6), 20)
    full = run(orc, cfg)
    for threads in (1, 2, 4, 8, 12):
        par = orc.pp_eval_threads(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs,
                                  0, cfg.n_alloc, cfg.n_samples, cfg.seed, threads=threads)
        assert np.array_equal(full.view(np.uint32), par.view(np.uint32))


def test_invocation_changes_stream(orc):
    cfg = W.pp_cfg1()
    a = run(orc, cfg, invocation=0)
    b = run(orc, cfg, invocation=1)
    assert not np.array_equal(a, b)


def test_golden_cfg1(orc):
    """Regression fixture written by tests/golden/make_golden.py (oracle only)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "pp_cfg1_costs.txt")
    want = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    C = run(orc, W.pp_cfg1())
    for i, h in want:
        assert float(C[int(i)]).hex() == h


def test_flop_count_per_sample_matches_hand_count(orc):
    """Counting build: 159 binary32 flops per PP sample (fma = 2), the figure
    DESIGN.md §6 derives by hand from spec/RNG.md + spec/MODELS.md:
    3 x (Box-Muller polar 27 (radius table cubic 7, sincos 20) + obs 5)
    + action 35 (one rsqrt_spec since R22b) + objective 28."""
    L = orc.lib(counting=True)
    assert L.od_is_counting_build() == 1
    cfg = W.pp_cfg3()

    def flops(S):
        L.od_flops_reset()
        orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, 10, S, 1, counting=True)
        return L.od_flops_read()

    assert (flops(101) - flops(100)) == 10 * 159
    per_alloc = (flops(100) - 10 * 100 * 159)
    # per call: u_star = action 35 + unit 22 = 57, plus dsig 1;
    # per allocation: 3 sigma fma (6) + K (5) + mean (2) = 13
    assert per_alloc == 58 + 10 * 13


def test_method_flop_count(orc):
    """The method count the roofline's headline fraction uses (SURVEY §8(d):
    fma = 2, add/mul = 1, a square root = 1, a divide = 1): the counting build in
    method mode scores sqrt_spec as 1 flop and rsqrt_spec as 2 (sqrt + divide)
    instead of their Newton steps.  PP: 131 per sample (159 executed: the 2 x 14
    Newton flops of the body's rsqrt_spec are implementation, not method), 13 per
    allocation, 30 per call; one sextet (6 accumulator normals): 87, no square
    root left in it since the radius became a table cubic (spec/RNG.md §3)."""
    L = orc.lib(counting=True)
    cfg = W.pp_cfg3()

    def flops(n, S):
        L.od_flops_reset()
        orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, n, S, 1, counting=True)
        return L.od_flops_read()

    try:
        L.od_flops_method(1)
        assert flops(10, 101) - flops(10, 100) == 10 * 131
        a, b = flops(10, 100) - 10 * 100 * 131, flops(20, 100) - 20 * 100 * 131
        assert (b - a) == 10 * 13 and a - 10 * 13 == 30
        z = np.zeros(6, np.float32)
        L.od_flops_reset()
        L.od_normal_acc(1, 5, 0, 1, z)
        assert L.od_flops_read() == 87
    finally:
        L.od_flops_method(0)
    L.od_flops_reset()
    L.od_normal_acc(1, 5, 0, 1, z)
    assert L.od_flops_read() == 87


def test_multi_invocation_is_the_listing1_loop(orc):
    """pp_eval_multi = one pp_eval per trial t on inputs[t % len] with invocation0 + t
    (reading Q17); distinct invocations draw distinct noise."""
    import workloads as W
    cfg = W.PPConfig("m", (3, 4, 2), 6)
    sets = W.pp_positions(3, seed=11)
    C = orc.pp_eval_multi(cfg.n_levels, cfg.levels, cfg.w, cfg.params, sets, 5, 0, cfg.n_alloc, 6, 9, invocation0=2)
    assert C.shape == (5, cfg.n_alloc)
    for t in range(5):
        want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, sets[t % 3], 0, cfg.n_alloc, 6, 9,
                           invocation=2 + t)
        assert np.array_equal(C[t].view(np.uint32), want.view(np.uint32))
    # same positions, different invocation -> different samples
    assert not np.array_equal(C[0], orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, sets[0], 0,
                                                 cfg.n_alloc, 6, 9, invocation=5))
    assert np.all(np.abs(sets) <= 10) and sets.dtype == np.float32


def test_noisy_prey_objective_matches_offset_gaussian_angle_law(orc):
    """Closed-form pin of the noisy PP path (Obs -> Action -> Objective):
    with kappa = 0 the action is the direction to the observed prey; with the
    player and predator noise-free (level 1, sigma_min = 0) and the prey at
    (r, 0) observed with std sigma (level 0), u* = (1, 0) and the objective
    |u - u*|^2 = 2 - 2 cos(Theta), Theta the angle of an offset 2-D Gaussian.
    E[cos Theta] = sqrt(pi/8) nu e^{-nu^2/4} [I0(nu^2/4) + I1(nu^2/4)], nu = r/sigma
    (cross-checked here by quadrature of the exact angle density).  64 allocations
    x 5000 samples; a variance-for-std mistake (nu halved) is rejected."""
    from scipy import integrate, special
    r, sig = 4.0, 2.0

    def ecos(nu):
        return math.sqrt(math.pi / 8) * nu * math.exp(-nu * nu / 4) * (special.i0(nu * nu / 4) + special.i1(nu * nu / 4))

    nu = r / sig

    def dens(t):
        c = math.cos(t)
        return (math.exp(-nu * nu / 2) / (2 * math.pi)
                * (1 + math.sqrt(2 * math.pi) * nu * c * math.exp(nu * nu * c * c / 2) * special.ndtr(nu * c)))

    assert abs(integrate.quad(lambda t: math.cos(t) * dens(t), -math.pi, math.pi, epsabs=1e-13)[0] - ecos(nu)) < 1e-10
    L = 64
    levels = np.array([0.0] * L + [1.0, 1.0], np.float32)
    C = orc.pp_eval((L, 1, 1), levels, np.zeros(3, np.float32), np.array([sig, 0.0, 0.0], np.float32),
                    np.array([r, 0, -3, 2, 0, 0], np.float32), 0, L, 5000, 7).astype(np.float64)
    se = C.std() / math.sqrt(L)
    want = 2 - 2 * ecos(nu)
    assert abs(C.mean() - want) <= 4 * se, (C.mean(), want, se)
    assert abs(C.mean() - (2 - 2 * ecos(r / sig ** 2))) > 20 * se


def test_noisy_predator_action_matches_angle_law_quadrature(orc):
    """Pin of the Action node's predator term under real noise (toward the
    prey, away from the predator): prey and player noise-free, the predator
    observed with std sigma.  Only the direction of the observed predator enters
    (unit(v_d)), and its angle around the true direction follows the exact
    offset-Gaussian angle density, so E[|u - u*|^2] is a 1-D integral over that
    density of |unit(u_p - kappa u(phi0 + psi)) - u*|^2 (scipy quadrature).
    The oracle's mean over 64 x 10^4 samples must match within 4 SE + 1 %;
    a flipped kappa sign (0.096 vs 0.036) is rejected."""
    from scipy import integrate, special
    sig, kap = 2.0, 0.5
    pp, pd = np.array([4.0, 0.0]), np.array([-3.0, 2.0])
    nu, phi0 = math.hypot(*pd) / sig, math.atan2(pd[1], pd[0])

    def dens(t):
        c = math.cos(t)
        return (math.exp(-nu * nu / 2) / (2 * math.pi)
                * (1 + math.sqrt(2 * math.pi) * nu * c * math.exp(nu * nu * c * c / 2) * special.ndtr(nu * c)))

    def unit(v):
        return v / math.hypot(*v)

    def expect(k):
        up = unit(pp)
        us = unit(up - k * np.array([math.cos(phi0), math.sin(phi0)]))

        def obj(psi):
            u = unit(up - k * np.array([math.cos(phi0 + psi), math.sin(phi0 + psi)]))
            return float(((u - us) ** 2).sum())
        return integrate.quad(lambda t: obj(t) * dens(t), -math.pi, math.pi, epsabs=1e-12, limit=200)[0]

    L = 64
    levels = np.array([1.0] + [0.0] * L + [1.0], np.float32)     # prey level 1, predator level 0, player level 1
    C = orc.pp_eval((1, L, 1), levels, np.zeros(3, np.float32), np.array([sig, 0.0, kap], np.float32),
                    np.array([4, 0, -3, 2, 0, 0], np.float32), 0, L, 10000, 11).astype(np.float64)
    se = C.std() / math.sqrt(L)
    want = expect(kap)
    assert abs(C.mean() - want) <= 4 * se + 0.01 * want, (C.mean(), want, se)
    assert abs(C.mean() - expect(-kap)) > 100 * se


def test_r21_fused_objective_step_is_closer_to_binary64(orc):
    """DESIGN.md reading R21, justified by accuracy rather than by the compiler:
    the objective's difference Delta = fma(d, y_d, -u*) (one rounding) is closer
    to the binary64 plain definition (od_pp_trace_f64) than the unfused
    u_hat = d*y_d, Delta = u_hat - u* (two roundings).  A second oracle build
    that differs only in that step (-DOD_UNFUSED_OBJECTIVE) is compared sample by
    sample on cfg3 inputs; tests/r21_error.py is the larger run
    (profiles/r02_r21_error.txt)."""
    import os
    import subprocess
    import tempfile
    import oracle
    so = os.path.join(tempfile.mkdtemp(), "liboracle_unfused.so")
    subprocess.check_call(["gcc", *oracle.CFLAGS, "-DOD_UNFUSED_OBJECTIVE", oracle._SRC, "-o", so, "-lm"])
    unfused = oracle._bind(so)
    cfg = W.pp_cfg3()
    idx = np.random.default_rng(7).choice(cfg.n_alloc, 600, replace=False)
    rf, ru = [], []
    for i in idx:
        args = (cfg.n_levels, cfg.levels, cfg.params, cfg.inputs, int(i), cfg.n_samples, cfg.seed)
        e64 = orc.pp_trace_f64(*args)
        rf.append(np.abs(orc.pp_trace(*args).astype(np.float64) - e64) / e64)
        ru.append(np.abs(orc.pp_trace(*args, lib_handle=unfused).astype(np.float64) - e64) / e64)
    rf, ru = np.concatenate(rf), np.concatenate(ru)
    assert not np.array_equal(rf, ru)                       # the two builds really differ
    closer, farther = np.mean(rf < ru), np.mean(rf > ru)
    assert closer > farther + 0.01, (closer, farther)
    assert np.median(rf) < np.median(ru)                    # (the mean is set by a few ill-conditioned samples)


def _objective_expectation_2d(noisy, sig, kap, P, h=0.004, span=6.0):
    """E[|unit(action(o)) - u*|^2] with entity `noisy` observed as p + sig z,
    z ~ N(0, I), by a midpoint sum over z in [-span, span]^2 (binary64; the
    integrand is bounded, the Gaussian weight beyond 6 sigma is < 1e-7)."""
    P = np.asarray(P, np.float64).reshape(3, 2)

    def unit(v):
        return v / np.linalg.norm(v, axis=-1, keepdims=True)

    def action(o0, o1, o2):
        return unit(o0 - o2) - kap * unit(o1 - o2)

    us = unit(action(P[0], P[1], P[2]))
    g = np.arange(-span + h / 2, span, h)
    zx, zy = np.meshgrid(g, g, indexing="ij")
    z = np.stack([zx.ravel(), zy.ravel()], axis=1)
    w = np.exp(-0.5 * (z ** 2).sum(1)) * h * h / (2 * math.pi)
    o = [np.broadcast_to(P[e], z.shape) for e in range(3)]
    o[noisy] = P[noisy] + sig * z
    u = unit(action(*o))
    e = ((u - us) ** 2).sum(1)
    return float((w * e).sum() / w.sum())


def test_noisy_player_objective_matches_2d_integral(orc):
    """Pin of the third Box-Muller pair of the sextet (the player's observation,
    angle packed from the low bytes of X0 and X1, spec/RNG.md §6) and of both
    Action terms at once: prey and predator noise-free, the player observed with
    std sigma, so v_p and v_d share the same noise.  The oracle's mean objective
    over 64 x 10^4 samples must match the binary64 2-D integral over the
    player's Gaussian within 4 SE + 1 %; the same noise applied to the prey or to
    the predator instead (a swapped entity in the sextet) is rejected."""
    sig, kap = 1.0, 0.5
    P = [4.0, 0.0, -3.0, 2.0, 0.0, 0.0]
    L = 64
    levels = np.array([1.0, 1.0] + [0.0] * L, np.float32)      # prey level 1, predator level 1, player level 0
    C = orc.pp_eval((1, 1, L), levels, np.zeros(3, np.float32), np.array([sig, 0.0, kap], np.float32),
                    np.array(P, np.float32), 0, L, 10000, 23).astype(np.float64)
    se = C.std() / math.sqrt(L)
    want = _objective_expectation_2d(2, sig, kap, P)
    assert abs(C.mean() - want) <= 4 * se + 0.01 * want, (C.mean(), want, se)
    for wrong in (0, 1):
        other = _objective_expectation_2d(wrong, sig, kap, P)
        assert abs(C.mean() - other) > 20 * se + 0.01 * want, (wrong, C.mean(), other)
