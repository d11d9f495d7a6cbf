"""Pins for the DDM, LCI and Stroop-LCA oracle (spec/MODELS.md §4-6).

DDM: deterministic first passage in binary32, the closed-form error rate and
decision time of the drift-diffusion model (Bogacz et al. 2006, the DDM the
paper cites at P:466) with the discrete-monitoring (Siegmund) correction, and
the exact Gaussian law of the Euler endpoint.  LCI: the Fig. 3 clone relation
(P:477).  Stroop: zero-noise determinism, the Stroop effect, conservation.
"""
import math

import numpy as np
import pytest
from scipy import stats

import workloads as W


def ddm(orc, **kw):
    c = W.DDMConfig(**kw)
    return c, orc.ddm_params(c.drift, c.noise, c.threshold, c.x0, c.dt, c.n_steps,
                             c.rt_bin_steps, c.n_x_bins, c.x_lo, c.x_hi)


@pytest.mark.parametrize("drift,dt,want", [(1.0, 0.01, 101), (1.0, 0.005, 201), (2.0, 0.01, 51),
                                           (-1.0, 0.01, 101)])
def test_ddm_zero_noise_first_passage_binary32(orc, drift, dt, want):
    """x_n = fma(dt, A, x) accumulated in binary32 crosses z = 1 at step 101 for
    A dt = 0.01 (100 in real arithmetic): the oracle mirrors binary32 exactly."""
    # reference: the same recurrence evaluated by numpy binary32 (dt*A is exact here)
    x = np.float32(0)
    n_ref = None
    for n in range(1, 2000):
        x = np.float32(x + np.float32(np.float32(dt) * np.float32(drift)))
        if abs(x) >= 1:
            n_ref = n
            break
    assert n_ref == want
    c, p = ddm(orc, drift=drift, noise=0.0, dt=dt, n_steps=1000)
    ch, st, _ = orc.ddm_trial(p, 1, 0)
    assert st == want and ch == (0 if drift > 0 else 1)


def _siegmund(A, s, z, dt):
    zp = z + 0.5826 * s * math.sqrt(dt)
    er = 1.0 / (1.0 + math.exp(2 * A * zp / s ** 2))
    rt = zp / A * math.tanh(A * zp / s ** 2)
    return er, rt


def test_ddm_closed_form_error_rate_and_decision_time(orc):
    c, p = ddm(orc)  # cfg2 parameters: A = sigma = z = 1, dt = 0.01, N = 1000
    n = 200_000
    rt_hist, rt_sum, x_hist = orc.ddm_batch(p, 11, 0, n, threads=8)
    nb = c.n_rt_bins
    up, lo, und = int(rt_hist[:nb].sum()), int(rt_hist[nb:2 * nb].sum()), int(rt_hist[2 * nb])
    assert up + lo + und == n and int(x_hist.sum()) == n
    er_mc = lo / (up + lo)
    rt_mc = (int(rt_sum[0]) + int(rt_sum[1])) / (up + lo) * c.dt
    er_cf, rt_cf = _siegmund(1.0, 1.0, 1.0, c.dt)
    se_er = math.sqrt(er_cf * (1 - er_cf) / n)
    assert abs(er_mc - er_cf) <= 4 * se_er + 0.005 * er_cf
    assert abs(rt_mc - rt_cf) <= 0.01 * rt_cf
    # the uncorrected continuous-time law is clearly rejected (the pin has power)
    er_raw = 1 / (1 + math.exp(2.0))
    assert abs(er_mc - er_raw) > 8 * se_er


def test_ddm_endpoint_is_exact_gaussian(orc):
    """Euler with Gaussian increments: x_N ~ N(x0 + A N dt, sigma^2 N dt) exactly."""
    c, p = ddm(orc, n_steps=200, drift=0.5, noise=1.3)
    xs = np.array([orc.ddm_trial(p, 5, t)[2] for t in range(4000)], np.float64)
    mu, sd = 0.5 * 200 * c.dt, 1.3 * math.sqrt(200 * c.dt)
    assert stats.kstest((xs - mu) / sd, "norm").pvalue > 1e-3


def test_ddm_histograms_conserve_and_add_over_shards(orc):
    c, p = ddm(orc, n_steps=300)
    full = orc.ddm_batch(p, 3, 0, 3000)
    a = orc.ddm_batch(p, 3, 0, 1234)
    b = orc.ddm_batch(p, 3, 1234, 3000)
    for f, x, y in zip(full, a, b):
        assert np.array_equal(f, x + y)
    assert int(full[0].sum()) == 3000 and int(full[2].sum()) == 3000
    # rt_sum is consistent with per-trial steps
    s = [0, 0]
    for t in range(3000):
        ch, st, _ = orc.ddm_trial(p, 3, t)
        if ch < 2:
            s[ch] += st
    assert [int(v) for v in full[1]] == s


def test_lci_is_a_bit_exact_clone_of_ddm(orc):
    """Fig. 3: rate_LCI = 0, offset = 0, noise N(0,1) vs rate_DDI = 1,
    noise 1 perform identical computation -> identical trajectories."""
    c, p = ddm(orc, drift=0.7, noise=1.0, threshold=1.0, n_steps=400)
    for t in range(300):
        d = orc.ddm_trial(p, 9, t)
        l = orc.lci_trial(0.7, 0.0, 0.0, 1.0, c.dt, 1.0, 400, 9, t)
        assert d[0] == l[0] and d[1] == l[1]
        assert np.float32(d[2]).view(np.uint32) == np.float32(l[2]).view(np.uint32)
    # and a leak breaks the equivalence
    diff = sum(orc.ddm_trial(p, 9, t)[2] != orc.lci_trial(0.7, 0.3, 0.0, 1.0, c.dt, 1.0, 400, 9, t)[2]
               for t in range(20))
    assert diff == 20


def test_stroop_zero_noise_deterministic_and_stroop_effect(orc):
    P = W.STROOP_PARAMS.copy()
    P[5] = 0.0  # noise off
    rts = {}
    for j in range(12):
        r, st = orc.stroop_trial(P, 1.0, 0.5, 1, 1000 + j, j)
        kind, colour = j % 3, (j // 3) % 2
        rts.setdefault(kind, set()).add(st)
        assert r == colour          # word at half strength (0.75 < 1.0) loses
        # without suppression the stronger word wins the incongruent trial: an error
        r0, _ = orc.stroop_trial(P, 1.0, 0.0, 1, 1000 + j, j)
        assert (r0 == colour) == (kind != 1)
    # deterministic: one RT per stimulus kind regardless of unit id / colour
    assert all(len(v) == 1 for v in rts.values())
    cong, incong, neut = rts[0].pop(), rts[1].pop(), rts[2].pop()
    assert cong < neut < incong, (cong, neut, incong)  # Stroop interference


def test_stroop_counts_conserve_and_add(orc):
    c = W.stroop_small()
    counts, net = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, 10, 20, c.n_trials, c.seed)
    a, _ = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, 10, 20, c.n_trials, c.seed, 0, 100)
    b, _ = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, 10, 20, c.n_trials, c.seed, 100, 300)
    assert np.array_equal(counts, a + b)
    assert (counts[:, 0] + counts[:, 1] <= c.n_trials).all()
    # rt_sum bounded by decided trials x N
    assert (counts[:, 2] <= (c.n_trials - counts[:, 1]) * c.n_steps).all()


def test_stroop_value_is_correctly_rounded_binary64_formula(orc):
    from fractions import Fraction as F
    P, w = W.STROOP_PARAMS, W.STROOP_W
    for nc, nu, rs in [(0, 0, 0), (150, 3, 9000), (299, 0, 12345)]:
        v = orc.stroop_value(P, w, 0.5, 0.25, 300, nc, nu, rs)
        exact = (F(float(P[8])) * nc / 300 - F(float(P[9])) * F(float(P[6])) * (rs + nu * 200) / 300
                 - (F(float(w[0])) * F(1, 2) + F(float(w[1])) * F(1, 4)))
        assert abs(F(float(v)) - exact) <= abs(exact) * F(1, 2 ** 23) + F(1, 2 ** 60)


def test_stroop_lca_unit_is_reflected_brownian_motion(orc):
    """Closed-form pin for the noisy, rectified LCA unit (spec/MODELS.md §6).

    With tau = 1 (pathway input reaches h in one step), no leak, no inhibition,
    and the competing unit held at 0 by a strongly negative word input
    (incongruent trial, g_w = -50), the colour unit is an Euler walk with drift
    mu = g_c u_c and noise sigma, projected onto x >= 0 and absorbed at theta:
    reflected Brownian motion with drift, whose mean first-passage time from 0 is
        E[T] = theta/mu - sigma^2/(2 mu^2) (1 - exp(-2 mu theta / sigma^2)).
    Discrete monitoring moves both barriers out by beta sigma sqrt(dt),
    beta = 0.5826 (Siegmund's correction at the absorbing barrier, as in the
    DDM pin; the same constant at the projected reflecting barrier), i.e.
    theta_eff = theta + 2 beta sigma sqrt(dt).  Without the rectification the
    mean would be theta_eff/mu (~0.26 s here) and without the discretisation
    shift 0.142 s: both are rejected by > 8 SE."""
    P = W.STROOP_PARAMS.copy()
    mu, sig, th, dt, N = 2.0, 1.0, 0.5, 5e-4, 3000
    P[0], P[1], P[2], P[3], P[4], P[5], P[6], P[7], P[10] = mu, -50.0, 1.0, 0.0, 0.0, sig, dt, th, N
    n = 8000
    resp, st = np.array([orc.stroop_trial(P, 1.0, 0.0, 5, u, 1) for u in range(n)]).T
    assert np.all(resp == 0)                     # the colour unit always answers
    T = st.astype(np.float64) * dt
    se = T.std() / math.sqrt(n)

    def ET(theta):
        return theta / mu - sig ** 2 / (2 * mu ** 2) * (1 - math.exp(-2 * mu * theta / sig ** 2))

    th_eff = th + 2 * 0.5826 * sig * math.sqrt(dt)
    assert abs(T.mean() - ET(th_eff)) <= 4 * se + 0.01 * ET(th_eff), (T.mean(), ET(th_eff), se)
    assert abs(T.mean() - th_eff / mu) > 50 * se          # power: rectification matters
    assert abs(T.mean() - ET(th)) > 8 * se                # power: the discretisation shift matters


def _golden(name):
    import os
    return open(os.path.join(os.path.dirname(__file__), "golden", name)).read().splitlines()


def test_golden_ddm_and_stroop(orc):
    """Regression fixtures written by tests/golden/make_golden.py (oracle only)."""
    d = W.DDMConfig(n_steps=250, n_trials=2000)
    p = orc.ddm_params(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                       d.x_lo, d.x_hi)
    got = orc.ddm_batch(p, d.seed, 0, d.n_trials)
    rows = {ln.split()[0]: [int(v) for v in ln.split()[1:]] for ln in _golden("ddm_small_hist.txt")
            if not ln.startswith("#")}
    for name, arr in zip(("rt_hist", "rt_sum", "x_hist"), got):
        assert [int(v) for v in arr] == rows[name], name
    lev = np.linspace(0, 1, 4).astype(np.float32)
    counts, net = orc.stroop_eval((4, 4), np.concatenate([lev, lev]), W.STROOP_W, W.STROOP_PARAMS, 0, 16, 60, W.SEED)
    for ln in _golden("stroop_small_counts.txt"):
        if ln.startswith("#"):
            continue
        i, nc, nu, rs, v = ln.split()
        i = int(i)
        assert [int(counts[i, 0]), int(counts[i, 1]), int(counts[i, 2])] == [int(nc), int(nu), int(rs)]
        assert float(net[i]) == float.fromhex(v)


def test_lci_with_leak_endpoint_is_the_ar1_law(orc):
    """LCI with a leak is Euler-discretised Ornstein-Uhlenbeck:
    x_{n+1} = (1 - lam dt) x_n + I dt + sigma sqrt(dt) g — an AR(1) whose
    endpoint from x_0 = 0 is exactly Gaussian with
        mean = I dt (1 - r^N) / (1 - r),  var = sigma^2 dt (1 - r^{2N}) / (1 - r^2),  r = 1 - lam dt.
    KS test of 4000 endpoints; a leak applied with the wrong sign is rejected."""
    I, lam, sig, dt, N = 0.8, 2.0, 0.7, 0.01, 300
    xs = np.array([orc.lci_trial(I, lam, 0.0, sig, dt, 1e9, N, 17, u)[2] for u in range(4000)], np.float64)
    r = 1 - lam * dt
    mean = I * dt * (1 - r ** N) / (1 - r)
    sd = math.sqrt(sig ** 2 * dt * (1 - r ** (2 * N)) / (1 - r ** 2))
    assert stats.kstest((xs - mean) / sd, "norm").pvalue > 1e-3
    r_bad = 1 + lam * dt
    mean_bad = I * dt * (1 - r_bad ** N) / (1 - r_bad)
    assert abs(xs.mean() - mean_bad) > 50 * xs.std() / math.sqrt(len(xs))


def test_stroop_energy_trace_closed_forms(orc):
    """Decision energy over time (spec/MODELS.md §6b): with zero noise, no
    leak, no inhibition and tau = 1, unit k integrates x_k(n) = n dt I_k, so an
    incongruent trial (both units driven, colour 0: I_0 = g_c u_c, I_1 = g_w (1 - u_s))
    has energy x0 x1 = n^2 dt^2 I_0 I_1 (binary32 accumulation within 1e-5), a
    congruent trial (only the colour unit driven) has energy 0 at every step, and
    sums over trial ranges add."""
    P = W.STROOP_PARAMS.copy()
    P[2], P[3], P[4], P[5], P[6], P[7], P[10] = 1.0, 0.0, 0.0, 0.0, 0.01, 1e9, 150
    u_c, u_s = 0.8, 0.25
    I0, I1 = P[0] * u_c, P[1] * (1 - u_s)
    e = orc.stroop_energy(P, u_c, u_s, 3, 7, 30, 1, 2)          # trial 1: incongruent, colour 0
    n = np.arange(1, 151, dtype=np.float64)
    want = n ** 2 * 0.01 ** 2 * I0 * I1 * 2 ** 24
    assert np.all(np.abs(e - want) <= 1e-5 * want + 1)
    assert not np.any(orc.stroop_energy(P, u_c, u_s, 3, 7, 30, 0, 1))   # trial 0: congruent -> 0
    Q = W.STROOP_PARAMS.copy()
    whole = orc.stroop_energy(Q, 0.6, 0.4, 11, 2, 90, 0, 90)
    parts = orc.stroop_energy(Q, 0.6, 0.4, 11, 2, 90, 0, 37) + orc.stroop_energy(Q, 0.6, 0.4, 11, 2, 90, 37, 90)
    assert np.array_equal(whole, parts) and whole[-1] > 0


def test_lci_batch_is_the_ddm_batch_at_zero_leak(orc):
    """Fig. 3 clone relation at batch level: LCI histograms with leak = 0,
    offset = 0 equal the DDM's bit for bit (same stream-2 normals); a leak changes them."""
    d = W.DDMConfig(n_steps=240, n_trials=600, x0=0.05)
    p = orc.ddm_params(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                       d.x_lo, d.x_hi)
    ddm = orc.ddm_batch(p, 13, 0, 600)
    lci = orc.ddm_batch(p, 13, 0, 600, lci=(0.0, 0.0))
    assert all(np.array_equal(a, b) for a, b in zip(ddm, lci))
    leaky = orc.ddm_batch(p, 13, 0, 600, lci=(1.5, 0.0))
    assert not np.array_equal(ddm[2], leaky[2])


def test_ddm_grid_zero_noise_passage_and_value(orc):
    """DDM control grid (spec/MODELS.md §6c): with zero noise, A = 1, dt = 0.01,
    z = 1 every trial crosses at step 101 in binary32 (not 100; the DDM pin's
    value); a negative drift gives errors at the same step; the value is the
    correctly rounded binary64 formula of the integer counts."""
    from fractions import Fraction as F
    P = W.DDMG_PARAMS.copy()
    P[0], P[1], P[2], P[3], P[6] = 0.0, 1.0, 0.0, 0.01, 300
    for u in range(5):
        assert orc.ddmg_trial(P, 1.0, 1.0, 3, u) == (1, 101)
    P[0] = -2.0                                   # A = -2 + 1 = -1
    assert orc.ddmg_trial(P, 1.0, 1.0, 3, 0) == (0, 101)
    w = W.DDMG_W
    for nc, nu, rs in [(0, 0, 0), (70, 3, 9000), (99, 0, 12345)]:
        v = orc.ddmg_value(W.DDMG_PARAMS, w, 0.5, 0.75, 100, nc, nu, rs)
        Q = W.DDMG_PARAMS
        exact = (F(float(Q[4])) * nc / 100 - F(float(Q[5])) * F(float(Q[3])) * (rs + nu * 400) / 100
                 - (F(float(w[0])) * F(1, 2) + F(float(w[1])) * F(3, 4)))
        assert abs(F(float(v)) - exact) <= abs(exact) * F(1, 2 ** 23) + F(1, 2 ** 60)


def test_ddm_grid_accuracy_and_decision_time_closed_forms(orc):
    """Per allocation the grid's DDM has drift A = A0 + g_a u0 and threshold z = u1:
    accuracy 1/(1 + exp(-2 A z'/sigma^2)) and decision time z' tanh(A z'/sigma^2)/A
    with z' = z + 0.5826 sigma sqrt(dt) (Siegmund, as the DDM pin), for three
    allocations; 2000 trials each, a horizon with no undecided trial."""
    P = W.DDMG_PARAMS.copy()
    P[6] = 3000
    sig, dt = float(P[2]), float(P[3])
    lev = np.array([0.0, 0.4, 1.0, 0.5, 1.0, 0.8], np.float32)      # u0 levels | u1 levels
    counts, _ = orc.ddmg_eval((3, 3), lev, W.DDMG_W, P, 0, 9, 2000, 17, threads=8)
    for i in (1, 5, 6):
        u0, u1 = float(lev[i // 3]), float(lev[3 + i % 3])
        A = float(np.float32(np.float32(P[1]) * np.float32(u0) + np.float32(P[0])))
        zp = u1 + 0.5826 * sig * math.sqrt(dt)
        nc, nu, rs = (int(v) for v in counts[i])
        assert nu == 0
        acc, acc_cf = nc / 2000, 1 / (1 + math.exp(-2 * A * zp / sig ** 2))
        assert abs(acc - acc_cf) <= 4 * math.sqrt(acc_cf * (1 - acc_cf) / 2000) + 0.01, (i, acc, acc_cf)
        dt_mc, dt_cf = rs / 2000 * dt, zp * math.tanh(A * zp / sig ** 2) / A
        assert abs(dt_mc - dt_cf) <= 0.05 * dt_cf, (i, dt_mc, dt_cf)


# ---------------------------------------------------------------------------
# Stroop-LCA closed forms with leak != inhibition, both nonzero, and tau < 1
# (spec/MODELS.md §6; the LCA of P:466, the Botvinick Stroop model of P:525).
#
# Pathway: h_k(n) = I_k (1 - (1 - tau)^n)  (h_k(0) = 0).
# Response layer, while neither unit is rectified:
#   x(n) = M x(n-1) + dt h(n),  M = [[1 - dt lam, -dt beta], [-dt beta, 1 - dt lam]]
# diagonalised on (1, 1) and (1, -1): s = x0 + x1 and d = x0 - x1 follow
#   s(n) = a_s s(n-1) + dt (h0 + h1)(n),  a_s = 1 - dt (lam + beta)
#   d(n) = a_d d(n-1) + dt (h0 - h1)(n),  a_d = 1 - dt (lam - beta)
# so with r = 1 - tau:  s(n) = dt (I0 + I1) G(a_s, n),  d(n) = dt (I0 - I1) G(a_d, n),
#   G(a, n) = sum_{m=1..n} a^{n-m} (1 - r^m) = (1 - a^n)/(1 - a) - r (a^n - r^n)/(a - r).
# With noise, the same linear system is an AR(1) pair: E[s], E[d] as above and
#   Var s(n) = Var d(n) = 2 nsd^2 (1 - a^{2n}) / (1 - a^2)  (a = a_s resp. a_d),
#   Cov(s, d) = 0  (the two unit noises are independent with equal variance).
# ---------------------------------------------------------------------------
_LAM, _BETA, _TAU, _DT = 0.4, 0.15, 0.3, 0.05


def _stroop_params(gc, gw, tau, lam, beta, sig, dt, theta, N):
    P = W.STROOP_PARAMS.copy()
    P[0], P[1], P[2], P[3], P[4], P[5], P[6], P[7], P[10] = gc, gw, tau, lam, beta, sig, dt, theta, N
    return P


def _G(a, r, n):
    n = np.asarray(n, np.float64)
    return (1 - a ** n) / (1 - a) - r * (a ** n - r ** n) / (a - r)


def _lca_closed_form(I0, I1, tau, lam, beta, dt, n):
    r = 1.0 - tau
    a_s, a_d = 1 - dt * (lam + beta), 1 - dt * (lam - beta)
    s = dt * (I0 + I1) * _G(a_s, r, n)
    d = dt * (I0 - I1) * _G(a_d, r, n)
    h0, h1 = I0 * (1 - r ** n), I1 * (1 - r ** n)
    return h0, h1, (s + d) / 2, (s - d) / 2


def test_stroop_lca_zero_noise_linear_recurrence_closed_form(orc):
    """Incongruent trial (colour 0, word 1), both units driven and never
    rectified: the oracle's pathway states and both response units follow the
    closed form to binary32 accumulation accuracy; the latch step is the closed
    form's first crossing.  Power: a swapped leak/inhibition, a flipped
    inhibition sign, self- instead of lateral inhibition and tau = 1 all miss
    by orders of magnitude more than the tolerance."""
    N, theta = 200, 1.0
    uc, us = 0.8, 0.3
    gc, gw = 1.0, 1.5
    P = _stroop_params(gc, gw, _TAU, _LAM, _BETA, 0.0, _DT, 1e6, N)
    I0, I1 = np.float64(np.float32(gc * uc)), np.float64(np.float32(np.float32(gw) * np.float32(1 - np.float32(us))))
    resp, st, tr = orc.stroop_trace(P, uc, us, 7, 123, 1)        # trial 1: incongruent, colour 0
    assert resp == -1 and st == 0                                 # theta out of reach
    n = np.arange(1, N + 1)
    h0, h1, x0, x1 = _lca_closed_form(I0, I1, _TAU, _LAM, _BETA, _DT, n)
    assert (x0 > 0).all() and (x1 > x0).all()                     # never rectified; word unit leads
    tol = 2e-5 * np.maximum(1.0, np.abs(x1))
    for got, want in ((tr[:, 0], h0), (tr[:, 1], h1), (tr[:, 2], x0), (tr[:, 3], x1)):
        assert np.max(np.abs(got - want)) < 2e-5, np.max(np.abs(got - want))
    # power: each plausible slip moves the trajectory far outside the tolerance
    wrong = {
        "leak<->inhibition": _lca_closed_form(I0, I1, _TAU, _BETA, _LAM, _DT, n),
        "inhibition sign": _lca_closed_form(I0, I1, _TAU, _LAM, -_BETA, _DT, n),
        "tau = 1": _lca_closed_form(I0, I1, 1.0, _LAM, _BETA, _DT, n),
    }
    for name, (_, _, y0, y1) in wrong.items():
        dev = max(np.max(np.abs(tr[:, 2] - y0)), np.max(np.abs(tr[:, 3] - y1)))
        assert dev > 1000 * tol.max(), (name, dev)
    # self-inhibition (x_k instead of x_{1-k}): both units decouple with a = 1 - dt (lam + beta)
    a = 1 - _DT * (_LAM + _BETA)
    y0 = _DT * I0 * _G(a, 1 - _TAU, n)
    assert np.max(np.abs(tr[:, 2] - y0)) > 1000 * tol.max()
    # the latch: with theta = 1 the word unit (1) crosses first, at the closed form's step
    P2 = _stroop_params(gc, gw, _TAU, _LAM, _BETA, 0.0, _DT, theta, N)
    r2, st2 = orc.stroop_trial(P2, uc, us, 7, 123, 1)
    n_cf = int(np.argmax(x1 >= theta)) + 1
    assert abs(x1[n_cf - 1] - theta) > 1e-3 and x0[n_cf - 1] < theta   # not a rounding-order tie
    assert (r2, st2) == (1, n_cf)


def test_stroop_lca_rectified_unit_closed_form(orc):
    """Congruent trial: unit 1 gets no input, so lateral inhibition drives it
    below 0 and the rectification holds it at exactly 0; unit 0 then follows
    the scalar leaky recurrence x0(n) = (1 - dt lam) x0 + dt h0(n) (no
    inhibition term, since x1 = 0) — pins the rectification and the leak on
    their own."""
    N = 150
    P = _stroop_params(1.0, 1.5, _TAU, _LAM, _BETA, 0.0, _DT, 1e6, N)
    uc, us = 0.6, 0.2
    _, _, tr = orc.stroop_trace(P, uc, us, 3, 45, 0)              # trial 0: congruent, colour 0 = word 0
    I0 = np.float64(np.float32(np.float32(0.6) + np.float32(np.float32(1.5) * np.float32(1 - np.float32(0.2)))))
    n = np.arange(1, N + 1)
    a = 1 - _DT * _LAM
    x0 = _DT * I0 * _G(a, 1 - _TAU, n)
    assert np.all(tr[:, 3] == 0.0)
    assert np.max(np.abs(tr[:, 2] - x0)) < 2e-5
    assert np.max(np.abs(tr[:, 1])) == 0.0                        # h1 = 0 exactly


def test_stroop_lca_noisy_ar1_moments(orc):
    """With noise, both units far from 0 (never rectified): the sum and
    difference coordinates are independent AR(1) processes with the closed-form
    means and variances above (Cov = 0).  A swapped leak/inhibition (a_d > 1)
    or a flipped inhibition sign (Var s and Var d exchanged) is rejected."""
    N, sig, tau = 100, 0.1, 0.9
    gc, gw, uc, us = 4.0, 5.0, 1.0, 0.0
    P = _stroop_params(gc, gw, tau, _LAM, _BETA, sig, _DT, 1e6, N)
    n_units = 4000
    X = np.empty((n_units, N, 2))
    for u in range(n_units):
        _, _, tr = orc.stroop_trace(P, uc, us, 11, u, 1)          # incongruent: I0 = gc uc, I1 = gw (1 - us)
        X[u] = tr[:, 2:4]
    assert (X > 0).all()                                          # rectification never engaged
    s, d = X[:, :, 0] + X[:, :, 1], X[:, :, 0] - X[:, :, 1]
    nsd2 = float(np.float32(sig) * np.sqrt(np.float32(_DT))) ** 2
    I0, I1 = gc * uc, gw * (1 - us)
    r = 1 - tau
    a_s, a_d = 1 - _DT * (_LAM + _BETA), 1 - _DT * (_LAM - _BETA)
    for k in (9, 39, 99):                                         # steps 10, 40, 100
        m = k + 1
        ms, md = _DT * (I0 + I1) * _G(a_s, r, m), _DT * (I0 - I1) * _G(a_d, r, m)
        vs = 2 * nsd2 * (1 - a_s ** (2 * m)) / (1 - a_s ** 2)
        vd = 2 * nsd2 * (1 - a_d ** (2 * m)) / (1 - a_d ** 2)
        assert abs(s[:, k].mean() - ms) < 4 * math.sqrt(vs / n_units)
        assert abs(d[:, k].mean() - md) < 4 * math.sqrt(vd / n_units)
        se_v = math.sqrt(2.0 / n_units)
        assert abs(s[:, k].var() / vs - 1) < 4 * se_v, (k, s[:, k].var(), vs)
        assert abs(d[:, k].var() / vd - 1) < 4 * se_v, (k, d[:, k].var(), vd)
        assert abs(np.corrcoef(s[:, k], d[:, k])[0, 1]) < 4 / math.sqrt(n_units)
    # power at step 100: flipped inhibition exchanges the two variances (ratio ~2)
    m = 100
    vs = 2 * nsd2 * (1 - a_s ** (2 * m)) / (1 - a_s ** 2)
    vd = 2 * nsd2 * (1 - a_d ** (2 * m)) / (1 - a_d ** 2)
    assert abs(s[:, 99].var() / vd - 1) > 10 * math.sqrt(2.0 / n_units)
    assert abs(d[:, 99].var() / vs - 1) > 10 * math.sqrt(2.0 / n_units)
    # swapped leak/inhibition: a_d' = 1 - dt (beta - lam) > 1, variance grows geometrically
    a_w = 1 - _DT * (_BETA - _LAM)
    vw = 2 * nsd2 * (a_w ** (2 * m) - 1) / (a_w ** 2 - 1)
    assert abs(d[:, 99].var() / vw - 1) > 10 * math.sqrt(2.0 / n_units)


def test_stroop_energy_noisy_gaussian_product_moments(orc):
    """Decision energy with noise (spec/MODELS.md §6b), in the linear
    regime of the AR(1) pin above (both units far from 0, theta out of reach):
    x0 = (s + d)/2 and x1 = (s - d)/2 are jointly Gaussian with s, d independent,
    so per step
        m_k = E[x_k],  v = Var x0 = Var x1 = (Var s + Var d)/4,  c = Cov(x0, x1) = (Var s - Var d)/4,
        E[x0 x1]   = m0 m1 + c,
        Var(x0 x1) = m0^2 v + m1^2 v + 2 m0 m1 c + v^2 + c^2   (product of bivariate normals).
    4000 single incongruent colour-0 trials (j = 1 mod 6), each its own energy
    trace; the mean and the variance of llrint(x0 x1 2^24)/2^24 at steps 1 … 100
    within 4.5 SE.  Power: a flipped inhibition sign, a swapped leak/inhibition
    and x0^2 instead of x0 x1 miss the mean; 10 % more noise misses the variance."""
    N, sig, tau = 100, 0.3, 0.9
    gc, gw, uc, us = 8.0, 10.0, 1.0, 0.0
    P = _stroop_params(gc, gw, tau, _LAM, _BETA, sig, _DT, 1e6, N)
    n = 4000
    T = 6 * n
    E = np.stack([orc.stroop_energy(P, uc, us, 11, 0, T, 1 + 6 * k, 2 + 6 * k)
                  for k in range(n)]).astype(np.float64) / 2 ** 24
    nsd2 = float(np.float32(sig) * np.sqrt(np.float32(_DT))) ** 2
    I0, I1, r = gc * uc, gw * (1 - us), 1 - tau

    def moments(m, lam=_LAM, beta=_BETA, noise2=nsd2):
        a_s, a_d = 1 - _DT * (lam + beta), 1 - _DT * (lam - beta)
        ms, md = _DT * (I0 + I1) * _G(a_s, r, m), _DT * (I0 - I1) * _G(a_d, r, m)
        vs = 2 * noise2 * (1 - a_s ** (2 * m)) / (1 - a_s ** 2)
        vd = 2 * noise2 * (1 - a_d ** (2 * m)) / (1 - a_d ** 2)
        m0, m1, v, c = (ms + md) / 2, (ms - md) / 2, (vs + vd) / 4, (vs - vd) / 4
        return m0, m1, v, c, m0 * m1 + c, m0 ** 2 * v + m1 ** 2 * v + 2 * m0 * m1 * c + v * v + c * c

    for k in (0, 4, 9, 39, 99):
        m = k + 1
        e = E[:, k]
        m0, m1, v, c, mean, var = moments(m)
        se_m = math.sqrt(var / n)
        se_v = math.sqrt(max(np.mean((e - e.mean()) ** 4) - e.var() ** 2, 0.0) / n)
        assert abs(e.mean() - mean) < 4.5 * se_m, (m, e.mean(), mean)
        assert abs(e.var() - var) < 4.5 * se_v, (m, e.var(), var)
        if m >= 40:
            # power: each plausible slip is > 10 SE away
            for wrong in (moments(m, beta=-_BETA)[4], moments(m, lam=_BETA, beta=_LAM)[4], m0 * m0 + v):
                assert abs(e.mean() - wrong) > 10 * se_m, (m, wrong)
            assert abs(e.var() - moments(m, noise2=1.21 * nsd2)[5]) > 6 * se_v
