"""The oracle's noisy accumulator models against the EXACT first-passage laws of
their Euler-discretised processes (tests/exact_law.py: Nystrom propagation of
the one-step Gaussian transition kernel, binary64, no simulation).

These pin the oracle at the bench constants themselves — the values
DESIGN.md §4 previously listed as "absolute values ... parity unpinned":
- DDM (spec/MODELS.md §4; §4.4): the whole RT histogram of cfg2;
- Stroop-LCA (spec/MODELS.md §6; P:466 LCA, P:525 Botvinick Stroop): per
  stimulus kind AND colour (the latch tests unit 0 first, so the colour unit's
  priority differs between colours; both laws are computed), the first-response
  law at the cfg4 constants, and the allocation value V;
- Extended Stroop (spec/MODELS.md §10): both DDMs' laws per kind, and
  the (n_both, n_undecided, rt_sum) counts;
- DDM control grid (spec/MODELS.md §6c): the per-allocation counts.
Each comparison is a Pearson chi-square (or z) test with a fixed seed; each
test also shows its power by rejecting mutated laws (a latch one step late, a
flipped inhibition sign, no rectification, tau = 1, a doubled leak, noise,
drift and threshold off by a few percent)."""
import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import exact_law as X
import workloads as W

P_OK = 1e-3          # a correct law: the fixed-seed chi-square p-value stays above this
P_REJECT = 1e-12     # a mutated law: its p-value must fall below this


# --------------------------------------------------------------- the law itself
def test_exact_laws_conserve_mass_and_converge():
    a = X.ddm_first_passage(1.0, 1.0, 1.0, 0.0, 0.01, 1000, nodes=300)
    b = X.ddm_first_passage(1.0, 1.0, 1.0, 0.0, 0.01, 1000, nodes=500)
    assert abs(a[0].sum() + a[1].sum() + a[2] - 1.0) < 1e-10
    assert np.abs(a[0] - b[0]).max() < 1e-12 and np.abs(a[1] - b[1]).max() < 1e-12
    P = W.STROOP_PARAMS
    gc, gw, tau, lam, beta, sig, dt, th = (float(v) for v in P[:8])
    c = X.lca2_first_passage(1.0, 1.5, tau, lam, beta, sig, dt, th, 200, nodes=36)
    d = X.lca2_first_passage(1.0, 1.5, tau, lam, beta, sig, dt, th, 200, nodes=64)
    assert abs(c[0].sum() + c[1].sum() + c[2] - 1.0) < 1e-10
    assert np.abs(c[0] - d[0]).max() < 1e-9 and np.abs(c[1] - d[1]).max() < 1e-9
    # no barrier within reach: everything stays undecided
    e = X.ddm_first_passage(0.0, 1.0, 50.0, 0.0, 0.01, 100, nodes=200)
    assert e[2] > 1 - 1e-12


def test_lca_law_matches_a_direct_simulation_with_library_normals():
    """The Nystrom law against the spec's equations simulated in binary64 with
    numpy's normal generator (nothing from the oracle): P(first response = unit
    0) and its mean step, incongruent inputs at the cfg4 constants."""
    P = W.STROOP_PARAMS
    gc, gw, tau, lam, beta, sig, dt, th = (float(v) for v in P[:8])
    N = int(P[10])
    I = np.array([1.0, 1.5])
    p0, p1, pu = X.lca2_first_passage(I[0], I[1], tau, lam, beta, sig, dt, th, N, nodes=48)
    rng = np.random.default_rng(20211029)
    n = 200_000
    x = np.zeros((n, 2))
    h = np.zeros(2)
    resp = np.full(n, -1)
    st = np.zeros(n)
    nsd = sig * math.sqrt(dt)
    for s in range(1, N + 1):
        h = h + tau * (I - h)
        q = np.stack([h[0] - lam * x[:, 0] - beta * x[:, 1], h[1] - lam * x[:, 1] - beta * x[:, 0]], 1)
        x = np.maximum(x + dt * q + nsd * rng.standard_normal((n, 2)), 0.0)
        und = resp < 0
        r0 = und & (x[:, 0] >= th)
        r1 = und & ~r0 & (x[:, 1] >= th)
        resp[r0], st[r0], resp[r1], st[r1] = 0, s, 1, s
    q = p0.sum()
    assert abs((resp == 0).mean() - q) < 4.5 * math.sqrt(q * (1 - q) / n)
    steps = np.arange(1, N + 1)
    m = (steps * p0).sum() / q
    v = (steps ** 2 * p0).sum() / q - m * m
    assert abs(st[resp == 0].mean() - m) < 4.5 * math.sqrt(v / (resp == 0).sum())


# --------------------------------------------------------------- DDM (cfg2)
def _ddm_p(orc, c):
    return orc.ddm_params(c.drift, c.noise, c.threshold, c.x0, c.dt, c.n_steps, c.rt_bin_steps, c.n_x_bins,
                          c.x_lo, c.x_hi)


def test_ddm_cfg2_rt_histogram_is_the_exact_discrete_law(orc):
    """All 201 cells of the cfg2 RT histogram (upper / lower first passage in
    10-step bins, undecided) from 2e5 oracle trials against the exact law of
    the Euler walk; a latch one step late, 5 % more noise or drift and a 2 %
    higher threshold are each rejected."""
    c = W.DDMConfig()
    rt, _, _ = orc.ddm_batch(_ddm_p(orc, c), 11, 0, 200_000, threads=16)
    law = X.ddm_first_passage(c.drift, c.noise, c.threshold, c.x0, c.dt, c.n_steps)
    stat, dof, p = X.chi2_pvalue(rt, X.binned(*law, c.rt_bin_steps))
    print(f"ddm cfg2: chi2 {stat:.1f} / {dof} dof, p = {p:.3g}")
    assert p > P_OK, (stat, dof, p)
    late = (np.concatenate([[0.0], law[0][:-1]]), np.concatenate([[0.0], law[1][:-1]]), law[2])
    assert X.chi2_pvalue(rt, X.binned(*late, c.rt_bin_steps))[2] < P_REJECT
    for drift, noise, z in [(1.05, 1.0, 1.0), (1.0, 1.05, 1.0), (1.0, 1.0, 1.02)]:
        m = X.ddm_first_passage(drift, noise, z, 0.0, c.dt, c.n_steps, nodes=300)
        assert X.chi2_pvalue(rt, X.binned(*m, c.rt_bin_steps))[2] < P_REJECT, (drift, noise, z)


# --------------------------------------------------------------- Stroop-LCA (cfg4 constants)
def _stroop_class_hist(orc, P, uc, us, i, T, kind, colour, n):
    """Oracle trials of one (kind, colour) class of allocation i (units i*T + j
    as in od_stroop_eval): per-step counts of correct / error responses."""
    N = int(P[10])
    js = [3 * m + kind for m in range(colour, 2 * n, 2)]

    def run(chunk):
        cc, ce, u = np.zeros(N), np.zeros(N), 0
        for j in chunk:
            r, st = orc.stroop_trial(P, uc, us, 42, i * T + j, j)
            if r < 0:
                u += 1
            elif r == colour:
                cc[st - 1] += 1
            else:
                ce[st - 1] += 1
        return cc, ce, u

    with ThreadPoolExecutor(8) as ex:
        parts = list(ex.map(run, [js[k::8] for k in range(8)]))
    return sum(p[0] for p in parts), sum(p[1] for p in parts), sum(p[2] for p in parts)


STROOP_ALLOCS = [(60, 30), (99, 0)]       # (u_c, u_s) level indices of cfg4's 100 x 100 grid


def test_stroop_lca_first_response_law_at_cfg4_constants(orc):
    """Per allocation, stimulus kind and colour: the binned first-response law
    (correct / error in 10-step bins, undecided) of 6000 oracle trials against
    the exact law, at the cfg4 constants (leak = inhibition = 0.2, tau = 0.1,
    sigma = 0.5, dt = 0.05, theta = 1, N = 200).  The 12 classes' chi-squares
    are summed; each mutation must be rejected by the sum."""
    from scipy.stats import chi2
    P = W.STROOP_PARAMS.copy()
    T = 100_000
    muts = {"inhibition sign": dict(inhibition=-float(P[4])), "no rectification": dict(rectify=False),
            "tau = 1": dict(tau=1.0), "leak x2": dict(leak=2 * float(P[3])), "noise x1.1": dict(noise=1.1 * float(P[5]))}
    tot = {k: [0.0, 0] for k in ["ok", *muts]}
    lev = W.stroop_cfg4().levels
    for k0, k1 in STROOP_ALLOCS:
        uc, us = float(lev[k0]), float(lev[100 + k1])
        i = k0 * 100 + k1
        for kind in range(3):
            for colour in range(2):
                cc, ce, u = _stroop_class_hist(orc, P, uc, us, i, T, kind, colour, 3000)
                obs = X.binned(cc, ce, u, 10)
                s, d, _ = X.chi2_pvalue(obs, X.binned(*X.stroop_class_law(P, uc, us, kind, colour), 10))
                tot["ok"][0] += s
                tot["ok"][1] += d
                for name, m in muts.items():
                    law = X.stroop_class_law(P, uc, us, kind, colour, **m)
                    s, d, _ = X.chi2_pvalue(obs, X.binned(*law, 10))
                    tot[name][0] += s
                    tot[name][1] += d
    p_ok = chi2.sf(*tot["ok"])
    print("stroop classes:", {k: (round(v[0], 1), v[1], float(f"{chi2.sf(*v):.3g}")) for k, v in tot.items()})
    assert p_ok > P_OK, tot["ok"]
    for name in muts:
        assert chi2.sf(*tot[name]) < P_REJECT, (name, tot[name])


def test_stroop_value_at_cfg4_constants_is_its_exact_expectation(orc):
    """od_stroop_eval's counts over T = 6e4 trials (all six classes, 1e4 each)
    against their exact expectations — n_correct, n_undecided and rt_sum within
    4.5 standard errors (stratified variance) — for the two allocations."""
    P = W.STROOP_PARAMS.copy()
    c = W.stroop_cfg4()
    T = 60_000
    for k0, k1 in STROOP_ALLOCS:
        i = k0 * 100 + k1
        counts, net = orc.stroop_eval(c.n_levels, c.levels, c.w, P, i, i + 1, T, 42, threads=1)
        uc, us = float(c.levels[k0]), float(c.levels[100 + k1])
        mean, var = X.stroop_expected_counts(P, uc, us, T)
        got = counts[0].astype(np.float64)
        z = X.zscores(got, mean, var)
        print(f"stroop value ({k0}, {k1}): counts {got}, expected {np.round(mean, 1)}, z {np.round(z, 2)}")
        assert np.all(np.abs(z[[0, 2]]) < 4.5), (k0, k1, got, mean, z)
        assert got[1] <= mean[1] + 4.5 * math.sqrt(var[1]) + 3, (got, mean)   # undecided: rare
        v = orc.stroop_value(P, c.w, uc, us, T, *(int(x) for x in counts[0]))
        assert net[0] == np.float32(v)


# --------------------------------------------------------------- Extended Stroop (§10)
def test_extended_stroop_ddms_follow_their_exact_laws(orc):
    """Per kind: each DDM's binned (upper, lower, undecided) first-passage law
    from 3000 trials of version A; and the per-allocation counts n_both,
    n_undecided, rt_sum = sum of max(n1, n2) from od_ext_stroop_eval over
    T = 6e4 trials against their exact expectations (the two DDMs are
    independent given the front-end)."""
    from scipy.stats import chi2
    P = W.EXT_STROOP_PARAMS.copy()
    Nd = int(P[10])
    uc, us = float(np.float32(0.7)), float(np.float32(0.4))
    tot = [0.0, 0]
    bad = [0.0, 0]
    for kind in range(3):
        A1, A2 = X.ext_stroop_drifts(P, uc, us, kind)
        laws = [X.ext_stroop_ddm_law(P, A1), X.ext_stroop_ddm_law(P, A2)]
        hist = [[np.zeros(Nd), np.zeros(Nd), 0] for _ in range(2)]
        for m in range(3000):
            j = 3 * m + kind
            hit, st = orc.ext_stroop_trial(0, P, uc, us, 42, 7_000_000 + j, j)
            for d in range(2):
                if hit[d] == 0:
                    hist[d][2] += 1
                else:
                    hist[d][hit[d] - 1][st[d] - 1] += 1
        for d in range(2):
            obs = X.binned(*hist[d], 5)
            s, k, _ = X.chi2_pvalue(obs, X.binned(*laws[d], 5))
            tot[0] += s
            tot[1] += k
            # power: the other DDM's law (drifts swapped between the DDMs)
            s, k, _ = X.chi2_pvalue(obs, X.binned(*laws[1 - d], 5))
            bad[0] += s
            bad[1] += k
    print(f"ext-stroop laws: chi2 {tot[0]:.1f} / {tot[1]} dof, p = {chi2.sf(*tot):.3g}; swapped p = {chi2.sf(*bad):.3g}")
    assert chi2.sf(*tot) > P_OK, tot
    assert chi2.sf(*bad) < P_REJECT, bad

    lev = np.array([0.0, uc, 0.0, us], np.float32)
    T = 60_000
    counts, _ = orc.ext_stroop_eval(0, (2, 2), lev, W.STROOP_W, P, 3, 4, T, 42, threads=1)
    mean, var = X.ext_stroop_expected_counts(P, uc, us, T)
    got = counts[0].astype(np.float64)
    z = X.zscores(got, mean, var)
    print(f"ext-stroop counts {got}, expected {np.round(mean, 1)}, z {np.round(z, 2)}")
    assert np.all(np.abs(z) < 4.5), (got, mean, z)


# --------------------------------------------------------------- DDM control grid (§6c)
def test_ddm_grid_counts_are_their_exact_expectations(orc):
    """Per allocation (attention u0 -> drift A0 + g_a u0, threshold u1) the
    counts n_correct, n_undecided, rt_sum over 2e4 trials at the grid's own
    horizon (N = 400, where some trials stay undecided) against the exact law."""
    P = W.DDMG_PARAMS.copy()
    lev = np.array([0.0, 0.5, 1.0, 0.3, 1.0, 2.0], np.float32)     # u0 levels | u1 levels
    T = 20_000
    counts, _ = orc.ddmg_eval((3, 3), lev, W.DDMG_W, P, 0, 9, T, 17, threads=9)
    swapped = []
    for i in range(9):
        u0, u1 = float(lev[i // 3]), float(lev[3 + i % 3])
        mean, var = X.ddmg_expected_counts(P, u0, u1, T)
        sd = np.sqrt(var)
        got = counts[i].astype(np.float64)
        z = X.zscores(got, mean, var)
        print(f"ddm grid alloc {i}: z {np.round(z, 2)}")
        assert np.all(np.abs(z) < 4.5), (i, got, mean, z)
        # power: the allocation decoded the other way round (u0 <-> u1 level indices)
        j = (i % 3) * 3 + i // 3
        if j != i:
            mj, _ = X.ddmg_expected_counts(P, float(lev[j // 3]), float(lev[3 + j % 3]), T)
            swapped.append(abs(got[2] - mj[2]) / sd[2])
    assert min(swapped) > 8, swapped
