"""Pins for the Extended Stroop A/B oracle (spec/MODELS.md §10)."""
import math

import numpy as np

import workloads as W


def test_versions_a_and_b_are_bit_identical(orc):
    """'conceptually different but computationally equivalent'."""
    c = W.ext_stroop_small()
    ca, na = orc.ext_stroop_eval(0, c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials, c.seed, threads=8)
    cb, nb = orc.ext_stroop_eval(1, c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials, c.seed, threads=8)
    assert np.array_equal(ca, cb)
    assert np.array_equal(na.view(np.uint32), nb.view(np.uint32))
    # and each trial individually
    for j in range(60):
        assert orc.ext_stroop_trial(0, c.params, 0.7, 0.3, 5, 1000 + j, j) == \
            orc.ext_stroop_trial(1, c.params, 0.7, 0.3, 5, 1000 + j, j)


def _zero_noise():
    P = W.EXT_STROOP_PARAMS.copy()
    P[7] = 0.0
    return P


def test_zero_noise_decisions_follow_drift_signs_and_conflict_slows_pointing(orc):
    P = _zero_noise()
    # no word suppression: the stronger word wins the incongruent colour decision
    (h_cong, st_cong) = orc.ext_stroop_trial(0, P, 1.0, 0.0, 1, 7, 0)      # congruent
    (h_inc, st_inc) = orc.ext_stroop_trial(0, P, 1.0, 0.0, 1, 7, 1)        # incongruent
    (h_neu, st_neu) = orc.ext_stroop_trial(0, P, 1.0, 0.0, 1, 7, 2)        # neutral
    assert h_cong == (1, 1) and h_neu == (1, 1)
    assert h_inc[0] == 2                      # colour DDM hits the lower (wrong) bound
    # conflict energy E = h0 h1 > 0 only with both pathways active -> pointing is slower
    (_, s_c) = orc.ext_stroop_trial(0, P, 1.0, 0.5, 1, 7, 0)
    (h_i, s_i) = orc.ext_stroop_trial(0, P, 1.0, 0.5, 1, 7, 1)
    (_, s_n) = orc.ext_stroop_trial(0, P, 1.0, 0.5, 1, 7, 2)
    assert h_i[1] == 1 and s_i[1] > s_c[1]
    assert s_c[1] == s_n[1]                   # E = 0 in both: same pointing drift


def test_zero_noise_first_passage_is_binary32_accumulation(orc):
    """Pointing DDM with zero noise: x_n = fma(dt, A2, x_{n-1}); first n with x >= z."""
    P = _zero_noise()
    (_, (_, n2)) = orc.ext_stroop_trial(0, P, 1.0, 0.0, 1, 3, 0)   # congruent: E = 0, A2 = a_p
    a2, dt, z = np.float32(P[5]), np.float32(P[8]), np.float32(P[9])
    x = np.float32(0)
    want = None
    for n in range(1, 1000):
        x = np.float32(np.float64(dt) * np.float64(a2) + np.float64(x))   # exact product, one rounding
        if x >= z:
            want = n
            break
    assert n2 == want


def test_counts_conserve(orc):
    c = W.ext_stroop_small()
    counts, _ = orc.ext_stroop_eval(0, c.n_levels, c.levels, c.w, c.params, 5, 17, c.n_trials, c.seed)
    assert (counts[:, 0] + counts[:, 1] <= c.n_trials).all()
    assert (counts[:, 2] <= (c.n_trials - counts[:, 1]) * int(c.params[10])).all()


def test_both_ddms_follow_the_closed_form_error_rates(orc):
    """Closed-form pin for Extended Stroop (spec/MODELS.md §10): the
    front-end is a geometric series, h_k = I_k (1 - (1 - tau)^N_h) in real
    arithmetic, so the two DDM drifts are A1 = (h_c - h_w) lambda and
    A2 = a_p - gamma h_c h_w; the DDMs draw disjoint normals, so
    P(both hit the upper bound) = (1 - ER(A1)) (1 - ER(A2)) with the DDM error
    rate ER(A) = 1 / (1 + exp(2 A z' / sigma^2)), z' = z + 0.5826 sigma sqrt(dt)
    (Siegmund, as in the DDM pin), over a horizon long enough that no trial is
    undecided.  Congruent and incongruent stimuli; a flipped conflict sign or
    swapped colour/word pathways is rejected."""
    P = W.EXT_STROOP_PARAMS.copy()
    dt = 0.002
    P[8], P[10] = dt, 2500
    g_c, g_w, tau, Nh, lam, a_p, gam, sig, _, z = (float(v) for v in P[:10])
    u_c, u_s = 1.0, 0.5
    ic, iw = g_c * u_c, g_w * (1 - u_s)
    f = 1 - (1 - tau) ** Nh
    zp = z + 0.5826 * sig * math.sqrt(dt)

    def er(A):
        return 1 / (1 + math.exp(2 * A * zp / sig ** 2))

    n = 4000
    for trial, (Ic, Iw) in ((0, (ic + iw, 0.0)), (1, (ic, iw))):     # congruent, incongruent (colour 0)
        hc, hw = Ic * f, Iw * f
        A1, A2 = (hc - hw) * lam, a_p - gam * hc * hw
        both = und = 0
        for u in range(n):
            (h1, h2), _ = orc.ext_stroop_trial(0, P, u_c, u_s, 9, u, trial)
            both += (h1 == 1 and h2 == 1)
            und += (h1 == 0 or h2 == 0)
        assert und == 0
        p = both / n
        pred = (1 - er(A1)) * (1 - er(A2))
        se = math.sqrt(pred * (1 - pred) / n)
        assert abs(p - pred) <= 4 * se + 0.005, (trial, p, pred, se)
        if trial == 1:
            wrong_sign = (1 - er(A1)) * (1 - er(a_p + gam * hc * hw))
            swapped = (1 - er(-A1)) * (1 - er(A2))
            assert abs(p - wrong_sign) > 4 * se and abs(p - swapped) > 4 * se


def test_ext_stroop_trial_subranges_add_up(orc):
    """Counts over trial sub-ranges sum to the whole-range counts (exact integers;
    the GPU's trial-range launches are checked against these)."""
    c = W.ext_stroop_small()
    full, net = orc.ext_stroop_eval(1, c.n_levels, c.levels, c.w, c.params, 3, 17, c.n_trials, c.seed)
    a, na = orc.ext_stroop_eval(1, c.n_levels, c.levels, c.w, c.params, 3, 17, c.n_trials, c.seed, trial_end=77)
    b, _ = orc.ext_stroop_eval(1, c.n_levels, c.levels, c.w, c.params, 3, 17, c.n_trials, c.seed, trial_begin=77)
    assert np.array_equal(full, a + b) and na is None and net is not None
