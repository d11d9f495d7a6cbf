"""Exact first-passage laws of the Euler-discretised accumulator models, by
Nystrom quadrature of the one-step transition kernel (test infrastructure).

This is an independent pin for the oracle's noisy accumulator models: it does
not simulate anything and shares nothing with `oracle/` (no normals, no
Philox, no binary32 arithmetic).  It propagates the probability law of the
discrete-time process the models define — the Euler update with Gaussian
increments of spec/MODELS.md §4 (DDM, §4.4), §6 (Stroop-LCA, §5)
and §10 (the two DDMs of the Extended Stroop model) — in binary64:

    mu_{n+1}(dy) = integral K(dy | x) mu_n(dx)    over the not-yet-absorbed states,

with the absorbed mass of each step recorded as that step's first-passage
probability.  K is Gaussian (mean = the Euler drift step, sd = sigma sqrt(dt)),
so every absorption probability is a normal tail (`scipy.special.ndtr`) and
the continuous part of mu_n is carried as its density at Gauss-Legendre nodes;
the density of a discrete-time walk is analytic on the closed interval, so
the quadrature converges spectrally (the tests check two node counts agree).
The Stroop-LCA unit is rectified (x = max(., 0)), so its law also has an atom
at 0 per coordinate, carried exactly.

The oracle simulates the same processes with Box-Muller normals in binary32;
its Monte Carlo histograms must agree with these laws within sampling error
(the test's chi-square / z bounds) — a dropped term, a wrong sign, a swapped
index, a latch one step late or a wrong noise scale all move the law by many
standard errors (each test also checks that a mutated law is rejected).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import ndtr


def _gl(n: int, lo: float, hi: float):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (hi - lo) * x + 0.5 * (hi + lo), 0.5 * (hi - lo) * w


def _phi(u):
    return np.exp(-0.5 * u * u) / math.sqrt(2.0 * math.pi)


def ddm_first_passage(drift: float, noise: float, z: float, x0: float, dt: float, n_steps: int,
                      nodes: int = 400):
    """First passage of x_n = x_{n-1} + dt A + sigma sqrt(dt) g_n, x_0 = x0,
    through +z (upper, tested first) or -z (spec/MODELS.md §4: latch the first
    x >= z or x <= -z).  Returns (p_up[n_steps], p_lo[n_steps], p_undecided):
    p_up[n-1] = P(first passage at step n through the upper boundary)."""
    s = noise * math.sqrt(dt)
    step = dt * drift
    y, w = _gl(nodes, -z, z)
    p_up = np.zeros(n_steps)
    p_lo = np.zeros(n_steps)
    if s == 0.0:
        raise ValueError("noise must be positive (use the zero-noise pins)")
    # step 1 from the point mass at x0
    m = x0 + step
    p_up[0] = ndtr((m - z) / s)
    p_lo[0] = ndtr((-z - m) / s)
    dens = _phi((y - m) / s) / s                         # density of the survivors at the nodes
    # kernel K[i, j] = density at node j from node i, times the source weight
    M = (y + step)[:, None]
    K = _phi((y[None, :] - M) / s) / s
    up = ndtr((M[:, 0] - z) / s)
    lo = ndtr((-z - M[:, 0]) / s)
    for n in range(1, n_steps):
        mass = w * dens
        p_up[n] = mass @ up
        p_lo[n] = mass @ lo
        dens = mass @ K
    p_und = float(w @ dens)
    return p_up, p_lo, p_und


def lca2_first_passage(I0: float, I1: float, tau: float, leak: float, inhibition: float, noise: float,
                       dt: float, theta: float, n_steps: int, nodes: int = 64, rectify: bool = True):
    """First response of the two-unit rectified LCA of spec/MODELS.md §6 with
    pathway inputs (I0, I1):
        h_k(n) = h_k(n-1) + tau (I_k - h_k(n-1)),  h(0) = 0
        x_k(n) = max(x_k + dt (h_k(n) - leak x_k - inhibition x_{1-k}) + sigma sqrt(dt) g_k, 0)
        respond 0 if x_0 >= theta, else 1 if x_1 >= theta (checked after each step).
    Returns (p_r0[n_steps], p_r1[n_steps], p_undecided)."""
    s = noise * math.sqrt(dt)
    if s == 0.0:
        raise ValueError("noise must be positive (use the zero-noise pins)")
    g, gw = _gl(nodes, 0.0, theta)
    x = np.concatenate([[0.0], g])                       # node 0 = the atom at 0
    W = np.concatenate([[1.0], gw])                      # atom weight 1, GL weights for densities
    X0, X1 = np.meshgrid(x, x, indexing="ij")
    X0, X1 = X0.ravel(), X1.ravel()
    WW = np.outer(W, W).ravel()
    # law: V[i0, i1] = a00 at (0,0); line densities on the axes; density inside
    V = np.zeros((nodes + 1, nodes + 1))
    V[0, 0] = 1.0
    p0 = np.zeros(n_steps)
    p1 = np.zeros(n_steps)
    h0 = h1 = 0.0
    for n in range(n_steps):
        h0 = h0 + tau * (I0 - h0)
        h1 = h1 + tau * (I1 - h1)
        m0 = X0 + dt * (h0 - leak * X0 - inhibition * X1)
        m1 = X1 + dt * (h1 - leak * X1 - inhibition * X0)
        src = WW * V.ravel()
        keep = src != 0.0
        src, m0, m1 = src[keep], m0[keep], m1[keep]
        q0 = ndtr((m0 - theta) / s)                      # x_0 >= theta
        q1 = ndtr((m1 - theta) / s)
        p0[n] = src @ q0
        p1[n] = src @ ((1.0 - q0) * q1)
        A0 = np.empty((src.size, nodes + 1))
        A1 = np.empty((src.size, nodes + 1))
        if rectify:
            A0[:, 0] = ndtr(-m0 / s)                         # atom: P(y_k <= 0)
            A1[:, 0] = ndtr(-m1 / s)
        else:
            A0[:, 0] = 0.0
            A1[:, 0] = 0.0
        A0[:, 1:] = _phi((g[None, :] - m0[:, None]) / s) / s
        A1[:, 1:] = _phi((g[None, :] - m1[:, None]) / s) / s
        V = A0.T @ (src[:, None] * A1)
    p_und = float(W @ V @ W)
    return p0, p1, p_und


def binned(p_a, p_b, p_und, bin_steps: int):
    """spec/MODELS.md §4's histogram layout: outcome a at (n-1)/B, outcome b at
    nb + (n-1)/B, undecided at 2 nb."""
    n = p_a.size
    nb = (n + bin_steps - 1) // bin_steps
    out = np.zeros(2 * nb + 1)
    idx = np.arange(n) // bin_steps
    np.add.at(out, idx, p_a)
    np.add.at(out, nb + idx, p_b)
    out[2 * nb] = p_und
    return out


def chi2_pvalue(counts, probs, min_expected: float = 5.0):
    """Pearson chi-square of integer counts against exact cell probabilities,
    adjacent cells pooled (in order) until each expected count >= min_expected.
    Returns (statistic, dof, p-value)."""
    from scipy.stats import chi2
    counts = np.asarray(counts, np.float64)
    probs = np.asarray(probs, np.float64)
    T = counts.sum()
    exp = probs / probs.sum() * T
    oc, ec = [], []
    o = e = 0.0
    for c, x in zip(counts, exp):
        o += c
        e += x
        if e >= min_expected:
            oc.append(o)
            ec.append(e)
            o = e = 0.0
    if e > 0 or o > 0:
        if ec:
            oc[-1] += o
            ec[-1] += e
        else:
            oc.append(o)
            ec.append(e)
    oc, ec = np.array(oc), np.array(ec)
    stat = float(((oc - ec) ** 2 / ec).sum())
    dof = max(len(ec) - 1, 1)
    return stat, dof, float(chi2.sf(stat, dof))


# ------------------------------------------------------------------ the models' expected counts
# Per-allocation outcome counts of spec/MODELS.md §6 / §6c / §10 over T trials
# follow from the per-trial laws above: trial j has kind j mod 3 and colour
# (j div 3) mod 2, so a class (kind, colour) is a residue of j mod 6.  The
# counts are sums of independent trials, so their mean and variance are the
# class-weighted sums of the per-trial moments (n_correct, n_undecided, rt_sum).

def _class_sizes(T: int):
    """{(kind, colour): number of trials j < T in that class}."""
    out = {}
    for r in range(6):
        k = (r % 3, r // 3)
        out[k] = out.get(k, 0) + T // 6 + (1 if r < T % 6 else 0)
    return out


def stroop_inputs(P, uc: float, us: float, kind: int, colour: int):
    """Pathway inputs (I_0, I_1) of spec/MODELS.md §6 for one trial class (binary32 products, as the model)."""
    ic = float(np.float32(P[0]) * np.float32(uc))
    iw = float(np.float32(P[1]) * (np.float32(1.0) - np.float32(us)))
    I = [0.0, 0.0]
    I[colour] += ic
    if kind == 0:
        I[colour] += iw
    elif kind == 1:
        I[1 - colour] += iw
    return I


def stroop_class_law(P, uc: float, us: float, kind: int, colour: int, nodes: int = 36, **mut):
    """(p_correct[N], p_error[N], p_undecided) of one Stroop-LCA trial class
    (the response that names the colour is correct)."""
    tau, lam, beta, sig, dt, th = (float(v) for v in P[2:8])
    a = dict(tau=tau, leak=lam, inhibition=beta, noise=sig, dt=dt, theta=th, n_steps=int(P[10]), nodes=nodes)
    a.update(mut)
    I = stroop_inputs(P, uc, us, kind, colour)
    r0, r1, und = lca2_first_passage(I[0], I[1], **a)
    return (r0, r1, und) if colour == 0 else (r1, r0, und)


def _moments(pc, pe, pu, N, n):
    steps = np.arange(1, N + 1, dtype=np.float64)
    q = pc.sum()
    r1 = (steps * (pc + pe)).sum()
    r2 = (steps ** 2 * (pc + pe)).sum()
    return n * np.array([q, pu, r1]), n * np.array([q * (1 - q), pu * (1 - pu), r2 - r1 * r1])


def stroop_expected_counts(P, uc: float, us: float, T: int, nodes: int = 36):
    """Mean and variance of (n_correct, n_undecided, rt_sum) over trials [0, T)."""
    mean, var = np.zeros(3), np.zeros(3)
    for (kind, colour), n in _class_sizes(T).items():
        m, v = _moments(*stroop_class_law(P, uc, us, kind, colour, nodes), int(P[10]), n)
        mean += m
        var += v
    return mean, var


def ext_stroop_drifts(P, uc: float, us: float, kind: int):
    """spec/MODELS.md §10 front-end in binary64 for colour 0 (the colour DDM's
    drift (h_c - h_{1-c}) lambda is the same for either colour): (A1, A2)."""
    I = stroop_inputs(P, uc, us, kind, 0)
    tau, Nh = float(P[2]), int(P[3])
    h = [x * (1.0 - (1.0 - tau) ** Nh) for x in I]
    return (h[0] - h[1]) * float(P[4]), float(P[5]) - float(P[6]) * (h[0] * h[1])


def ext_stroop_ddm_law(P, A: float, nodes: int = 300):
    return ddm_first_passage(A, float(P[7]), float(P[9]), 0.0, float(P[8]), int(P[10]), nodes=nodes)


def ext_stroop_expected_counts(P, uc: float, us: float, T: int):
    """Mean and variance of (n_both, n_undecided, rt_sum = sum of max(n1, n2)
    over trials where both DDMs decided) over trials [0, T)."""
    Nd = int(P[10])
    steps = np.arange(1, Nd + 1, dtype=np.float64)
    mean, var = np.zeros(3), np.zeros(3)
    sizes = _class_sizes(T)
    for kind in range(3):
        n = sizes[(kind, 0)] + sizes[(kind, 1)]
        A1, A2 = ext_stroop_drifts(P, uc, us, kind)
        (u1, l1, n1), (u2, l2, n2) = ext_stroop_ddm_law(P, A1), ext_stroop_ddm_law(P, A2)
        pb = u1.sum() * u2.sum()
        pu = 1.0 - (1.0 - n1) * (1.0 - n2)
        F = np.cumsum(u1 + l1) * np.cumsum(u2 + l2)                 # P(max(n1, n2) <= n, both decided)
        pmax = np.diff(np.concatenate([[0.0], F]))
        r1, r2 = (steps * pmax).sum(), (steps ** 2 * pmax).sum()
        mean += n * np.array([pb, pu, r1])
        var += n * np.array([pb * (1 - pb), pu * (1 - pu), r2 - r1 * r1])
    return mean, var


def ddmg_expected_counts(P, u0: float, u1: float, T: int, nodes: int = 300):
    """spec/MODELS.md §6c: drift A0 + g_a u0 (binary32, as the model), threshold u1."""
    A = float(np.float32(np.float32(P[1]) * np.float32(u0) + np.float32(P[0])))
    up, lo, und = ddm_first_passage(A, float(P[2]), float(u1), 0.0, float(P[3]), int(P[6]), nodes=nodes)
    return _moments(up, lo, und, int(P[6]), T)


def zscores(got, mean, var):
    got = np.asarray(got, np.float64)
    sd = np.sqrt(np.maximum(var, 0.0))
    return np.where(sd > 0, (got - mean) / np.where(sd > 0, sd, 1.0), np.where(got == mean, 0.0, np.inf))
