"""GPU outputs at the bench's FULL sizes against the exact first-passage laws of
the models (tests/exact_law.py) — a property that holds at any size and needs
no oracle run: the DDM cfg2 histogram of all 1e6 trials, and for the Stroop
cfg4 grid (1e4 allocations x 1e5 trials), the Extended Stroop grid and the DDM
control grid (1e4 x 1e4 each), the counts of the GPU's own argmax allocation
and of sampled allocations, each within 4.5 standard errors of its exact
expectation (spec/MODELS.md §4, §6, §6c, §10)."""
import numpy as np
import pytest

import exact_law as X
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no fallback)"
    torch.cuda.set_device(0)
    import paper_2110_15425_b200 as D
    return D


def test_ddm_cfg2_full_histogram_is_the_exact_law(D):
    import torch
    d = W.ddm_cfg2()
    rh, rs, xh = (torch.zeros(n, dtype=torch.int64, device="cuda") for n in d.hist_sizes)
    D.ddm_batch(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                d.x_lo, d.x_hi, 0, d.n_trials, d.seed, rh, rs, xh)
    torch.cuda.synchronize()
    rt = rh.cpu().numpy()
    law = X.ddm_first_passage(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps)
    stat, dof, p = X.chi2_pvalue(rt, X.binned(*law, d.rt_bin_steps))
    assert p > 1e-3, (stat, dof, p)
    late = (np.concatenate([[0.0], law[0][:-1]]), np.concatenate([[0.0], law[1][:-1]]), law[2])
    assert X.chi2_pvalue(rt, X.binned(*late, d.rt_bin_steps))[2] < 1e-12


def _grid_counts(D, kind, c):
    import torch
    m = D.load_model(kind, c.n_levels, c.levels, c.w, c.params, device=0)
    n = c.n_alloc
    net = torch.empty(n, dtype=torch.float32, device="cuda")
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    counts = torch.zeros(3 * n, dtype=torch.int64, device="cuda")
    D.eval_grid(m, None, c.n_trials, c.seed, 0, n, net=net, best=best, counts=counts)
    torch.cuda.synchronize()
    return counts.cpu().numpy().reshape(n, 3), int(best.item()) & 0xFFFFFFFF


SAMPLED = [0, 99, 1234, 5050, 7007, 9900, 9999]


@pytest.mark.parametrize("model", ["stroop_cfg4", "ext_stroop", "ddm_grid"])
def test_full_grid_counts_match_the_exact_law(D, model):
    if model == "stroop_cfg4":
        c, kind = W.stroop_cfg4(), W.KIND_STROOP_LCA
        expect = lambda u0, u1: X.stroop_expected_counts(c.params, u0, u1, c.n_trials)   # noqa: E731
    elif model == "ext_stroop":
        c, kind = W.ext_stroop_grid(), W.KIND_EXT_STROOP_A
        expect = lambda u0, u1: X.ext_stroop_expected_counts(c.params, u0, u1, c.n_trials)   # noqa: E731
    else:
        c, kind = W.ddmg_grid(), W.KIND_DDM_GRID
        expect = lambda u0, u1: X.ddmg_expected_counts(c.params, u0, u1, c.n_trials)   # noqa: E731
    counts, best = _grid_counts(D, kind, c)
    L1 = c.n_levels[1]
    for i in [best, *SAMPLED]:
        u0, u1 = float(c.levels[i // L1]), float(c.levels[c.n_levels[0] + i % L1])
        mean, var = expect(u0, u1)
        z = X.zscores(counts[i], mean, var)
        assert np.all(np.abs(z) < 4.5), (model, i, counts[i], mean, z)
