"""Small driver for ncu captures of the DDM and Stroop kernels (tools only).

    python tools/profile_extras.py [--pp]      # cfg2 DDM batch + 100-allocation slices of cfg4 (around its optimum) and the Ext Stroop grid
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2110_15425_b200 as D  # noqa: E402
import workloads as W  # noqa: E402


def main():
    torch.cuda.set_device(0)
    if "--pp" in sys.argv:      # one cfg3 grid search first (for metric-only captures)
        c3 = W.pp_cfg3()
        mp = D.load_model(W.KIND_PREDATOR_PREY, c3.n_levels, c3.levels, c3.w, c3.params, device=0)
        pnet = torch.empty(c3.n_alloc, device="cuda")
        pbest = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        for _ in range(2):
            D.eval_grid(mp, c3.inputs, c3.n_samples, c3.seed, net=pnet, best=pbest)
    d = W.ddm_cfg2()
    rh, rs, xh = (torch.zeros(n, dtype=torch.int64, device="cuda") for n in d.hist_sizes)
    for _ in range(2):
        D.ddm_batch(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                    d.x_lo, d.x_hi, 0, d.n_trials, d.seed, rh, rs, xh)
    c = W.stroop_cfg4()
    m = D.load_model(W.KIND_STROOP_LCA, c.n_levels, c.levels, c.w, c.params, device=0)
    n = 100
    net = torch.empty(n, device="cuda")
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    counts = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    for _ in range(2):       # a slice around the cfg4 optimum (allocation 8083): representative response times
        D.eval_grid(m, None, c.n_trials, c.seed, 8000, 8000 + n, net=net, best=best, counts=counts)
    if "--stroop-full" in sys.argv:   # the whole cfg4 grid in the library's launch shape
        nf = c.n_alloc
        netf = torch.empty(nf, device="cuda")
        countsf = torch.empty(3 * nf, dtype=torch.int64, device="cuda")
        D.eval_grid(m, None, c.n_trials, c.seed, 0, nf, net=netf, best=best, counts=countsf)
    g = W.ext_stroop_grid()
    mx = D.load_model(W.KIND_EXT_STROOP_A, g.n_levels, g.levels, g.w, g.params, device=0)
    for _ in range(2):
        D.eval_grid(mx, None, g.n_trials, g.seed, 0, n, net=net, best=best, counts=counts)
    if "--more" in sys.argv:   # the round's additions: DDM grid slice, LCI batch, energy trace
        gd = W.ddmg_grid()
        mg = D.load_model(W.KIND_DDM_GRID, gd.n_levels, gd.levels, gd.w, gd.params, device=0)
        for _ in range(2):
            D.eval_grid(mg, None, gd.n_trials, gd.seed, 0, n, net=net, best=best, counts=counts)
        for _ in range(2):
            D.ddm_batch(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                        d.x_lo, d.x_hi, 0, d.n_trials, d.seed, rh, rs, xh, lci=(0.5, 0.0))
        for _ in range(2):
            D.stroop_energy(m, 8083, c.n_trials, c.seed)
    torch.cuda.synchronize()
    print("ok", int(rh.sum()), float(net[0]))


if __name__ == "__main__":
    main()
