"""Exercise every kernel of libdistill.so on small inputs (for compute-sanitizer runs; tools only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2110_15425_b200 as D  # noqa: E402
import workloads as W  # noqa: E402


def main():
    torch.cuda.set_device(0)
    cfg = W.PPConfig("s", (7, 5, 3), 6)
    m = D.load_model(W.KIND_PREDATOR_PREY, cfg.n_levels, cfg.levels, cfg.w, cfg.params, device=0)
    net = torch.empty(cfg.n_alloc, device="cuda")
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.eval_grid(m, cfg.inputs, 6, 1, net=net, best=best)
    D.eval_grid(m, cfg.inputs, 5, 1, 3, 77, net=net, best=best)
    D.argmax(net, 0, best)
    tie = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.argmax_ties(net, 0, 3, 0, best, tie)
    D.eval_grid_host(m, cfg.inputs, 6, 1, net_out=np.empty(cfg.n_alloc, np.float32))
    D.pp_episode(m, cfg.inputs, 5, 4, 2)
    D.pp_amr(m, cfg.inputs, (0, 0, 0), (1, 1, 1), 3, 4, 2)
    d = W.DDMConfig(n_steps=50)
    rh, rs, xh = (torch.zeros(n, dtype=torch.int64, device="cuda") for n in d.hist_sizes)
    D.ddm_batch(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins, d.x_lo,
                d.x_hi, 0, 700, 1, rh, rs, xh)
    c = W.StroopConfig("s", (3, 4), 50)
    ms = D.load_model(W.KIND_STROOP_LCA, c.n_levels, c.levels, c.w, c.params, device=0)
    sn = torch.empty(c.n_alloc, device="cuda")
    D.eval_grid(ms, None, c.n_trials, 1, net=sn, best=best)
    for kind in (W.KIND_EXT_STROOP_A, W.KIND_EXT_STROOP_B):
        mx = D.load_model(kind, c.n_levels, c.levels, c.w, W.EXT_STROOP_PARAMS, device=0)
        D.eval_grid(mx, None, 30, 1, net=sn, best=best)
    sets = torch.from_numpy(W.pp_positions(3)).cuda()
    mnet = torch.empty((4, cfg.n_alloc), device="cuda")
    mbest = torch.full((4,), -1, dtype=torch.int64, device="cuda")
    D.eval_grid_multi(m, sets, 4, 5, 1, net=mnet, best=mbest)
    run = D.EpisodeRun(m, cfg.inputs, 3, 4, 2)
    for t in range(3):
        run.search(t, 0, 50)
        run.search(t, 50, cfg.n_alloc)
        run.advance(t)
    D.eval_grid_host(m, cfg.inputs, 6, 1, net_out=torch.empty(cfg.n_alloc, pin_memory=True).numpy())
    D.ddm_batch(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins, d.x_lo,
                d.x_hi, 0, 700, 1, rh, rs, xh, lci=(0.5, 0.01))
    D.stroop_energy(ms, 3, c.n_trials, 1)
    gd = W.ddmg_grid(4, 60)
    mdg = D.load_model(W.KIND_DDM_GRID, gd.n_levels, gd.levels, gd.w, gd.params, device=0)
    D.eval_grid(mdg, None, gd.n_trials, 1, net=torch.empty(gd.n_alloc, device="cuda"), best=best)
    torch.cuda.synchronize()
    print("sanitize-small ok", int(best.item()), int(rh.sum()))


if __name__ == "__main__":
    main()
