"""Small driver for ncu captures of the DDM and Stroop kernels (tools only).

    python tools/profile_extras.py       # cfg2 DDM batch + a 100-allocation slice of cfg4
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
    for _ in range(2):
        D.eval_grid(m, None, c.n_trials, c.seed, 0, n, net=net, best=best, counts=counts)
    torch.cuda.synchronize()
    print("ok", int(rh.sum()), float(net[0]))


if __name__ == "__main__":
    main()
