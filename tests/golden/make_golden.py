"""Writes tests/golden/*.txt from the ORACLE ONLY (never from the CUDA path).

pp_cfg1_costs.txt: binary32 cost C of every cfg1 allocation (hex-float).
ddm_small_hist.txt: DDM histograms of 2000 cfg2-parameter trials of 250 steps.
stroop_small_counts.txt: Stroop integer outcomes of a 4x4 grid x 60 trials.
All are regression fixtures (they catch an unintended change of the oracle's
arithmetic or RNG stream layout); their correctness rests on the pins in
tests/test_oracle_*.py, not on these files.
"""
import numpy as np
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
import workloads as W  # noqa: E402


def main():
    cfg = W.pp_cfg1()
    C = oracle.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc,
                       cfg.n_samples, cfg.seed)
    key, _ = oracle.argmax_net(-C)
    with open(os.path.join(HERE, "pp_cfg1_costs.txt"), "w") as f:
        f.write("# cfg1 (workloads.pp_cfg1, seed 42): index  cost-hex ; written by make_golden.py\n")
        f.write(f"# best key 0x{key:016x} -> index {key & 0xffffffff}\n")
        for i, c in enumerate(C):
            f.write(f"{i} {float(c).hex()}\n")
    d = W.DDMConfig(n_steps=250, n_trials=2000)
    p = oracle.ddm_params(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                          d.x_lo, d.x_hi)
    rh, rs, xh = oracle.ddm_batch(p, d.seed, 0, d.n_trials)
    with open(os.path.join(HERE, "ddm_small_hist.txt"), "w") as f:
        f.write("# DDMConfig(n_steps=250, n_trials=2000), seed 42: rt_hist / rt_sum / x_hist ; make_golden.py\n")
        for name, arr in (("rt_hist", rh), ("rt_sum", rs), ("x_hist", xh)):
            f.write(name + " " + " ".join(str(int(v)) for v in arr) + "\n")
    lev = np.linspace(0, 1, 4).astype(np.float32)
    counts, net = oracle.stroop_eval((4, 4), np.concatenate([lev, lev]), W.STROOP_W, W.STROOP_PARAMS, 0, 16, 60,
                                     W.SEED)
    with open(os.path.join(HERE, "stroop_small_counts.txt"), "w") as f:
        f.write("# Stroop 4x4 grid (levels k/3), 60 trials, seed 42: index n_correct n_undecided rt_sum V-hex\n")
        for i in range(16):
            f.write(f"{i} {int(counts[i, 0])} {int(counts[i, 1])} {int(counts[i, 2])} {float(net[i]).hex()}\n")


if __name__ == "__main__":
    main()
