"""Writes tests/golden/*.txt from the ORACLE ONLY (never from the CUDA path).

pp_cfg1_costs.txt: binary32 cost C of every cfg1 allocation (hex-float), a
regression fixture — its correctness rests on the pins in
tests/test_oracle_pp.py, not on this file.
"""
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


if __name__ == "__main__":
    main()
