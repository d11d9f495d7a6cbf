"""Test infrastructure (it runs the CPU oracle, so it lives under tests/; not a
pytest module — `test_r21_fused_objective_step_is_closer_to_binary64` is the
pinned version).  DESIGN.md reading R21: is the fused objective step Delta = fma(d, y_d, -u*)
closer to the plain binary64 definition than the unfused u_hat = d*y_d; Delta =
u_hat - u* ?  (Test infrastructure: runs only the CPU oracle.)

Builds a second copy of the oracle with -DOD_UNFUSED_OBJECTIVE (only the
objective's rounding differs), evaluates per-sample objectives e_s of the same
allocations with both, and compares each against the binary64 re-evaluation
od_pp_trace_f64 (same Philox bits, libm Box-Muller, exact 1/sqrt).  Prints the
error statistics; `profiles/r02_r21_error.txt` holds the committed output.

    python tests/r21_error.py [n_alloc]
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402


def unfused_lib():
    out = os.path.join(tempfile.gettempdir(), "liboracle_unfused.so")
    subprocess.check_call(["gcc", *oracle.CFLAGS, "-DOD_UNFUSED_OBJECTIVE", oracle._SRC, "-o", out, "-lm"])
    return oracle._bind(out)


def main():
    n_alloc = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
    oracle.build()
    fused, unfused = oracle.lib(), unfused_lib()
    cfg = W.pp_cfg3()
    rng = np.random.default_rng(2110)
    idx = rng.choice(cfg.n_alloc, n_alloc, replace=False)
    ef, eu, e64 = [], [], []
    for i in idx:
        args = (cfg.n_levels, cfg.levels, cfg.params, cfg.inputs, int(i), cfg.n_samples, cfg.seed)
        ef.append(oracle.pp_trace(*args, lib_handle=fused))
        eu.append(oracle.pp_trace(*args, lib_handle=unfused))
        e64.append(oracle.pp_trace_f64(*args))
    ef, eu, e64 = (np.concatenate(v).astype(np.float64) for v in (ef, eu, e64))
    rf, ru = np.abs(ef - e64) / e64, np.abs(eu - e64) / e64
    print(f"cfg3 inputs, {n_alloc} random allocations x {cfg.n_samples} samples = {ef.size} per-sample objectives")
    print("relative error vs binary64        fused Delta (R21)    unfused u_hat - u*")
    for name, f in (("mean", np.mean), ("median", np.median), ("p99", lambda a: np.quantile(a, 0.99)),
                    ("max", np.max)):
        print(f"  {name:<8}                        {f(rf):.3e}            {f(ru):.3e}")
    small = e64 < np.quantile(e64, 0.1)
    print(f"  mean, smallest decile of e       {rf[small].mean():.3e}            {ru[small].mean():.3e}")
    print(f"fused strictly closer on {np.mean(rf < ru):.3f} of samples, farther on {np.mean(rf > ru):.3f}")
    # the allocation costs (sum of 100 samples / S + K) against od_pp_eval_f64
    cf = oracle.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, 2000, cfg.n_samples, cfg.seed)
    lib_u = unfused
    cu = np.zeros(2000, np.float32)
    lib_u.od_pp_eval(oracle._u32(cfg.n_levels), oracle._f32(cfg.levels), oracle._f32(cfg.w),
                     oracle._f32(cfg.params), oracle._f32(cfg.inputs), 0, 2000, cfg.n_samples, cfg.seed, 0,
                     cu.ctypes.data)
    c64 = oracle.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, 2000, cfg.n_samples,
                         cfg.seed, f64=True)
    print(f"allocation costs [0, 2000): mean rel. error fused {np.mean(np.abs(cf - c64) / c64):.3e}, "
          f"unfused {np.mean(np.abs(cu - c64) / c64):.3e}")


if __name__ == "__main__":
    main()
