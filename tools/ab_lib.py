#!/usr/bin/env python
"""A/B two builds of libdistill.so on the hot workloads (tools only).

    python tools/ab_lib.py LIB_A.so LIB_B.so [--rounds 3]

Each round loads every library in a fresh subprocess (one CUDA context per
build, alternating A B A B ...) and times, with CUDA events on the launching
stream: PP cfg3 (20 graph-replayed grid searches, median), DDM cfg2 (graph:
zeroing + kernel, median of 5), a Stroop cfg4 slice (allocations [8000, 8100)
x 1e5 trials, median of 3), Extended Stroop A, the DDM control grid and the
whole cfg4 grid (one pass each).  Every output array is hashed: the two builds must agree bit for
bit, so an A/B is only reported for equivalent code.
"""
from __future__ import annotations

import hashlib
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib_path: str) -> dict:
    sys.path.insert(0, ROOT)
    import torch
    import paper_2110_15425_b200._abi as A
    A.LIB_PATH = os.path.abspath(lib_path)
    import paper_2110_15425_b200 as D
    import workloads as W

    dev = torch.device("cuda", 0)
    out = {}

    def h(*ts):
        m = hashlib.sha1()
        for t in ts:
            m.update(t.detach().cpu().numpy().tobytes())
        return m.hexdigest()[:16]

    def ev():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # PP cfg3
    c = W.pp_cfg3()
    m = D.load_model(W.KIND_PREDATOR_PREY, c.n_levels, c.levels, c.w, c.params, device=0)
    net = torch.empty(c.n_alloc, dtype=torch.float32, device=dev)
    best = torch.empty(1, dtype=torch.int64, device=dev)

    def pp():
        D.key_reset(best)
        D.eval_grid(m, c.inputs, c.n_samples, c.seed, net=net, best=best)

    pp()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        pp()
    ts = []
    for _ in range(20):
        e0, e1 = ev()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["pp_cfg3_ms"] = statistics.median(ts)
    out["pp_hash"] = h(net, best)

    # PP latency mode: the paper's PP-L (6^3 = 216 allocations) and a 40^3 grid (4-lane
    # mode), 20 graph-replayed grid searches, device time per search in microseconds
    for name, L in (("pp_L_us", 6), ("pp_40c_us", 40)):
        cs = W.PPConfig(f"pp_{L}", (L, L, L), 100)
        ms2 = D.load_model(W.KIND_PREDATOR_PREY, cs.n_levels, cs.levels, cs.w, cs.params, device=0)
        n2 = torch.empty(cs.n_alloc, dtype=torch.float32, device=dev)
        b2 = torch.empty(1, dtype=torch.int64, device=dev)

        def small():
            D.key_reset(b2)
            D.eval_grid(ms2, cs.inputs, cs.n_samples, cs.seed, net=n2, best=b2)

        small()
        torch.cuda.synchronize()
        g3 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g3):
            for _ in range(20):
                small()
        g3.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = ev()
            e0.record()
            g3.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 20)
        out[name] = statistics.median(ts)
        out[name.replace("_us", "_hash")] = h(n2, b2)

    # DDM cfg2
    d = W.ddm_cfg2()
    hbuf = torch.zeros(sum(d.hist_sizes), dtype=torch.int64, device=dev)
    rh, rs, xh = torch.split(hbuf, list(d.hist_sizes))

    def ddm():
        hbuf.zero_()
        D.ddm_batch(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                    d.x_lo, d.x_hi, 0, d.n_trials, d.seed, rh, rs, xh)

    ddm()
    torch.cuda.synchronize()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        ddm()
    ts = []
    for _ in range(5):
        e0, e1 = ev()
        e0.record()
        g2.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["ddm_cfg2_ms"] = statistics.median(ts)
    out["ddm_hash"] = h(hbuf)

    # Stroop cfg4 slice
    s = W.stroop_cfg4()
    ms_ = D.load_model(W.KIND_STROOP_LCA, s.n_levels, s.levels, s.w, s.params, device=0)
    b, e = 8000, 8100
    snet = torch.empty(e - b, dtype=torch.float32, device=dev)
    sbest = torch.empty(1, dtype=torch.int64, device=dev)
    scounts = torch.empty(3 * (e - b), dtype=torch.int64, device=dev)
    ts = []
    for _ in range(3):
        D.key_reset(sbest)
        e0, e1 = ev()
        e0.record()
        D.eval_grid(ms_, None, s.n_trials, s.seed, b, e, net=snet, best=sbest, counts=scounts)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out["stroop_slice_ms"] = statistics.median(ts)
    out["stroop_hash"] = h(snet, sbest, scounts)

    # Extended Stroop A, the DDM control grid and the whole cfg4 grid, one timed pass each
    for name, cfg, kind in (("ext_stroop", W.ext_stroop_grid(), W.KIND_EXT_STROOP_A),
                            ("ddm_grid", W.ddmg_grid(), W.KIND_DDM_GRID),
                            ("stroop_cfg4", W.stroop_cfg4(), W.KIND_STROOP_LCA)):
        mm = D.load_model(kind, cfg.n_levels, cfg.levels, cfg.w, cfg.params, device=0)
        xn = torch.empty(cfg.n_alloc, dtype=torch.float32, device=dev)
        xb = torch.empty(1, dtype=torch.int64, device=dev)
        xc = torch.empty(3 * cfg.n_alloc, dtype=torch.int64, device=dev)
        D.key_reset(xb)
        D.eval_grid(mm, None, cfg.n_trials, cfg.seed, net=xn, best=xb, counts=xc)   # warm
        D.key_reset(xb)
        e0, e1 = ev()
        e0.record()
        D.eval_grid(mm, None, cfg.n_trials, cfg.seed, net=xn, best=xb, counts=xc)
        e1.record()
        torch.cuda.synchronize()
        out[f"{name}_ms"] = e0.elapsed_time(e1)
        out[f"{name}_hash"] = h(xn, xb, xc)
    return out


def main():
    if len(sys.argv) >= 3 and sys.argv[1] == "--child":
        print(json.dumps(child(sys.argv[2])), flush=True)
        return 0
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    libs, rounds = args.libs, args.rounds
    res = {lib: [] for lib in libs}
    for _ in range(rounds):
        for lib in libs:
            p = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", lib],
                               capture_output=True, text=True, timeout=600)
            if p.returncode != 0:
                print(p.stderr[-3000:])
                return 1
            res[lib].append(json.loads(p.stdout.strip().splitlines()[-1]))
    keys = [k for k in res[libs[0]][0] if k.endswith("_ms") or k.endswith("_us")]
    print("build".ljust(28) + "".join(k.rjust(18) for k in keys))
    for lib in libs:
        row = [statistics.median(r[k] for r in res[lib]) for k in keys]
        print(os.path.basename(lib).ljust(28) + "".join(f"{v:18.4f}" for v in row))
    hk = [k for k in res[libs[0]][0] if k.endswith("_hash")]
    same = all(res[lib][i][k] == res[libs[0]][0][k] for lib in libs for i in range(rounds) for k in hk)
    print("outputs bit-identical across builds and rounds:", same)
    if not same:
        for lib in libs:
            print(lib, {k: res[lib][0][k] for k in hk})
    return 0 if same else 2


if __name__ == "__main__":
    sys.exit(main())
