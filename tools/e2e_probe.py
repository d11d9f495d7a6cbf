#!/usr/bin/env python
"""Where the end-to-end host-buffer call spends its time beyond the kernel (tools only).

    python tools/e2e_probe.py

cfg3 on one GPU: (1) the device-resident step replayed from a CUDA graph (events);
(2) distill_eval_grid_host through the binding (events around the call, as bench.py's
e2e); (3) the same call timed with the host clock, with and without the net values.
"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2110_15425_b200 as D
    import workloads as W
    c = W.pp_cfg3()
    m = D.load_model(W.KIND_PREDATOR_PREY, c.n_levels, c.levels, c.w, c.params, device=0)
    dev = torch.device("cuda", 0)
    net_d = torch.empty(c.n_alloc, dtype=torch.float32, device=dev)
    net_h = torch.empty(c.n_alloc, dtype=torch.float32, pin_memory=True)
    best = torch.empty(1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream()

    def ev():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, n=30):
        ts = []
        for _ in range(n):
            e0, e1 = ev()
            e0.record(st)
            fn()
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    def dev_step(net):
        D.key_reset(best)
        D.eval_grid(m, c.inputs, c.n_samples, c.seed, net=net, best=best)

    for _ in range(3):
        dev_step(net_d)
    torch.cuda.synchronize()
    print(f"kernel + reset, net -> device memory      {timed(lambda: dev_step(net_d)):.4f} ms")
    h = net_h.numpy()
    D.eval_grid_host(m, c.inputs, c.n_samples, c.seed, net_out=h)
    print(f"eval_grid_host (events, bench e2e)        {timed(lambda: D.eval_grid_host(m, c.inputs, c.n_samples, c.seed, net_out=h)):.4f} ms")
    ts = []
    for _ in range(30):
        t = time.perf_counter()
        D.eval_grid_host(m, c.inputs, c.n_samples, c.seed, net_out=h)
        ts.append(1e3 * (time.perf_counter() - t))
    print(f"eval_grid_host (host clock)               {statistics.median(ts):.4f} ms")
    ts = []
    for _ in range(30):
        t = time.perf_counter()
        D.eval_grid_host(m, c.inputs, c.n_samples, c.seed, net_out=None)
        ts.append(1e3 * (time.perf_counter() - t))
    print(f"eval_grid_host, key only (host clock)     {statistics.median(ts):.4f} ms")


if __name__ == "__main__":
    main()
