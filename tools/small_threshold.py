"""Grid-search device time vs grid size (CUDA-graph replay), for choosing the
latency-mode threshold of distill.cu (tools only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2110_15425_b200 as D  # noqa: E402
import workloads as W  # noqa: E402


def main():
    torch.cuda.set_device(0)
    for L in (4, 6, 10, 13, 16, 18, 20, 22, 24, 26, 28, 32, 40, 50, 64, 100):
        c = W.PPConfig(f"L{L}", (L, L, L), 100)
        m = D.load_model(W.KIND_PREDATOR_PREY, c.n_levels, c.levels, c.w, c.params, device=0)
        net = torch.empty(c.n_alloc, device="cuda")
        best = torch.empty(1, dtype=torch.int64, device="cuda")
        D.eval_grid(m, c.inputs, 100, 1, net=net, best=best)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                D.eval_grid(m, c.inputs, 100, 1, net=net, best=best)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"L={L:4d} allocations {c.n_alloc:8d}  {ms * 1e3:9.2f} us  {c.evals / (ms / 1e3):.3e} evals/s")


if __name__ == "__main__":
    main()
