#!/usr/bin/env python
"""A/B of distill_argmax (K2) between library builds (tools only).

    python tools/argmax_ab.py LIB_A.so LIB_B.so

Each build in a fresh process: the argmax over 128e6 values (512 MB, one call)
and over 8 x 16e6 values (8 calls on 64 MB copies, one CUDA graph), CUDA-event
medians of 5 passes; then the NEXT-2 tie pass (distill_argmax_ties) over the
512 MB; the keys must agree across builds.
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(lib_path):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2110_15425_b200._abi as A
    A.LIB_PATH = os.path.abspath(lib_path)
    import paper_2110_15425_b200 as D
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(7)
    nv = 16_000_000
    base = -torch.rand(nv, generator=g, device=dev)
    base[::97] = float("nan")
    big = base.repeat(8)
    kk = torch.full((9,), -1, dtype=torch.int64, device=dev)
    D.argmax(big, 0, kk[8:9])
    ga = torch.cuda.CUDAGraph()
    with torch.cuda.graph(ga):
        for c in range(8):
            D.argmax(big[c * nv:(c + 1) * nv], 0, kk[c:c + 1])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    one, gr = [], []
    for r in range(6):
        kk.fill_(-1)
        e0.record()
        D.argmax(big, 0, kk[8:9])
        e1.record()
        torch.cuda.synchronize()
        if r:
            one.append(e0.elapsed_time(e1))
        e0.record()
        ga.replay()
        e1.record()
        torch.cuda.synchronize()
        if r:
            gr.append(e0.elapsed_time(e1) / 8)
    # NEXT-2's second pass over the same 512 MB (distill_argmax_ties; ~0 ties: the scan itself)
    tie = torch.full((1,), -1, dtype=torch.int64, device=dev)
    tt = []
    for r in range(6):
        tie.fill_(-1)
        e0.record()
        D.argmax_ties(big, 0, 5, 0, kk[8:9], tie)
        e1.record()
        torch.cuda.synchronize()
        if r:
            tt.append(e0.elapsed_time(e1))
    keys = sorted({int(x) & (2 ** 64 - 1) for x in kk.cpu().numpy()}) + [int(tie.item()) & (2 ** 64 - 1)]
    print(json.dumps({"one_512MB_ms": statistics.median(one), "graph_64MB_ms": statistics.median(gr),
                      "ties_512MB_ms": statistics.median(tt), "keys": keys}))


def main():
    if sys.argv[1] == "--child":
        return child(sys.argv[2])
    res = {}
    for _ in range(2):
        for lib in sys.argv[1:]:
            out = subprocess.run([sys.executable, __file__, "--child", lib], capture_output=True, text=True,
                                 check=True)
            res.setdefault(lib, []).append(json.loads(out.stdout.strip().splitlines()[-1]))
    keys = {json.dumps(r["keys"]) for rs in res.values() for r in rs}
    print(f"{'build':30s} {'512 MB, one call':>18s} {'GB/s':>7s} {'64 MB (graph of 8)':>20s} {'GB/s':>7s}"
          f" {'ties 512 MB':>14s} {'GB/s':>7s}")
    for lib, rs in res.items():
        a = statistics.median(r["one_512MB_ms"] for r in rs)
        b = statistics.median(r["graph_64MB_ms"] for r in rs)
        c = statistics.median(r["ties_512MB_ms"] for r in rs)
        print(f"{os.path.basename(lib):30s} {a:15.4f} ms {512e6 / a / 1e6:7.0f} {b:17.4f} ms {64e6 / b / 1e6:7.0f}"
              f" {c:11.4f} ms {512e6 / c / 1e6:7.0f}")
    print("keys identical across builds and rounds:", len(keys) == 1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
