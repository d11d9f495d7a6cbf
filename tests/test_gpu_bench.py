"""bench.py's own arm on the GPU: one short run, JSON line checked against the
driver contract (keys, roofline / cpu_baseline / e2e / clocks objects, launch
accounting)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_json_contract_on_gpu():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--no-extras"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["config"]["workload"].startswith("pp_cfg3") and d["vs_baseline"] is None
    per_gpu = d["timing"]["allocations_per_gpu"]
    assert per_gpu == d["config"]["allocations"] == 10 ** 6
    assert "CUDA graph" in d["timing"]["step"]
    r = d["roofline"]
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s" and 0 < r["frac_counted_method"] < r["frac_executed"] < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and r["frac_method"] == r["frac"]
    assert r["cost_array_write"]["bytes_per_launch"] == 4 * per_gpu
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] >= 4 * per_gpu
    assert 0 < e["value"] <= d["value"] * 1.05
    # the pipelined host-buffer calls (distill_eval_grid_host_async) each returned the step's key;
    # the one-call-per-step synchronous figure is reported beside it
    assert e["keys_match_step"] is True and 0 < e["sync"]["value"] <= e["value"] * 1.05
    assert d["gpu_launches"] == d["steps"]                 # one fused kernel per step
    assert d["clocks"]["sm_max_mhz"] > 0
    # the best allocation of the timed grid search decodes inside the grid, and the
    # key of the graph-captured, signed-order step IS the oracle's cfg3 key
    assert 0 <= d["result"]["best_index"] < d["config"]["allocations"]
    sys.path.insert(0, ROOT)
    import oracle
    import workloads as W
    c = W.pp_cfg3()
    full = oracle.pp_eval_threads(c.n_levels, c.levels, c.w, c.params, c.inputs, 0, c.n_alloc, c.n_samples, c.seed,
                                  threads=os.cpu_count() or 8)
    assert d["result"]["key"] == f"{oracle.argmax_net(-full)[0]:016x}"


@pytest.mark.parametrize("n", [2, 8])
def test_bench_self_spawns_ranks_and_reproduces_the_single_gpu_key(n):
    """`bench.py --gpus N` without torchrun launches N ranks itself (here all on
    GPU 0 over gloo: the multi-rank code path, not a timing): n_gpus = N, the cfg5
    grid sharded N ways, and the combined key equal to cfg5 evaluated whole on one
    GPU (itself bit-exact against the oracle, test_pp_cfg5_whole_grid_one_gpu)."""
    import torch
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "3",
                          "--warmup", "3", "--no-extras", "--no-cpu-baseline", "--dist-backend", "gloo",
                          "--device", "0"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["scaling"] == "strong" and d["config"]["workload"].startswith("pp_cfg5")
    assert d["timing"]["allocations_per_gpu"] == 8_000_000 // n
    sys.path.insert(0, ROOT)
    import paper_2110_15425_b200 as D
    import workloads as W
    c5 = W.pp_cfg5()
    m = D.load_model(W.KIND_PREDATOR_PREY, c5.n_levels, c5.levels, c5.w, c5.params, device=0)
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.eval_grid(m, c5.inputs, c5.n_samples, c5.seed, best=best)
    assert d["result"]["key"] == f"{D.key_from_tensor(best):016x}"


def test_bench_graph_captures_the_nccl_allreduce_on_one_gpu():
    """The multi-GPU step's riskiest piece — the NCCL key all-reduce captured in
    the CUDA graph with the kernel, and the capture agreement — run on one GPU
    as a one-rank NCCL group (--collective-at-1): the graph is used, and the
    all-reduced key is the oracle's cfg3 key (as at N = 1 without the collective)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--no-extras", "--no-cpu-baseline", "--collective-at-1"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert "captured in one CUDA graph" in d["timing"]["step"] and "collective-at-1" in d["timing"]["step"]
    sys.path.insert(0, ROOT)
    import oracle
    import workloads as W
    c = W.pp_cfg3()
    full = oracle.pp_eval_threads(c.n_levels, c.levels, c.w, c.params, c.inputs, 0, c.n_alloc, c.n_samples, c.seed,
                                  threads=os.cpu_count() or 8)
    assert d["result"]["key"] == f"{oracle.argmax_net(-full)[0]:016x}"
