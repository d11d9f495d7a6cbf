"""bench.py's reference arm runs on CPU (it times the oracle): check the JSON
line against the driver contract (keys, units, impl tag, zero-copy e2e)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--ref-budget-s", "2"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "evals/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("pp_cfg3")
    import bench
    import workloads as W
    assert d["config"] == bench.workload_config(W.pp_cfg3(), 1)      # the same config object as our arm
    assert d["metric"] == bench.METRIC
    baseline = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == baseline["metric"]


def test_bench_host_helpers(monkeypatch):
    """Host-side helpers of the GPU arm: nvidia-smi's -i follows CUDA_VISIBLE_DEVICES
    (each rank samples its own physical GPU), the workload per world size (N = 1 cfg3,
    N > 1 cfg5 strong, --weak ~1e6 per GPU) and the contiguous 4-aligned shards."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    import paper_2110_15425_b200 as D
    monkeypatch.delenv("CUDA_VISIBLE_DEVICES", raising=False)
    assert bench.smi_device(3) == "3"
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "4,5,6,7")
    assert [bench.smi_device(r) for r in range(4)] == ["4", "5", "6", "7"]
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "GPU-abc, GPU-def")
    assert bench.smi_device(1) == "GPU-def"
    args = argparse.Namespace(weak=False, strong=False)
    assert bench.workload(1, args)[0].n_alloc == 10 ** 6 and bench.workload(1, args)[1] == "weak"
    for n in (2, 4, 8):
        cfg, scaling = bench.workload(n, args)
        assert cfg.n_alloc == 8 * 10 ** 6 and scaling == "strong"
        shards = [D.shard_range(cfg.n_alloc, r, n) for r in range(n)]
        assert shards[0][0] == 0 and shards[-1][1] == cfg.n_alloc
        assert all(a[1] == b[0] for a, b in zip(shards, shards[1:])) and all(b % 4 == 0 for b, _ in shards)
    args.weak = True
    assert bench.workload(8, args)[0].n_alloc == 8 * 10 ** 6 and bench.workload(8, args)[1] == "weak"
