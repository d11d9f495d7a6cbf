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
    r = d["roofline"]
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["cost_array_write"]["bytes_per_launch"] == 4 * d["config"]["allocations_per_gpu"]
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] >= 4 * d["config"]["allocations_per_gpu"]
    assert 0 < e["value"] <= d["value"] * 1.05
    assert d["gpu_launches"] == d["steps"]                 # one fused kernel per step
    assert d["clocks"]["sm_max_mhz"] > 0
    # the best allocation of the timed grid search decodes inside the grid
    assert 0 <= d["config"]["best"]["index"] < d["config"]["allocations"]
