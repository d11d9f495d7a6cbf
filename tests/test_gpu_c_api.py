"""The C ABI used from plain C (examples/c_api_demo.c, no Python in the call
path): compiled with gcc against include/distill.h and libdistill.so, its
cfg1 grid search must print the oracle's 27 costs and best key bit for bit, and
its host-buffer calls (synchronous and two in flight) the same key."""
import os
import subprocess

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_c_program_through_the_abi(orc, tmp_path):
    exe = str(tmp_path / "c_api_demo")
    lib_dir = os.path.join(ROOT, "paper_2110_15425_b200")
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(ROOT, "examples", "c_api_demo.c"), "-L", lib_dir, "-ldistill",
                           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    host = [l for l in lines if l.startswith("host ")]
    lines = [l for l in lines if not l.startswith("host ")]
    costs = np.array([float.fromhex(l.split()[1]) for l in lines[:-1]], np.float32)
    cfg = W.pp_cfg1()
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc, cfg.n_samples,
                       cfg.seed)
    assert np.array_equal(costs.view(np.uint32), want.view(np.uint32))
    key = int(lines[-1].split()[-1], 16)
    assert key == orc.argmax_net(-want)[0]
    # the synchronous host-buffer call and two in-flight async calls: the same key and net values
    f = host[0].split()
    assert len(host) == 1 and [int(f[2], 16), int(f[4], 16), int(f[5], 16)] == [key] * 3 and f[-1] == "same"
