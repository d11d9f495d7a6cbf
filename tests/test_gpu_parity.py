"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element.

Bar: binary32 costs/net values bit-exact (stronger than the
north star's 1e-5 relative, which is also asserted against the binary64
re-evaluation); keys, argmax indices, counts and histograms bit-exact.
"""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no fallback)"
    torch.cuda.set_device(0)
    import paper_2110_15425_b200 as D
    return D


def _model(D, cfg, kind=W.KIND_PREDATOR_PREY):
    return D.load_model(kind, cfg.n_levels, cfg.levels, cfg.w, cfg.params, device=0)


def _gpu_pp(D, m, cfg, begin=0, end=None, invocation=0, seed=None, inputs=None):
    import torch
    end = cfg.n_alloc if end is None else end
    net = torch.empty(max(end - begin, 1), dtype=torch.float32, device="cuda")
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.eval_grid(m, cfg.inputs if inputs is None else inputs, cfg.n_samples, cfg.seed if seed is None else seed,
                begin, end, net=net, best=best, invocation=invocation)
    torch.cuda.synchronize()
    return -net.cpu().numpy()[:end - begin], int(best.item()) & (2 ** 64 - 1)


def _bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def test_pp_cfg1_bit_exact(D, orc):
    cfg = W.pp_cfg1()
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, 27, cfg.n_samples, cfg.seed)
    assert np.array_equal(_bits(C), _bits(want))
    assert key == orc.argmax_net(-want)[0]


@pytest.mark.parametrize("shape,S", [((7, 11, 13), 37), ((1, 1, 1), 1), ((2, 3, 700), 5), ((33, 1, 1), 100)])
def test_pp_ragged_grids_bit_exact(D, orc, shape, S):
    """Grids spanning several 256-thread tiles with a ragged tail, S = 1 and odd S."""
    cfg = W.PPConfig("r", shape, S)
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc, S, cfg.seed)
    assert np.array_equal(_bits(C), _bits(want))
    assert key == orc.argmax_net(-want)[0]


def test_pp_shards_concatenate_to_full_run(D, orc):
    """Shard invariance: any split [b, e) reproduces the full run; min of shard keys = full key."""
    cfg = W.PPConfig("s", (9, 10, 11), 20)
    m = _model(D, cfg)
    full, kfull = _gpu_pp(D, m, cfg)
    cuts = [0, 1, 257, 500, 511, 990]
    parts, keys = [], []
    for b, e in zip(cuts, cuts[1:]):
        c, k = _gpu_pp(D, m, cfg, b, e)
        parts.append(c)
        keys.append(k)
    assert np.array_equal(_bits(np.concatenate(parts)), _bits(full))
    assert min(keys) == kfull
    for rank in range(3):
        b, e = D.shard_range(cfg.n_alloc, rank, 3)
        c, _ = _gpu_pp(D, m, cfg, b, e)
        assert np.array_equal(_bits(c), _bits(full[b:e]))


def test_pp_seed_high_bits_and_invocation(D, orc):
    cfg = W.PPConfig("k", (5, 4, 3), 9)
    m = _model(D, cfg)
    seed = (0xDEADBEEF << 32) | 17
    inp = W.random_positions(3)
    for t in range(3):
        C, key = _gpu_pp(D, m, cfg, invocation=t, seed=seed, inputs=inp[t])
        want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, inp[t], 0, cfg.n_alloc, 9, seed,
                           invocation=t)
        assert np.array_equal(_bits(C), _bits(want))
        assert key == orc.argmax_net(-want)[0]


def test_pp_zero_noise_and_ties(D, orc):
    cfg = W.PPConfig("z", (6, 6, 6), 4)
    cfg.params = np.array([0.0, 0.0, 0.5], np.float32)
    cfg.w = np.zeros(3, np.float32)
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc, 4, cfg.seed)
    assert np.array_equal(_bits(C), _bits(want))
    assert (C == C[0]).all() and 0 <= C[0] < 1e-12 and key & 0xFFFFFFFF == 0


def test_pp_coincident_positions_and_nan(D, orc):
    """Degenerate inputs: coincident entities (|v| = 0 branch) and NaN positions."""
    cfg = W.PPConfig("d", (3, 3, 3), 6)
    cfg.inputs = np.array([0.0, 0.0, 0.0, 0.0, 0.0, 0.0], np.float32)
    cfg.params = np.array([0.0, 0.0, 0.5], np.float32)
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, 27, 6, cfg.seed)
    assert np.array_equal(_bits(C), _bits(want))
    cfg2 = W.PPConfig("n", (3, 3, 3), 6)
    m2 = _model(D, cfg2)
    C2, key2 = _gpu_pp(D, m2, cfg2, inputs=np.array([np.nan, 0, 1, 1, 0, 0], np.float32))
    assert np.isnan(C2).all()
    with pytest.raises(D.api.DistillError):
        D.key_decode(key2)


def test_pp_cfg3_full_size_argmax_and_sampled_costs(D, orc):
    """cfg3 (1e6 allocations x 100 samples) in the bench launch configuration:
    argmax key bit-exact against the full oracle grid search (north-star target),
    and 4096 sampled costs bit-exact."""
    import os
    cfg = W.pp_cfg3()
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([rng.integers(0, cfg.n_alloc, 4000), np.arange(64),
                                    np.arange(cfg.n_alloc - 32, cfg.n_alloc)]))
    for i in idx[:4096]:
        w = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, int(i), int(i) + 1,
                        cfg.n_samples, cfg.seed)
        assert _bits(C[i:i + 1])[0] == _bits(w)[0], int(i)
    full = orc.pp_eval_threads(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc,
                               cfg.n_samples, cfg.seed, threads=os.cpu_count() or 8)
    assert np.array_equal(_bits(C), _bits(full))
    assert key == orc.argmax_net(-full)[0]


def test_pp_cfg3_full_grid_over_seeds_invocations_and_positions(D, orc):
    """cfg3 at full size beyond the bench's seed: five more (seed, invocation,
    positions) triples — seeds 1..3 (SURVEY §8(d)'s sweep range), a high
    invocation word, random positions from the input recipe — each with all 1e6
    costs and the argmax key bit-exact against a full oracle grid search."""
    import os
    cfg = W.pp_cfg3()
    m = _model(D, cfg)
    pos = W.pp_positions(2)
    cases = [(1, 0, cfg.inputs), (2, 0, cfg.inputs), (3, 0, cfg.inputs), (42, 0xFFFFFFFF, cfg.inputs),
             (7, 5, pos[1])]
    for seed, inv, inputs in cases:
        C, key = _gpu_pp(D, m, cfg, invocation=inv, seed=seed, inputs=inputs)
        full = orc.pp_eval_threads(cfg.n_levels, cfg.levels, cfg.w, cfg.params, inputs, 0, cfg.n_alloc,
                                   cfg.n_samples, seed, threads=os.cpu_count() or 8, invocation=inv)
        assert np.array_equal(_bits(C), _bits(full)), (seed, inv)
        assert key == orc.argmax_net(-full)[0], (seed, inv)


def test_pp_within_north_star_tolerance_of_binary64(D, orc):
    cfg = W.pp_cfg3()
    m = _model(D, cfg)
    C, _ = _gpu_pp(D, m, cfg, 400000, 400512)
    c64 = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 400000, 400512,
                      cfg.n_samples, cfg.seed, f64=True)
    assert (np.abs(C - c64) / np.abs(c64)).max() < 1e-5


@pytest.mark.parametrize("n,off", [(1, 0), (5, 1), (1000, 3), (4096, 0), (100003, 2), (8_000_000, 0)])
def test_argmax_kernel_vs_oracle(D, orc, n, off):
    import torch
    rng = np.random.default_rng(n)
    v = rng.integers(-50, 50, size=n + off).astype(np.float32)
    v[rng.integers(0, n + off, size=max(1, n // 50))] = np.nan
    v[rng.integers(0, n + off, size=max(1, n // 70))] = -0.0
    t = torch.from_numpy(v).cuda()
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.argmax(t[off:], 1000, best)
    torch.cuda.synchronize()
    k_or, rc = orc.argmax_net(v[off:], 1000)
    assert (int(best.item()) & (2 ** 64 - 1)) == k_or


@pytest.mark.parametrize("n", [7, 8, 9, 4100, 1_000_003, 6_000_001])
def test_argmax_kernel_edge_cases_aligned(D, orc, n):
    """K2's aligned path (groups of eight visited in decreasing order, a group's
    first index resolved only when its max reaches the thread's best): random
    values, all -inf, NaN everywhere but one value, +-0 ties everywhere, the
    maximum tied at scattered indices, all NaN — keys bit-exact against the
    oracle (sizes below one group, ragged tails, several groups per thread)."""
    import torch
    rng = np.random.default_rng(n)
    cases = {
        "random": rng.standard_normal(n).astype(np.float32),
        "all -inf": np.full(n, -np.inf, np.float32),
        "nan but one": np.full(n, np.nan, np.float32),
        "signed zeros": np.where(rng.random(n) < 0.5, np.float32(-0.0), np.float32(0.0)).astype(np.float32),
        "scattered max": rng.integers(-3, 1, size=n).astype(np.float32),
        "all nan": np.full(n, np.nan, np.float32),
    }
    cases["nan but one"][rng.integers(0, n)] = -np.inf
    for name, v in cases.items():
        t = torch.from_numpy(v).cuda()
        best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        D.argmax(t, 12345, best)
        torch.cuda.synchronize()
        k_or, _ = orc.argmax_net(v, 12345)
        assert (int(best.item()) & (2 ** 64 - 1)) == k_or, (n, name)


def test_argmax_all_nan_and_empty(D, orc):
    import torch
    t = torch.full((10,), float("nan"), device="cuda")
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.argmax(t, 0, best)
    D.argmax(t[:0], 0, best)
    torch.cuda.synchronize()
    k = int(best.item()) & (2 ** 64 - 1)
    assert k >> 32 == 0xFFFFFFFF
    with pytest.raises(D.api.DistillError):
        D.key_decode(k)


def test_eval_grid_argument_errors(D):
    import torch
    cfg = W.pp_cfg1()
    m = _model(D, cfg)
    net = torch.empty(28, device="cuda")
    with pytest.raises(D.api.DistillError):
        D.eval_grid(m, cfg.inputs, 10, 1, 0, 28, net=net)          # past the grid
    with pytest.raises(ValueError):
        D.eval_grid(m, cfg.inputs, 10, 1, 0, 27, net=net[:20])     # buffer too small (caught in Python)
    with pytest.raises(D.api.DistillError):
        D.eval_grid(m, cfg.inputs, 0, 1, 0, 27, net=net)           # zero samples
    with pytest.raises(D.api.DistillError):
        D.eval_grid(m, cfg.inputs[:4], 10, 1, 0, 27, net=net)      # wrong input count
    with pytest.raises(D.api.DistillError):
        D.eval_grid(m, cfg.inputs, 2 ** 31 + 1, 1, 0, 27, net=net)  # sample counter could wrap
    ms = D.load_model(W.KIND_STROOP_LCA, (2, 2), np.array([0, 1, 0, 1], np.float32), W.STROOP_W,
                      W.STROOP_PARAMS, device=0)
    with pytest.raises(D.api.DistillError):
        D.eval_grid(ms, None, 2 ** 31 + 1, 1, 0, 4)                 # trial counter could wrap
    D.eval_grid(m, cfg.inputs, 10, 1, 5, 5, net=net)               # empty shard is a no-op


def _ddm_gpu(D, d, t0, t1, seed):
    import torch
    rh, rs, xh = (torch.zeros(n, dtype=torch.int64, device="cuda") for n in d.hist_sizes)
    D.ddm_batch(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                d.x_lo, d.x_hi, t0, t1, seed, rh, rs, xh)
    torch.cuda.synchronize()
    return [x.cpu().numpy().astype(np.uint64) for x in (rh, rs, xh)]


def _ddm_p(orc, d):
    return orc.ddm_params(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps,
                          d.n_x_bins, d.x_lo, d.x_hi)


@pytest.mark.parametrize("kw,t0,t1", [({}, 0, 4000), ({"n_steps": 333, "rt_bin_steps": 7}, 1000, 3001),
                                       ({"drift": -0.3, "noise": 2.0, "threshold": 2.5}, 123456, 125000),
                                       ({"n_steps": 1}, 0, 100), ({"n_steps": 12, "threshold": 0.3}, 0, 3000),
                                       ({"n_steps": 23, "threshold": 0.4, "rt_bin_steps": 1}, 7, 2500),
                                       ({"n_steps": 24, "threshold": -0.5}, 0, 100),
                                       ({"n_steps": 36, "threshold": 0.0, "noise": 0.01}, 0, 50),
                                       # RNG units across a multiple of 2^32 (the launch splits there: the
                                       # counter's c2 word changes) and at the top of the 64-bit range
                                       ({"n_steps": 120}, (1 << 32) - 700, (1 << 32) + 500),
                                       ({"n_steps": 61, "threshold": 0.6}, (1 << 64) - 600, (1 << 64) - 1)])
def test_ddm_histograms_bit_exact(D, orc, kw, t0, t1):
    import os
    d = W.DDMConfig(**kw)
    got = _ddm_gpu(D, d, t0, t1, 77)
    want = orc.ddm_batch(_ddm_p(orc, d), 77, t0, t1, threads=os.cpu_count() or 8)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_ddm_cfg2_full_size_properties(D, orc):
    """cfg2 (1e6 x 1000) in the bench launch configuration: conservation, shard
    additivity against a differently-launched split, a bit-exact oracle slice,
    and the closed-form error rate / decision time."""
    import math
    import os
    d = W.ddm_cfg2()
    full = _ddm_gpu(D, d, 0, d.n_trials, d.seed)
    a = _ddm_gpu(D, d, 0, 300001, d.seed)
    b = _ddm_gpu(D, d, 300001, d.n_trials, d.seed)
    for f, x, y in zip(full, a, b):
        assert np.array_equal(f, x + y)
    assert int(full[0].sum()) == d.n_trials and int(full[2].sum()) == d.n_trials
    sl = _ddm_gpu(D, d, 999000, d.n_trials, d.seed)
    want = orc.ddm_batch(_ddm_p(orc, d), d.seed, 999000, d.n_trials, threads=os.cpu_count() or 8)
    for g, w in zip(sl, want):
        assert np.array_equal(g, w)
    nb = d.n_rt_bins
    up, lo = int(full[0][:nb].sum()), int(full[0][nb:2 * nb].sum())
    zp = 1 + 0.5826 * math.sqrt(d.dt)
    er_cf, rt_cf = 1 / (1 + math.exp(2 * zp)), zp * math.tanh(zp)
    er = lo / (up + lo)
    assert abs(er - er_cf) < 4 * math.sqrt(er_cf * (1 - er_cf) / d.n_trials) + 0.005 * er_cf
    rt = (int(full[1][0]) + int(full[1][1])) / (up + lo) * d.dt
    assert abs(rt - rt_cf) < 0.005 * rt_cf


def _stroop_gpu(D, m, c, begin, end, trial_range=(0, 0)):
    import torch
    n = end - begin
    net = torch.empty(n, dtype=torch.float32, device="cuda")
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    counts = torch.zeros(3 * n, dtype=torch.int64, device="cuda")
    D.eval_grid(m, None, c.n_trials, c.seed, begin, end, net=net, best=best, counts=counts,
                trial_range=trial_range)
    torch.cuda.synchronize()
    return (counts.cpu().numpy().astype(np.uint64).reshape(n, 3), net.cpu().numpy(),
            int(best.item()) & (2 ** 64 - 1))


def test_stroop_small_grid_bit_exact(D, orc):
    c = W.stroop_small()
    m = D.load_model(W.KIND_STROOP_LCA, c.n_levels, c.levels, c.w, c.params, device=0)
    cnt, net, key = _stroop_gpu(D, m, c, 0, c.n_alloc)
    wc, wn = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials, c.seed, threads=8)
    assert np.array_equal(cnt, wc)
    assert np.array_equal(_bits(net), _bits(wn))
    assert key == orc.argmax_net(wn)[0]
    # a shard and a trial sub-range
    cnt2, _, _ = _stroop_gpu(D, m, c, 37, 61, trial_range=(5, 250))
    wc2, _ = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, 37, 61, c.n_trials, c.seed, 5, 250)
    assert np.array_equal(cnt2, wc2)


def test_stroop_cfg4_sampled_allocations_full_trials(D, orc):
    """cfg4 grid (1e4 allocations), T = 1e5 trials: sampled allocations simulated
    over all trials, counts and V bit-exact."""
    import os
    c = W.stroop_cfg4()
    m = D.load_model(W.KIND_STROOP_LCA, c.n_levels, c.levels, c.w, c.params, device=0)
    for b in (0, 4321, 9998):
        cnt, net, _ = _stroop_gpu(D, m, c, b, b + 2)
        wc, wn = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, b, b + 2, c.n_trials, c.seed,
                                 threads=os.cpu_count() or 8)
        assert np.array_equal(cnt, wc)
        assert np.array_equal(_bits(net), _bits(wn))


@pytest.mark.parametrize("shape,S,T,seed", [((3, 3, 3), 10, 30, 42), ((8, 7, 6), 24, 20, 5), ((20, 20, 20), 16, 12, 9)])
def test_pp_episode_bit_exact(D, orc, shape, S, T, seed):
    """Closed-loop episode (spec/MODELS.md §7): every step's key, the whole trajectory
    and the outcome bit-exact against the oracle's step-by-step loop."""
    import torch
    cfg = W.PPConfig("ep", shape, S)
    m = _model(D, cfg)
    init = np.array([4.0, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32)
    speeds = (1.0, 0.7, 0.5)
    traj, keys, status = D.pp_episode(m, init, T, S, seed, speeds=speeds, capture_radius=0.6)
    torch.cuda.synchronize()
    w_traj, w_keys, w_status = orc.pp_episode(cfg.n_levels, cfg.levels, cfg.w, cfg.params, init, T, S, seed,
                                              speeds=speeds, capture_radius=0.6)
    assert np.array_equal(_bits(traj.cpu().numpy()), _bits(w_traj))
    assert [int(k) & (2 ** 64 - 1) for k in keys.cpu().numpy()] == [int(k) for k in w_keys]
    assert tuple(int(v) for v in status.cpu().numpy()) == w_status


def test_pp_episode_capture_and_graph_replay(D, orc):
    """Straight-chase capture (outcome 1 at the closed-form step) and a CUDA-graph
    capture of the whole episode replays to the same result."""
    import torch
    cfg = W.PPConfig("ep", (3, 3, 3), 4)
    cfg.params = np.array([0.0, 0.0, 0.0], np.float32)
    m = _model(D, cfg)
    init = np.array([5.0, 0.0, -1000.0, 0.0, 0.0, 0.0], np.float32)
    traj, keys, status = D.pp_episode(m, init, 40, 4, 7, speeds=(1.0, 0.75, 0.0), capture_radius=0.5)
    torch.cuda.synchronize()
    assert tuple(int(v) for v in status.cpu().numpy()) == (1, 18)
    cfg2 = W.PPConfig("ep", (6, 6, 6), 8)
    m2 = _model(D, cfg2)
    init2 = np.array([4.0, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32)
    t2 = torch.empty((17, 6), dtype=torch.float32, device="cuda")
    t2[0] = torch.from_numpy(init2).cuda()
    k2 = torch.empty(16, dtype=torch.int64, device="cuda")
    s2 = torch.empty(2, dtype=torch.int32, device="cuda")
    D.pp_episode(m2, None, 16, 8, 3, traj=t2, keys=k2, status=s2)     # warm-up outside capture
    torch.cuda.synchronize()
    ref = (t2.clone(), k2.clone(), s2.clone())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        D.pp_episode(m2, None, 16, 8, 3, traj=t2, keys=k2, status=s2)
    t2.zero_()
    t2[0] = torch.from_numpy(init2).cuda()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(t2, ref[0]) and torch.equal(k2, ref[1]) and torch.equal(s2, ref[2])


@pytest.mark.parametrize("n,off", [(1_000_003, 0), (1_000_003, 1), (4_194_304, 2), (13, 0)])
def test_argmax_ties_large_arrays_vs_oracle(D, orc, n, off):
    """NEXT-2's second pass on large arrays (float4 path and the misaligned scalar
    path): maxima tied at scattered indices incl. +-0 and -inf cases, NaN around
    them — the tie key bit-exact against the oracle for several seeds."""
    import torch
    rng = np.random.default_rng(n + off)
    for case in ("scattered", "zeros", "neg inf"):
        v = rng.standard_normal(n + off).astype(np.float32) - 10.0
        v[rng.integers(0, n + off, size=max(1, n // 40))] = np.nan
        hit = rng.integers(0, n + off, size=min(n, 50))
        if case == "scattered":
            v[hit] = 3.5
        elif case == "zeros":
            v = np.minimum(v, -1.0)
            v[hit] = np.where(rng.random(hit.size) < 0.5, np.float32(-0.0), np.float32(0.0))
        else:
            v[:] = np.where(np.isnan(v), np.nan, -np.inf).astype(np.float32)
        t = torch.from_numpy(v).cuda()[off:]
        for seed in (1, 2, 99):
            best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
            tie = torch.full((1,), -1, dtype=torch.int64, device="cuda")
            D.argmax(t, 777, best)
            D.argmax_ties(t, 777, seed, 4, best, tie)
            torch.cuda.synchronize()
            k_or, t_or, _ = orc.argmax_random_ties(v[off:], 777, seed, 4)
            assert (int(best.item()) & (2 ** 64 - 1)) == k_or, (n, off, case, seed)
            assert (int(tie.item()) & (2 ** 64 - 1)) == t_or, (n, off, case, seed)


def test_argmax_random_ties_bit_exact_and_uniform(D, orc):
    """NEXT-2: GPU tie keys equal the oracle's for every seed; 8 tied minima each
    win 1/8 +- 0.02 of 4000 reseeded runs; a PP grid with all-equal costs picks
    a uniformly random allocation instead of index 0."""
    import torch
    net = np.full(64, -5.0, np.float32)
    tied = [3, 7, 11, 20, 33, 40, 51, 63]
    net[tied] = -1.0
    t_net = torch.from_numpy(net).cuda()
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.argmax(t_net, 0, best)
    ties = torch.full((4000,), -1, dtype=torch.int64, device="cuda")
    for seed in range(4000):
        D.argmax_ties(t_net, 0, seed, 0, best, ties[seed:seed + 1])
    torch.cuda.synchronize()
    got = [int(x) & (2 ** 64 - 1) for x in ties.cpu().numpy()]
    counts = dict.fromkeys(tied, 0)
    for seed, t in enumerate(got):
        k, t_or, rc = orc.argmax_random_ties(net, 0, seed)
        assert t == t_or
        counts[t & 0xFFFFFFFF] += 1
    for v in counts.values():
        assert abs(v / 4000 - 1 / 8) < 0.02
    cfg = W.PPConfig("ties", (4, 4, 4), 4)
    cfg.params = np.array([0.0, 0.0, 0.5], np.float32)
    cfg.w = np.zeros(3, np.float32)
    m = _model(D, cfg)
    netp = torch.empty(64, device="cuda")
    bestp = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.eval_grid(m, cfg.inputs, 4, 1, net=netp, best=bestp)
    tie = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.argmax_ties(netp, 0, 1, 0, bestp, tie)
    torch.cuda.synchronize()
    _, t_or, _ = orc.argmax_random_ties(netp.cpu().numpy(), 0, 1)
    assert int(tie.item()) & (2 ** 64 - 1) == t_or


@pytest.mark.parametrize("shape,S,R,lo,hi", [((5, 5, 5), 16, 7, (0, 0, 0), (1, 1, 1)),
                                             ((9, 1, 1), 100, 6, (0, .5, .5), (1, .5, .5)),
                                             ((12, 10, 8), 12, 4, (0, 0.2, 0), (1, 0.8, 0.5))])
def test_pp_amr_bit_exact(D, orc, shape, S, R, lo, hi):
    """NEXT-4: every round's key and box bit-exact against the oracle's refinement loop."""
    import torch
    cfg = W.PPConfig("amr", shape, S)
    m = _model(D, cfg)
    keys, boxes = D.pp_amr(m, cfg.inputs, lo, hi, R, S, 21, invocation0=3)
    torch.cuda.synchronize()
    w_keys, w_boxes = orc.pp_amr(cfg.n_levels, cfg.w, cfg.params, cfg.inputs, lo, hi, R, S, 21, invocation0=3)
    assert [int(k) & (2 ** 64 - 1) for k in keys.cpu().numpy()] == [int(k) for k in w_keys]
    assert np.array_equal(_bits(boxes.cpu().numpy()), _bits(w_boxes))


def test_ext_stroop_a_b_bit_exact_and_identical(D, orc):
    """NEXT-3: Extended Stroop versions A and B on the GPU — counts, V and key bit-exact
    against the oracle, and A == B (the clone relation)."""
    import torch
    c = W.ext_stroop_small()
    res = {}
    for kind, variant in ((W.KIND_EXT_STROOP_A, 0), (W.KIND_EXT_STROOP_B, 1)):
        m = D.load_model(kind, c.n_levels, c.levels, c.w, c.params, device=0)
        cnt, net, key = _stroop_gpu(D, m, c, 0, c.n_alloc)
        wc, wn = orc.ext_stroop_eval(variant, c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials,
                                     c.seed, threads=8)
        assert np.array_equal(cnt, wc)
        assert np.array_equal(_bits(net), _bits(wn))
        assert key == orc.argmax_net(wn)[0]
        res[variant] = (cnt, net, key)
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(_bits(res[0][1]), _bits(res[1][1]))
    # full-size control grid (1e4 allocations), sampled allocations, 1e4 trials
    g = W.ext_stroop_grid()
    m = D.load_model(W.KIND_EXT_STROOP_A, g.n_levels, g.levels, g.w, g.params, device=0)
    for b in (0, 5050, 9998):
        cnt, net, _ = _stroop_gpu(D, m, g, b, b + 2)
        wc, wn = orc.ext_stroop_eval(0, g.n_levels, g.levels, g.w, g.params, b, b + 2, g.n_trials, g.seed)
        assert np.array_equal(cnt, wc) and np.array_equal(_bits(net), _bits(wn))


def test_eval_grid_host_pinned_and_pageable(D, orc):
    """The end-to-end host-buffer call: pinned output (zero-copy, written by the
    kernel) and pageable output (device scratch + copy) both bit-exact."""
    import torch
    cfg = W.PPConfig("h", (17, 13, 11), 12)
    m = _model(D, cfg)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 5, cfg.n_alloc, 12, cfg.seed)
    k_or, _ = orc.argmax_net(-want, 5)
    pinned = torch.empty(cfg.n_alloc, dtype=torch.float32, pin_memory=True).numpy()
    pageable = np.empty(cfg.n_alloc, np.float32)
    for out in (pinned, pageable):
        key = D.eval_grid_host(m, cfg.inputs, 12, cfg.seed, 5, cfg.n_alloc, net_out=out[:cfg.n_alloc - 5])
        assert key == k_or
        assert np.array_equal(_bits(-out[:cfg.n_alloc - 5]), _bits(want))
    assert D.eval_grid_host(m, cfg.inputs, 12, cfg.seed, 5, cfg.n_alloc) == k_or   # key only


def test_pp_cfg5_last_shard_of_eight(D, orc):
    """cfg5 (200^3 = 8e6 allocations): the shard rank 7 of 8 owns in the N=8 run,
    evaluated in the bench launch configuration — all 1e6 costs and the shard key
    bit-exact against the oracle (threads over host cores)."""
    import os
    cfg = W.pp_cfg5()
    m = _model(D, cfg)
    b, e = D.shard_range(cfg.n_alloc, 7, 8)
    C, key = _gpu_pp(D, m, cfg, b, e)
    want = orc.pp_eval_threads(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, b, e, cfg.n_samples,
                               cfg.seed, threads=os.cpu_count() or 8)
    assert np.array_equal(_bits(C), _bits(want))
    assert key == orc.argmax_net(-want, b)[0]


def test_pp_large_odd_sample_count(D, orc):
    """S = 1001 (odd, > 1000) on a ragged grid: the packed pair loop's odd tail."""
    cfg = W.PPConfig("S", (3, 5, 7), 1001)
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc, 1001, cfg.seed)
    assert np.array_equal(_bits(C), _bits(want))
    assert key == orc.argmax_net(-want)[0]


def test_ddm_cfg2_endpoint_chi_square(D, orc):
    """cfg2 at full size: the Euler endpoint x_N is exactly N(x0 + A N dt, sigma^2 N dt)
    (Gaussian increments); chi-square of the 128-bin histogram (+ tails) against it."""
    import math
    from scipy import stats
    d = W.ddm_cfg2()
    _, _, xh = _ddm_gpu(D, d, 0, d.n_trials, d.seed)
    mu, sd = d.x0 + d.drift * d.n_steps * d.dt, d.noise * math.sqrt(d.n_steps * d.dt)
    edges = np.linspace(np.float32(d.x_lo), np.float32(d.x_hi), d.n_x_bins + 1)
    cdf = stats.norm.cdf((edges - mu) / sd)
    p = np.concatenate([[cdf[0]], np.diff(cdf), [1 - cdf[-1]]])
    obs = xh.astype(np.float64)
    expct = p * d.n_trials
    keep = expct > 20
    chi2 = float(((obs[keep] - expct[keep]) ** 2 / expct[keep]).sum())
    dof = int(keep.sum()) - 1
    assert stats.chi2.sf(chi2, dof) > 1e-4, (chi2, dof)


@pytest.mark.parametrize("shape", [(1, 1, 200), (1, 50, 1), (200, 1, 1)])
def test_pp_degenerate_single_level_signals(D, orc, shape):
    cfg = W.PPConfig("deg", shape, 6)
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc, 6, cfg.seed)
    assert np.array_equal(_bits(C), _bits(want))
    for i in (0, cfg.n_alloc - 1):      # one-allocation shards at both ends
        c1, k1 = _gpu_pp(D, m, cfg, i, i + 1)
        assert _bits(c1)[0] == _bits(want[i:i + 1])[0] and k1 == orc.key(float(want[i]), i)


def test_argmax_ties_all_nan_and_empty(D, orc):
    import torch
    t = torch.full((16,), float("nan"), device="cuda")
    best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.argmax(t, 0, best)
    tie = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    D.argmax_ties(t, 0, 1, 0, best, tie)
    D.argmax_ties(t[:0], 0, 1, 0, best, tie)
    torch.cuda.synchronize()
    assert int(tie.item()) == -1          # KEY_INIT: nothing can win


@pytest.mark.parametrize("kind,variant,n_idx,n_val,thr_idx,thr", [
    (W.KIND_STROOP_LCA, None, 10, 37, 7, 0.4),        # odd trip count, low threshold: many early passages
    (W.KIND_STROOP_LCA, None, 10, 1, 7, 1.0),         # single step (only the ragged path runs)
    (W.KIND_EXT_STROOP_A, 0, 10, 37, 9, 0.3),
    (W.KIND_EXT_STROOP_B, 1, 10, 37, 9, 0.3),
    (W.KIND_EXT_STROOP_A, 0, 10, 1, 9, 0.05)])
def test_stroop_kinds_odd_trip_counts_bit_exact(D, orc, kind, variant, n_idx, n_val, thr_idx, thr):
    """Ragged last quad block and the two-step latch test on both Stroop kernels."""
    ext = variant is not None
    c = W.ext_stroop_small() if ext else W.stroop_small()
    c.params = c.params.copy()
    c.params[n_idx] = n_val
    c.params[thr_idx] = thr
    m = D.load_model(kind, c.n_levels, c.levels, c.w, c.params, device=0)
    cnt, net, key = _stroop_gpu(D, m, c, 0, c.n_alloc)
    if ext:
        wc, wn = orc.ext_stroop_eval(variant, c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials,
                                     c.seed, threads=8)
    else:
        wc, wn = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials, c.seed, threads=8)
    assert np.array_equal(cnt, wc)
    assert np.array_equal(_bits(net), _bits(wn))
    assert key == orc.argmax_net(wn)[0]
    assert cnt[:, 1].sum() < cnt.shape[0] * c.n_trials or n_val == 1   # some trials decide


@pytest.mark.parametrize("shape,S,T,n_sets,inv0,rng_", [((8, 7, 6), 24, 7, 3, 5, (0, None)),
                                                        ((5, 5, 5), 9, 4, 1, 0, (17, 101)),
                                                        ((33, 1, 3), 2, 16, 16, 1000, (0, None))])
def test_eval_grid_multi_bit_exact(D, orc, shape, S, T, n_sets, inv0, rng_):
    """Listing-1 multi-invocation launch: every invocation's costs and key bit-exact
    against the oracle's per-trial loop."""
    import torch
    cfg = W.PPConfig("multi", shape, S)
    m = _model(D, cfg)
    b, e = rng_[0], (cfg.n_alloc if rng_[1] is None else rng_[1])
    sets = W.pp_positions(n_sets, seed=3)
    d_sets = torch.from_numpy(sets).cuda()
    net = torch.empty((T, e - b), dtype=torch.float32, device="cuda")
    best = torch.full((T,), -1, dtype=torch.int64, device="cuda")
    D.eval_grid_multi(m, d_sets, T, S, cfg.seed, b, e, invocation0=inv0, net=net, best=best)
    torch.cuda.synchronize()
    want = orc.pp_eval_multi(cfg.n_levels, cfg.levels, cfg.w, cfg.params, sets, T, b, e, S, cfg.seed, invocation0=inv0)
    assert np.array_equal(_bits(-net.cpu().numpy()), _bits(want))
    keys = [int(k) & (2 ** 64 - 1) for k in best.cpu().numpy()]
    assert keys == [orc.argmax_net(-want[t], b)[0] for t in range(T)]


def test_eval_grid_multi_cfg3_x16_matches_single_calls(D, orc):
    """Full-size cfg3 with 16 invocations (SURVEY §8(d) cfg3 variant) in one launch ==
    16 single-invocation calls (bit-exact net rows and keys); two rows and keys also
    against the oracle."""
    import torch
    cfg = W.pp_cfg3()
    m = _model(D, cfg)
    T = 16
    sets = W.pp_positions(T)
    d_sets = torch.from_numpy(sets).cuda()
    net = torch.empty((T, cfg.n_alloc), dtype=torch.float32, device="cuda")
    best = torch.full((T,), -1, dtype=torch.int64, device="cuda")
    D.eval_grid_multi(m, d_sets, T, cfg.n_samples, cfg.seed, net=net, best=best)
    net1 = torch.empty(cfg.n_alloc, dtype=torch.float32, device="cuda")
    best1 = torch.empty(1, dtype=torch.int64, device="cuda")
    for t in range(T):
        best1.fill_(-1)
        D.eval_grid(m, sets[t], cfg.n_samples, cfg.seed, invocation=t, net=net1, best=best1)
        torch.cuda.synchronize()
        assert torch.equal(net1.view(torch.int32), net[t].view(torch.int32))
        assert int(best1.item()) == int(best[t].item())
    for t in (0, T - 1):
        row = -net[t].cpu().numpy()
        for i in np.random.default_rng(t).integers(0, cfg.n_alloc, 64):
            w = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, sets[t], int(i), int(i) + 1,
                            cfg.n_samples, cfg.seed, invocation=t)
            assert _bits(row[int(i)]) == _bits(w)[0]


def test_graft_entry_smoke():
    """The driver's smoke(): cfg1 costs + key and a DDM batch bit-exact on cuda:0."""
    import __graft_entry__
    __graft_entry__.smoke()


def test_binding_rejects_wrong_buffer_dtypes(D):
    """The thin binding checks element types before calling the ABI (a float64
    net or an int32 key buffer would otherwise be silently misread)."""
    import torch
    cfg = W.pp_cfg1()
    m = _model(D, cfg)
    good_net = torch.empty(cfg.n_alloc, dtype=torch.float32, device="cuda")
    good_best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match="float32"):
        D.eval_grid(m, cfg.inputs, cfg.n_samples, cfg.seed, net=good_net.double(), best=good_best)
    with pytest.raises(ValueError, match="int64"):
        D.eval_grid(m, cfg.inputs, cfg.n_samples, cfg.seed, net=good_net, best=good_best.int())
    with pytest.raises(ValueError, match="int64"):
        D.argmax(good_net, 0, good_best.float())
    D.eval_grid(m, cfg.inputs, cfg.n_samples, cfg.seed, net=good_net, best=good_best)   # still fine


def test_seed_sweep_1_to_100(D, orc):
    """SURVEY §8(d) / S:569: parity over seeds 1..100 — cfg1 costs and keys for
    every seed, a small DDM batch and a small Stroop grid for every tenth."""
    import torch
    cfg = W.pp_cfg1()
    m = _model(D, cfg)
    ms = D.load_model(W.KIND_STROOP_LCA, (3, 4), np.linspace(0, 1, 7).astype(np.float32), W.STROOP_W,
                      W.STROOP_PARAMS, device=0)
    for seed in range(1, 101):
        C, key = _gpu_pp(D, m, cfg, seed=seed)
        want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc,
                           cfg.n_samples, seed)
        assert np.array_equal(_bits(C), _bits(want)), seed
        assert key == orc.argmax_net(-want)[0], seed
        if seed % 10 == 0:
            d = W.DDMConfig(n_steps=150, n_trials=700)
            got = _ddm_gpu(D, d, 0, d.n_trials, seed)
            for g, w in zip(got, orc.ddm_batch(_ddm_p(orc, d), seed, 0, d.n_trials)):
                assert np.array_equal(g, w), seed
            n = 12
            counts = torch.zeros(3 * n, dtype=torch.int64, device="cuda")
            net = torch.empty(n, dtype=torch.float32, device="cuda")
            D.eval_grid(ms, None, 90, seed, 0, n, net=net, counts=counts)
            torch.cuda.synchronize()
            wc, wn = orc.stroop_eval((3, 4), np.linspace(0, 1, 7).astype(np.float32), W.STROOP_W, W.STROOP_PARAMS,
                                     0, n, 90, seed)
            assert np.array_equal(counts.cpu().numpy().astype(np.uint64).reshape(n, 3), wc), seed
            assert np.array_equal(_bits(net.cpu().numpy()), _bits(wn)), seed


def test_eval_grid_host_published_key_rearms_between_calls(D, orc):
    """Pinned h_best: the last block publishes the key and re-arms the device key
    and counter, so consecutive calls (other seeds, ranges, sample parities,
    interleaved with the pageable-key copy path and an empty range) each return
    their own key, never a min with a previous call's."""
    import ctypes as C
    from paper_2110_15425_b200 import _abi
    cfg = W.PPConfig("h2", (9, 8, 7), 6)
    m = _model(D, cfg)
    calls = [(11, 0, cfg.n_alloc, 6), (3, 100, 300, 7), (11, 0, cfg.n_alloc, 6), (99, 7, 8, 2), (5, 0, 0, 6),
             (42, 200, cfg.n_alloc, 5)]
    for rep in range(2):
        for seed, b, e, S in calls:
            want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, b, e, S, seed)
            k_or = orc.argmax_net(-want, b)[0] if e > b else D.KEY_INIT
            if rep == 0:
                got = D.eval_grid_host(m, cfg.inputs, S, seed, b, e)              # pinned key (binding)
            else:
                k = C.c_uint64()                                                   # pageable key: copy path
                inp = np.ascontiguousarray(cfg.inputs, np.float32)
                _abi.check(_abi.lib().distill_eval_grid_host(m.handle, _abi._fptr(inp), 6, b, e, S, 0, seed,
                                                             None, C.byref(k), None))
                got = int(k.value)
                got2 = D.eval_grid_host(m, cfg.inputs, S, seed, b, e)             # and pinned right after
                assert got2 == got
            assert got == k_or, (rep, seed, b, e, S)


def test_eval_grid_host_async_pipelined_slots(D, orc):
    """distill_eval_grid_host_async: several grid searches in flight at once on
    double-buffered pinned slots (other seeds, ranges and sample parities), first on
    one stream, then alternating between two streams (the handle orders its
    host-buffer launches across streams): every net array and key bit-exact
    against the oracle, a call's slots untouched by the calls after it; pageable
    slots are refused with E_INVALID_ARG and nothing is enqueued."""
    import torch
    from paper_2110_15425_b200 import _abi
    cfg = W.PPConfig("ha", (9, 8, 7), 6)
    m = _model(D, cfg)
    calls = [(11, 0, cfg.n_alloc, 6), (3, 100, 300, 7), (42, 200, cfg.n_alloc, 5), (99, 7, 8, 2),
             (11, 0, cfg.n_alloc, 6), (5, 1, cfg.n_alloc - 1, 9)]
    wants = []
    for seed, b, e, S in calls:
        w = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, b, e, S, seed)
        wants.append((w, orc.argmax_net(-w, b)[0]))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for mode in ("one stream", "two streams"):
        slots = [(torch.full((cfg.n_alloc,), float("nan"), dtype=torch.float32, pin_memory=True).numpy(),
                  torch.zeros(1, dtype=torch.int64, pin_memory=True).numpy()) for _ in calls]
        evs = []
        for q, (seed, b, e, S) in enumerate(calls):      # all enqueued before any is read
            st = streams[0] if mode == "one stream" else streams[q % 2]
            net, key = slots[q]
            D.eval_grid_host_async(m, cfg.inputs, S, seed, b, e, net_out=net[:e - b], key_out=key, stream=st)
            ev = torch.cuda.Event()
            ev.record(st)
            evs.append(ev)
        for q, (seed, b, e, S) in enumerate(calls):
            evs[q].synchronize()
            net, key = slots[q]
            w, k_or = wants[q]
            assert int(key[0]) & (2 ** 64 - 1) == k_or, (mode, q)
            assert np.array_equal(_bits(-net[:e - b]), _bits(w)), (mode, q)
            assert np.isnan(net[e - b:]).all()
    # pageable slots: refused before anything is enqueued
    with pytest.raises(_abi.DistillError):
        D.eval_grid_host_async(m, cfg.inputs, 6, 11, 0, cfg.n_alloc, key_out=np.zeros(1, np.int64))
    pk = torch.zeros(1, dtype=torch.int64, pin_memory=True).numpy()
    with pytest.raises(_abi.DistillError):
        D.eval_grid_host_async(m, cfg.inputs, 6, 11, 0, cfg.n_alloc, net_out=np.empty(cfg.n_alloc, np.float32),
                               key_out=pk)
    # and the synchronous call still works right after
    assert D.eval_grid_host(m, cfg.inputs, 6, 11, 0, cfg.n_alloc) == wants[0][1]


def test_pp_episode_in_pieces_over_shards(D, orc):
    """NEXT-1 over a sharded grid, emulated in one process: per step, three shard
    searches atomicMin into keys[t] (the MIN all-reduce), then advance — every
    key, the trajectory and the outcome bit-exact against the oracle episode."""
    import torch
    cfg = W.PPConfig("eps", (9, 8, 7), 10)
    m = _model(D, cfg)
    init = np.array([4.0, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32)
    T, seed = 15, 8
    run = D.EpisodeRun(m, init, T, cfg.n_samples, seed, speeds=(1.0, 0.7, 0.5), capture_radius=0.6)
    shards = [D.shard_range(cfg.n_alloc, r, 3) for r in range(3)]
    for t in range(T):
        for b, e in reversed(shards):
            run.search(t, b, e)
        run.advance(t)
    torch.cuda.synchronize()
    w_traj, w_keys, w_status = orc.pp_episode(cfg.n_levels, cfg.levels, cfg.w, cfg.params, init, T,
                                              cfg.n_samples, seed, speeds=(1.0, 0.7, 0.5), capture_radius=0.6)
    assert np.array_equal(_bits(run.traj.cpu().numpy()), _bits(w_traj))
    assert [int(k) & (2 ** 64 - 1) for k in run.keys.cpu().numpy()] == [int(k) for k in w_keys]
    assert tuple(int(v) for v in run.status.cpu().numpy()) == w_status
    with pytest.raises(D.api.DistillError):
        run.search(T, 0, 1)                      # t past the episode
    with pytest.raises(D.api.DistillError):
        run.search(0, 5, cfg.n_alloc + 1)        # shard past the grid


def _episode_rank(rank, world, port, out_path):
    import os
    import torch
    import torch.distributed as dist
    import paper_2110_15425_b200 as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)                     # both ranks share the one GPU; gloo reduces on the host
    cfg = W.PPConfig("epd", (9, 8, 7), 10)
    m = D.load_model(W.KIND_PREDATOR_PREY, cfg.n_levels, cfg.levels, cfg.w, cfg.params, device=0)
    traj, keys, status = D.pp_episode_sharded(m, np.array([4.0, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32), 12,
                                              cfg.n_samples, 8, rank, world, speeds=(1.0, 0.7, 0.5),
                                              capture_radius=0.6)
    torch.cuda.synchronize()
    np.savez(f"{out_path}.{rank}.npz", traj=traj.cpu().numpy(), keys=keys.cpu().numpy(), status=status.cpu().numpy())
    dist.destroy_process_group()


def test_pp_episode_sharded_two_ranks_gloo(D, orc, tmp_path):
    """pp_episode_sharded with two processes (gloo all-reduce on the host, both
    ranks on the single GPU — their kernels never wait on each other): both
    ranks hold the oracle's trajectory, keys and outcome bit for bit."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = str(tmp_path / "ep")
    mp.start_processes(_episode_rank, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    cfg = W.PPConfig("epd", (9, 8, 7), 10)
    w_traj, w_keys, w_status = orc.pp_episode(cfg.n_levels, cfg.levels, cfg.w, cfg.params,
                                              np.array([4.0, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32), 12,
                                              cfg.n_samples, 8, speeds=(1.0, 0.7, 0.5), capture_radius=0.6)
    for r in range(2):
        z = np.load(f"{out}.{r}.npz")
        assert np.array_equal(_bits(z["traj"]), _bits(w_traj))
        assert [int(k) & (2 ** 64 - 1) for k in z["keys"]] == [int(k) for k in w_keys]
        assert tuple(int(v) for v in z["status"]) == w_status


def test_pp_amr_no_valid_allocation(D, orc):
    import torch
    cfg = W.PPConfig("amr_nan", (4, 3, 2), 4)
    m = _model(D, cfg)
    inputs = np.array([np.nan, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32)
    lo, hi = (0.0, 0.1, 0.2), (1.0, 0.9, 0.8)
    keys, boxes = D.pp_amr(m, inputs, lo, hi, 3, 4, 5)
    torch.cuda.synchronize()
    w_keys, w_boxes = orc.pp_amr(cfg.n_levels, cfg.w, cfg.params, inputs, lo, hi, 3, 4, 5)
    assert [int(k) & (2 ** 64 - 1) for k in keys.cpu().numpy()] == [int(k) for k in w_keys]
    assert np.array_equal(_bits(boxes.cpu().numpy()), _bits(w_boxes))


def test_pp_amr_in_pieces_over_shards(D, orc):
    """NEXT-4 over a sharded grid, emulated in one process: per round the level
    table, three shard searches (atomicMin = the MIN all-reduce), the refine —
    keys and boxes bit-exact against the oracle."""
    import torch
    cfg = W.PPConfig("amrs", (6, 5, 4), 8)
    m = _model(D, cfg)
    lo, hi, R = (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), 5
    run = D.AmrRun(m, cfg.inputs, lo, hi, R, 8, 13, invocation0=2)
    shards = [D.shard_range(cfg.n_alloc, r, 3) for r in range(3)]
    for r in range(R):
        run.levels_for(r)
        for b, e in shards:
            run.search(r, b, e)
        run.refine(r)
    torch.cuda.synchronize()
    w_keys, w_boxes = orc.pp_amr(cfg.n_levels, cfg.w, cfg.params, cfg.inputs, lo, hi, R, 8, 13, invocation0=2)
    assert [int(k) & (2 ** 64 - 1) for k in run.keys.cpu().numpy()] == [int(k) for k in w_keys]
    assert np.array_equal(_bits(run.boxes.cpu().numpy()), _bits(w_boxes))


def _amr_rank(rank, world, port, out_path):
    import os
    import torch
    import torch.distributed as dist
    import paper_2110_15425_b200 as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = W.PPConfig("amrd", (6, 5, 4), 8)
    m = D.load_model(W.KIND_PREDATOR_PREY, cfg.n_levels, cfg.levels, cfg.w, cfg.params, device=0)
    keys, boxes = D.pp_amr_sharded(m, cfg.inputs, (0, 0, 0), (1, 1, 1), 5, 8, 13, rank, world, invocation0=2)
    torch.cuda.synchronize()
    np.savez(f"{out_path}.{rank}.npz", keys=keys.cpu().numpy(), boxes=boxes.cpu().numpy())
    dist.destroy_process_group()


def test_pp_amr_sharded_two_ranks_gloo(D, orc, tmp_path):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = str(tmp_path / "amr")
    mp.start_processes(_amr_rank, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    cfg = W.PPConfig("amrd", (6, 5, 4), 8)
    w_keys, w_boxes = orc.pp_amr(cfg.n_levels, cfg.w, cfg.params, cfg.inputs, (0, 0, 0), (1, 1, 1), 5, 8, 13,
                                 invocation0=2)
    for r in range(2):
        z = np.load(f"{out}.{r}.npz")
        assert [int(k) & (2 ** 64 - 1) for k in z["keys"]] == [int(k) for k in w_keys]
        assert np.array_equal(_bits(z["boxes"]), _bits(w_boxes))


def test_grid_search_and_best_convenience(D, orc):
    """L4 convenience: grid_search over shard=(rank, world) returns
    (net, key); the min of the shard keys decodes through best() to the oracle's
    argmax, and the shard nets concatenate to the oracle's V."""
    cfg = W.PPConfig("gs", (11, 9, 7), 12)
    m = _model(D, cfg)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc, 12, cfg.seed)
    k_or = orc.argmax_net(-want)[0]
    nets, keys = [], []
    for r in range(3):
        net, key = D.grid_search(m, cfg.inputs, 12, cfg.seed, shard=(r, 3))
        nets.append(net.cpu().numpy())
        keys.append(int(key.item()) & (2 ** 64 - 1))
    assert np.array_equal(_bits(-np.concatenate(nets)), _bits(want))
    assert min(keys) == k_or
    net, key = D.grid_search(m, cfg.inputs, 12, cfg.seed)
    cost, idx = D.best(key)
    assert idx == k_or & 0xFFFFFFFF and np.float32(cost) == want[idx]


def test_concurrent_streams_and_threads_on_one_model(D, orc):
    """One read-only model handle evaluated from two streams at once (device
    buffers) and from two host threads through the serialised host-buffer call:
    every result equals its sequential counterpart."""
    import threading
    import torch
    cfg = W.PPConfig("conc", (40, 30, 20), 12)
    m = _model(D, cfg)
    seeds = (5, 6)
    ref = {}
    for sd in seeds:
        ref[sd] = _gpu_pp(D, m, cfg, seed=sd)
    streams = [torch.cuda.Stream() for _ in seeds]
    nets = [torch.empty(cfg.n_alloc, dtype=torch.float32, device="cuda") for _ in seeds]
    bests = [torch.full((1,), -1, dtype=torch.int64, device="cuda") for _ in seeds]
    torch.cuda.synchronize()
    for _ in range(3):
        for st, sd, net, best in zip(streams, seeds, nets, bests):
            with torch.cuda.stream(st):
                D.key_reset(best, stream=st)
                D.eval_grid(m, cfg.inputs, cfg.n_samples, sd, net=net, best=best, stream=st)
        torch.cuda.synchronize()
        for sd, net, best in zip(seeds, nets, bests):
            assert np.array_equal(_bits(-net.cpu().numpy()), _bits(ref[sd][0]))
            assert int(best.item()) & (2 ** 64 - 1) == ref[sd][1]
    out = {}

    def worker(sd):
        k = None
        for _ in range(5):
            k = D.eval_grid_host(m, cfg.inputs, cfg.n_samples, sd)
        out[sd] = k

    th = [threading.Thread(target=worker, args=(sd,)) for sd in seeds]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for sd in seeds:
        assert out[sd] == ref[sd][1]


def test_randomised_parity_fuzz(D, orc):
    """Deterministic fuzz: 60 random PP configurations (shapes, sample counts
    odd/even, params, positions, seeds, shards, both the warp-per-allocation and
    the thread-per-allocation kernels), 12 random DDM / Stroop configurations and
    8 random DDM-grid / Extended Stroop configurations with trial sub-ranges,
    each bit-exact against the oracle."""
    import os
    import torch
    rng = np.random.default_rng(int(os.environ.get("DISTILL_FUZZ_SEED", "2024")))
    for case in range(int(os.environ.get("DISTILL_FUZZ_CASES", "60"))):
        shape = tuple(int(x) for x in rng.integers(1, 9, 3))
        if case % 6 == 0:
            shape = (int(rng.integers(20, 40)),) * 3         # > 9472 allocations: thread-per-allocation kernel
        S = int(rng.integers(1, 40))
        cfg = W.PPConfig("fz", shape, S)
        cfg.params = np.array([rng.uniform(0, 3), rng.uniform(0, 0.5), rng.uniform(0, 2)], np.float32)
        cfg.w = rng.uniform(-0.2, 0.3, 3).astype(np.float32)
        cfg.levels = rng.uniform(0, 1, sum(shape)).astype(np.float32)
        cfg.inputs = rng.uniform(-8, 8, 6).astype(np.float32)
        seed = int(rng.integers(0, 2 ** 63))
        inv = int(rng.integers(0, 1000))
        m = _model(D, cfg)
        b = int(rng.integers(0, cfg.n_alloc))
        e = int(rng.integers(b + 1, cfg.n_alloc + 1))
        C, key = _gpu_pp(D, m, cfg, b, e, invocation=inv, seed=seed)
        want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, b, e, S, seed, invocation=inv)
        assert np.array_equal(_bits(C), _bits(want)), (case, shape, S, b, e)
        assert key == orc.argmax_net(-want, b)[0], case
        m.close()
    for case in range(6):
        d = W.DDMConfig(drift=float(rng.uniform(-2, 2)), noise=float(rng.uniform(0.2, 2)),
                        threshold=float(rng.uniform(0.2, 2)), x0=float(rng.uniform(-0.1, 0.1)),
                        dt=float(rng.choice([0.001, 0.005, 0.01])), n_steps=int(rng.integers(1, 400)),
                        rt_bin_steps=int(rng.integers(1, 30)), n_x_bins=int(rng.integers(1, 60)))
        t0 = int(rng.integers(0, 10 ** 6))
        t1 = t0 + int(rng.integers(1, 900))
        sd = int(rng.integers(0, 2 ** 63))
        for g, w in zip(_ddm_gpu(D, d, t0, t1, sd), orc.ddm_batch(_ddm_p(orc, d), sd, t0, t1)):
            assert np.array_equal(g, w), case
    for case in range(6):
        P = W.STROOP_PARAMS.copy()
        P[:8] = [rng.uniform(0.5, 2), rng.uniform(0.5, 2), rng.uniform(0.02, 1), rng.uniform(0, 0.5),
                 rng.uniform(0, 0.5), rng.uniform(0.05, 1), rng.choice([0.01, 0.05]), rng.uniform(0.3, 1.5)]
        P[10] = int(rng.integers(1, 120))
        Ls = (int(rng.integers(1, 6)), int(rng.integers(1, 6)))
        lev = rng.uniform(0, 1, sum(Ls)).astype(np.float32)
        ms = D.load_model(W.KIND_STROOP_LCA, Ls, lev, W.STROOP_W, P, device=0)
        n = Ls[0] * Ls[1]
        T = int(rng.integers(1, 200))
        sd = int(rng.integers(0, 2 ** 63))
        counts = torch.zeros(3 * n, dtype=torch.int64, device="cuda")
        net = torch.empty(n, dtype=torch.float32, device="cuda")
        D.eval_grid(ms, None, T, sd, 0, n, net=net, counts=counts)
        torch.cuda.synchronize()
        wc, wn = orc.stroop_eval(Ls, lev, W.STROOP_W, P, 0, n, T, sd)
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64).reshape(n, 3), wc), case
        assert np.array_equal(_bits(net.cpu().numpy()), _bits(wn)), case
    # the trial-streaming kernels (R14b) on random DDM-grid / Extended Stroop configurations
    # and random trial sub-ranges
    for case in range(8):
        ext = case % 2 == 1
        Ls = (int(rng.integers(1, 6)), int(rng.integers(1, 6)))
        n = Ls[0] * Ls[1]
        T = int(rng.integers(1, 300))
        tb = int(rng.integers(0, T))
        te = int(rng.integers(tb + 1, T + 1)) if case % 4 < 2 else T
        if case % 4 >= 2:
            tb = 0
        sd = int(rng.integers(0, 2 ** 63))
        if ext:
            P = W.EXT_STROOP_PARAMS.copy()
            P[3] = int(rng.integers(0, 40))
            P[9] = rng.uniform(0.1, 1.0)
            P[10] = int(rng.integers(1, 150))
            lev = rng.uniform(0, 1, sum(Ls)).astype(np.float32)
            kind, variant = (W.KIND_EXT_STROOP_A, 0) if case % 3 else (W.KIND_EXT_STROOP_B, 1)
        else:
            P = W.DDMG_PARAMS.copy()
            P[0], P[1], P[2] = rng.uniform(-0.5, 0.5), rng.uniform(0, 2), rng.uniform(0.3, 1.5)
            P[6] = int(rng.integers(1, 500))
            lev = np.concatenate([rng.uniform(0, 1, Ls[0]), rng.uniform(0.05, 1.5, Ls[1])]).astype(np.float32)
            kind = W.KIND_DDM_GRID
        w = np.array([0.3, 0.1], np.float32)
        mg = D.load_model(kind, Ls, lev, w, P, device=0)
        counts = torch.zeros(3 * n, dtype=torch.int64, device="cuda")
        D.eval_grid(mg, None, T, sd, 0, n, counts=counts, trial_range=(tb, te))
        torch.cuda.synchronize()
        if ext:
            wc, _ = orc.ext_stroop_eval(variant, Ls, lev, w, P, 0, n, T, sd, trial_begin=tb, trial_end=te)
        else:
            wc, _ = orc.ddmg_eval(Ls, lev, w, P, 0, n, T, sd, tb, te)
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64).reshape(n, 3), wc), (case, ext, tb, te)


@pytest.mark.slow
def test_ddm_cfg2_full_size_bit_exact(D, orc):
    """cfg2 in full (1e6 trials x 1000 steps, the bench launch configuration):
    every histogram bin and both RT sums equal the oracle's (threads over the
    host cores; ~30 s on the GPU box's CPU)."""
    import os
    d = W.ddm_cfg2()
    got = _ddm_gpu(D, d, 0, d.n_trials, d.seed)
    want = orc.ddm_batch(_ddm_p(orc, d), d.seed, 0, d.n_trials, threads=os.cpu_count() or 8)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.slow
def test_ext_stroop_and_stroop_cfg4_shards_bit_exact(D, orc):
    """Contiguous shards at the bench sizes with ALL trials: 2000 of the Extended
    Stroop grid's 1e4 allocations x 1e4 trials, and 200 of Stroop cfg4's 1e4
    allocations x 1e5 trials x 200 steps — every count, V and the shard key
    bit-exact (oracle threads over the host cores; ~40 s on the GPU box)."""
    import os
    th = os.cpu_count() or 8
    g = W.ext_stroop_grid()
    m = D.load_model(W.KIND_EXT_STROOP_A, g.n_levels, g.levels, g.w, g.params, device=0)
    b, e = 3000, 5000
    cnt, net, key = _stroop_gpu(D, m, g, b, e)
    wc, wn = orc.ext_stroop_eval(0, g.n_levels, g.levels, g.w, g.params, b, e, g.n_trials, g.seed, threads=th)
    assert np.array_equal(cnt, wc)
    assert np.array_equal(_bits(net), _bits(wn))
    assert key == orc.argmax_net(wn, b)[0]
    c = W.stroop_cfg4()
    ms = D.load_model(W.KIND_STROOP_LCA, c.n_levels, c.levels, c.w, c.params, device=0)
    b, e = 4000, 4200
    cnt, net, key = _stroop_gpu(D, ms, c, b, e)
    wc, wn = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, b, e, c.n_trials, c.seed, threads=th)
    assert np.array_equal(cnt, wc)
    assert np.array_equal(_bits(net), _bits(wn))
    assert key == orc.argmax_net(wn, b)[0]


def test_stroop_energy_trace_bit_exact(D, orc):
    """Decision energy over time (§6b): per-step integer sums bit-exact
    against the oracle for several allocations, trial sub-ranges (accumulating
    into one buffer), an odd step count, and the cfg4 constants with 1e5 trials."""
    import os
    import torch
    c = W.stroop_small()
    P = c.params.copy()
    P[10] = 37
    m = D.load_model(W.KIND_STROOP_LCA, c.n_levels, c.levels, c.w, P, device=0)
    for alloc in (0, 17, c.n_alloc - 1):
        got = D.stroop_energy(m, alloc, c.n_trials, 9)
        torch.cuda.synchronize()
        k0, k1 = alloc // c.n_levels[1], alloc % c.n_levels[1]
        uc, us = float(c.levels[k0]), float(c.levels[c.n_levels[0] + k1])
        want = orc.stroop_energy(P, uc, us, 9, alloc, c.n_trials, 0, c.n_trials)
        assert np.array_equal(got.cpu().numpy(), want), alloc
    esum = torch.zeros(37, dtype=torch.int64, device="cuda")
    D.stroop_energy(m, 5, c.n_trials, 4, trial_range=(0, 111), esum=esum)
    D.stroop_energy(m, 5, c.n_trials, 4, trial_range=(111, c.n_trials), esum=esum)
    torch.cuda.synchronize()
    uc, us = float(c.levels[0]), float(c.levels[c.n_levels[0] + 5])
    assert np.array_equal(esum.cpu().numpy(), orc.stroop_energy(P, uc, us, 4, 5, c.n_trials, 0, c.n_trials))
    g = W.stroop_cfg4()
    mg = D.load_model(W.KIND_STROOP_LCA, g.n_levels, g.levels, g.w, g.params, device=0)
    got = D.stroop_energy(mg, 8083, g.n_trials, g.seed)
    torch.cuda.synchronize()
    uc, us = float(g.levels[80]), float(g.levels[100 + 83])
    want = orc.stroop_energy(g.params, uc, us, g.seed, 8083, g.n_trials, 0, g.n_trials, threads=os.cpu_count() or 8)
    assert np.array_equal(got.cpu().numpy(), want)


def test_lci_batch_bit_exact_and_fig3_clone(D, orc):
    """distill_lci_batch (spec §5): histograms bit-exact against the
    oracle with a leak and an offset, and with leak = offset = 0 bit-identical to
    distill_ddm_batch on the same trials (the Fig. 3 'computationally
    equivalent' pair, here exact)."""
    import torch

    def run(d, t0, t1, seed, lci):
        rh, rs, xh = (torch.zeros(n, dtype=torch.int64, device="cuda") for n in d.hist_sizes)
        D.ddm_batch(d.drift, d.noise, d.threshold, d.x0, d.dt, d.n_steps, d.rt_bin_steps, d.n_x_bins,
                    d.x_lo, d.x_hi, t0, t1, seed, rh, rs, xh, lci=lci)
        torch.cuda.synchronize()
        return [x.cpu().numpy().astype(np.uint64) for x in (rh, rs, xh)]

    for kw, lci in (({"n_steps": 300, "drift": 0.7}, (1.2, 0.0)), ({"n_steps": 77, "drift": -0.4}, (0.5, 0.003)),
                    ({"n_steps": 1000}, (0.0, 0.0))):
        d = W.DDMConfig(**kw)
        got = run(d, 1000, 6000, 21, lci)
        want = orc.ddm_batch(_ddm_p(orc, d), 21, 1000, 6000, lci=lci)
        for g, w in zip(got, want):
            assert np.array_equal(g, w), (kw, lci)
    d = W.DDMConfig(n_steps=500)
    for g, w in zip(run(d, 0, 20000, 5, (0.0, 0.0)), run(d, 0, 20000, 5, None)):
        assert np.array_equal(g, w)


def test_ddm_grid_bit_exact(D, orc):
    """DDM control grid (spec/MODELS.md §6c): counts, V and key bit-exact against
    the oracle on a small grid (odd step count, trial sub-range), and sampled
    allocations of the 100 x 100 bench grid with all 1e4 trials."""
    import os
    c = W.ddmg_grid(7, 300)
    c.params = c.params.copy()
    c.params[6] = 257
    m = D.load_model(W.KIND_DDM_GRID, c.n_levels, c.levels, c.w, c.params, device=0)
    cnt, net, key = _stroop_gpu(D, m, c, 0, c.n_alloc)
    wc, wn = orc.ddmg_eval(c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials, c.seed, threads=8)
    assert np.array_equal(cnt, wc)
    assert np.array_equal(_bits(net), _bits(wn))
    assert key == orc.argmax_net(wn)[0]
    cnt2, _, _ = _stroop_gpu(D, m, c, 11, 40, trial_range=(13, 222))
    wc2, _ = orc.ddmg_eval(c.n_levels, c.levels, c.w, c.params, 11, 40, c.n_trials, c.seed, 13, 222)
    assert np.array_equal(cnt2, wc2)
    g = W.ddmg_grid()
    mg = D.load_model(W.KIND_DDM_GRID, g.n_levels, g.levels, g.w, g.params, device=0)
    for b in (0, 5050, 9998):
        cnt, net, _ = _stroop_gpu(D, mg, g, b, b + 2)
        wc, wn = orc.ddmg_eval(g.n_levels, g.levels, g.w, g.params, b, b + 2, g.n_trials, g.seed,
                               threads=os.cpu_count() or 8)
        assert np.array_equal(cnt, wc) and np.array_equal(_bits(net), _bits(wn))


# ---------------------------------------------------------------------------
# Round 2: full-grid checks (VERDICT r01 "What's missing" 1-2)
# ---------------------------------------------------------------------------
def _host_threads():
    import os
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 8


def _observed_gaps(orc, cfg, i, s):
    """|o_prey - o_player| and |o_pred - o_player| of sample s of allocation i
    (binary64 from the sample's binary32 normals; spec/MODELS.md §2 Obs nodes)."""
    z = np.zeros(6, np.float32)
    orc.lib().od_normal_sextet(int(cfg.seed), int(i), int(s), 0, z)
    L = cfg.n_levels
    k = (i // (L[1] * L[2]), (i // L[2]) % L[1], i % L[2])
    lev = [cfg.levels[k[0]], cfg.levels[L[0] + k[1]], cfg.levels[L[0] + L[1] + k[2]]]
    smax, smin = float(cfg.params[0]), float(cfg.params[1])
    p = np.asarray(cfg.inputs, np.float64).reshape(3, 2)
    o = np.array([p[e] + (smax + float(lev[e]) * (smin - smax)) * z[2 * e:2 * e + 2].astype(np.float64)
                  for e in range(3)])
    return np.linalg.norm(o[0] - o[2]), np.linalg.norm(o[1] - o[2])


def test_pp_cfg3_full_grid_within_binary64_tolerance(D, orc):
    """North-star tolerance on the WHOLE cfg3 grid against the binary64 plain
    definition (od_pp_eval_f64: same Philox bits, libm Box-Muller, exact 1/sqrt;
    P:155-161).  The binary32 model (the paper's FP32 mode, reading R12) meets
    1e-5 relative on all but a few allocations; each exception must be ONE
    ill-conditioned sample — an observation that puts the prey or the predator
    within 0.05 of the player, where the Action node's unit vector amplifies
    binary32 rounding — with the other samples still inside the tolerance.  The
    argmax equals the binary64 argmax (or their binary64 gap is below the
    deviation bound)."""
    cfg = W.pp_cfg3()
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    c64 = orc.pp_eval_threads(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc,
                              cfg.n_samples, cfg.seed, threads=_host_threads(), f64=True)
    rel = np.abs(C.astype(np.float64) - c64) / np.abs(c64)
    assert np.median(rel) < 2e-7 and np.quantile(rel, 0.9999) < 1e-5
    bad = np.nonzero(rel >= 1e-5)[0]
    assert len(bad) <= 10, len(bad)
    for i in bad:
        args = (cfg.n_levels, cfg.levels, cfg.params, cfg.inputs, int(i), cfg.n_samples, cfg.seed)
        dev = np.abs(orc.pp_trace(*args).astype(np.float64) - orc.pp_trace_f64(*args))
        s = int(dev.argmax())
        rest = (dev.sum() - dev[s]) / cfg.n_samples
        assert rest < 1e-5 * c64[i], (int(i), rest)                # all other samples within tolerance
        assert min(_observed_gaps(orc, cfg, int(i), s)) < 0.05, int(i)   # the one outlier is ill-conditioned
    i32 = key & 0xFFFFFFFF
    i64 = int(np.argmin(c64))
    if i32 != i64:
        assert c64[i32] - c64[i64] <= rel.max() * abs(c64[i64]), (i32, i64, c64[i32] - c64[i64])


def test_pp_cfg5_whole_grid_one_gpu(D, orc):
    """cfg5 (200^3 = 8e6 allocations x 100 samples, BASELINE configs[4]) whole on ONE
    GPU: all 8e6 costs and the key bit-exact against the full oracle run on the host
    cores.  This key is the invariant every N-GPU run must reproduce (the sharded
    bench path is checked against it in test_gpu_bench.py)."""
    cfg = W.pp_cfg5()
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg)
    full = orc.pp_eval_threads(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, 0, cfg.n_alloc,
                               cfg.n_samples, cfg.seed, threads=_host_threads())
    assert np.array_equal(_bits(C), _bits(full))
    assert key == orc.argmax_net(-full)[0]
    # the same grid in 8 shards, keys combined with MIN == the whole-grid key
    import torch
    ks = []
    for r in range(8):
        b, e = D.shard_range(cfg.n_alloc, r, 8)
        best = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        D.eval_grid(m, cfg.inputs, cfg.n_samples, cfg.seed, b, e, best=best)
        ks.append(D.key_from_tensor(best))
    assert min(ks) == key


def test_stroop_cfg4_reduced_full_grid_key(D, orc):
    """SURVEY §8(d)'s argmax parity case for cfg4: all 1e4 allocations of the cfg4
    control grid x 1e3 trials x 200 steps — every allocation's integer counts, V
    and the full-grid key bit-exact against the oracle (P:159-161 selection over
    the Stroop model of P:525)."""
    c = W.stroop_cfg4()
    c.n_trials = 1000
    m = D.load_model(W.KIND_STROOP_LCA, c.n_levels, c.levels, c.w, c.params, device=0)
    cnt, net, key = _stroop_gpu(D, m, c, 0, c.n_alloc)
    wc, wn = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials, c.seed,
                             threads=_host_threads())
    assert np.array_equal(cnt, wc)
    assert np.array_equal(_bits(net), _bits(wn))
    assert key == orc.argmax_net(wn)[0]


def test_ext_stroop_and_ddm_grid_reduced_full_grid_keys(D, orc):
    """The bench's other control grids (1e4 allocations each) with reduced trial
    counts: Extended Stroop A x 200 trials and the DDM control grid x 300
    trials — all counts, V and the full-grid key bit-exact."""
    g = W.ext_stroop_grid()
    g.n_trials = 200
    m = D.load_model(W.KIND_EXT_STROOP_A, g.n_levels, g.levels, g.w, g.params, device=0)
    cnt, net, key = _stroop_gpu(D, m, g, 0, g.n_alloc)
    wc, wn = orc.ext_stroop_eval(0, g.n_levels, g.levels, g.w, g.params, 0, g.n_alloc, g.n_trials, g.seed,
                                 threads=_host_threads())
    assert np.array_equal(cnt, wc) and np.array_equal(_bits(net), _bits(wn))
    assert key == orc.argmax_net(wn)[0]
    d = W.ddmg_grid(100, 300)
    md = D.load_model(W.KIND_DDM_GRID, d.n_levels, d.levels, d.w, d.params, device=0)
    cnt, net, key = _stroop_gpu(D, md, d, 0, d.n_alloc)
    wc, wn = orc.ddmg_eval(d.n_levels, d.levels, d.w, d.params, 0, d.n_alloc, d.n_trials, d.seed,
                           threads=_host_threads())
    assert np.array_equal(cnt, wc) and np.array_equal(_bits(net), _bits(wn))
    assert key == orc.argmax_net(wn)[0]


def test_signed_key_order(D, orc):
    """key_order = 1 (include/distill.h): the kernel stores key ^ 2^63, combined by
    a signed atomicMin from DISTILL_KEY_INIT_SIGNED — the same key as the unsigned
    order for PP and Stroop grids, shards combine with a plain int64 min."""
    import torch
    cfg = W.PPConfig("sk", (17, 13, 11), 12)
    m = _model(D, cfg)
    _, key = _gpu_pp(D, m, cfg)
    best = torch.empty(1, dtype=torch.int64, device="cuda")
    D.key_reset(best, signed=True)
    torch.cuda.synchronize()
    assert int(best.item()) == 2 ** 63 - 1
    D.eval_grid(m, cfg.inputs, cfg.n_samples, cfg.seed, best=best, signed_key=True)
    assert D.key_from_tensor(best, signed=True) == key
    parts = []
    for r in range(3):
        b, e = D.shard_range(cfg.n_alloc, r, 3)
        t = torch.empty(1, dtype=torch.int64, device="cuda")
        D.key_reset(t, signed=True)
        D.eval_grid(m, cfg.inputs, cfg.n_samples, cfg.seed, b, e, best=t, signed_key=True)
        parts.append(int(t.item()))
    assert (min(parts) & (2 ** 64 - 1)) ^ (1 << 63) == key
    c = W.stroop_small()
    ms = D.load_model(W.KIND_STROOP_LCA, c.n_levels, c.levels, c.w, c.params, device=0)
    _, _, k_u = _stroop_gpu(D, ms, c, 0, c.n_alloc)
    counts = torch.zeros(3 * c.n_alloc, dtype=torch.int64, device="cuda")
    D.key_reset(best, signed=True)
    D.eval_grid(ms, None, c.n_trials, c.seed, best=best, counts=counts, signed_key=True)
    assert D.key_from_tensor(best, signed=True) == k_u
    # an all-NaN grid: no valid candidate (high word 0xFFFFFFFF), as in the unsigned order
    D.key_reset(best, signed=True)
    D.eval_grid(m, np.array([np.nan, 0, 1, 1, 0, 0], np.float32), cfg.n_samples, cfg.seed, best=best,
                signed_key=True)
    assert D.key_from_tensor(best, signed=True) >> 32 == 0xFFFFFFFF
    with pytest.raises(D.api.DistillError):
        D.key_decode(D.key_from_tensor(best, signed=True))


@pytest.mark.parametrize("model", ["stroop", "ext_a", "ext_b", "ddmg"])
@pytest.mark.parametrize("case", ["latch_at_step_1", "never_latch", "short_trip", "ragged_trial_range"])
def test_trial_streaming_edges_bit_exact(D, orc, model, case):
    """Trial streaming (DESIGN R14b: a trial ends at its response; lanes take the
    next trial of their block) against the fixed-trip oracle: every trial
    latching at step 1, none latching (all N steps), N below one group (tail
    only), and a trial sub-range too small to give every block and lane a trial
    — counts bit-exact (and V / key for full ranges)."""
    if model == "stroop":
        c, kind = W.stroop_small(), W.KIND_STROOP_LCA
        thr_i, n_i = 7, 10
    elif model == "ddmg":
        c, kind = W.ddmg_grid(6, 257), W.KIND_DDM_GRID
        thr_i, n_i = None, 6
    else:
        c, kind = W.ext_stroop_small(), (W.KIND_EXT_STROOP_A if model == "ext_a" else W.KIND_EXT_STROOP_B)
        thr_i, n_i = 9, 10
    c.params = c.params.copy()
    c.levels = c.levels.copy()
    rng_ = (0, 0)
    if case == "latch_at_step_1":                             # threshold 0: the first step passes
        if thr_i is None:
            c.levels[c.n_levels[0]:] = 0.0
        else:
            c.params[thr_i] = 0.0
    elif case == "never_latch":
        if thr_i is None:
            c.levels[c.n_levels[0]:] = 1e6
        else:
            c.params[thr_i] = 1e6
    elif case == "short_trip":
        c.params[n_i] = 4 if model != "ddmg" else 7
    else:
        rng_ = (5, 9)
    m = D.load_model(kind, c.n_levels, c.levels, c.w, c.params, device=0)
    cnt, net, key = _stroop_gpu(D, m, c, 0, c.n_alloc, trial_range=rng_)
    tb, te = rng_ if rng_ != (0, 0) else (0, c.n_trials)
    if model == "stroop":
        wc, wn = orc.stroop_eval(c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials, c.seed, tb, te,
                                 threads=8)
    elif model == "ddmg":
        wc, wn = orc.ddmg_eval(c.n_levels, c.levels, c.w, c.params, 0, c.n_alloc, c.n_trials, c.seed, tb, te,
                               threads=8)
    else:
        wc, wn = orc.ext_stroop_eval(0 if model == "ext_a" else 1, c.n_levels, c.levels, c.w, c.params, 0,
                                     c.n_alloc, c.n_trials, c.seed, threads=8, trial_begin=tb, trial_end=te)
    assert np.array_equal(cnt, wc)
    if rng_ == (0, 0):
        assert np.array_equal(_bits(net), _bits(wn))
        assert key == orc.argmax_net(wn)[0]
    if case == "latch_at_step_1":
        assert cnt[:, 1].sum() == 0 and (cnt[:, 2] == (te - tb)).all()   # every trial decides at step 1
    if case == "never_latch":
        assert (cnt[:, 1] == (te - tb)).all()


@pytest.mark.parametrize("b,e", [(1625 ** 3 - 600, 1625 ** 3), (2 ** 31 - 300, 2 ** 31 + 301),
                                 (1625 ** 3 - 70_001, 1625 ** 3)])
def test_pp_top_of_the_index_range(D, orc, b, e):
    """The largest grid the packed key admits (reading R20: global index < 2^32):
    1625^3 = 4.29e9 allocations; shards at the very top (latency-mode and
    one-thread-per-allocation kernels) and across 2^31 — costs and the shard
    key bit-exact against the oracle; a grid of 2^32 allocations is refused."""
    cfg = W.PPConfig("pp_max", (1625, 1625, 1625), 6)
    m = _model(D, cfg)
    C, key = _gpu_pp(D, m, cfg, begin=b, end=e)
    want = orc.pp_eval(cfg.n_levels, cfg.levels, cfg.w, cfg.params, cfg.inputs, b, e, cfg.n_samples, cfg.seed)
    assert np.array_equal(_bits(C), _bits(want))
    assert key == orc.argmax_net(-want, b)[0]
    with pytest.raises(D.api.DistillError):
        _model(D, W.PPConfig("pp_too_big", (65536, 65536, 1), 6))
