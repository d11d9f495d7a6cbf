"""Pins for the closed-loop predator-prey episode oracle (spec/MODELS.md §7)."""
import numpy as np

import workloads as W


def _cfg(sig=(0.0, 0.0), kappa=0.0, L=3):
    c = W.PPConfig("ep", (L, L, L), 4)
    c.params = np.array([sig[0], sig[1], kappa], np.float32)
    return c


def test_straight_chase_capture_time_closed_form(orc):
    """Zero noise, kappa = 0, prey straight ahead fleeing along the same line: the
    gap shrinks by v_pl - v_py per step, so capture happens at the first t with
    d0 - t (v_pl - v_py) <= r_c."""
    c = _cfg()
    init = np.array([5.0, 0.0, -1000.0, 0.0, 0.0, 0.0], np.float32)  # predator far behind
    traj, keys, (outcome, steps) = orc.pp_episode(c.n_levels, c.levels, c.w, c.params, init, 40, 4, 7,
                                                  speeds=(1.0, 0.75, 0.0), capture_radius=0.5)
    d0, closure, rc = 5.0, 0.25, 0.5
    t_star = int(np.ceil((d0 - rc) / closure))   # 18
    assert outcome == 1 and steps == t_star
    gaps = traj[:t_star + 1, 0] - traj[:t_star + 1, 4]
    assert np.allclose(gaps, d0 - closure * np.arange(t_star + 1), atol=1e-4)
    # frozen afterwards, no more grid searches
    assert (traj[t_star:] == traj[t_star]).all()
    assert (keys[t_star:] == 0xFFFFFFFFFFFFFFFF).all() and (keys[:t_star] != 0xFFFFFFFFFFFFFFFF).all()


def test_predator_capture_in_one_step(orc):
    c = _cfg()
    init = np.array([100.0, 0.0, 1.2, 0.0, 0.0, 0.0], np.float32)
    traj, keys, (outcome, steps) = orc.pp_episode(c.n_levels, c.levels, c.w, c.params, init, 10, 4, 7,
                                                  speeds=(1.0, 0.0, 0.5), capture_radius=0.5)
    assert (outcome, steps) == (2, 1)
    assert np.allclose(traj[1], [100.0, 0.0, 0.7, 0.0, 1.0, 0.0], atol=1e-6)


def test_zero_noise_best_allocation_is_cheapest(orc):
    """With no observation noise every allocation sees the same move, so the grid
    search picks the cheapest attention (index 0 for w >= 0) at every step."""
    c = _cfg()
    init = np.array([8.0, 3.0, -4.0, 1.0, 0.0, 0.0], np.float32)
    _, keys, _ = orc.pp_episode(c.n_levels, c.levels, c.w, c.params, init, 6, 4, 7)
    assert all(int(k) & 0xFFFFFFFF == 0 for k in keys)


def test_noisy_episode_keys_match_single_grid_searches(orc):
    """Each step's key is the argmin of an ordinary grid search (invocation t) on
    that step's positions."""
    c = W.PPConfig("ep2", (5, 5, 5), 16)
    init = np.array([4.0, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32)
    traj, keys, _ = orc.pp_episode(c.n_levels, c.levels, c.w, c.params, init, 6, 16, 11)
    for t in range(6):
        C = orc.pp_eval(c.n_levels, c.levels, c.w, c.params, traj[t], 0, c.n_alloc, 16, 11, invocation=t)
        k, _ = orc.argmax_net(-C)
        assert k == int(keys[t])
