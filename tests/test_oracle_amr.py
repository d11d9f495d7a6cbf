"""Pins for the coarse-to-fine refinement oracle (spec/MODELS.md §9)."""
import numpy as np

import workloads as W


def test_amr_zero_noise_converges_to_planted_corner(orc):
    """Zero noise -> C = K exactly; with w = (-0.1, 0.2, 0.05) the optimum is the
    corner (1, 0, 0) and every round's best allocation sits on it while the box
    shrinks geometrically toward it."""
    params = np.array([0.0, 0.0, 0.5], np.float32)
    w = np.array([-0.1, 0.2, 0.05], np.float32)
    keys, boxes = orc.pp_amr((5, 5, 5), w, params, W.pp_cfg1().inputs, [0, 0, 0], [1, 1, 1], 7, 4, 3)
    for r in range(7):
        c, idx = orc.key_decode(int(keys[r]))
        assert idx == 4 * 25                       # (top level, 0, 0)
    widths = boxes[:, :, 1] - boxes[:, :, 0]
    assert np.allclose(widths[1:, 0], [0.25 / 4 ** r for r in range(7)], rtol=1e-5)
    assert np.allclose(boxes[-1, 0], [1 - 0.25 / 4 ** 6, 1.0], atol=1e-6)
    assert (boxes[-1, 1] == [0, 0.25 / 4 ** 6]).all() or np.allclose(boxes[-1, 1], [0, 0.25 / 4 ** 6])


def test_amr_matches_fine_scan_of_prey_attention(orc):
    """Fig. 4 analogue: refining the prey attention (others fixed at 0.5) in rounds
    of 5 levels lands within 0.1 of the argmin of a 101-level scan with the same
    sample budget per point (the objective is noisy and flat near its minimum)."""
    cfg = W.pp_cfg1()
    S = 3000
    keys, boxes = orc.pp_amr((5, 1, 1), cfg.w, cfg.params, cfg.inputs, [0, 0.5, 0.5], [1, 0.5, 0.5], 6, S, 5)
    final_lo, final_hi = boxes[-1, 0]
    a_amr = 0.5 * (final_lo + final_hi)
    fine = W.PPConfig("scan", (101, 1, 1), S)
    fine.levels = np.concatenate([W.linear_levels(101), [0.5], [0.5]]).astype(np.float32)
    C = orc.pp_eval(fine.n_levels, fine.levels, fine.w, fine.params, fine.inputs, 0, 101, S, 5)
    a_scan = fine.levels[int(np.argmin(C))]
    assert 0.3 < a_scan < 0.95            # interior optimum (reading R4)
    assert abs(a_amr - a_scan) < 0.1, (a_amr, a_scan)


def test_amr_no_valid_allocation_keeps_the_box(orc):
    """All costs NaN (NaN prey position): every round's key has the NaN high word
    and the box is carried over unchanged (spec/MODELS.md §9)."""
    cfg = W.PPConfig("amr_nan", (4, 3, 2), 4)
    inputs = np.array([np.nan, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32)
    lo, hi = (0.0, 0.1, 0.2), (1.0, 0.9, 0.8)
    keys, boxes = orc.pp_amr(cfg.n_levels, cfg.w, cfg.params, inputs, lo, hi, 3, 4, 5)
    assert all(int(k) >> 32 == 0xFFFFFFFF for k in keys)
    for r in range(4):
        assert np.array_equal(boxes[r], np.array([lo, hi], np.float32).T)
