"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This module holds the *inputs* of each BASELINE.json configuration — level
tables, positions, model constants, seeds — and none of the method's
arithmetic (no RNG draws of the method, no model equations).  It is the only
module both the oracle side and the CUDA side import (DESIGN.md §5 states the
recipe and where every number comes from).

Configs (BASELINE.json ``configs``, in order):
  cfg1  predator-prey 3 signals x 3 levels (27 allocations) x 10 samples
  cfg2  DDM 1e6 trials x 1000 Euler steps, RT/accuracy histograms
  cfg3  predator-prey 3 x 100 levels (1e6 allocations) x 100 samples, 1 GPU
  cfg4  Stroop-LCA 1e4 allocations (2 x 100 levels) x 1e5 trials x 200 steps
  cfg5  predator-prey XL 3 x 200 levels (8e6 allocations) x 100 samples, 2/4/8 GPUs
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED = 42

# model-kind ids (mirrors the enum both sides define independently)
KIND_PREDATOR_PREY = 1
KIND_STROOP_LCA = 2


def linear_levels(L: int) -> np.ndarray:
    """a_k = k / (L-1) in binary32 (reading R2: levels evenly spaced in [0, 1])."""
    if L == 1:
        return np.zeros(1, np.float32)
    return (np.arange(L, dtype=np.float32) / np.float32(L - 1)).astype(np.float32)


@dataclass
class PPConfig:
    name: str
    n_levels: tuple
    n_samples: int
    # inputs = prey.xy, predator.xy, player.xy
    inputs: np.ndarray = field(default_factory=lambda: np.array([4.0, 1.0, -3.0, 2.0, 0.0, 0.0], np.float32))
    # params = sigma_max, sigma_min, kappa (reading R3)
    params: np.ndarray = field(default_factory=lambda: np.array([2.0, 0.1, 0.5], np.float32))
    # linear attention cost per entity (reading R4: 0.1, not SPEC's 0.3)
    w: np.ndarray = field(default_factory=lambda: np.array([0.1, 0.1, 0.1], np.float32))
    seed: int = SEED
    levels: np.ndarray = None

    def __post_init__(self):
        if self.levels is None:
            self.levels = np.concatenate([linear_levels(L) for L in self.n_levels]).astype(np.float32)

    @property
    def n_alloc(self) -> int:
        return int(np.prod(self.n_levels))

    @property
    def evals(self) -> int:
        return self.n_alloc * self.n_samples


def pp_cfg1() -> PPConfig:
    return PPConfig("pp_cfg1_3x3x3_s10", (3, 3, 3), 10)


def pp_positions(n_sets: int, seed: int = SEED) -> np.ndarray:
    """Synthetic multi-invocation inputs (SURVEY §8(d) cfg3 16-invocation variant):
    prey, predator, player positions uniform in [-10, 10]^2, float32 [n_sets, 6]."""
    return np.random.default_rng(seed).uniform(-10.0, 10.0, size=(int(n_sets), 6)).astype(np.float32)


def pp_cfg3() -> PPConfig:
    return PPConfig("pp_cfg3_100^3_s100", (100, 100, 100), 100)


def pp_cfg5() -> PPConfig:
    return PPConfig("pp_cfg5_200^3_s100", (200, 200, 200), 100)


def pp_weak(n_gpus: int) -> PPConfig:
    """Weak-scaling family: ~1e6 allocations per GPU. N=1 -> cfg3, N=8 -> cfg5."""
    if n_gpus == 1:
        return pp_cfg3()
    if n_gpus == 8:
        return pp_cfg5()
    L = int(round(100 * n_gpus ** (1.0 / 3.0)))
    return PPConfig(f"pp_weak{n_gpus}_{L}^3_s100", (L, L, L), 100)


def random_positions(n_invocations: int, seed: int = 7, span: float = 10.0) -> np.ndarray:
    """Per-invocation true positions, uniform in [-span, span]^2 (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-span, span, size=(n_invocations, 6)).astype(np.float32)


@dataclass
class DDMConfig:
    name: str = "ddm_cfg2_1e6x1000"
    drift: float = 1.0
    noise: float = 1.0
    threshold: float = 1.0
    x0: float = 0.0
    dt: float = 0.01
    n_steps: int = 1000
    rt_bin_steps: int = 10
    n_x_bins: int = 128
    n_trials: int = 1_000_000
    seed: int = SEED

    @property
    def x_lo(self) -> float:
        m, sd = self.x0 + self.drift * self.n_steps * self.dt, self.noise * math.sqrt(self.n_steps * self.dt)
        return float(np.float32(m - 6 * sd))

    @property
    def x_hi(self) -> float:
        m, sd = self.x0 + self.drift * self.n_steps * self.dt, self.noise * math.sqrt(self.n_steps * self.dt)
        return float(np.float32(m + 6 * sd))

    @property
    def n_rt_bins(self) -> int:
        return (self.n_steps + self.rt_bin_steps - 1) // self.rt_bin_steps

    @property
    def hist_sizes(self):
        return 2 * self.n_rt_bins + 1, 2, self.n_x_bins + 2


def ddm_cfg2() -> DDMConfig:
    return DDMConfig()


# Stroop-LCA surrogate constants (reading R15; spec/MODELS.md §6), frozen:
# g_c, g_w, tau, leak, inhibition, noise, dt, threshold, reward, rt_cost, n_steps
STROOP_PARAMS = np.array([1.0, 1.5, 0.1, 0.2, 0.2, 0.5, 0.05, 1.0, 1.0, 0.1, 200.0], np.float32)
STROOP_W = np.array([0.3, 0.1], np.float32)


@dataclass
class StroopConfig:
    name: str
    n_levels: tuple
    n_trials: int
    params: np.ndarray = field(default_factory=lambda: STROOP_PARAMS.copy())
    w: np.ndarray = field(default_factory=lambda: STROOP_W.copy())
    seed: int = SEED
    levels: np.ndarray = None

    def __post_init__(self):
        if self.levels is None:
            self.levels = np.concatenate([linear_levels(L) for L in self.n_levels]).astype(np.float32)

    @property
    def n_alloc(self) -> int:
        return int(np.prod(self.n_levels))

    @property
    def n_steps(self) -> int:
        return int(self.params[10])

    @property
    def evals(self) -> int:
        return self.n_alloc * self.n_trials


def stroop_cfg4() -> StroopConfig:
    return StroopConfig("stroop_cfg4_1e4x1e5x200", (100, 100), 100_000)


def stroop_small() -> StroopConfig:
    return StroopConfig("stroop_small_10x10x300", (10, 10), 300)


# DDM control grid constants (spec/MODELS.md §6c): A0, g_a, sigma, dt, R, c_rt, N;
# signals: attention u0 in [0, 1] (drift A = A0 + g_a u0), threshold u1 in [0.3, 1.5]
DDMG_PARAMS = np.array([0.2, 1.5, 1.0, 0.01, 1.0, 0.5, 400.0], np.float32)
DDMG_W = np.array([0.05, 0.05], np.float32)
KIND_DDM_GRID = 5


def ddmg_grid(L: int = 100, n_trials: int = 10_000) -> "StroopConfig":
    """DDM control grid: L attention levels k/(L-1) x L thresholds 0.3 + 1.2 k/(L-1)."""
    lev = np.concatenate([linear_levels(L), (0.3 + 1.2 * linear_levels(L)).astype(np.float32)]).astype(np.float32)
    return StroopConfig(f"ddm_grid_{L}x{L}x{n_trials}", (L, L), n_trials, params=DDMG_PARAMS.copy(),
                        w=DDMG_W.copy(), levels=lev)


# Extended Stroop A/B constants (reading R26; spec/MODELS.md §10):
# g_c, g_w, tau, N_h, lambda, a_p, gamma, sigma_d, dt_d, z_d, N_d, reward, rt_cost
EXT_STROOP_PARAMS = np.array([1.0, 1.5, 0.1, 30.0, 2.0, 1.2, 0.8, 1.0, 0.01, 0.5, 100.0, 1.0, 0.2], np.float32)
KIND_EXT_STROOP_A = 3
KIND_EXT_STROOP_B = 4


def ext_stroop_small() -> StroopConfig:
    return StroopConfig("ext_stroop_small_8x8x240", (8, 8), 240, params=EXT_STROOP_PARAMS.copy())


def ext_stroop_grid() -> StroopConfig:
    """Bench/next-row configuration: the cfg4 control grid (1e4 allocations) x 1e4 trials."""
    return StroopConfig("ext_stroop_1e4x1e4", (100, 100), 10_000, params=EXT_STROOP_PARAMS.copy())
