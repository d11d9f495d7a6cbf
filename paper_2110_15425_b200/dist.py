"""Multi-GPU plumbing: contiguous grid shards and the single key all-reduce.

The paper gives each CPU thread "a segment of the grid search space"
(P:349-352); here each rank (one process per GPU) owns one contiguous shard
of the global allocation range, runs the fused kernel on it, and the shards'
best keys are combined with ONE all-reduce of an int64 (NCCL over NVLink /
NVSwitch; gloo in the CPU tests).  DDM trial shards combine their u64
histograms with one SUM all-reduce.  Both reductions are associative and
commutative over exact integers, so results are bit-identical for any world
size (spec/MODELS.md §3).
"""
from __future__ import annotations

from typing import Tuple

SIGN = 1 << 63
MASK = (1 << 64) - 1


def shard_range(n: int, rank: int, world: int, align: int = 4) -> Tuple[int, int]:
    """Contiguous shard [b, e) of [0, n) for `rank`: ceil(n/world) rounded up to
    a multiple of `align` per rank (the last ranks may be short or empty)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    per = -(-n // world)
    per = -(-per // align) * align
    b = min(n, rank * per)
    e = min(n, b + per)
    return b, e


def key_to_i64(key: int) -> int:
    """Unsigned key -> signed int64 with the same order (flip bit 63)."""
    v = (int(key) & MASK) ^ SIGN
    return v - (1 << 64) if v >= SIGN else v


def i64_to_key(v: int) -> int:
    return (int(v) & MASK) ^ SIGN


def best_allreduce(best, group=None, signed: bool = False):
    """In-place: global min key across ranks.  `best` is an int64 tensor with the
    raw key bits; flips bit 63 so signed MIN == unsigned min, all-reduces, flips back.
    signed=True: `best` already holds the signed key order (eval_grid(...,
    signed_key=True) writes it from the kernel), so it is ONE all-reduce and nothing else."""
    import torch
    import torch.distributed as dist
    if signed:
        dist.all_reduce(best, op=dist.ReduceOp.MIN, group=group)
        return best
    flip = torch.tensor(-(1 << 63), dtype=torch.int64, device=best.device)
    best.bitwise_xor_(flip)
    dist.all_reduce(best, op=dist.ReduceOp.MIN, group=group)
    best.bitwise_xor_(flip)
    return best


def hist_allreduce(tensors, group=None):
    """SUM all-reduce of int64 histograms (DDM trial shards), fused into one call."""
    import torch
    import torch.distributed as dist
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    off = 0
    for t in tensors:
        n = t.numel()
        t.copy_(flat[off:off + n].view_as(t))
        off += n
    return tensors


def pp_episode_sharded(model, init, n_steps: int, n_samples: int, seed: int, rank: int, world: int, group=None,
                       speeds=(1.0, 0.8, 0.6), capture_radius: float = 0.5, stream=None):
    """Closed-loop episode over a grid sharded across ranks (SURVEY §8(f) NEXT-1:
    one grid search + all-reduce per time step).  Each rank searches its
    contiguous shard for step t, the keys are MIN-all-reduced, and every rank
    advances the identical trajectory.  Returns (traj, keys, status) tensors."""
    from .api import EpisodeRun
    b, e = shard_range(model.n_alloc, rank, world)
    run = EpisodeRun(model, init, n_steps, n_samples, seed, speeds, capture_radius, stream=stream)
    for t in range(int(n_steps)):
        run.search(t, b, e)
        if world > 1:
            best_allreduce(run.keys[t:t + 1], group)
        run.advance(t)
    return run.traj, run.keys, run.status


def pp_amr_sharded(model, inputs, lo, hi, rounds: int, n_samples: int, seed: int, rank: int, world: int,
                   group=None, invocation0: int = 0, stream=None):
    """Coarse-to-fine refinement over a grid sharded across ranks: per round the
    level table (replicated), a shard search, one key all-reduce and the
    (replicated) box refinement.  Returns (keys, boxes) tensors, identical on
    every rank."""
    from .api import AmrRun
    b, e = shard_range(model.n_alloc, rank, world)
    run = AmrRun(model, inputs, lo, hi, rounds, n_samples, seed, invocation0, stream=stream)
    for r in range(int(rounds)):
        run.levels_for(r)
        run.search(r, b, e)
        if world > 1:
            best_allreduce(run.keys[r:r + 1], group)
        run.refine(r)
    return run.keys, run.boxes
