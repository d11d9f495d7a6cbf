"""B200-native grid-search hot path of Distill (arXiv 2110.15425).

Public Python API (thin wrappers over the C ABI in include/distill.h):

    load_model(kind, n_levels, levels, cost_weights, params, device=0) -> Model
    grid_search(model, inputs, n_samples, seed, shard=(rank, world)) -> (net, key)
    best(key, group=None) -> (cost, index)        # all-reduce across ranks + decode
    eval_grid(model, inputs, n_samples, seed, begin=0, end=None, net=None, best=None, ...)
    eval_grid_host(model, inputs, n_samples, seed, ...)   # host buffers, end to end
    eval_grid_host_async(model, inputs, ..., net_out=, key_out=)   # the same, enqueue only (pinned slots)
    eval_grid_multi(model, d_inputs, n_invocations, n_samples, seed, ...)   # many invocations, one launch
    argmax(values, index_base, best) / argmax_ties(values, base, seed, t, best, tie)
    key_reset(best) / key_decode(key)
    ddm_batch(..., lci=None | (leak, offset))      # DDM / leaky competing integrator batches
    stroop_energy(model, alloc, n_trials, seed)   # decision energy over time
    rng_rad(words) / rng_normals_acc(...) / rng_normals_pp(...)   # rows a2/a3 on their own

Model kinds: 1 predator-prey, 2 Stroop-LCA, 3/4 Extended Stroop A/B, 5 DDM
control grid (workloads.KIND_*); eval_grid evaluates any of them.
    pp_episode(model, init, n_steps, n_samples, seed, ...)   # closed loop, on the device
    pp_amr(model, inputs, lo, hi, rounds, n_samples, seed)   # coarse-to-fine refinement
    shard_range(n, rank, world) / best_allreduce(key, group)   # multi-GPU plumbing
    pp_episode_sharded(model, init, T, S, seed, rank, world)  # closed loop over a sharded grid

Importing this package does not touch the GPU; the shared library is loaded
on first use and there is no CPU fallback.
"""
from .api import (KEY_INIT, key_from_tensor, AmrRun, EpisodeRun, Model, best, grid_search, stroop_energy, argmax, argmax_ties, ddm_batch, eval_grid, eval_grid_host, eval_grid_host_async, eval_grid_multi, key_decode,
                  key_reset, launch_count, load_model, pp_amr, pp_episode, rng_normals_acc, rng_normals_pp, rng_rad)
from .dist import (best_allreduce, hist_allreduce, key_to_i64, i64_to_key, pp_amr_sharded, pp_episode_sharded,
                   shard_range)

__all__ = ["KEY_INIT", "key_from_tensor", "Model", "best", "grid_search", "stroop_energy", "argmax", "argmax_ties", "ddm_batch", "eval_grid", "eval_grid_host", "eval_grid_host_async", "eval_grid_multi", "key_decode", "pp_episode", "pp_amr",
           "key_reset", "launch_count", "load_model", "best_allreduce", "hist_allreduce", "key_to_i64",
           "i64_to_key", "shard_range", "pp_episode_sharded", "EpisodeRun", "pp_amr_sharded", "AmrRun",
           "rng_rad", "rng_normals_acc", "rng_normals_pp"]
