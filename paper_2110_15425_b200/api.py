"""Python face of the C ABI: the same calls, torch tensors for device memory.

Each function only marshals arguments and forwards to libdistill.so
(include/distill.h documents semantics, layouts, ownership and errors).
Keys live in int64 tensors holding the raw unsigned 64-bit pattern.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _abi
from ._abi import KEY_INIT, DistillError, check, lib

import threading as _threading

_INIT_LOCK = _threading.Lock()


def _stream_handle(stream, device: Optional[int] = None) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream


def _on_device(t):
    """The library's model-less entries launch on the current device: make it the tensor's."""
    import contextlib
    import torch
    return torch.cuda.device(t.device) if getattr(t, "is_cuda", False) else contextlib.nullcontext()


def _on_stream(stream):
    """Context for library-side temporaries: allocate (and zero) them on the
    stream the kernels run on, so the caching allocator cannot hand their memory
    to another stream while those kernels still use it."""
    import contextlib
    import torch
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


# element type each named buffer must have (the C ABI's float* / u64* / int*);
# u64 buffers are int64 tensors holding the raw bit pattern
_BUF_DTYPE = {"esum": "int64", "net": "float32", "values": "float32", "inputs": "float32", "traj": "float32",
              "boxes": "float32", "levels": "float32", "rad": "float32",
              "best": "int64", "tie": "int64", "keys": "int64", "counts": "int64",
              "rt_hist": "int64", "rt_sum": "int64", "x_hist": "int64", "status": "int32"}


def _dev_ptr(t, name: str, numel: Optional[int] = None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} buffer must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} buffer must be contiguous")
    want = _BUF_DTYPE.get(name)
    if want is not None and str(t.dtype) != f"torch.{want}":
        raise ValueError(f"{name} buffer must be {want}, got {t.dtype}")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} buffer too small: {t.numel()} < {numel}")
    return t.data_ptr()


class Model:
    """Owns a distill_model handle (device read-only block)."""

    def __init__(self, kind: int, n_levels, levels, cost_weights, params, device: int = 0):
        self.kind = int(kind)
        self.n_levels = np.ascontiguousarray(np.asarray(n_levels, np.uint32))
        self.levels = np.ascontiguousarray(np.asarray(levels, np.float32))
        self.cost_weights = np.ascontiguousarray(np.asarray(cost_weights, np.float32))
        self.params = np.ascontiguousarray(np.asarray(params, np.float32))
        self.device = int(device)
        desc = _abi.ModelDesc(self.kind, self.n_levels.size, _abi._uptr(self.n_levels), _abi._fptr(self.levels),
                              _abi._fptr(self.cost_weights), _abi._fptr(self.params), self.params.size)
        h = C.c_void_p()
        check(lib().distill_load_model(C.byref(desc), self.device, C.byref(h)))
        self._h = h
        n = C.c_uint64()
        check(lib().distill_grid_size(self._h, C.byref(n)))
        self.n_alloc = int(n.value)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().distill_free_model(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def load_model(kind, n_levels, levels, cost_weights, params, device: int = 0) -> Model:
    return Model(kind, n_levels, levels, cost_weights, params, device)


def eval_grid(model: Model, inputs, n_samples: int, seed: int, begin: int = 0, end: Optional[int] = None,
              net=None, best=None, invocation: int = 0, counts=None, trial_range=(0, 0), stream=None,
              signed_key: bool = False) -> None:
    """distill_eval_grid: allocations [begin, end) -> net[end-begin] (V = -C), best (atomicMin key).

    signed_key: best holds key ^ 2^63 (key_order = 1; reset it with key_reset(best, signed=True)),
    so an int64 MIN all-reduce combines shards with no conversion."""
    end = model.n_alloc if end is None else int(end)
    n = end - int(begin)
    inp = np.ascontiguousarray(np.asarray(inputs if inputs is not None else np.zeros(0), np.float32))
    a = _abi.EvalArgs()
    a.inputs = _abi._fptr(inp) if inp.size else None
    a.n_inputs = inp.size
    a.begin, a.end = int(begin), end
    a.n_samples, a.invocation, a.seed = int(n_samples), int(invocation), int(seed) & (2 ** 64 - 1)
    a.d_net = _dev_ptr(net, "net", n)
    a.d_best = _dev_ptr(best, "best", 1)
    a.trial_begin, a.trial_end = int(trial_range[0]), int(trial_range[1])
    a.key_order = 1 if signed_key else 0
    if counts is None and model.kind != _abi.MODEL_PREDATOR_PREY:
        import torch
        with _on_stream(stream):      # freed on return: stream-ordered reuse only
            counts = torch.empty(3 * max(n, 1), dtype=torch.int64, device=torch.device("cuda", model.device))
            a.d_counts = _dev_ptr(counts, "counts", 3 * n)
            check(lib().distill_eval_grid(model.handle, C.byref(a), _stream_handle(stream, model.device)))
        return
    a.d_counts = _dev_ptr(counts, "counts", 3 * n)
    check(lib().distill_eval_grid(model.handle, C.byref(a), _stream_handle(stream, model.device)))


def grid_search(model: Model, inputs, n_samples: int, seed: int, shard=None, invocation: int = 0, stream=None):
    """One grid search with library-allocated outputs (SURVEY §8(b) L4 shape):
    evaluates this rank's shard (shard = (rank, world), contiguous 4-aligned
    ranges; None = the whole grid) and returns (net, key): net = V for the
    shard's allocations (float32 CUDA tensor), key = the shard's best key
    (int64 CUDA tensor, raw bits; combine across ranks with best())."""
    import torch
    from .dist import shard_range
    b, e = (0, model.n_alloc) if shard is None else shard_range(model.n_alloc, int(shard[0]), int(shard[1]))
    dev = torch.device("cuda", model.device)
    with _on_stream(stream):
        net = torch.empty(max(e - b, 1), dtype=torch.float32, device=dev)
        key = torch.full((1,), -1, dtype=torch.int64, device=dev)
    eval_grid(model, inputs, n_samples, seed, b, e, net=net, best=key, invocation=invocation, stream=stream)
    return net[:e - b], key


def best(key, group=None):
    """Global best allocation from a shard key tensor: MIN all-reduce across the
    process group when torch.distributed is initialised with world size > 1
    (in place), then decode -> (cost C, global index); V = -C."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        from .dist import best_allreduce
        best_allreduce(key, group)
    return key_decode(key_from_tensor(key))


def eval_grid_multi(model: Model, inputs, n_invocations: int, n_samples: int, seed: int, begin: int = 0,
                    end: Optional[int] = None, invocation0: int = 0, net=None, best=None, stream=None) -> None:
    """distill_eval_grid_multi: invocation t on position set t mod n_sets, RNG invocation invocation0 + t.

    `inputs` is a CUDA float32 tensor [n_sets, 6]; net [T, end-begin] and best [T] as in eval_grid."""
    end = model.n_alloc if end is None else int(end)
    n, T = end - int(begin), int(n_invocations)
    if inputs.dim() != 2 or inputs.shape[1] != 6:
        raise ValueError("inputs must be a float32 CUDA tensor of shape [n_sets, 6]")
    a = _abi.MultiArgs(_dev_ptr(inputs, "inputs"), int(inputs.shape[0]), T, int(invocation0), int(n_samples),
                       int(begin), end, int(seed) & (2 ** 64 - 1), _dev_ptr(net, "net", T * n),
                       _dev_ptr(best, "best", T))
    check(lib().distill_eval_grid_multi(model.handle, C.byref(a), _stream_handle(stream, model.device)))


def eval_grid_host(model: Model, inputs, n_samples: int, seed: int, begin: int = 0, end: Optional[int] = None,
                   net_out: Optional[np.ndarray] = None, invocation: int = 0, stream=None) -> int:
    """distill_eval_grid_host: host inputs in, host V (optional) and best key out; synchronous."""
    end = model.n_alloc if end is None else int(end)
    inp = np.asarray(inputs, np.float32).reshape(-1)
    if getattr(model, "_h_key", None) is None:      # pinned: the kernel publishes the key into it
        with _INIT_LOCK:
            if getattr(model, "_h_key", None) is None:
                import threading
                import torch
                model._h_key_lock = threading.Lock()
                hk = torch.empty(1, dtype=torch.int64, pin_memory=True)
                # per-model host slots and their ctypes pointers, made once: the call
                # itself then only copies the 6 positions and reads the key back
                model._h_key_np = hk.numpy()
                model._h_key_ptr = C.cast(hk.data_ptr(), C.POINTER(C.c_uint64))
                model._h_inp = np.zeros(6, np.float32)
                model._h_inp_ptr = _abi._fptr(model._h_inp)
                model._h_key = hk
    net_ptr = None
    if net_out is not None:
        if net_out.dtype != np.float32 or not net_out.flags.c_contiguous or net_out.size < end - begin:
            raise ValueError("net_out must be a contiguous float32 array of end-begin elements")
        net_ptr = net_out.ctypes.data
    # The pinned key slot (and the positions slot) are per model: hold them from the
    # call until the key is read, so a concurrent call on another thread cannot publish
    # over them in between (the library itself serialises host-buffer calls per handle).
    with model._h_key_lock:
        if inp.size == 6:
            model._h_inp[:] = inp
            inp_ptr = model._h_inp_ptr
        else:                                        # the library rejects it (needs 6 inputs)
            inp = np.ascontiguousarray(inp)
            inp_ptr = _abi._fptr(inp) if inp.size else None
        check(lib().distill_eval_grid_host(model.handle, inp_ptr, inp.size, int(begin), end,
                                           int(n_samples), int(invocation), int(seed) & (2 ** 64 - 1), net_ptr,
                                           model._h_key_ptr, _stream_handle(stream, model.device)))
        return int(model._h_key_np[0]) & (2 ** 64 - 1)


def eval_grid_host_async(model: Model, inputs, n_samples: int, seed: int, begin: int = 0,
                         end: Optional[int] = None, net_out: Optional[np.ndarray] = None, key_out=None,
                         invocation: int = 0, stream=None) -> None:
    """distill_eval_grid_host_async: the end-to-end call without the final synchronisation.
    net_out (optional) and key_out (>= 1 int64 element) must be pinned host memory (e.g. the
    .numpy() view of a torch pin_memory tensor); they hold V and the raw key bits once
    `stream` has passed the call (record an event after it and wait for that).  Keep two
    sets of slots to have the next grid search in flight while reading this one."""
    end = model.n_alloc if end is None else int(end)
    inp = np.ascontiguousarray(np.asarray(inputs, np.float32).reshape(-1))
    if key_out is None or key_out.dtype != np.int64 or not key_out.flags.c_contiguous or key_out.size < 1:
        raise ValueError("key_out must be a contiguous int64 array (pinned) of at least one element")
    net_ptr = None
    if net_out is not None:
        if net_out.dtype != np.float32 or not net_out.flags.c_contiguous or net_out.size < end - begin:
            raise ValueError("net_out must be a contiguous float32 array of end-begin elements")
        net_ptr = net_out.ctypes.data
    check(lib().distill_eval_grid_host_async(model.handle, _abi._fptr(inp) if inp.size else None, inp.size,
                                             int(begin), end, int(n_samples), int(invocation),
                                             int(seed) & (2 ** 64 - 1), net_ptr, key_out.ctypes.data,
                                             _stream_handle(stream, model.device)))


def stroop_energy(model: Model, alloc: int, n_trials: int, seed: int, trial_range=None, esum=None, stream=None):
    """distill_stroop_energy: per-step sums of llrint(x0·x1·2^24) over the trials of
    one Stroop-LCA allocation (int64 CUDA tensor [N], accumulated; zeroed if allocated here)."""
    import torch
    N = int(model.params[10])
    if esum is None:                  # zeroed on the kernel's stream (ordered before it)
        with _on_stream(stream):
            esum = torch.zeros(N, dtype=torch.int64, device=torch.device("cuda", model.device))
    t0, t1 = (0, int(n_trials)) if trial_range is None else (int(trial_range[0]), int(trial_range[1]))
    check(lib().distill_stroop_energy(model.handle, int(alloc), int(n_trials), t0, t1, int(seed) & (2 ** 64 - 1),
                                      _dev_ptr(esum, "esum", N), _stream_handle(stream, model.device)))
    return esum


def argmax(values, index_base: int, best, stream=None) -> None:
    """distill_argmax: atomicMin of key(-values[j], index_base + j) into best."""
    with _on_device(values):
        check(lib().distill_argmax(_dev_ptr(values, "values"), values.numel(), int(index_base),
                                   _dev_ptr(best, "best", 1), _stream_handle(stream, values.device.index)))


def argmax_ties(values, index_base: int, seed: int, invocation: int, best, tie, stream=None) -> None:
    """distill_argmax_ties: random tie-break among the minimal costs (spec/MODELS.md §8)."""
    with _on_device(values):
        check(lib().distill_argmax_ties(_dev_ptr(values, "values"), values.numel(), int(index_base),
                                        int(seed) & (2 ** 64 - 1), int(invocation), _dev_ptr(best, "best", 1),
                                        _dev_ptr(tie, "tie", 1), _stream_handle(stream, values.device.index)))


def key_reset(best, stream=None, signed: bool = False) -> None:
    """best <- DISTILL_KEY_INIT (or DISTILL_KEY_INIT_SIGNED for the signed key order)."""
    fn = lib().distill_key_reset_signed if signed else lib().distill_key_reset
    with _on_device(best):
        check(fn(_dev_ptr(best, "best", 1), _stream_handle(stream, best.device.index)))


def key_decode(key: int):
    """-> (cost C, global index); raises DistillError(E_NO_VALID) for an all-NaN/empty key."""
    c = C.c_float()
    idx = C.c_uint64()
    st = lib().distill_key_decode(int(key) & (2 ** 64 - 1), C.byref(c), C.byref(idx))
    check(st)
    return c.value, int(idx.value)


def ddm_batch(drift, noise, threshold, x0, dt, n_steps, rt_bin_steps, n_x_bins, x_lo, x_hi,
              trial_begin, trial_end, seed, rt_hist, rt_sum, x_hist, stream=None, lci=None) -> None:
    """distill_ddm_batch: histograms (int64 tensors) accumulated on the device."""
    a = _abi.DdmArgs(drift, noise, threshold, x0, dt, int(n_steps), int(rt_bin_steps), int(n_x_bins),
                     x_lo, x_hi, int(trial_begin), int(trial_end), int(seed) & (2 ** 64 - 1),
                     _dev_ptr(rt_hist, "rt_hist"), _dev_ptr(rt_sum, "rt_sum", 2), _dev_ptr(x_hist, "x_hist"))
    nb = (int(n_steps) + int(rt_bin_steps) - 1) // int(rt_bin_steps)
    if rt_hist.numel() < 2 * nb + 1 or x_hist.numel() < int(n_x_bins) + 2:
        raise ValueError("histogram buffers too small")
    with _on_device(rt_hist):
        if lci is None:
            check(lib().distill_ddm_batch(C.byref(a), _stream_handle(stream, rt_hist.device.index)))
        else:                               # distill_lci_batch: drift is the input I, lci = (leak, offset)
            check(lib().distill_lci_batch(C.byref(a), float(lci[0]), float(lci[1]),
                                          _stream_handle(stream, rt_hist.device.index)))


def _episode_args(model: Model, init, n_steps: int, n_samples: int, seed: int, speeds, capture_radius,
                  traj, keys, status, stream=None):
    import torch
    dev = torch.device("cuda", model.device)
    T = int(n_steps)
    with _on_stream(stream):
        traj = torch.empty((T + 1, 6), dtype=torch.float32, device=dev) if traj is None else traj
        keys = torch.empty(T, dtype=torch.int64, device=dev) if keys is None else keys
        status = torch.empty(2, dtype=torch.int32, device=dev) if status is None else status
    init_arr = None if init is None else np.ascontiguousarray(np.asarray(init, np.float32))
    a = _abi.EpisodeArgs(T, int(n_samples), int(seed) & (2 ** 64 - 1), float(speeds[0]), float(speeds[1]),
                         float(speeds[2]), float(capture_radius),
                         _abi._fptr(init_arr) if init_arr is not None else None,
                         _dev_ptr(traj, "traj", 6 * (T + 1)), _dev_ptr(keys, "keys", T),
                         _dev_ptr(status, "status", 2))
    return a, init_arr, traj, keys, status


class EpisodeRun:
    """A closed-loop episode driven step by step (distill_pp_episode_begin /
    _search / _advance), for grids sharded across ranks: between search(t) and
    advance(t) the caller all-reduces keys[t:t+1] (dist.best_allreduce)."""

    def __init__(self, model: Model, init, n_steps: int, n_samples: int, seed: int, speeds=(1.0, 0.8, 0.6),
                 capture_radius: float = 0.5, traj=None, keys=None, status=None, stream=None):
        self.model, self.stream = model, stream
        self._a, self._init, self.traj, self.keys, self.status = _episode_args(
            model, init, n_steps, n_samples, seed, speeds, capture_radius, traj, keys, status, stream)
        check(lib().distill_pp_episode_begin(model.handle, C.byref(self._a), _stream_handle(stream, model.device)))

    def search(self, t: int, begin: int = 0, end: Optional[int] = None) -> None:
        end = self.model.n_alloc if end is None else int(end)
        check(lib().distill_pp_episode_search(self.model.handle, C.byref(self._a), int(t), int(begin), end,
                                              _stream_handle(self.stream, self.model.device)))

    def advance(self, t: int) -> None:
        check(lib().distill_pp_episode_advance(self.model.handle, C.byref(self._a), int(t),
                                               _stream_handle(self.stream, self.model.device)))


def pp_episode(model: Model, init, n_steps: int, n_samples: int, seed: int, speeds=(1.0, 0.8, 0.6),
               capture_radius: float = 0.5, traj=None, keys=None, status=None, stream=None):
    """distill_pp_episode: closed-loop episode on the device (spec/MODELS.md §7).

    Returns (traj[(T+1),6] float32, keys[T] int64 raw key bits, status[2] int32) CUDA tensors.
    If `init` is None, traj[0] must already hold the initial positions."""
    a, _keep, traj, keys, status = _episode_args(model, init, n_steps, n_samples, seed, speeds, capture_radius,
                                                 traj, keys, status, stream)
    check(lib().distill_pp_episode(model.handle, C.byref(a), _stream_handle(stream, model.device)))
    return traj, keys, status


def _amr_args(model: Model, inputs, lo, hi, rounds: int, n_samples: int, seed: int, invocation0: int,
              keys, boxes, levels, stream=None):
    import torch
    dev = torch.device("cuda", model.device)
    R = int(rounds)
    with _on_stream(stream):
        keys = torch.empty(R, dtype=torch.int64, device=dev) if keys is None else keys
        boxes = torch.empty((R + 1, 3, 2), dtype=torch.float32, device=dev) if boxes is None else boxes
        levels = torch.empty(int(model.n_levels.sum()), dtype=torch.float32, device=dev) if levels is None else levels
    inp = np.ascontiguousarray(np.asarray(inputs, np.float32))
    a = _abi.AmrArgs(_abi._fptr(inp), inp.size, (C.c_float * 3)(*[float(x) for x in lo]),
                     (C.c_float * 3)(*[float(x) for x in hi]), R, int(n_samples), int(invocation0),
                     int(seed) & (2 ** 64 - 1), _dev_ptr(keys, "keys", R), _dev_ptr(boxes, "boxes", 6 * (R + 1)),
                     _dev_ptr(levels, "levels", int(model.n_levels.sum())))
    return a, inp, keys, boxes, levels


def pp_amr(model: Model, inputs, lo, hi, rounds: int, n_samples: int, seed: int, invocation0: int = 0,
           keys=None, boxes=None, levels=None, stream=None):
    """distill_pp_amr: coarse-to-fine refinement on the device (spec/MODELS.md §9).

    Returns (keys[R] int64 raw key bits, boxes[R+1, 3, 2] float32) CUDA tensors."""
    a, _keep, keys, boxes, levels = _amr_args(model, inputs, lo, hi, rounds, n_samples, seed, invocation0,
                                              keys, boxes, levels, stream)
    check(lib().distill_pp_amr(model.handle, C.byref(a), _stream_handle(stream, model.device)))
    return keys, boxes


class AmrRun:
    """Coarse-to-fine refinement driven round by round (distill_pp_amr_begin /
    _levels / _search / _refine), for grids sharded across ranks: between
    search(r) and refine(r) the caller all-reduces keys[r:r+1]."""

    def __init__(self, model: Model, inputs, lo, hi, rounds: int, n_samples: int, seed: int,
                 invocation0: int = 0, stream=None):
        self.model, self.stream = model, stream
        self._a, self._inp, self.keys, self.boxes, self.levels = _amr_args(
            model, inputs, lo, hi, rounds, n_samples, seed, invocation0, None, None, None, stream)
        check(lib().distill_pp_amr_begin(model.handle, C.byref(self._a), _stream_handle(stream, model.device)))

    def levels_for(self, r: int) -> None:
        check(lib().distill_pp_amr_levels(self.model.handle, C.byref(self._a), int(r), _stream_handle(self.stream, self.model.device)))

    def search(self, r: int, begin: int = 0, end: Optional[int] = None) -> None:
        end = self.model.n_alloc if end is None else int(end)
        check(lib().distill_pp_amr_search(self.model.handle, C.byref(self._a), int(r), int(begin), end,
                                          _stream_handle(self.stream, self.model.device)))

    def refine(self, r: int) -> None:
        check(lib().distill_pp_amr_refine(self.model.handle, C.byref(self._a), int(r), _stream_handle(self.stream, self.model.device)))


def rng_rad(words, device: int = 0, out=None, stream=None):
    """distill_rng_rad: rad_spec of raw radius words -> float32 CUDA tensor.  `words`: uint32
    bit patterns as an int32 CUDA tensor, or any host array (copied to `device`)."""
    import torch
    if not getattr(words, "is_cuda", False):
        w = np.ascontiguousarray(np.asarray(words, dtype=np.uint32)).view(np.int32)
        words = torch.from_numpy(w).to(torch.device("cuda", device))
    if words.dtype != torch.int32 or not words.is_contiguous():
        raise ValueError("words must be a contiguous int32 CUDA tensor of uint32 bit patterns")
    with _on_device(words), _on_stream(stream):
        out = torch.empty(words.numel(), dtype=torch.float32, device=words.device) if out is None else out
        check(lib().distill_rng_rad(words.data_ptr(), words.numel(), _dev_ptr(out, "rad", words.numel()),
                                    _stream_handle(stream, words.device.index)))
    return out


def rng_normals_acc(seed: int, unit_begin: int, n_units: int, n_per_unit: int, device: int = 0, stream=None):
    """distill_rng_normals_acc: stream-2 normals 0..n_per_unit-1 of RNG units
    [unit_begin, unit_begin + n_units) -> float32 CUDA tensor [n_units, n_per_unit]."""
    import torch
    with torch.cuda.device(device), _on_stream(stream):
        out = torch.empty((max(int(n_units), 1), int(n_per_unit)), dtype=torch.float32,
                          device=torch.device("cuda", device))
        check(lib().distill_rng_normals_acc(int(seed) & (2 ** 64 - 1), int(unit_begin), int(n_units),
                                            int(n_per_unit), out.data_ptr(), _stream_handle(stream, device)))
    return out[:int(n_units)]


def rng_normals_pp(seed: int, alloc_begin: int, n_alloc: int, n_samples: int, invocation: int = 0,
                   device: int = 0, stream=None):
    """distill_rng_normals_pp: the predator-prey observation noise (stream 1) of
    allocations [alloc_begin, alloc_begin + n_alloc) -> float32 CUDA tensor [n_alloc, n_samples, 6]."""
    import torch
    with torch.cuda.device(device), _on_stream(stream):
        out = torch.empty((max(int(n_alloc), 1), int(n_samples), 6), dtype=torch.float32,
                          device=torch.device("cuda", device))
        check(lib().distill_rng_normals_pp(int(seed) & (2 ** 64 - 1), int(alloc_begin), int(n_alloc),
                                           int(n_samples), int(invocation), out.data_ptr(),
                                           _stream_handle(stream, device)))
    return out[:int(n_alloc)]


def sm_clock_mhz(micros: int = 200, stream=None) -> float:
    """distill_sm_clock_probe: median effective SM clock in MHz (measurement utility)."""
    v = C.c_double()
    check(lib().distill_sm_clock_probe(int(micros), C.byref(v), _stream_handle(stream)))
    return float(v.value)


def launch_count() -> int:
    return int(lib().distill_launch_count())


def key_from_tensor(best, signed: bool = False) -> int:
    """Raw unsigned key from an int64 tensor (one device->host read); signed=True
    undoes the signed key order (bit 63 flipped)."""
    k = int(best.reshape(-1)[0].item()) & (2 ** 64 - 1)
    return k ^ (1 << 63) if signed else k


__all__ = ["KEY_INIT", "stroop_energy", "AmrRun", "DistillError", "EpisodeRun", "Model", "grid_search", "best", "load_model", "eval_grid", "eval_grid_host", "eval_grid_multi", "argmax",
           "key_reset", "key_decode", "ddm_batch", "launch_count", "key_from_tensor", "pp_episode", "argmax_ties", "pp_amr", "sm_clock_mhz",
           "rng_rad", "rng_normals_acc", "rng_normals_pp"]
