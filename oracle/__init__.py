"""CPU oracle for the Distill grid-search hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2110_15425_b200`` never imports it and the two share
no code (see ``distill_oracle.h``).

This module only builds ``distill_oracle.c`` with gcc and marshals numpy
arrays through ctypes; every arithmetic step is in the C file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "distill_oracle.c")
_HDR = os.path.join(_HERE, "distill_oracle.h")
# DISTILL_ORACLE_SANITIZE=1: build and load ASan/UBSan-instrumented copies
# (`make sanitize-oracle` runs the CPU suite that way; needs libasan preloaded)
_SAN = os.environ.get("DISTILL_ORACLE_SANITIZE") == "1"
_SUFFIX = "_asan" if _SAN else ""
LIB = os.path.join(_HERE, f"liboracle{_SUFFIX}.so")
LIB_COUNT = os.path.join(_HERE, f"liboracle_count{_SUFFIX}.so")
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-mfma",
          "-fPIC", "-shared", "-Wall"]
SAN_CFLAGS = ["-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined"]


def build(force: bool = False) -> None:
    """Compile the oracle (and its flop-counting twin) with gcc."""
    san = SAN_CFLAGS if _SAN else []
    for out, extra in ((LIB, san), (LIB_COUNT, ["-DOD_COUNT_FLOPS", *san])):
        if (not force and os.path.exists(out)
                and os.path.getmtime(out) >= max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))):
            continue
        tmp = f"{out}.{os.getpid()}.tmp"          # per-process name: concurrent builders never share a file
        subprocess.check_call(["gcc", *CFLAGS, *extra, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, out)


_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


class DdmParams(C.Structure):
    _fields_ = [("drift", C.c_float), ("noise", C.c_float), ("threshold", C.c_float),
                ("x0", C.c_float), ("dt", C.c_float), ("n_steps", C.c_uint32),
                ("rt_bin_steps", C.c_uint32), ("n_x_bins", C.c_uint32),
                ("x_lo", C.c_float), ("x_hi", C.c_float)]


def _bind(path: str) -> C.CDLL:
    lib = C.CDLL(path)
    u64, u32, f32 = C.c_uint64, C.c_uint32, C.c_float
    sig = {
        "od_philox4x32_10": (None, [_u32p, _u32p, _u32p]),
        "od_rad": (f32, [u32]),
        "od_rad_array": (None, [_u32p, _f32p, u64]),
        "od_rad_table": (None, [_f32p]),
        "od_rsqrt": (f32, [f32]),
        "od_sincos2pi": (None, [u32, C.POINTER(f32), C.POINTER(f32)]),
        "od_rsqrt_array": (None, [_f32p, _f32p, u64]),
        "od_sincos2pi_array": (None, [_u32p, _f32p, _f32p, u64]),
        "od_normal_acc": (None, [u64, u64, u64, u64, _f32p]),
        "od_normal_sextet": (None, [u64, u32, u32, u32, _f32p]),
        "od_pp_eval": (C.c_int, [_u32p, _f32p, _f32p, _f32p, _f32p, u64, u64, u32, u64, u32, C.c_void_p]),
        "od_pp_trace": (C.c_int, [_u32p, _f32p, _f32p, _f32p, u64, u32, u64, u32, _f32p]),
        "od_pp_trace_f64": (C.c_int, [_u32p, _f32p, _f32p, _f32p, u64, u32, u64, u32, _f64p]),
        "od_pp_eval_f64": (C.c_int, [_u32p, _f32p, _f32p, _f32p, _f32p, u64, u64, u32, u64, u32, C.c_void_p]),
        "od_key": (u64, [f32, u32]),
        "od_argmax_random_ties": (C.c_int, [_f32p, u64, u64, u64, u32, C.POINTER(u64), C.POINTER(u64)]),
        "od_argmax_net": (C.c_int, [_f32p, u64, u64, C.POINTER(u64)]),
        "od_ddm_trial": (None, [C.POINTER(DdmParams), u64, u64, C.POINTER(C.c_int), C.POINTER(u32), C.POINTER(f32)]),
        "od_ddm_batch": (C.c_int, [C.POINTER(DdmParams), u64, u64, u64, _u64p, _u64p, _u64p]),
        "od_lci_batch": (C.c_int, [C.POINTER(DdmParams), f32, f32, u64, u64, u64, _u64p, _u64p, _u64p]),
        "od_lci_trial": (None, [f32, f32, f32, f32, f32, f32, u32, u64, u64,
                                C.POINTER(C.c_int), C.POINTER(u32), C.POINTER(f32)]),
        "od_stroop_eval": (C.c_int, [_u32p, _f32p, _f32p, _f32p, u64, u64, u32, u32, u32, u64, C.c_void_p, C.c_void_p]),
        "od_stroop_value": (f32, [_f32p, _f32p, f32, f32, u32, u64, u64, u64]),
        "od_stroop_trial": (None, [_f32p, f32, f32, u64, u64, u32, C.POINTER(C.c_int), C.POINTER(u32)]),
        "od_stroop_trace": (None, [_f32p, f32, f32, u64, u64, u32, C.POINTER(C.c_int), C.POINTER(u32), _f32p]),
        "od_ddmg_trial": (None, [_f32p, f32, f32, u64, u64, C.POINTER(C.c_int), C.POINTER(u32)]),
        "od_ddmg_value": (f32, [_f32p, _f32p, f32, f32, u32, u64, u64, u64]),
        "od_ddmg_eval": (C.c_int, [_u32p, _f32p, _f32p, _f32p, u64, u64, u32, u32, u32, u64, C.c_void_p,
                                   C.c_void_p]),
        "od_stroop_energy": (None, [_f32p, f32, f32, u64, u64, u32, u32, u32,
                                    np.ctypeslib.ndpointer(np.int64, flags="C")]),
        "od_pp_episode": (C.c_int, [_u32p, _f32p, _f32p, _f32p, _f32p, u32, u32, u64, _f32p, f32,
                                    _f32p, _u64p, np.ctypeslib.ndpointer(np.int32, flags="C")]),
        "od_pp_amr": (C.c_int, [_u32p, _f32p, _f32p, _f32p, _f32p, _f32p, u32, u32, u64, u32, _u64p, _f32p]),
        "od_ext_stroop_eval": (C.c_int, [C.c_int, _u32p, _f32p, _f32p, _f32p, u64, u64, u32, u64,
                                         C.c_void_p, C.c_void_p]),
        "od_ext_stroop_eval_range": (C.c_int, [C.c_int, _u32p, _f32p, _f32p, _f32p, u64, u64, u32, u32, u32, u64,
                                               C.c_void_p, C.c_void_p]),
        "od_ext_stroop_trial_a": (None, [_f32p, f32, f32, u64, u64, u32, np.ctypeslib.ndpointer(np.int32, flags="C"),
                                         _u32p]),
        "od_ext_stroop_trial_b": (None, [_f32p, f32, f32, u64, u64, u32, np.ctypeslib.ndpointer(np.int32, flags="C"),
                                         _u32p]),
        "od_flops_read": (C.c_ulonglong, []),
        "od_flops_reset": (None, []),
        "od_flops_method": (None, [C.c_int]),
        "od_is_counting_build": (C.c_int, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None
_lib_count = None
_lock = threading.Lock()


def lib(counting: bool = False) -> C.CDLL:
    global _lib, _lib_count
    with _lock:
        if counting:
            if _lib_count is None:
                build()
                _lib_count = _bind(LIB_COUNT)
            return _lib_count
        if _lib is None:
            build()
            _lib = _bind(LIB)
        return _lib


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


# ---------------------------------------------------------------- RNG

def philox(ctr, key) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    lib().od_philox4x32_10(_u32(ctr), _u32(key), out)
    return out


def rad(R: int) -> float:
    """rad_spec (spec/RNG.md §3): the Box-Muller radius sqrt(-2 ln u1(R))."""
    return lib().od_rad(int(R))


def rsqrt(x: float) -> float:
    return lib().od_rsqrt(float(x))


def sincos2pi(a: int):
    c, s = C.c_float(), C.c_float()
    lib().od_sincos2pi(int(a), C.byref(c), C.byref(s))
    return c.value, s.value


def rad_array(R) -> np.ndarray:
    R = _u32(R)
    y = np.empty(R.size, np.float32)
    lib().od_rad_array(R, y, R.size)
    return y


def rad_table() -> np.ndarray:
    """The 736 x 4 coefficient table RT of spec/RNG.md §3 as this oracle built it."""
    out = np.zeros((736, 4), np.float32)
    lib().od_rad_table(out)
    return out


def rsqrt_array(x) -> np.ndarray:
    x = _f32(x)
    y = np.empty_like(x)
    lib().od_rsqrt_array(x, y, x.size)
    return y


def sincos2pi_array(a):
    a = _u32(a)
    c = np.empty(a.size, np.float32)
    s = np.empty(a.size, np.float32)
    lib().od_sincos2pi_array(a, c, s, a.size)
    return c, s


def normal_acc(seed: int, unit: int, first: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float32)
    lib().od_normal_acc(seed, unit, first, n, out)
    return out


def normal_sextet(seed: int, alloc: int, sample: int, invocation: int = 0) -> np.ndarray:
    out = np.zeros(6, np.float32)
    lib().od_normal_sextet(seed, alloc, sample, invocation, out)
    return out


# ---------------------------------------------------------------- predator-prey

def pp_eval_multi(n_levels, levels, w, params, input_sets, n_invocations, begin, end, n_samples, seed,
                  invocation0=0):
    """PAPER.md Listing 1: one controller invocation per trial t with
    inputs[t % len] (reading Q17); here invocation t uses set t mod n_sets and RNG
    invocation word invocation0 + t.  Returns float32 costs C [T, end-begin]."""
    sets = np.asarray(input_sets, np.float32).reshape(-1, 6)
    return np.stack([pp_eval(n_levels, levels, w, params, sets[t % len(sets)], begin, end, n_samples, seed,
                             invocation=invocation0 + t) for t in range(int(n_invocations))]) \
        if n_invocations else np.zeros((0, int(end) - int(begin)), np.float32)


def pp_eval(n_levels, levels, w, params, inputs, begin, end, n_samples, seed,
            invocation=0, f64=False, counting=False) -> np.ndarray:
    n = int(end) - int(begin)
    out = np.zeros(max(n, 0), np.float64 if f64 else np.float32)
    L = lib(counting)
    fn = L.od_pp_eval_f64 if f64 else L.od_pp_eval
    rc = fn(_u32(n_levels), _f32(levels), _f32(w), _f32(params), _f32(inputs),
            int(begin), int(end), int(n_samples), int(seed), int(invocation),
            out.ctypes.data_as(C.c_void_p))
    if rc != 0:
        raise ValueError("od_pp_eval rejected its arguments")
    return out


def pp_trace(n_levels, levels, params, inputs, i, n_samples, seed, invocation=0, lib_handle=None) -> np.ndarray:
    """Per-sample objective e_s of allocation i (debug/tests)."""
    out = np.zeros(int(n_samples), np.float32)
    (lib_handle or lib()).od_pp_trace(_u32(n_levels), _f32(levels), _f32(params), _f32(inputs), int(i), int(n_samples),
                      int(seed), int(invocation), out)
    return out


def pp_trace_f64(n_levels, levels, params, inputs, i, n_samples, seed, invocation=0, lib_handle=None) -> np.ndarray:
    """Per-sample binary64 objective of allocation i (the plain definition)."""
    out = np.zeros(int(n_samples), np.float64)
    (lib_handle or lib()).od_pp_trace_f64(_u32(n_levels), _f32(levels), _f32(params), _f32(inputs), int(i),
                                          int(n_samples), int(seed), int(invocation), out)
    return out


def pp_eval_threads(n_levels, levels, w, params, inputs, begin, end, n_samples, seed,
                    invocation=0, threads=1, f64=False) -> np.ndarray:
    """Contiguous segments over Python threads (ctypes drops the GIL) — the
    paper's multicore scheme; f64 = the binary64 re-evaluation."""
    n = int(end) - int(begin)
    out = np.zeros(n, np.float64 if f64 else np.float32)
    threads = max(1, min(int(threads), max(n, 1)))
    seg = (n + threads - 1) // threads
    args = (_u32(n_levels), _f32(levels), _f32(w), _f32(params), _f32(inputs))
    L = lib()

    def work(t):
        b = begin + t * seg
        e = min(begin + n, b + seg)
        if e <= b:
            return
        view = out[b - begin:e - begin]
        (L.od_pp_eval_f64 if f64 else L.od_pp_eval)(*args, b, e, int(n_samples), int(seed), int(invocation),
                                                   view.ctypes.data_as(C.c_void_p))

    ts = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return out


def key(cost: float, index: int) -> int:
    return int(lib().od_key(float(cost), int(index)))


def argmax_net(net, base=0):
    k = C.c_uint64()
    arr = _f32(net)
    rc = lib().od_argmax_net(arr, arr.size, int(base), C.byref(k))
    return int(k.value), rc


def argmax_random_ties(net, base=0, seed=0, invocation=0):
    """(best key, tie key, rc); winner index = tie & 0xffffffff (spec/MODELS.md §8)."""
    k, t = C.c_uint64(), C.c_uint64()
    arr = _f32(net)
    rc = lib().od_argmax_random_ties(arr, arr.size, int(base), int(seed), int(invocation), C.byref(k), C.byref(t))
    return int(k.value), int(t.value), rc


def key_decode(k: int):
    hi = (k >> 32) & 0xFFFFFFFF
    idx = k & 0xFFFFFFFF
    if hi == 0xFFFFFFFF:
        return float("nan"), idx
    b = (hi & 0x7FFFFFFF) if (hi >> 31) else (~hi & 0xFFFFFFFF)
    return float(np.array([b], np.uint32).view(np.float32)[0]), idx


def pp_episode(n_levels, levels, w, params, init, n_steps, n_samples, seed, speeds=(1.0, 0.8, 0.6),
               capture_radius=0.5):
    """Closed-loop episode (spec/MODELS.md §7): (traj[T+1,6], keys[T], (outcome, steps))."""
    traj = np.zeros((int(n_steps) + 1) * 6, np.float32)
    keys = np.zeros(int(n_steps), np.uint64)
    status = np.zeros(2, np.int32)
    rc = lib().od_pp_episode(_u32(n_levels), _f32(levels), _f32(w), _f32(params), _f32(init), int(n_steps),
                             int(n_samples), int(seed), _f32(speeds), float(capture_radius), traj, keys, status)
    if rc != 0:
        raise ValueError("od_pp_episode rejected its arguments")
    return traj.reshape(-1, 6), keys, (int(status[0]), int(status[1]))


def pp_amr(n_levels, w, params, inputs, lo, hi, rounds, n_samples, seed, invocation0=0):
    """Coarse-to-fine refinement (spec/MODELS.md §9): (keys[R], boxes[R+1, 3, 2])."""
    keys = np.zeros(int(rounds), np.uint64)
    boxes = np.zeros((int(rounds) + 1) * 6, np.float32)
    rc = lib().od_pp_amr(_u32(n_levels), _f32(w), _f32(params), _f32(inputs), _f32(lo), _f32(hi), int(rounds),
                         int(n_samples), int(seed), int(invocation0), keys, boxes)
    if rc != 0:
        raise ValueError("od_pp_amr rejected its arguments")
    return keys, boxes.reshape(-1, 3, 2)


# ---------------------------------------------------------------- DDM / LCI

def ddm_params(drift, noise, threshold, x0, dt, n_steps, rt_bin_steps, n_x_bins, x_lo, x_hi):
    return DdmParams(drift, noise, threshold, x0, dt, n_steps, rt_bin_steps, n_x_bins, x_lo, x_hi)


def ddm_trial(p: DdmParams, seed: int, trial: int):
    ch, st, xe = C.c_int(), C.c_uint32(), C.c_float()
    lib().od_ddm_trial(C.byref(p), seed, trial, C.byref(ch), C.byref(st), C.byref(xe))
    return ch.value, st.value, xe.value


def ddm_hist_sizes(p: DdmParams):
    nb = (p.n_steps + p.rt_bin_steps - 1) // p.rt_bin_steps
    return 2 * nb + 1, 2, p.n_x_bins + 2


def ddm_batch(p: DdmParams, seed: int, t0: int, t1: int, threads: int = 1, lci=None):
    """DDM batch histograms (spec/MODELS.md §4); with lci = (leak, offset) the
    LCI update of §5 instead (drift = input I), binned identically."""
    a, b, c = ddm_hist_sizes(p)
    threads = max(1, min(int(threads), max(t1 - t0, 1)))
    seg = (t1 - t0 + threads - 1) // threads
    parts = [(np.zeros(a, np.uint64), np.zeros(b, np.uint64), np.zeros(c, np.uint64)) for _ in range(threads)]
    L = lib()

    def work(t):
        s = t0 + t * seg
        e = min(t1, s + seg)
        if e > s:
            if lci is None:
                L.od_ddm_batch(C.byref(p), seed, s, e, *parts[t])
            else:
                L.od_lci_batch(C.byref(p), float(lci[0]), float(lci[1]), seed, s, e, *parts[t])

    ts = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return tuple(sum(p_[k] for p_ in parts) for k in range(3))


def lci_trial(inp, leak, offset, noise, dt, threshold, n_steps, seed, unit):
    ch, st, xe = C.c_int(), C.c_uint32(), C.c_float()
    lib().od_lci_trial(inp, leak, offset, noise, dt, threshold, n_steps, seed, unit,
                       C.byref(ch), C.byref(st), C.byref(xe))
    return ch.value, st.value, xe.value


# ---------------------------------------------------------------- Stroop

def stroop_eval(n_levels, levels, w, params, begin, end, n_trials, seed,
                trial_begin=0, trial_end=None, threads=1):
    """Returns (counts[n,3] uint64, net[n] float32 or None if a trial sub-range)."""
    if trial_end is None:
        trial_end = n_trials
    n = int(end) - int(begin)
    counts = np.zeros((n, 3), np.uint64)
    full = (trial_begin == 0 and trial_end == n_trials)
    net = np.zeros(n, np.float32) if full else None
    args = (_u32(n_levels), _f32(levels), _f32(w), _f32(params))
    L = lib()
    threads = max(1, min(int(threads), max(n, 1)))
    seg = (n + threads - 1) // threads

    def work(t):
        b = begin + t * seg
        e = min(begin + n, b + seg)
        if e <= b:
            return
        cv = counts[b - begin:e - begin]
        nv = net[b - begin:e - begin].ctypes.data_as(C.c_void_p) if full else None
        rc = L.od_stroop_eval(*args, b, e, int(n_trials), int(trial_begin), int(trial_end),
                              int(seed), cv.ctypes.data_as(C.c_void_p), nv)
        if rc != 0:
            raise ValueError("od_stroop_eval rejected its arguments")

    ts = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return counts, net


def ddmg_trial(params, u0, u1, seed, unit):
    """DDM control grid trial (spec/MODELS.md §6c): (resp 1 correct / 0 error / -1 undecided, step)."""
    r, st = C.c_int(), C.c_uint32()
    lib().od_ddmg_trial(_f32(params), float(u0), float(u1), int(seed), int(unit), C.byref(r), C.byref(st))
    return r.value, st.value


def ddmg_value(params, w, u0, u1, n_trials, n_correct, n_undecided, rt_sum):
    return lib().od_ddmg_value(_f32(params), _f32(w), float(u0), float(u1), int(n_trials), int(n_correct),
                               int(n_undecided), int(rt_sum))


def ddmg_eval(n_levels, levels, w, params, begin, end, n_trials, seed, trial_begin=0, trial_end=None, threads=1):
    """Returns (counts[n,3] uint64 {n_correct, n_undecided, rt_sum}, net[n] float32 or None)."""
    if trial_end is None:
        trial_end = n_trials
    n = int(end) - int(begin)
    counts = np.zeros((n, 3), np.uint64)
    full = (trial_begin == 0 and trial_end == n_trials)
    net = np.zeros(n, np.float32) if full else None
    args = (_u32(n_levels), _f32(levels), _f32(w), _f32(params))
    threads = max(1, min(int(threads), max(n, 1)))
    seg = (n + threads - 1) // threads

    def work(t):
        b = begin + t * seg
        e = min(begin + n, b + seg)
        if e <= b:
            return
        cv = counts[b - begin:e - begin]
        nv = net[b - begin:e - begin].ctypes.data_as(C.c_void_p) if full else None
        if lib().od_ddmg_eval(*args, b, e, int(n_trials), int(trial_begin), int(trial_end), int(seed),
                              cv.ctypes.data_as(C.c_void_p), nv) != 0:
            raise ValueError("od_ddmg_eval rejected its arguments")

    ts = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return counts, net


def stroop_energy(params, u_c, u_s, seed, i, n_trials, t0, t1, threads=1):
    """Decision-energy trace (spec/MODELS.md §6b; "predict decision energy
    over time"): int64 sums over trials [t0, t1) of llrint(x0(n) x1(n) 2^24)."""
    N = int(np.float32(params[10]))
    P = np.ascontiguousarray(np.asarray(params, np.float32))
    threads = max(1, min(int(threads), max(int(t1) - int(t0), 1)))
    seg = (int(t1) - int(t0) + threads - 1) // threads
    parts = [np.zeros(N, np.int64) for _ in range(threads)]

    def work(k):
        s0 = int(t0) + k * seg
        s1 = min(int(t1), s0 + seg)
        if s1 > s0:
            lib().od_stroop_energy(P, float(u_c), float(u_s), int(seed), int(i), int(n_trials), s0, s1, parts[k])

    import threading
    ts = [threading.Thread(target=work, args=(k,)) for k in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return np.sum(parts, axis=0)


def stroop_trial(params, u_c, u_s, seed, unit, trial):
    r, st = C.c_int(), C.c_uint32()
    lib().od_stroop_trial(_f32(params), u_c, u_s, seed, unit, trial, C.byref(r), C.byref(st))
    return r.value, st.value


def stroop_trace(params, u_c, u_s, seed, unit, trial):
    """od_stroop_trace: (resp, step, states[N, 4] = (h0, h1, x0, x1) after each step)."""
    P = _f32(params)
    tr = np.zeros(4 * int(P[10]), np.float32)
    r, st = C.c_int(), C.c_uint32()
    lib().od_stroop_trace(P, u_c, u_s, seed, unit, trial, C.byref(r), C.byref(st), tr)
    return r.value, st.value, tr.reshape(-1, 4)


def stroop_value(params, w, u_c, u_s, n_trials, n_correct, n_undecided, rt_sum):
    return lib().od_stroop_value(_f32(params), _f32(w), u_c, u_s, n_trials,
                                 int(n_correct), int(n_undecided), int(rt_sum))


# ---------------------------------------------------------------- Extended Stroop A/B

def ext_stroop_eval(variant, n_levels, levels, w, params, begin, end, n_trials, seed, threads=1,
                    trial_begin=0, trial_end=None):
    """variant 0 = A, 1 = B (spec/MODELS.md §10): (counts[n,3] uint64, net[n] float32 or None for a
    trial sub-range)."""
    if trial_end is None:
        trial_end = n_trials
    n = int(end) - int(begin)
    counts = np.zeros((n, 3), np.uint64)
    full = (trial_begin == 0 and trial_end == n_trials)
    net = np.zeros(n, np.float32)
    args = (_u32(n_levels), _f32(levels), _f32(w), _f32(params))
    L = lib()
    threads = max(1, min(int(threads), max(n, 1)))
    seg = (n + threads - 1) // threads

    def work(t):
        b = begin + t * seg
        e = min(begin + n, b + seg)
        if e <= b:
            return
        rc = L.od_ext_stroop_eval_range(int(variant), *args, b, e, int(n_trials), int(trial_begin), int(trial_end),
                                        int(seed), counts[b - begin:e - begin].ctypes.data_as(C.c_void_p),
                                        net[b - begin:e - begin].ctypes.data_as(C.c_void_p) if full else None)
        if rc != 0:
            raise ValueError("od_ext_stroop_eval rejected its arguments")

    ts = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return counts, (net if full else None)


def ext_stroop_trial(variant, params, u_c, u_s, seed, unit, trial):
    hit = np.zeros(2, np.int32)
    st = np.zeros(2, np.uint32)
    fn = lib().od_ext_stroop_trial_a if variant == 0 else lib().od_ext_stroop_trial_b
    fn(_f32(params), float(u_c), float(u_s), int(seed), int(unit), int(trial), hit, st)
    return (int(hit[0]), int(hit[1])), (int(st[0]), int(st[1]))
