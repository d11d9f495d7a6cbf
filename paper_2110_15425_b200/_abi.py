"""ctypes binding of libdistill.so (include/distill.h) — argument marshalling only.

Names mirror the C ABI (``distill_load_model`` -> ``load_model`` ...).  Device
buffers are torch CUDA tensors (PyTorch is plumbing: memory, streams, process
groups); every step of the hot path runs in the library's kernels.  There is
no CPU fallback: if the shared library is missing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DISTILL_LIB selects another build of the same library (e.g. the bounds-checked debug
# build, -DDISTILL_BOUNDS_CHECK=1, tools/gpu/r2_bounds.sh); default: the in-tree product build
LIB_PATH = os.environ.get("DISTILL_LIB") or os.path.join(_HERE, "libdistill.so")

OK, E_INVALID_ARG, E_OVERFLOW, E_UNSUPPORTED, E_CUDA, E_NO_VALID = range(6)
MODEL_PREDATOR_PREY = 1
MODEL_STROOP_LCA = 2
KEY_INIT = 0xFFFFFFFFFFFFFFFF
KEY_INIT_SIGNED = 0x7FFFFFFFFFFFFFFF      # signed key order: stored word = key ^ 2^63
ABI_VERSION = 3                           # include/distill.h DISTILL_ABI_VERSION


class DistillError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"distill status {status}: {msg}")
        self.status = status


class ModelDesc(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("n_signals", C.c_uint32),
                ("n_levels", C.POINTER(C.c_uint32)), ("levels", C.POINTER(C.c_float)),
                ("cost_weights", C.POINTER(C.c_float)), ("params", C.POINTER(C.c_float)),
                ("n_params", C.c_uint32)]


class EvalArgs(C.Structure):
    _fields_ = [("inputs", C.POINTER(C.c_float)), ("n_inputs", C.c_uint32),
                ("begin", C.c_uint64), ("end", C.c_uint64),
                ("n_samples", C.c_uint32), ("invocation", C.c_uint32), ("seed", C.c_uint64),
                ("d_net", C.c_void_p), ("d_best", C.c_void_p), ("d_counts", C.c_void_p),
                ("trial_begin", C.c_uint32), ("trial_end", C.c_uint32), ("key_order", C.c_uint32)]


class DdmArgs(C.Structure):
    _fields_ = [("drift", C.c_float), ("noise", C.c_float), ("threshold", C.c_float),
                ("x0", C.c_float), ("dt", C.c_float), ("n_steps", C.c_uint32),
                ("rt_bin_steps", C.c_uint32), ("n_x_bins", C.c_uint32),
                ("x_lo", C.c_float), ("x_hi", C.c_float),
                ("trial_begin", C.c_uint64), ("trial_end", C.c_uint64), ("seed", C.c_uint64),
                ("d_rt_hist", C.c_void_p), ("d_rt_sum", C.c_void_p), ("d_x_hist", C.c_void_p)]


class EpisodeArgs(C.Structure):
    _fields_ = [("n_steps", C.c_uint32), ("n_samples", C.c_uint32), ("seed", C.c_uint64),
                ("v_player", C.c_float), ("v_prey", C.c_float), ("v_predator", C.c_float),
                ("capture_radius", C.c_float), ("h_init", C.POINTER(C.c_float)),
                ("d_traj", C.c_void_p), ("d_keys", C.c_void_p), ("d_status", C.c_void_p)]


class AmrArgs(C.Structure):
    _fields_ = [("inputs", C.POINTER(C.c_float)), ("n_inputs", C.c_uint32),
                ("lo", C.c_float * 3), ("hi", C.c_float * 3),
                ("rounds", C.c_uint32), ("n_samples", C.c_uint32), ("invocation0", C.c_uint32),
                ("seed", C.c_uint64), ("d_keys", C.c_void_p), ("d_boxes", C.c_void_p), ("d_levels", C.c_void_p)]


class MultiArgs(C.Structure):
    _fields_ = [("d_inputs", C.c_void_p), ("n_sets", C.c_uint32), ("n_invocations", C.c_uint32),
                ("invocation0", C.c_uint32), ("n_samples", C.c_uint32),
                ("begin", C.c_uint64), ("end", C.c_uint64), ("seed", C.c_uint64),
                ("d_net", C.c_void_p), ("d_best", C.c_void_p)]


EXPORTS = {
    "distill_abi_version": (C.c_int, []),
    "distill_last_error": (C.c_char_p, []),
    "distill_load_model": (C.c_int, [C.POINTER(ModelDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "distill_free_model": (None, [C.c_void_p]),
    "distill_grid_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "distill_eval_grid": (C.c_int, [C.c_void_p, C.POINTER(EvalArgs), C.c_void_p]),
    "distill_eval_grid_host": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.c_uint32, C.c_uint64, C.c_uint64,
                                         C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p,
                                         C.POINTER(C.c_uint64), C.c_void_p]),
    "distill_eval_grid_host_async": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.c_uint32, C.c_uint64,
                                               C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p,
                                               C.c_void_p, C.c_void_p]),
    "distill_argmax": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]),
    "distill_argmax_ties": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
    "distill_key_reset": (C.c_int, [C.c_void_p, C.c_void_p]),
    "distill_key_reset_signed": (C.c_int, [C.c_void_p, C.c_void_p]),
    "distill_key_decode": (C.c_int, [C.c_uint64, C.POINTER(C.c_float), C.POINTER(C.c_uint64)]),
    "distill_ddm_batch": (C.c_int, [C.POINTER(DdmArgs), C.c_void_p]),
    "distill_launch_count": (C.c_uint64, []),
    "distill_sm_clock_probe": (C.c_int, [C.c_uint32, C.POINTER(C.c_double), C.c_void_p]),
    "distill_rng_rad": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "distill_rng_normals_acc": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p]),
    "distill_rng_normals_pp": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                         C.c_void_p]),
    "distill_pp_amr": (C.c_int, [C.c_void_p, C.POINTER(AmrArgs), C.c_void_p]),
    "distill_pp_amr_begin": (C.c_int, [C.c_void_p, C.POINTER(AmrArgs), C.c_void_p]),
    "distill_pp_amr_levels": (C.c_int, [C.c_void_p, C.POINTER(AmrArgs), C.c_uint32, C.c_void_p]),
    "distill_pp_amr_search": (C.c_int, [C.c_void_p, C.POINTER(AmrArgs), C.c_uint32, C.c_uint64, C.c_uint64,
                                        C.c_void_p]),
    "distill_pp_amr_refine": (C.c_int, [C.c_void_p, C.POINTER(AmrArgs), C.c_uint32, C.c_void_p]),
    "distill_eval_grid_multi": (C.c_int, [C.c_void_p, C.POINTER(MultiArgs), C.c_void_p]),
    "distill_lci_batch": (C.c_int, [C.POINTER(DdmArgs), C.c_float, C.c_float, C.c_void_p]),
    "distill_stroop_energy": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                        C.c_void_p, C.c_void_p]),
    "distill_pp_episode": (C.c_int, [C.c_void_p, C.POINTER(EpisodeArgs), C.c_void_p]),
    "distill_pp_episode_begin": (C.c_int, [C.c_void_p, C.POINTER(EpisodeArgs), C.c_void_p]),
    "distill_pp_episode_search": (C.c_int, [C.c_void_p, C.POINTER(EpisodeArgs), C.c_uint32, C.c_uint64, C.c_uint64,
                                            C.c_void_p]),
    "distill_pp_episode_advance": (C.c_int, [C.c_void_p, C.POINTER(EpisodeArgs), C.c_uint32, C.c_void_p]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libdistill.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.distill_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {L.distill_abi_version()}, the binding needs {ABI_VERSION}: rebuild")
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != OK:
        raise DistillError(status, lib().distill_last_error().decode(errors="replace"))


def _fptr(arr):
    return arr.ctypes.data_as(C.POINTER(C.c_float))


def _uptr(arr):
    return arr.ctypes.data_as(C.POINTER(C.c_uint32))
