"""CPU-only checks of the boundary: libdistill.so loads, exports every symbol
include/distill.h declares, validates arguments before touching CUDA, and its
pure host key decoder agrees with the oracle's key encoder.  No kernel runs."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def abi():
    import __graft_entry__ as g
    g.build_cuda()
    from paper_2110_15425_b200 import _abi
    return _abi


def test_every_declared_symbol_is_exported(abi):
    hdr = open(os.path.join(ROOT, "include", "distill.h")).read()
    names = set(re.findall(r"\b(distill_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 12
    L = abi.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(abi.EXPORTS) == names


def test_abi_version_matches_header(abi):
    hdr = open(os.path.join(ROOT, "include", "distill.h")).read()
    v = int(re.search(r"#define DISTILL_ABI_VERSION (\d+)", hdr).group(1))
    assert abi.lib().distill_abi_version() == v


def test_library_has_sm100a_code():
    import subprocess
    lib = os.path.join(ROOT, "paper_2110_15425_b200", "libdistill.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _desc(abi, kind=1, D=3, L=(2, 2, 2), n_params=3):
    L = np.asarray(L, np.uint32)
    lev = np.zeros(int(L.sum()), np.float32)
    w = np.zeros(D, np.float32)
    p = np.zeros(max(n_params, 1), np.float32)
    keep = (L, lev, w, p)
    d = abi.ModelDesc(kind, D, abi._uptr(L), abi._fptr(lev), abi._fptr(w), abi._fptr(p), n_params)
    return d, keep


@pytest.mark.parametrize("kw,status", [
    (dict(kind=99), 3),                               # unknown kind -> UNSUPPORTED
    (dict(D=2, L=(2, 2)), 3),                         # PP needs 3 signals
    (dict(L=(2, 0, 2)), 1),                           # zero levels -> INVALID_ARG
    (dict(n_params=2), 1),                            # wrong param count
    (dict(L=(65536, 65536, 2)), 2),                   # > 2^32-1 allocations -> OVERFLOW
])
def test_load_model_validates_before_cuda(abi, kw, status):
    import ctypes as C
    d, keep = _desc(abi, **kw)
    h = C.c_void_p()
    st = abi.lib().distill_load_model(C.byref(d), 0, C.byref(h))
    assert st == status, abi.lib().distill_last_error()
    assert not h.value
    assert abi.lib().distill_last_error()


def test_null_arguments_rejected(abi):
    import ctypes as C
    L = abi.lib()
    assert L.distill_load_model(None, 0, None) == abi.E_INVALID_ARG
    assert L.distill_eval_grid(None, None, None) == abi.E_INVALID_ARG
    assert L.distill_ddm_batch(None, None) == abi.E_INVALID_ARG
    assert L.distill_argmax(None, 10, 0, None, None) == abi.E_INVALID_ARG
    k = C.c_uint64()
    for fn in (L.distill_eval_grid_host, L.distill_eval_grid_host_async):
        assert fn(None, None, 6, 0, 1, 1, 0, 0, None, C.byref(k), None) == abi.E_INVALID_ARG
        assert "NULL" in L.distill_last_error().decode()
    L.distill_free_model(None)  # NULL-safe


def test_key_decode_inverts_oracle_keys(abi, orc):
    import ctypes as C
    rng = np.random.default_rng(1)
    vals = list(rng.normal(size=50).astype(np.float32) * 1e3) + [0.0, -0.0, np.inf, -np.inf, 1e-40]
    for i, v in enumerate(vals):
        k = orc.key(float(v), 1000 + i)
        c, idx = C.c_float(), C.c_uint64()
        assert abi.lib().distill_key_decode(k, C.byref(c), C.byref(idx)) == abi.OK
        assert idx.value == 1000 + i
        assert c.value == (0.0 if v == 0 else float(np.float32(v)))
    c, idx = C.c_float(), C.c_uint64()
    assert abi.lib().distill_key_decode(orc.key(float("nan"), 3), C.byref(c), C.byref(idx)) == abi.E_NO_VALID


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2110_15425_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|distill_oracle|\bod_[a-z])", src), f


def test_next_row_entry_points_validate_before_cuda(abi):
    """NEXT-1/2/4 entry points reject bad arguments with E_INVALID_ARG and never abort."""
    import ctypes as C
    L = abi.lib()
    e = abi.EpisodeArgs()
    assert L.distill_pp_episode(None, C.byref(e), None) == abi.E_INVALID_ARG
    g = abi.AmrArgs()
    assert L.distill_pp_amr(None, C.byref(g), None) == abi.E_INVALID_ARG
    assert L.distill_argmax_ties(None, 5, 0, 0, 0, None, None, None) == abi.E_INVALID_ARG
    # empty input is a no-op (no CUDA call needed)
    dummy = C.c_uint64(0)
    assert L.distill_argmax_ties(None, 0, 0, 0, 0, C.addressof(dummy), C.addressof(dummy), None) == abi.OK
    assert L.distill_argmax(None, 0, 0, C.addressof(dummy), None) == abi.OK
    assert L.distill_argmax(None, 1, 0xFFFFFFFF, C.addressof(dummy), None) == abi.E_INVALID_ARG
    assert L.distill_sm_clock_probe(0, None, None) == abi.E_INVALID_ARG


def test_eval_grid_multi_validates_before_cuda(abi):
    import ctypes as C
    L = abi.lib()
    a = abi.MultiArgs()
    assert L.distill_eval_grid_multi(None, C.byref(a), None) == abi.E_INVALID_ARG
    assert L.distill_eval_grid_multi(None, None, None) == abi.E_INVALID_ARG


def test_binding_buffer_checks_on_cpu():
    """The binding's buffer checks run before any ABI call: host tensors, wrong
    element types, non-contiguous or short buffers are rejected with ValueError."""
    import pytest
    import torch
    from paper_2110_15425_b200 import api
    with pytest.raises(ValueError, match="CUDA"):
        api._dev_ptr(torch.zeros(4), "net", 4)
    assert api._dev_ptr(None, "net", 4) is None
    t = torch.zeros(4, dtype=torch.float64)
    t.is_cuda                                   # host tensor: the CUDA check fires first
    with pytest.raises(ValueError):
        api._dev_ptr(t, "net", 4)
    assert set(api._BUF_DTYPE.values()) == {"float32", "int64", "int32"}


def test_ddm_grid_model_validation_without_gpu(abi):
    """Kind 5 (DDM control grid) needs 2 signals and 7 params with an integer step count."""
    import ctypes as C
    import numpy as np
    L = abi.lib()
    nl = np.array([3, 4], np.uint32)
    lev = np.zeros(7, np.float32)
    w = np.zeros(2, np.float32)
    for params, want in ((np.zeros(6, np.float32), abi.E_INVALID_ARG),
                         (np.array([0.2, 1.5, 1.0, 0.01, 1.0, 0.5, 0.5], np.float32), abi.E_INVALID_ARG)):
        d = abi.ModelDesc(5, 2, abi._uptr(nl), abi._fptr(lev), abi._fptr(w), abi._fptr(params), params.size)
        h = C.c_void_p()
        assert L.distill_load_model(C.byref(d), 0, C.byref(h)) == want


def test_round2_entry_validation_without_gpu(abi):
    """Round-2 boundary additions reject bad arguments synchronously, before any
    CUDA call: the signed key reset (NULL, misaligned), misaligned histogram
    buffers of the DDM batch, and the binding's ABI-version guard."""
    import ctypes as C
    L = abi.lib()
    assert L.distill_key_reset_signed(None, None) == abi.E_INVALID_ARG
    assert L.distill_key_reset_signed(C.c_void_p(0x1003), None) == abi.E_INVALID_ARG
    assert "misaligned" in L.distill_last_error().decode()
    a = abi.DdmArgs(1.0, 1.0, 1.0, 0.0, 0.01, 10, 1, 4, -1.0, 1.0, 0, 10, 1,
                    C.c_void_p(0x1004), C.c_void_p(0x2000), C.c_void_p(0x3000))
    assert L.distill_ddm_batch(C.byref(a), None) == abi.E_INVALID_ARG
    assert "aligned" in L.distill_last_error().decode()
    assert abi.ABI_VERSION == L.distill_abi_version() == 3
    assert abi.KEY_INIT_SIGNED == (1 << 63) - 1
    # the eval-args struct carries key_order at the end (include/distill.h, ABI 2)
    assert abi.EvalArgs._fields_[-1][0] == "key_order"


def test_rng_entry_validation_without_gpu(abi):
    """Rows a2/a3 on their own (distill_rng_*): NULL / misaligned buffers, empty
    ranges, zero per-unit counts and index overflow are decided synchronously,
    before any CUDA call (include/distill.h)."""
    import ctypes as C
    L = abi.lib()
    ok, bad, ovf = 0, abi.E_INVALID_ARG, abi.E_OVERFLOW
    assert L.distill_rng_rad(None, 0, None, None) == ok                  # empty: nothing enqueued
    assert L.distill_rng_rad(None, 5, C.c_void_p(0x1000), None) == bad
    assert L.distill_rng_rad(C.c_void_p(0x1002), 5, C.c_void_p(0x1000), None) == bad
    assert "aligned" in L.distill_last_error().decode()
    assert L.distill_rng_normals_acc(1, 0, 0, 12, None, None) == ok
    assert L.distill_rng_normals_acc(1, 0, 4, 12, None, None) == bad
    assert L.distill_rng_normals_acc(1, 0, 4, 0, C.c_void_p(0x1000), None) == bad
    assert L.distill_rng_normals_acc(1, 0, 1 << 40, 1 << 30, C.c_void_p(0x1000), None) == ovf
    assert L.distill_rng_normals_acc(1, (1 << 64) - 2, 4, 12, C.c_void_p(0x1000), None) == ovf
    assert L.distill_rng_normals_pp(1, 0, 0, 10, 0, None, None) == ok
    assert L.distill_rng_normals_pp(1, 0, 4, 0, 0, C.c_void_p(0x1000), None) == bad
    assert L.distill_rng_normals_pp(1, 0xFFFFFFF0, 32, 10, 0, C.c_void_p(0x1000), None) == ovf
    assert L.distill_rng_normals_pp(1, 0, 4, 10, 0, C.c_void_p(0x1001), None) == bad
