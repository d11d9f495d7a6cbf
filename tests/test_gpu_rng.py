"""GPU parity of rows a2 (Philox4x32-10) and a3 (uniform -> normal) on their own.

The hot kernels inline these device functions; here they run over chosen
inputs through the C ABI (distill_rng_*) and are compared bit for bit with the
oracle's spec/RNG.md functions: the radius over every radius value, and the
stream-1 / stream-2 normals over many RNG units, including the 32-bit
boundaries of the unit and allocation words and the ragged tails.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 0x9E3779B97F4A7C15


@pytest.fixture(scope="module")
def D():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no fallback)"
    torch.cuda.set_device(0)
    import paper_2110_15425_b200 as D
    return D


def _bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def test_rad_every_radius_value_bit_exact(D, orc):
    """rad_spec depends on the 24 bits R >> 8 (region bit + 23 uniform bits):
    all 2^24 of them, with random low bytes, against od_rad (spec/RNG.md §3)."""
    rng = np.random.default_rng(11)
    R = (np.arange(1 << 24, dtype=np.uint32) << np.uint32(8)) | rng.integers(0, 256, 1 << 24, dtype=np.uint32)
    gpu = D.rng_rad(R).cpu().numpy()
    ref = orc.rad_array(R)
    bad = np.flatnonzero(_bits(gpu) != _bits(ref))
    assert bad.size == 0, f"{bad.size} mismatches, first R=0x{int(R[bad[0]]):08x}: {gpu[bad[0]]} vs {ref[bad[0]]}"
    # both regions and the octave ends are in the sweep
    assert gpu.min() > 0 and np.isfinite(gpu).all()


@pytest.mark.parametrize("n", [0, 1, 2, 3, 255, 257])
def test_rad_ragged_lengths(D, orc, n):
    """Two words per thread: odd counts and lengths that do not fill a block."""
    R = np.random.default_rng(n).integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    gpu = D.rng_rad(R).cpu().numpy()
    assert gpu.size == n
    if n:
        assert np.array_equal(_bits(gpu), _bits(orc.rad_array(R)))


@pytest.mark.parametrize("per_unit", [1, 6, 7, 12, 19, 24, 30])
def test_normals_acc_bit_exact(D, orc, per_unit):
    """Stream-2 normals (DDM / Stroop / LCI noise): the acc_normals12 groups and
    both ragged-tail paths (<= 6: one Philox block; 7..11: two), for units that
    straddle the 32-bit boundary of the unit word (c0 / c2 of the counter)."""
    begin, n_units = (1 << 32) - 700, 1400
    gpu = D.rng_normals_acc(SEED, begin, n_units, per_unit).cpu().numpy()
    ref = np.stack([orc.normal_acc(SEED, begin + u, 0, per_unit) for u in range(n_units)])
    assert np.array_equal(_bits(gpu), _bits(ref))


def test_normals_acc_angle_coverage(D, orc):
    """Enough pairs (240k) that nearly every one of the 65536 16-bit angle words of
    the sextet packing and every radius-table row is exercised."""
    n_units, per = 40_000, 12
    gpu = D.rng_normals_acc(SEED + 1, 123, n_units, per).cpu().numpy()
    ref = np.stack([orc.normal_acc(SEED + 1, 123 + u, 0, per) for u in range(n_units)])
    assert np.array_equal(_bits(gpu), _bits(ref))
    z = gpu.ravel().astype(np.float64)
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1.0) < 0.01


@pytest.mark.parametrize("n_samples,invocation", [(1, 0), (7, 5), (10, 0xFFFFFFFF)])
def test_normals_pp_bit_exact(D, orc, n_samples, invocation):
    """Stream-1 sextets (predator-prey observation noise), samples in lane pairs
    with an odd tail, allocations up to the top of the 32-bit range."""
    begin, n_alloc = (1 << 32) - 300, 300
    gpu = D.rng_normals_pp(SEED, begin, n_alloc, n_samples, invocation).cpu().numpy()
    ref = np.stack([np.stack([orc.normal_sextet(SEED, begin + t, s, invocation) for s in range(n_samples)])
                    for t in range(n_alloc)])
    assert np.array_equal(_bits(gpu), _bits(ref))
