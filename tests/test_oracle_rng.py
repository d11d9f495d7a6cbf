"""Pins for the oracle's counter-based normal generator (spec/RNG.md).

Each pin is something other than the oracle itself: published known-answer
vectors, binary64 libm, the normal law's moments and CDF.
"""
import math

import numpy as np
import pytest
from scipy import stats


# Random123 kat_vectors for philox4x32-10 (spec/RNG.md §1)
KATS = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


@pytest.mark.parametrize("ctr,key,want", KATS)
def test_philox_known_answers(orc, ctr, key, want):
    assert [int(v) for v in orc.philox(ctr, key)] == want


def _ulp32(ref):
    return np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)


def test_philox_matches_curand_host_generator(orc):
    """Library pin: cuRAND's host-side PHILOX4_32_10 generator (default ordering)
    emits block t = Philox4x32-10(ctr = (t >> 16, 0, t & 0xFFFF, 0), key = seed)
    — 70,000 blocks (both sides of the 2^16 subsequence wrap) must equal the oracle."""
    import ctypes
    import os
    path = "/usr/local/cuda/lib64/libcurand.so"
    if not os.path.exists(path):
        pytest.skip("libcurand not present")
    cr = ctypes.CDLL(path)
    for seed in (0, 0xDEADBEEF12345678):
        gen = ctypes.c_void_p()          # a fresh generator per seed (offset 0)
        assert cr.curandCreateGeneratorHost(ctypes.byref(gen), 161) == 0     # CURAND_RNG_PSEUDO_PHILOX4_32_10
        try:
            assert cr.curandSetPseudoRandomGeneratorSeed(gen, ctypes.c_ulonglong(seed)) == 0
            n = 70_000
            out = np.zeros(4 * n, np.uint32)
            assert cr.curandGenerate(gen, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(4 * n)) == 0
        finally:
            cr.curandDestroyGenerator(gen)
        blk = out.reshape(-1, 4)
        key = (seed & 0xFFFFFFFF, seed >> 32)
        for t in list(range(0, n, 37)) + [65535, 65536, n - 1]:
            assert np.array_equal(blk[t], orc.philox((t >> 16, 0, t & 0xFFFF, 0), key)), (seed, t)


def test_rad_exhaustive_over_all_radius_words(orc):
    """rad_spec (spec/RNG.md §3) for every one of the 2^23 radius values
    N = (R >> 8) | 1: within 4 * 2^-24 relative of sqrt(-2 ln(N 2^-24)) in
    binary64 libm (the plain definition of the Box-Muller radius)."""
    N = np.arange(1, 2 ** 24, 2, dtype=np.uint64)
    R = (N << np.uint64(8)).astype(np.uint32)          # (R >> 8) | 1 == N
    y = orc.rad_array(R).astype(np.float64)
    ref = np.sqrt(-2.0 * np.log(N.astype(np.float64) * 2.0 ** -24))
    rel = np.abs(y - ref) / ref
    assert rel.max() <= 4 * 2.0 ** -24, rel.max() / 2.0 ** -24
    # the low byte of the word and its lowest retained bit do not matter: N is forced odd
    assert np.array_equal(orc.rad_array(R | np.uint32(0xFF)), y.astype(np.float32))
    assert np.array_equal(orc.rad_array(R ^ np.uint32(0x100)), y.astype(np.float32))


def test_rad_table_is_the_interpolating_cubic(orc):
    """Independent check of the table RT: in every segment (region r, octave e,
    sub-segment j) the stored cubic, evaluated in binary64 from its binary32
    coefficients, passes through sqrt(-2 ln u1) at the four nodes
    t = (-3, -1, 1, 3)/128 (numpy's own interpolant through those points agrees
    coefficient by coefficient to binary32 rounding)."""
    T = orc.rad_table().astype(np.float64)
    tau = np.array([-3, -1, 1, 3], np.float64) / 128
    worst_val, worst_coef = 0.0, 0.0
    for r in (0, 1):
        for e in range(23):
            for j in range(16):
                c = 1 + (2 * j + 1) / 32
                x = (c + tau) * 2.0 ** e
                Nk = 2.0 ** 24 - x if r else x
                f = np.sqrt(-2 * np.log(Nk * 2.0 ** -24))
                row = T[368 * r + 16 * e + j]
                p = row[0] + tau * (row[1] + tau * (row[2] + tau * row[3]))
                worst_val = max(worst_val, float(np.max(np.abs(p - f) / f)))
                want = np.polyfit(tau, f, 3)[::-1]
                scale = np.abs(want) * np.array([1, 1 / 32, 1 / 32 ** 2, 1 / 32 ** 3]) / abs(want[0])
                dev = np.abs(row - want) * np.array([1, 1 / 32, 1 / 32 ** 2, 1 / 32 ** 3]) / abs(want[0])
                worst_coef = max(worst_coef, float(dev.max()))
    assert worst_val < 2e-7, worst_val
    assert worst_coef < 1e-7, worst_coef


def test_rsqrt_dense(orc):
    worst = 0.0
    for e in range(-60, 60, 3):
        b0 = np.float32(2.0 ** e).view(np.uint32)
        b1 = np.float32(2.0 ** (e + 2)).view(np.uint32)
        x = np.arange(b0, b1, 5, dtype=np.uint32).view(np.float32)
        y = orc.rsqrt_array(x).astype(np.float64)
        ref = 1.0 / np.sqrt(x.astype(np.float64))
        worst = max(worst, float((np.abs(y - ref) / ref).max()))
    assert worst <= 4 * 2.0 ** -24, worst


def test_sincos2pi_exhaustive_24bit(orc):
    """All 2^24 angle words with the low byte clear."""
    a = (np.arange(2 ** 24, dtype=np.uint64) << 8).astype(np.uint32)
    c, s = orc.sincos2pi_array(a)
    th = a.astype(np.float64) * (2 * math.pi / 2.0 ** 32) - math.pi / 2
    assert np.abs(c - np.cos(th)).max() <= 4 * 2.0 ** -24
    assert np.abs(s - np.sin(th)).max() <= 4 * 2.0 ** -24
    # half-turn symmetry is exact: A and A + 2^31 give negated pairs
    c2, s2 = orc.sincos2pi_array(a ^ np.uint32(0x80000000))
    assert np.array_equal(c2, -c) and np.array_equal(s2, -s)
    # phi = 0 at A = 2^30 (r = 0): exactly (1, 0)
    assert orc.sincos2pi(1 << 30) == (1.0, 0.0)


def test_accumulator_normals_match_definition(orc):
    """Stream-2 (accumulator) normals 6k..6k+5 of a unit are the sextet of block
    Philox(key, (U_lo, k, U_hi, 2)): sqrt(-2 ln u1)(cos, sin)(2 pi A / 2^32 - pi/2)
    from the raw words (binary64 libm), within the primitives' error bounds, and
    a 64-bit unit id splits into (lo, hi) counter words."""
    seed = 12345
    for unit in (77, (5 << 32) | 9):
        z = orc.normal_acc(seed, unit, 0, 6 * 64)
        for blk in range(64):
            X = [int(v) for v in orc.philox([unit & 0xFFFFFFFF, blk, unit >> 32, 2], [seed & 0xFFFFFFFF, seed >> 32])]
            A = [(X[3] << 16) & 0xFFFFFFFF, X[3] & 0xFFFF0000, ((X[0] << 24) | ((X[1] & 0xFF) << 16)) & 0xFFFFFFFF]
            for e in range(3):
                u1 = ((X[e] >> 8) | 1) * 2.0 ** -24
                rad = math.sqrt(-2 * math.log(u1))
                th = 2 * math.pi * A[e] / 2.0 ** 32 - math.pi / 2
                assert abs(z[6 * blk + 2 * e] - rad * math.cos(th)) <= 1e-6 * max(1, rad)
                assert abs(z[6 * blk + 2 * e + 1] - rad * math.sin(th)) <= 1e-6 * max(1, rad)
        # any window [first, first+n) is the same stream
        assert np.array_equal(orc.normal_acc(seed, unit, 17, 50), z[17:67])


def test_sextet_packing_matches_definition(orc):
    seed = 42
    for i, s in [(0, 0), (5, 3), (123456, 99), (999999, 0)]:
        X = [int(v) for v in orc.philox([i, s, 0, 1], [seed, 0])]
        A = [(X[3] << 16) & 0xFFFFFFFF, X[3] & 0xFFFF0000,
             ((X[0] << 24) | ((X[1] & 0xFF) << 16)) & 0xFFFFFFFF]
        z = orc.normal_sextet(seed, i, s, 0)
        for e in range(3):
            rad = math.sqrt(-2 * math.log(((X[e] >> 8) | 1) * 2.0 ** -24))
            th = 2 * math.pi * A[e] / 2.0 ** 32 - math.pi / 2
            assert abs(z[2 * e] - rad * math.cos(th)) <= 1e-6 * max(1, rad)
            assert abs(z[2 * e + 1] - rad * math.sin(th)) <= 1e-6 * max(1, rad)


def test_accumulator_normals_moments_and_ks(orc):
    """10^6 normals: mean within +-0.004, variance within +-0.01 (S:343 bounds),
    kurtosis 3, KS vs Phi."""
    z = np.concatenate([orc.normal_acc(7, u, 0, 10000) for u in range(100)]).astype(np.float64)
    assert abs(z.mean()) < 0.004
    assert abs(z.var() - 1) < 0.01
    assert abs(((z - z.mean()) ** 4).mean() - 3) < 0.05
    assert stats.kstest(z, "norm").pvalue > 1e-3


def test_sextet_normals_moments_independence(orc):
    z = np.array([orc.normal_sextet(3, i, s) for i in range(2000) for s in range(50)], np.float64)
    assert np.abs(z.mean(0)).max() < 0.02
    assert np.abs(z.var(0) - 1).max() < 0.03
    cc = np.corrcoef(z.T)
    assert np.abs(cc - np.eye(6)).max() < 0.02
    assert stats.kstest(z.ravel(), "norm").pvalue > 1e-3


def test_uniform_endpoints(orc):
    """u1 = 2^-24 (N = 1) gives the largest radius sqrt(48 ln 2); u1 = 1 - 2^-24
    (N = 2^24 - 1) the smallest, sqrt(-2 ln(1 - 2^-24)) ~ 2^-11.5."""
    big = orc.rad(0)
    assert abs(big - math.sqrt(48 * math.log(2))) <= 4 * 2.0 ** -24 * big
    small = orc.rad(0xFFFFFFFF)
    ref = math.sqrt(-2 * math.log1p(-2.0 ** -24))
    assert abs(small - ref) <= 4 * 2.0 ** -24 * ref
