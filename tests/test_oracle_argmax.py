"""Pins for the (value, index) key of spec/MODELS.md §3 against brute force."""
import math

import numpy as np


def test_key_order_equals_value_then_index_order(orc):
    rng = np.random.default_rng(0)
    vals = list(rng.normal(size=200).astype(np.float32)) + [np.float32(x) for x in
                                                             (0.0, -0.0, np.inf, -np.inf, 1e-45, -1e-45, 3.4e38)]
    items = [(float(v), i) for i, v in enumerate(vals)]
    by_key = sorted(items, key=lambda t: orc.key(t[0], t[1]))
    by_val = sorted(items, key=lambda t: (t[0], t[1]))
    assert by_key == by_val


def test_minus_zero_equals_plus_zero(orc):
    assert orc.key(-0.0, 5) == orc.key(0.0, 5)
    k, rc = orc.argmax_net(np.array([0.0, -0.0, -0.0], np.float32))
    assert rc == 0 and k & 0xFFFFFFFF == 0


def test_nan_never_wins_and_all_nan_is_no_valid(orc):
    net = np.array([np.nan, -5.0, np.nan, -7.0], np.float32)
    k, rc = orc.argmax_net(net)
    assert rc == 0 and k & 0xFFFFFFFF == 1
    k, rc = orc.argmax_net(np.array([np.nan, np.nan], np.float32))
    assert rc == 1
    k, rc = orc.argmax_net(np.zeros(0, np.float32))
    assert rc == 1 and k == 0xFFFFFFFFFFFFFFFF


def test_argmax_equals_brute_force_with_ties(orc):
    rng = np.random.default_rng(3)
    for _ in range(50):
        net = rng.integers(-3, 3, size=rng.integers(1, 60)).astype(np.float32)
        base = int(rng.integers(0, 1000))
        k, rc = orc.argmax_net(net, base)
        best = max(range(len(net)), key=lambda j: (net[j], -j))
        assert rc == 0 and (k & 0xFFFFFFFF) == base + best
        c, idx = orc.key_decode(k)
        assert c == -float(net[best]) and idx == base + best


def test_signed_int64_flip_preserves_order(orc):
    """Cross-rank combine: int64(key ^ 2^63) with signed MIN == unsigned min."""
    rng = np.random.default_rng(5)
    keys = [orc.key(float(v), i) for i, v in enumerate(rng.normal(size=100).astype(np.float32))]
    flipped = [((k ^ (1 << 63)) - (1 << 64)) if (k ^ (1 << 63)) >= (1 << 63) else (k ^ (1 << 63)) for k in keys]
    j = int(np.argmin(flipped))
    assert keys[j] == min(keys)
    assert math.isnan(orc.key_decode(orc.key(float("nan"), 3))[0])


def test_random_ties_uniform_frequency(orc):
    """8 tied minima among 64: over 10,000 reseeded runs each wins with
    frequency 1/8 +- 0.02 (P:306 'randomly pick one')."""
    net = np.full(64, -5.0, np.float32)
    tied = [3, 7, 11, 20, 33, 40, 51, 63]
    net[tied] = -1.0
    counts = dict.fromkeys(tied, 0)
    for seed in range(10000):
        k, t, rc = orc.argmax_random_ties(net, 0, seed)
        assert rc == 0 and k & 0xFFFFFFFF == 3       # plain rule: lowest index
        counts[t & 0xFFFFFFFF] += 1
    assert set(counts) == set(tied)
    for v in counts.values():
        assert abs(v / 10000 - 1 / 8) < 0.02


def test_random_ties_unique_minimum_wins_regardless_of_seed(orc):
    """One strictly minimal cost at index 5 -> it wins for every seed."""
    net = np.linspace(-3, -1, 40).astype(np.float32)
    net[5] = 1.0
    for seed in range(200):
        _, t, _ = orc.argmax_random_ties(net, 100, seed)
        assert t & 0xFFFFFFFF == 105


def test_random_ties_shard_combine(orc):
    """min over shards of the tie keys == tie key of the whole array (second all-reduce)."""
    rng = np.random.default_rng(2)
    net = rng.integers(-3, 1, 500).astype(np.float32)
    k_full, t_full, _ = orc.argmax_random_ties(net, 0, 77)
    parts = []
    for b, e in [(0, 123), (123, 300), (300, 500)]:
        kb, _, _ = orc.argmax_random_ties(net[b:e], b, 77)
        parts.append(kb)
    kmin = min(parts)
    assert kmin == k_full
    # pass B on each shard restricted to the global minimum value
    ties = []
    for b, e in [(0, 123), (123, 300), (300, 500)]:
        sub = net[b:e].copy()
        sub[-sub > orc.key_decode(kmin)[0]] = -np.inf       # only global minima can win
        _, tb, rc = orc.argmax_random_ties(sub, b, 77)
        if rc == 0 and orc.argmax_net(sub, b)[0] >> 32 == kmin >> 32:
            ties.append(tb)
    assert min(ties) == t_full
