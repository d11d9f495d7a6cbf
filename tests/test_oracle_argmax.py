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
