"""Pins for oracle.stats (C2): the RoutingStats
conservation invariants, k = 1 as a bincount, brute force, multi-rank sums."""

import itertools

import numpy as np

from oracle import stats


def _rand_idx(rng, T, E, k):
    if T == 0:
        return np.zeros((0, k), np.int32)
    return np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)


def test_conservation_invariants():
    rng = np.random.default_rng(0)
    for (T, E, k) in [(500, 8, 2), (300, 64, 8), (50, 5, 5), (0, 8, 2)]:
        a = _rand_idx(rng, T, E, k) if T else np.zeros((0, k), np.int32)
        b = _rand_idx(rng, T, E, k) if T else np.zeros((0, k), np.int32)
        load_a, coact = stats.route_stats(a, b, E)
        load_b = stats.load_counts(b, E)
        assert load_a.sum() == k * T
        assert coact.sum() == k * k * T
        assert np.array_equal(coact.sum(1), k * load_a)
        assert np.array_equal(coact.sum(0), k * load_b)
        assert load_a.dtype == np.int64 and coact.dtype == np.int64


def test_k1_is_bincount():
    rng = np.random.default_rng(1)
    E = 8
    a = rng.integers(0, E, size=(1000, 1)).astype(np.int32)
    b = rng.integers(0, E, size=(1000, 1)).astype(np.int32)
    coact = stats.coactivation_counts(a, b, E)
    ref = np.bincount(a[:, 0] * E + b[:, 0], minlength=E * E).reshape(E, E)
    assert np.array_equal(coact, ref)
    assert np.array_equal(stats.load_counts(a, E), np.bincount(a[:, 0], minlength=E))


def test_brute_force_tiny():
    rng = np.random.default_rng(2)
    E, k, T = 5, 3, 40
    a, b = _rand_idx(rng, T, E, k), _rand_idx(rng, T, E, k)
    ref = [[0] * E for _ in range(E)]
    for t in range(T):
        for j1, j2 in itertools.product(range(k), range(k)):
            ref[a[t][j1]][b[t][j2]] += 1
    assert stats.coactivation_counts(a, b, E).tolist() == ref


def test_multirank_sum_equals_concatenation():
    rng = np.random.default_rng(3)
    E, k = 8, 2
    parts = [(_rand_idx(rng, n, E, k), _rand_idx(rng, n, E, k)) for n in (100, 37, 0, 64)]
    tot_l = sum(stats.load_counts(a, E) for a, _ in parts)
    tot_c = sum(stats.coactivation_counts(a, b, E) for a, b in parts)
    A = np.concatenate([a for a, _ in parts])
    B = np.concatenate([b for _, b in parts])
    assert np.array_equal(tot_l, stats.load_counts(A, E))
    assert np.array_equal(tot_c, stats.coactivation_counts(A, B, E))
