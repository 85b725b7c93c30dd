"""Pins for the host placement utility (ILP 1 exact): SPEC's worked
example, brute force over all labeled surjective assignments,
E == G, dominance over the contiguous baseline."""

import itertools

import numpy as np
import pytest

from paper_2502_06643_b200 import placement


def test_spec_worked_example():
    a, o1 = placement.ilp1_exact([7, 1, 1, 1], 2)
    assert a.tolist() == [0, 1, 1, 1] and o1 == 4.0


def test_partition_count_is_stirling():
    # S(8,4) = 1701 canonical partitions
    assert sum(1 for _ in placement._restricted_growth_strings(8, 4)) == 1701


@pytest.mark.parametrize("E,G", [(5, 2), (6, 3), (7, 4), (6, 6)])
def test_matches_brute_force(E, G):
    rng = np.random.default_rng(E * 10 + G)
    for _ in range(5):
        load = rng.integers(0, 100, size=E)
        _, o1 = placement.ilp1_exact(load, G)
        best = None
        for a in itertools.product(range(G), repeat=E):
            if len(set(a)) != G:
                continue                       # Eq. (7): every cluster non-empty
            T = np.bincount(a, weights=load, minlength=G)
            v = np.abs(T - load.sum() / G).sum()
            best = v if best is None else min(best, v)
        assert o1 == pytest.approx(best, abs=1e-9)


def test_dominates_contiguous():
    rng = np.random.default_rng(0)
    for _ in range(10):
        load = rng.integers(0, 5000, size=8)
        _, o1 = placement.ilp1_exact(load, 4)
        c = placement.contiguous(8, 4)
        assert o1 <= placement.o1_times_G(load, c, 4) / 4 + 1e-9


def test_heuristic_never_beats_exact_and_is_valid():
    rng = np.random.default_rng(5)
    for E, G in [(6, 2), (8, 4), (9, 3), (10, 4)]:
        for _ in range(5):
            load = rng.integers(0, 1000, size=E)
            a_h, o_h = placement.ilp1_heuristic(load, G)
            _, o_x = placement.ilp1_exact(load, G)
            assert o_h >= o_x - 1e-9
            assert sorted(set(a_h.tolist())) == list(range(G))          # Eq. (7)
            assert o_h == pytest.approx(placement.o1_times_G(load, a_h, G) / G)


def test_heuristic_uniform_is_perfect_and_large_e_is_fast():
    a, o = placement.ilp1_heuristic([5] * 64, 8)
    assert o == 0.0 and np.bincount(a).tolist() == [8] * 8
    load = (1000 / (np.arange(64) + 1.0) ** 1.6).astype(int)
    a = placement.balanced(load, 4)          # S(64,4) is astronomically large -> heuristic
    assert len(a) == 64 and sorted(set(a.tolist())) == [0, 1, 2, 3]
    assert placement.stirling2(8, 4) == 1701


def test_skewed_load_isolates_hot_expert():
    # the SURVEY App. A.1 seed-0 counts at s = 1.6
    load = [13514, 7477, 4032, 2562, 1882, 1345, 1085, 871]
    a = placement.balanced(load, 4)
    assert a.tolist() == [0, 1, 2, 2, 3, 2, 3, 3]
    assert sum(1 for v in a if v == a[0]) == 1


# ---------------------------------------------------------------- ILP 2 (host tooling, NEXT-4)
def test_comm_costs_spec_examples_and_conservation():
    rng = np.random.default_rng(3)
    L, E, G = 4, 8, 4
    coact = rng.integers(0, 30, (L - 1, E, E))
    assign = np.stack([rng.permutation(np.arange(E) % G) for _ in range(L)])
    C = placement.comm_costs(coact, assign, G)
    assert C.shape == (L - 1, G, G)
    for l in range(L - 1):                                     # S: sum C[l] == sum transitions[l]
        assert C[l].sum() == coact[l].sum()
        ref = np.zeros((G, G), np.int64)                         # naive quadruple loop
        for e1 in range(E):
            for e2 in range(E):
                ref[assign[l][e1], assign[l + 1][e2]] += coact[l][e1][e2]
        assert np.array_equal(C[l], ref)
    one = placement.comm_costs(coact, np.zeros((L, E), int), 1)  # G = 1: all mass in C[l][0][0]
    assert np.array_equal(one[:, 0, 0], coact.sum(axis=(1, 2)))
    two = placement.comm_costs(np.array([[[10, 0], [0, 10]]]), np.array([[0, 1], [0, 1]]), 2)
    assert two.tolist() == [[[10, 0], [0, 10]]]


def test_objective_o2_spec_examples():
    C = np.array([[[10, 0], [0, 10]]])
    assert placement.objective_o2(C, [[0, 1], [0, 1]]) == 0      # heavy pairs co-located
    assert placement.objective_o2(C, [[0, 1], [1, 0]]) == 10     # crossing permutation
    assert placement.objective_o2(np.zeros((0, 2, 2)), [[0, 1]]) == 0   # L = 1: empty sum


def test_ilp2_dp_matches_exhaustive():
    import itertools
    rng = np.random.default_rng(4)
    for G, L in [(2, 3), (3, 3), (3, 4), (4, 3)]:
        perms = list(itertools.permutations(range(G)))
        for _ in range(6):
            C = rng.integers(0, 40, (L - 1, G, G))
            best = min(placement.objective_o2(C, [perms[i] for i in seq])
                       for seq in itertools.product(range(len(perms)), repeat=L))
            got = placement.ilp2_dp(C, G, L)
            assert all(sorted(p) == list(range(G)) for p in got)   # Eqs. 14-15
            assert placement.objective_o2(C, got) == best
            # ties: the lexicographically smallest optimal permutation sequence
            first = min(seq for seq in itertools.product(range(len(perms)), repeat=L)
                        if placement.objective_o2(C, [perms[i] for i in seq]) == best)
            assert got.tolist() == [list(perms[i]) for i in first]
    # the case where a forward DP with a final argmin picks the later layer's choice
    assert placement.ilp2_dp(np.array([[[0, 10], [10, 0]]]), 2, 2).tolist() == [[0, 1], [1, 0]]


def test_expert_to_gpu_and_balance():
    assign = np.array([[0, 0, 1, 1], [1, 0, 0, 1]])
    goc = np.array([[1, 0], [0, 1]])
    e2g = placement.expert_to_gpu(assign, goc)
    assert e2g.tolist() == [[1, 1, 0, 0], [1, 0, 0, 1]]
    assert placement.balance_slack(e2g, 2) == 0.0
    assert placement.balance_slack(np.array([[0, 0, 0, 1]]), 2) == 1.0


def test_placement_json_roundtrip_and_errors():
    """SPEC's portable placement file: the per-layer expert -> GPU maps
    round-trip; ragged or negative maps are rejected."""
    import json
    e2g = np.array([[0, 1, 2, 2, 3, 2, 3, 3], [1, 0, 3, 3, 2, 3, 2, 2]])
    goc = np.array([[0, 1, 2, 3], [1, 0, 3, 2]])
    text = placement.to_json(e2g, goc, objective=42.0)
    d = json.loads(text)
    assert set(d) == {"balance_slack", "objective", "gpu_of_cluster", "expert_to_gpu"}
    back, parsed = placement.from_json(text)
    assert back.dtype == np.int32 and back.tolist() == e2g.tolist()
    assert parsed["gpu_of_cluster"] == goc.tolist() and parsed["objective"] == 42.0
    assert parsed["balance_slack"] == placement.balance_slack(e2g, 4)
    for bad in ['{"expert_to_gpu": [[0, 1], [0]]}', '{"expert_to_gpu": [[0, -1]]}', '{"expert_to_gpu": []}']:
        with pytest.raises(ValueError):
            placement.from_json(bad)
