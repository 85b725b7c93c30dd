"""Pins for oracle.plan (C3): bijection and conservation
invariants, the Megatron 'naive mapping' (contiguous placement == stable
sort by expert), brute-force receive order, zero-expert ranks."""

import json
import os

import numpy as np
import pytest

from oracle import plan
from paper_2502_06643_b200 import placement

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _idx(rng, T, E, k):
    return np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32) if T else np.zeros((0, k), np.int32)


def test_worked_contiguous_placement():
    assert placement.contiguous(8, 4).tolist() == GOLDEN["contiguous_placement_E8_G4"]["value"]
    with pytest.raises(ValueError):
        placement.contiguous(6, 4)


@pytest.mark.parametrize("G,P", [(1, [0] * 8), (4, [0, 0, 1, 1, 2, 2, 3, 3]),
                                 (4, [0, 1, 2, 2, 3, 2, 3, 3]), (3, [2, 2, 2, 0, 0, 0, 0, 0])])
def test_invariants(G, P):
    rng = np.random.default_rng(G)
    E, k = 8, 2
    T_s = [50, 13, 0, 31][:G]
    idxs = [_idx(rng, n, E, k) for n in T_s]
    pl = plan.plan(idxs, P, G)
    for s in range(G):
        n = T_s[s] * k
        assert sorted(pl["slot"][s].ravel().tolist()) == list(range(n))        # bijection
        assert pl["cnt"][s].sum() == n
    assert np.array_equal(pl["recv_counts"], pl["send_counts"].sum(0))
    assert pl["recv_counts"].sum() == sum(T_s) * k
    # every item appears exactly once in exactly one receive list, at recv_pos
    seen = set()
    for g in range(G):
        for r, (s, t, j, e) in enumerate(pl["recv"][g]):
            assert P[e] == g and pl["recv_pos"][s][t, j] == r
            seen.add((s, t, j))
    assert len(seen) == sum(T_s) * k
    # a rank that hosts no expert receives nothing (reading G13)
    for g in range(G):
        if g not in P:
            assert pl["recv_counts"][g] == 0


def test_contiguous_is_stable_sort_by_expert():
    """Megatron naive mapping: with a contiguous placement the send order
    is exactly the stable argsort of the flattened expert ids."""
    rng = np.random.default_rng(7)
    for G in (1, 2, 4, 8):
        P = placement.contiguous(8, G)
        idx = _idx(rng, 97, 8, 2)
        pl = plan.plan([idx] + [np.zeros((0, 2), np.int32)] * (G - 1), P, G)
        order = np.argsort(idx.ravel(), kind="stable")
        inv = np.empty_like(order)
        inv[order] = np.arange(len(order))
        assert np.array_equal(pl["slot"][0].ravel(), inv)


def test_receive_order_brute_force():
    rng = np.random.default_rng(9)
    G, E, k = 3, 7, 3
    P = [1, 0, 2, 1, 1, 0, 2]
    idxs = [_idx(rng, n, E, k) for n in (20, 9, 15)]
    pl = plan.plan(idxs, P, G)
    for g in range(G):
        items = [(e, s, t, j) for s in range(G) for t in range(len(idxs[s])) for j in range(k)
                 for e in [idxs[s][t][j]] if P[e] == g]
        items.sort()
        assert [(s, t, j, e) for (e, s, t, j) in items] == pl["recv"][g]


@pytest.mark.parametrize("G,P", [(4, [0, 1, 2, 2, 3, 2, 3, 3]),       # ILP-1 balanced, non-monotone
                                 (3, [2, 2, 2, 0, 0, 0, 0, 0]),       # destinations in descending expert order
                                 (3, [1, 0, 2, 1, 1, 0, 2]),          # E = 7, interleaved
                                 (4, [3, 3, 3, 3, 3, 3, 1, 1])])      # ranks hosting no expert (G13)
def test_send_order_groups_by_destination(G, P):
    """G9 send order (tokens are sent to the GPU hosting their assigned
    expert): a source's send buffer is one contiguous run per destination rank, the
    runs in rank order, so the run for rank g starts at sum_{g' < g} send_counts[s][g']
    and has send_counts[s][g] items; inside a run the items are ordered by
    (expert, token, slot j).  Non-monotone placements make this differ from a plain
    sort by expert id."""
    rng = np.random.default_rng(len(P) * 10 + G)
    E, k = len(P), 3
    T_s = [40, 17, 29, 0][:G]
    idxs = [_idx(rng, n, E, k) for n in T_s]
    pl = plan.plan(idxs, P, G)
    for s in range(G):
        idx = idxs[s]
        start = 0
        for g in range(G):
            n = int(pl["send_counts"][s][g])
            items = [(int(idx[t, j]), t, j) for t in range(idx.shape[0]) for j in range(k) if P[idx[t, j]] == g]
            assert len(items) == n
            slots = sorted(int(pl["slot"][s][t, j]) for (_, t, j) in items)
            assert slots == list(range(start, start + n))           # contiguous run, in rank order
            by_slot = sorted(items, key=lambda it: pl["slot"][s][it[1], it[2]])
            assert by_slot == sorted(items)                          # (e, t, j) order inside the run
            start += n


def test_token_blocks():
    assert plan.token_blocks(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert plan.token_blocks(3, 4) == [(0, 1), (1, 2), (2, 3), (3, 3)]


def test_invalid_placement():
    with pytest.raises(ValueError):
        plan.plan([np.zeros((1, 2), np.int32)] * 2, [0, 2, 1, 1], 2)
