"""Pins for oracle.layer.layer_ep_tp / swiglu_tp_experts (tensor parallelism
inside the experts, reading G20):
  * tp = 1 reduces to the plain EP layer bit-exactly;
  * an expert whose TP slice 0 is the identity and whose other slices return 0
    gives out == x bit-exactly for every (G, tp, placement) -- pins the
    W = G*tp source blocks, the per-group receive layout and the per-slice
    return into send order;
  * the h of a slice is exactly the matching columns of the full h, and the sum
    of the bf16 partials is within the bf16 rounding bound of the exact
    (unrounded) h W2^T -- pins the F split of W1/W3 rows and W2 columns;
  * the TP layer equals the direct definition (C8) within the bound derived
    from the extra bf16 rounding of each partial;
  * C3 with S = 2G sources keeps the brute-force receive order (e, s, t).
"""

import numpy as np
import pytest
import torch

import synth
from oracle import bf16, ffn, layer, plan as oplan
from paper_2502_06643_b200 import placement


def _np(t):
    return bf16.from_bits(t.view(torch.int16).numpy().view(np.uint16))


def _weights(E, H, F, seed):
    ws = [synth.expert_weights(e, H, F, seed) for e in range(E)]
    return [_np(w[0]) for w in ws], [_np(w[1]) for w in ws], [_np(w[2]) for w in ws]


def _case(T, H, F, E, s, seed):
    x = _np(synth.hidden_states(T, H, seed=seed))
    w1, w3, w2 = _weights(E, H, F, seed)
    logits = synth.zipf_logits(T, E, s, seed=seed).numpy()
    return x, w1, w3, w2, logits


def test_tp1_is_plain_ep():
    T, H, F, E, k = 157, 64, 128, 8, 2
    x, w1, w3, w2, logits = _case(T, H, F, E, 1.6, 11)
    P = np.array([0, 1, 2, 2, 3, 2, 3, 3])
    ref, *_ = layer.layer_ep(x, logits, k, P, 4, layer.swiglu_experts(w1, w3, w2))
    out, *_ = layer.layer_ep_tp(x, logits, k, P, 4, 1, layer.swiglu_tp_experts(w1, w3, w2, 1))
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("G,tp,P", [(1, 2, [0] * 8), (2, 2, [0, 0, 0, 0, 1, 1, 1, 1]),
                                    (2, 4, [1, 0, 1, 1, 0, 1, 1, 1]), (3, 2, [2, 2, 2, 2, 2, 2, 1, 1])])
def test_identity_slice0_returns_x_bit_exact(G, tp, P):
    T, H, E, k = 211, 64, 8, 2
    x = _np(synth.hidden_states(T, H, seed=12))
    logits = synth.zipf_logits(T, E, 1.6, seed=12).numpy()

    def part(e, rows, q):
        return rows.copy() if q == 0 else np.zeros_like(rows)

    out, idx, w, pl = layer.layer_ep_tp(x, logits, k, np.array(P), G, tp, part)
    assert np.array_equal(out, x)
    # every one of the W = G*tp ranks is a source with its own G7 token block
    assert pl["cnt"].shape == (G * tp, E) and pl["cnt"].sum() == T * k
    assert pl["send_counts"].shape == (G * tp, G)


def test_slices_partition_h_and_sum_to_y():
    n, H, F, tp = 37, 64, 256, 4
    x = _np(synth.hidden_states(n, H, seed=13))
    w1, w3, w2 = _weights(1, H, F, 13)
    h_full, _ = ffn.swiglu(x, w1[0], w3[0], w2[0])
    exact = h_full @ w2[0].T                         # unrounded h W2^T
    fn = layer.swiglu_tp_experts(w1, w3, w2, tp)
    f = F // tp
    parts = []
    for q in range(tp):
        hq, _ = ffn.swiglu(x, w1[0][q * f:(q + 1) * f], w3[0][q * f:(q + 1) * f], w2[0][:, q * f:(q + 1) * f])
        assert np.array_equal(hq, h_full[:, q * f:(q + 1) * f])
        p = fn(0, x, q)
        assert np.array_equal(bf16.round_to_bf16(p), p)
        # partial q is the bf16 rounding of h_q W2_q^T (half an ulp, ulp <= 2^-7 |p|)
        pq_exact = h_full[:, q * f:(q + 1) * f] @ w2[0][:, q * f:(q + 1) * f].T
        assert np.all(np.abs(p - pq_exact) <= np.abs(pq_exact) * 2.0 ** -8 + 1e-30)
        parts.append(p)
    s = np.sum(parts, axis=0)
    bound = sum(np.abs(p) for p in parts) * 2.0 ** -8 + 1e-12
    assert np.all(np.abs(s - exact) <= bound)
    # a transposed or shifted W2 slice would break the sum by O(|y|), not O(ulp)
    assert np.abs(s - exact).max() < 1e-2 * np.abs(exact).max()


@pytest.mark.parametrize("G,tp", [(2, 2), (1, 4), (4, 2)])
def test_tp_layer_matches_direct_within_partial_rounding(G, tp):
    T, H, F, E, k = 97, 64, 256, 8, 2
    x, w1, w3, w2, logits = _case(T, H, F, E, 1.6, 14)
    P = placement.contiguous(E, G) if G > 1 else np.zeros(E, int)
    direct, idx, w = layer.layer_direct(x, logits, k, layer.swiglu_experts(w1, w3, w2))
    fn = layer.swiglu_tp_experts(w1, w3, w2, tp)
    out, idx2, w2_, _ = layer.layer_ep_tp(x, logits, k, np.asarray(P), G, tp, fn)
    assert np.array_equal(idx, idx2) and np.array_equal(w, w2_)
    # bound per element: each partial rounded once (<= 2^-8 |p|), y rounded once in
    # the direct path (<= 2^-8 |y|), two final roundings (<= 2^-8 |out| each)
    w64 = w.astype(np.float64)
    bound = (np.abs(out) + np.abs(direct)) * 2.0 ** -8
    for t in range(T):
        for j in range(k):
            e = idx[t, j]
            ps = [fn(e, x[t:t + 1], q)[0] for q in range(tp)]
            y = layer.swiglu_experts(w1, w3, w2)(e, x[t:t + 1])[0]
            bound[t] += w64[t, j] * (sum(np.abs(p) for p in ps) + np.abs(y)) * 2.0 ** -8
    assert np.all(np.abs(out - direct) <= bound + 1e-30)
    rel = np.abs(out - direct).max() / np.abs(direct).max()
    assert rel < 2e-2


def test_plan_more_sources_than_groups_brute_force():
    rng = np.random.default_rng(15)
    G, tp, E, k = 2, 3, 6, 2
    W = G * tp
    P = np.array([1, 0, 1, 0, 0, 1])
    idx_by = [np.stack([rng.permutation(E)[:k] for _ in range(n)]) if n else np.zeros((0, k), int)
              for n in (5, 0, 7, 3, 4, 6)]
    pl = oplan.plan(idx_by, P, G)
    for g in range(G):
        items = [(e, s, t, j) for s in range(W) for t in range(len(idx_by[s])) for j in range(k)
                 for e in [idx_by[s][t, j]] if P[e] == g]
        items.sort(key=lambda it: (it[0], it[1], it[2]))
        assert [(s, t, j, e) for (e, s, t, j) in items] == pl["recv"][g]
    assert pl["recv_counts"].sum() == sum(len(i) for i in idx_by) * k
