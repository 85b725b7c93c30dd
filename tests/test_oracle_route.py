"""Pins for oracle.route (C1): special cases that reduce to
argmax / a full sort, forced ties, a torch.topk+softmax cross-check, invariants,
and the Plackett-Luce closed form of Gumbel-top-k on Zipf logits against the
paper's printed 64% skew."""

import json
import os

import numpy as np
import pytest
import torch

import synth
from oracle import route
from paper_2502_06643_b200 import placement

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_k1_is_argmax():
    rng = np.random.default_rng(0)
    L = rng.integers(-3, 3, size=(500, 8)).astype(np.float32)   # many ties
    idx, w = route.route(L, 1)
    assert np.array_equal(idx[:, 0], np.argmax(L, axis=1))        # first max = lowest id
    assert np.all(w == 1.0)


def test_k_equals_E_is_full_descending_stable_order():
    rng = np.random.default_rng(1)
    L = rng.integers(-4, 4, size=(300, 6)).astype(np.float32)
    idx, _ = route.route(L, 6)
    for t in range(L.shape[0]):
        order = np.lexsort((np.arange(6), -L[t].astype(np.float64)))
        assert list(idx[t]) == list(order)


def test_forced_ties_and_signed_zero():
    L = np.array([[0.0, -0.0, 1.0, 1.0],
                  [-0.0, 0.0, -1.0, -1.0],
                  [2.0, 2.0, 2.0, 2.0]], dtype=np.float32)
    idx, w = route.route(L, 3)
    assert idx.tolist() == [[2, 3, 0], [0, 1, 2], [0, 1, 2]]
    assert w[0, 0] == w[0, 1]
    assert w[1, 0] == w[1, 1]
    assert np.allclose(w[2], 1 / 3, rtol=0, atol=1e-7)


def test_against_torch_topk_softmax_on_tie_free_rows():
    g = torch.Generator().manual_seed(3)
    L = torch.randn(2000, 64, generator=g)
    for k in (1, 2, 8):
        idx, w = route.route(L.numpy(), k)
        v, i = torch.topk(L.double(), k, dim=1)      # sorted=True, distinct values
        ws = torch.softmax(v, dim=1)
        assert np.array_equal(idx, i.numpy().astype(np.int32))
        assert np.allclose(w, ws.numpy(), rtol=1e-6, atol=1e-7)


def test_weight_invariants():
    L = synth.zipf_logits(4096, 8, 1.6, seed=0).numpy()
    idx, w = route.route(L, 2)
    assert np.all(np.abs(w.astype(np.float64).sum(1) - 1.0) < 1e-6)
    assert np.all(w[:, 0] >= w[:, 1])
    assert np.all(idx[:, 0] != idx[:, 1])


def test_k_out_of_range_is_an_error():
    with pytest.raises(ValueError):
        route.route(np.zeros((2, 4), np.float32), 5)
    with pytest.raises(ValueError):
        route.route(np.zeros((2, 4), np.float32), 0)


def plackett_luce_top2_marginals(p):
    """P(e in top-2) for sampling without replacement with probabilities p
    (closed form: p_e + sum_{e' != e} p_e' * p_e / (1 - p_e'))."""
    E = len(p)
    return np.array([p[e] + sum(p[f] * p[e] / (1 - p[f]) for f in range(E) if f != e)
                     for e in range(E)])


def test_zipf_gumbel_top2_matches_closed_form_and_paper_skew():
    """Gumbel-top-k of log p is Plackett-Luce sampling; the oracle's top-2 shares
    must match the closed form within 5 sigma, and s = 1.6 reproduces the
    paper's 'experts 0 and 1 process 64% of the total tokens'."""
    E, k, T, s = 8, 2, 16384, 1.6
    p = np.exp(synth.zipf_log_probs(E, s).double().numpy())
    p = p / p.sum()                                 # float32 log-probs -> exact normalisation
    marg = plackett_luce_top2_marginals(p)          # P(e selected), sums to 2
    assert abs(marg.sum() - 2.0) < 1e-12
    L = synth.zipf_logits(T, E, s, seed=0).numpy()
    idx, _ = route.route(L, k)
    counts = np.bincount(idx.ravel(), minlength=E)
    share = counts / T
    sigma = np.sqrt(marg * (1 - marg) / T)
    assert np.all(np.abs(share - marg) < 5 * sigma + 1e-12)
    # contiguous GPU-0 (experts 0 and 1) share of routed items
    P = placement.contiguous(E, 4)
    gpu0 = counts[P == 0].sum() / (k * T)
    assert abs((marg[0] + marg[1]) / k - GOLDEN["layer14_experts01_share"]["value"]) < 0.002
    assert abs(gpu0 - GOLDEN["layer14_experts01_share"]["value"]) < 0.01
