"""The oracle's pins are sharp: each test here plants one plausible mistake in
an oracle function (a wrong tie rule, a dropped term, a transposed operand, a
wrong loop order, truncation instead of round-to-nearest-even) and checks that
the pin written for that function fails.  If a pin stopped catching its
mutation, the oracle could drift from the paper unnoticed.
"""

import math

import numpy as np
import pytest

from oracle import bf16, ffn, layer, plan, route, stats
from tests import test_oracle_bf16 as t_bf16
from tests import test_oracle_ffn_layer as t_ffn
from tests import test_oracle_plan as t_plan
from tests import test_oracle_route as t_route
from tests import test_oracle_stats as t_stats


def _fails(fn, *args):
    with pytest.raises(AssertionError):
        fn(*args)


def test_route_tie_to_higher_id_is_caught(monkeypatch):
    def bad_row(row, k):                    # ties to the HIGHER expert id (not G2)
        pairs = sorted(((float(row[e]) + 0.0, e) for e in range(len(row))), key=lambda p: (-p[0], -p[1]))
        top = pairs[:k]
        num = [math.exp(l - top[0][0]) for l, _ in top]
        return [e for _, e in top], [n / sum(num) for n in num]
    monkeypatch.setattr(route, "route_row", bad_row)
    _fails(t_route.test_forced_ties_and_signed_zero)


def test_route_softmax_over_all_experts_is_caught(monkeypatch):
    orig = route.route_row

    def bad_row(row, k):                    # normalises over all E logits, not the top k (not G1)
        experts, _ = orig(row, k)
        ex = [math.exp(float(v) - float(max(row))) for v in row]
        return experts, [ex[e] / sum(ex) for e in experts]
    monkeypatch.setattr(route, "route_row", bad_row)
    _fails(t_route.test_against_torch_topk_softmax_on_tie_free_rows)


def test_swiglu_without_silu_is_caught(monkeypatch):
    def bad(x, w1, w3, w2):                 # gate applied linearly (dropped silu)
        h = bf16.round_to_bf16((x @ w1.T) * (x @ w3.T))
        return h, bf16.round_to_bf16(h @ w2.T)
    monkeypatch.setattr(ffn, "swiglu", bad)
    _fails(t_ffn.test_dense_swiglu_vs_torch_fp32)


def test_swiglu_swapped_gate_and_up_is_caught(monkeypatch):
    orig = ffn.swiglu

    def bad(x, w1, w3, w2):                 # silu on the up projection instead of the gate
        return orig(x, w3, w1, w2)
    monkeypatch.setattr(ffn, "swiglu", bad)
    _fails(t_ffn.test_dense_swiglu_vs_torch_fp32)


def test_receive_order_source_major_is_caught(monkeypatch):
    orig = plan.plan

    def bad(idx_by_source, P, G):           # receive rows ordered (s, e, t) instead of (e, s, t) (not G9)
        pl = orig(idx_by_source, P, G)
        pl["recv"] = [sorted(rows, key=lambda it: (it[0], it[3], it[1], it[2])) for rows in pl["recv"]]
        return pl
    monkeypatch.setattr(plan, "plan", bad)
    _fails(t_plan.test_receive_order_brute_force)


def test_send_order_by_expert_only_is_caught(monkeypatch):
    orig = plan.plan

    def bad(idx_by_source, P, G):           # send order keyed by e alone, not (P[e], e) (not G9)
        pl = orig(idx_by_source, P, G)
        for s, idx in enumerate(idx_by_source):
            idx = np.asarray(idx)
            order = np.argsort(idx.ravel(), kind="stable")
            sl = np.empty(len(order), dtype=np.int64)
            sl[order] = np.arange(len(order))
            pl["slot"][s] = sl.reshape(idx.shape)
        return pl
    monkeypatch.setattr(plan, "plan", bad)
    _fails(t_plan.test_send_order_groups_by_destination, 4, [0, 1, 2, 2, 3, 2, 3, 3])


def test_unpermute_without_gate_weights_is_caught(monkeypatch):
    def bad(ret_rows, w):                   # sums the k expert rows, drops the gate weights
        acc = np.zeros_like(ret_rows[0])
        for r in ret_rows:
            acc = acc + r
        return bf16.round_to_bf16(acc)
    monkeypatch.setattr(layer, "unpermute", bad)
    _fails(t_ffn.test_identity_expert_returns_x_bit_exact, 1.6)


def test_coactivation_transposed_is_caught(monkeypatch):
    orig = stats.coactivation_counts

    def bad(idx_l, idx_l1, E):              # R[e2][e1] instead of R[e1][e2]
        return orig(idx_l, idx_l1, E).T.copy()
    monkeypatch.setattr(stats, "coactivation_counts", bad)
    _fails(t_stats.test_brute_force_tiny)


def test_bf16_truncation_is_caught(monkeypatch):
    def bad(x):                             # truncates the mantissa (round toward zero), not RNE
        x = np.asarray(x, dtype=np.float64)
        u = x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFF0000)
        return u.view(np.float32).astype(np.float64)
    monkeypatch.setattr(bf16, "round_to_bf16", bad)
    _fails(t_bf16.test_matches_torch_on_fp32_values)
