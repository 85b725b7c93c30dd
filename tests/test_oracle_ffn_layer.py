"""Pins for oracle.ffn (C5) and oracle.layer (C4/C6/C7/C8):
  * E = 1, k = 1 reduces the layer to a dense SwiGLU MLP -> torch CPU float32
    reference (library routine), within the bf16 storage tolerance;
  * identity experts -> out == x bit-exactly (sum of gate weights is 1);
  * W2 = 0 -> out == 0;
  * the step-by-step EP algorithm == the direct definition (C7 == C8),
    bit-exactly, for every placement and G (placement invariance).
"""

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

import synth
from oracle import bf16, ffn, layer
from paper_2502_06643_b200 import placement


def _np(t):
    return bf16.from_bits(t.view(torch.int16).numpy().view(np.uint16))


def _weights(E, H, F, seed):
    ws = [synth.expert_weights(e, H, F, seed) for e in range(E)]
    return ([_np(w[0]) for w in ws], [_np(w[1]) for w in ws], [_np(w[2]) for w in ws], ws)


def test_silu_special_values():
    z = np.array([0.0, 50.0, -800.0, 1.0])
    s = ffn.silu(z)
    assert s[0] == 0.0 and s[1] == pytest.approx(50.0) and s[2] == 0.0
    assert s[3] == pytest.approx(1 / (1 + np.exp(-1.0)))


def test_dense_swiglu_vs_torch_fp32():
    H, F, n = 128, 256, 64
    x_t = synth.hidden_states(n, H, seed=5)
    w1, w3, w2, ws = _weights(1, H, F, seed=5)
    h, y = ffn.swiglu(_np(x_t), w1[0], w3[0], w2[0])
    assert np.array_equal(bf16.round_to_bf16(h), h) and np.array_equal(bf16.round_to_bf16(y), y)
    xf = x_t.float()
    W1, W3, W2 = (w.float() for w in ws[0])
    ref = ((Fn.silu(xf @ W1.T) * (xf @ W3.T)) @ W2.T).double().numpy()
    err = np.abs(y - ref).max() / np.abs(ref).max()
    assert err < 2e-2
    row = (np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1)).max()
    assert row < 2e-2


def test_layer_e1_k1_is_dense_mlp():
    H, F, T = 64, 128, 50
    x = _np(synth.hidden_states(T, H, seed=2))
    w1, w3, w2, _ = _weights(1, H, F, seed=2)
    logits = np.zeros((T, 1), np.float32)
    out, idx, w = layer.layer_direct(x, logits, 1, layer.swiglu_experts(w1, w3, w2))
    _, y = ffn.swiglu(x, w1[0], w3[0], w2[0])
    assert np.array_equal(out, y) and np.all(idx == 0) and np.all(w == 1.0)


@pytest.mark.parametrize("s", [0.0, 1.6])
def test_identity_expert_returns_x_bit_exact(s):
    T, H, E, k = 300, 64, 8, 2
    x = _np(synth.hidden_states(T, H, seed=1))
    logits = synth.zipf_logits(T, E, s, seed=1).numpy()
    out, *_ = layer.layer_ep(x, logits, k, placement.contiguous(E, 4), 4, layer.identity_expert)
    assert np.array_equal(out, x)
    out2, *_ = layer.layer_direct(x, logits, k, layer.identity_expert)
    assert np.array_equal(out2, x)


def test_zero_w2_gives_zero():
    T, H, F, E, k = 40, 64, 128, 4, 2
    x = _np(synth.hidden_states(T, H, seed=3))
    w1, w3, w2, _ = _weights(E, H, F, seed=3)
    w2 = [np.zeros_like(m) for m in w2]
    logits = synth.zipf_logits(T, E, 0.0, seed=3).numpy()
    out, *_ = layer.layer_ep(x, logits, k, [0, 1, 1, 0], 2, layer.swiglu_experts(w1, w3, w2))
    assert np.all(out == 0)


def test_ep_equals_direct_for_all_placements():
    T, H, F, E, k = 203, 64, 128, 8, 2
    x = _np(synth.hidden_states(T, H, seed=4))
    w1, w3, w2, _ = _weights(E, H, F, seed=4)
    fn = layer.swiglu_experts(w1, w3, w2)
    logits = synth.zipf_logits(T, E, 1.6, seed=4).numpy()
    direct, *_ = layer.layer_direct(x, logits, k, fn)
    for G, P in [(1, [0] * 8), (2, placement.contiguous(8, 2)), (4, placement.contiguous(8, 4)),
                 (4, [0, 1, 2, 2, 3, 2, 3, 3]), (3, [2, 2, 2, 2, 2, 2, 1, 1])]:
        out, *_ = layer.layer_ep(x, logits, k, np.array(P), G, fn)
        assert np.array_equal(out, direct), (G, P)
