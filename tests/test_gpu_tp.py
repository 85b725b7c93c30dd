"""GPU parity of tensor parallelism inside the experts (the
paper's "4EP-2TP"; reading G20) on virtual ranks:
G EP groups x tp ranks emulated on one GPU with the same kernels, counts,
slots and receive layout as G*tp real ranks.  Compared with the oracle's
step-by-step TP layer (oracle.layer.layer_ep_tp) and plan over W = G*tp
sources; integer/index work bit-exact, floats within 2e-2 (G16).  Real-rank TP
(P2P over NVLink) is covered by tests/test_multigpu.py.
"""

import numpy as np
import pytest
import torch

from oracle import layer as olayer
from oracle import plan as oplan
from oracle import route as oroute
from tests._util import Inputs, assert_close_layer, bf16_to_f64

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _moe():
    from paper_2502_06643_b200 import moe
    return moe


def make_layer(T, H, F, E, k, G, tp):
    return _moe().MoeLayer(max_tokens=max(T, 1), hidden=H, ffn=F, num_experts=E, max_k=k,
                           virtual_ranks=G * tp, tp=tp)


CASES = [  # (G EP groups, tp, placement over groups)
    (1, 2, [0] * 8),
    (2, 2, [0, 0, 0, 0, 1, 1, 1, 1]),
    (2, 2, [1, 0, 1, 1, 0, 1, 0, 1]),
    (4, 2, [0, 1, 2, 2, 3, 2, 3, 3]),
    (2, 4, [1, 1, 1, 1, 1, 1, 1, 1]),      # group 0 hosts no expert (G13)
]


@pytest.mark.parametrize("G,tp,P", CASES)
@pytest.mark.parametrize("T", [1000, 77])
def test_tp_plan_bit_exact(cuda_ok, G, tp, P, T):
    E, k, H = 8, 2, 64
    W = G * tp
    inp = Inputs(T, H, 128 * tp, E, k, s=1.6, seed=W * 10 + T, with_weights=False)
    lay = make_layer(T, H, 128 * tp, E, k, G, tp)
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, k)
    info = lay.dispatch(x, idx, P, info=True)
    dr, rp, ss, cnt = lay.debug_plan()
    ridx, _ = oroute.route(inp.logits.numpy(), k)
    blocks = oplan.token_blocks(T, W)
    pl = oplan.plan([ridx[a:b] for a, b in blocks], np.array(P), G)
    assert np.array_equal(cnt, pl["cnt"])                 # [W][E]: every rank is a source
    for s, (a, b) in enumerate(blocks):
        assert np.array_equal(ss[a:b], pl["slot"][s])
        assert np.array_equal(rp[a:b], pl["recv_pos"][s])
        assert np.array_equal(dr[a:b], np.array(P)[ridx[a:b]])
    assert list(info.recv_counts)[:G] == pl["recv_counts"].tolist()
    rows = lay.debug_recv()
    xb = inp.x.view(torch.int16).numpy().view(np.uint16)
    ref = np.concatenate([xb[[blocks[s][0] + t for (s, t, j, e) in pl["recv"][g]]].reshape(-1, H)
                          for g in range(G)])
    assert np.array_equal(rows, ref)


@pytest.mark.parametrize("G,tp,P", CASES)
def test_tp_identity_round_trip_bit_exact(cuda_ok, G, tp, P):
    """TP slice 0 returns its rows, the other slices zeros: out == x bit-exactly."""
    T, E, k, H = 999, 8, 2, 256
    inp = Inputs(T, H, 128 * tp, E, k, s=1.6, seed=5, with_weights=False)
    lay = make_layer(T, H, 128 * tp, E, k, G, tp)
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, k)
    lay.dispatch(x, idx, P)
    lay.identity_ffn()
    out = lay.combine(w)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), x.view(torch.int16))


@pytest.mark.parametrize("T,H,F,E,k,G,tp,P", [
    (1024, 64, 256, 8, 2, 2, 2, [0, 0, 0, 0, 1, 1, 1, 1]),     # tiny config, 2EP-2TP
    (1500, 256, 512, 8, 2, 1, 4, [0] * 8),                     # 1EP-4TP, several tiles, ragged tails
    (900, 128, 384, 8, 2, 2, 2, [1, 0, 1, 1, 0, 1, 0, 1]),       # F/tp = 192: 128-wide SwiGLU tiles
    (700, 128, 256, 16, 4, 4, 2, [e % 4 for e in range(16)]),  # 4EP-2TP (the paper's layout)
    (600, 128, 256, 64, 8, 2, 2, [e // 32 for e in range(64)]),  # E64 top-8 family
])
def test_tp_layer_parity(cuda_ok, T, H, F, E, k, G, tp, P):
    inp = Inputs(T, H, F, E, k, s=1.6, seed=23)
    lay = make_layer(T, H, F, E, k, G, tp)
    moe = _moe()
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, k)
    lay.dispatch(x, idx, P)
    w1, w3, w2 = inp.device_weights(DEV, list(range(E)))
    lay.expert_ffn(moe.pack_w13(w1, w3), w2)
    out = lay.combine(w)
    lay.sync()
    xo, lo = bf16_to_f64(inp.x), inp.logits.numpy()
    ref, ridx, _, _ = olayer.layer_ep_tp(xo, lo, k, np.array(P), G, tp, inp.oracle_tp_fn(tp))
    assert np.array_equal(idx.cpu().numpy(), ridx)
    assert_close_layer(bf16_to_f64(out), ref)
    # and the plain definition (C8) within the same tolerance
    direct, _, _ = olayer.layer_direct(xo, lo, k, inp.oracle_expert_fn())
    assert_close_layer(bf16_to_f64(out), direct)


def test_tp_decode_tiles(cuda_ok, monkeypatch):
    """TP with 128-row GEMM tiles on one CTA (decode-sized contexts)."""
    monkeypatch.setenv("MOE_GEMM_CG", "1")
    T, H, F, E, k, G, tp = 333, 128, 512, 8, 2, 2, 2
    P = [0, 1, 1, 0, 1, 0, 0, 1]
    inp = Inputs(T, H, F, E, k, s=1.6, seed=41)
    lay = make_layer(T, H, F, E, k, G, tp)
    moe = _moe()
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, k)
    lay.dispatch(x, idx, P)
    w1, w3, w2 = inp.device_weights(DEV, list(range(E)))
    lay.expert_ffn(moe.pack_w13(w1, w3), w2)
    out = lay.combine(w)
    lay.sync()
    ref, _, _, _ = olayer.layer_ep_tp(bf16_to_f64(inp.x), inp.logits.numpy(), k, np.array(P), G, tp,
                                      inp.oracle_tp_fn(tp))
    assert_close_layer(bf16_to_f64(out), ref)


def test_tp_bad_configs(cuda_ok):
    moe = _moe()
    kw = dict(max_tokens=64, hidden=64, num_experts=8, max_k=2)
    with pytest.raises(moe.MoeError) as ei:                   # tp does not divide the ranks
        moe.MoeLayer(ffn=256, virtual_ranks=6, tp=4, **kw)
    assert ei.value.status == 1
    with pytest.raises(moe.MoeError) as ei:                   # F / tp not a multiple of 64
        moe.MoeLayer(ffn=192, virtual_ranks=4, tp=2, **kw)
    assert ei.value.status == 5
    lay = moe.MoeLayer(ffn=256, virtual_ranks=4, tp=2, **kw)
    x = torch.zeros(8, 64, dtype=torch.bfloat16, device=DEV)
    idx = torch.zeros(8, 2, dtype=torch.int32, device=DEV)
    lay.dispatch(x, idx, [0, 0, 1, 1, 2, 2, 0, 0])            # placement value >= G/tp groups
    with pytest.raises(moe.MoeError) as ei:                   # (device-validated: latched)
        lay.sync()
    assert ei.value.status == 6 and "expert_to_rank value" in str(ei.value)
