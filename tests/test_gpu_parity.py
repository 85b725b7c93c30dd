"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by
element on the same seeded inputs.

Bars (BASELINE north_star): bit-exact for routing indices, permutation, per-GPU
splits and co-activation counts; within 2e-2 (tests/_util.py, reading G16) for
gate weights and layer outputs.  Sizes span several tiles with ragged tails;
the full BASELINE configuration (Mixtral layer, T = 16384, the bench's launch
configuration at N = 1) is checked on sampled tokens.
"""

import numpy as np
import pytest
import torch

import synth
from oracle import layer as olayer
from oracle import plan as oplan
from oracle import route as oroute
from oracle import stats as ostats
from paper_2502_06643_b200 import placement
from tests._util import Inputs, assert_close_layer, bf16_to_f64

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _moe():
    from paper_2502_06643_b200 import moe
    return moe


def make_layer(T, H, F, E, k, G=1):
    moe = _moe()
    return moe.MoeLayer(max_tokens=max(T, 1), hidden=H, ffn=F, num_experts=E, max_k=k, virtual_ranks=G)


# ------------------------------------------------------------------ a1
@pytest.mark.parametrize("T,E,k", [(1000, 8, 2), (4096, 8, 2), (777, 4, 1), (513, 16, 4), (1031, 64, 8),
                                   (300, 128, 16), (257, 256, 8), (65, 3, 3)])
def test_route_bit_exact_indices(cuda_ok, T, E, k):
    lay = make_layer(T, 64, 64, E, k)
    logits = synth.zipf_logits(T, E, 1.2, seed=T + E)
    # force ties and signed zeros on some rows
    logits[::7, :2] = 0.5
    logits[::11, 0] = 0.0
    logits[::11, 1] = -0.0
    logits[::13] = logits[::13].round()
    idx, w = lay.route(logits.to(DEV), k)
    torch.cuda.synchronize()
    ridx, rw = oroute.route(logits.numpy(), k)
    assert np.array_equal(idx.cpu().numpy(), ridx)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=2e-2, atol=0)
    assert np.abs(w.cpu().numpy().astype(np.float64) - rw).max() < 1e-5


def test_route_empty(cuda_ok):
    lay = make_layer(16, 64, 64, 8, 2)
    idx, w = lay.route(torch.zeros(0, 8, device=DEV), 2)
    assert idx.shape == (0, 2)


def test_route_nan_logit_latches_device_error(cuda_ok):
    """Reading G3: router logits are finite; a NaN latches MOE_ERR_DEVICE."""
    moe = _moe()
    lay = make_layer(64, 64, 64, 8, 2)
    logits = torch.randn(64, 8, device=DEV)
    logits[5, 3] = float("nan")
    lay.route(logits, 2)
    with pytest.raises(moe.MoeError) as ei:
        lay.sync()
    assert ei.value.status == 6 and "NaN" in str(ei.value)
    lay.route(torch.randn(64, 8, device=DEV), 2)     # the error word was cleared
    lay.sync()


# ------------------------------------------------------------------ a2
@pytest.mark.parametrize("T,E,k", [(5000, 8, 2), (1031, 64, 8), (333, 128, 4), (1, 8, 2), (777, 256, 16), (300, 200, 3)])
def test_route_stats_bit_exact(cuda_ok, T, E, k):
    lay = make_layer(T, 64, 64, E, k)
    l0 = synth.zipf_logits(T, E, 1.6, seed=1)
    l1 = synth.zipf_logits(T, E, 1.0, seed=2)
    a, _ = oroute.route(l0.numpy(), k)
    b, _ = oroute.route(l1.numpy(), k)
    load = torch.zeros(E, dtype=torch.int64, device=DEV)
    coact = torch.zeros(E, E, dtype=torch.int64, device=DEV)
    ia, ib = torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV)
    lay.route_stats(ia, ib, load, coact)
    lay.route_stats(ia, ib, load, coact)          # accumulates
    lay.sync()
    rl, rc = ostats.route_stats(a, b, E)
    assert np.array_equal(load.cpu().numpy(), 2 * rl)
    assert np.array_equal(coact.cpu().numpy(), 2 * rc)
    # idx_l1 = NULL: load only
    load2 = torch.zeros(E, dtype=torch.int64, device=DEV)
    lay.route_stats(ia, None, load2, None)
    lay.sync()
    assert np.array_equal(load2.cpu().numpy(), rl)


def test_route_stats_bad_expert_latches_device_error(cuda_ok):
    moe = _moe()
    lay = make_layer(100, 64, 64, 8, 2)
    idx = torch.zeros(100, 2, dtype=torch.int32, device=DEV)
    idx[5, 1] = 9
    load = torch.zeros(8, dtype=torch.int64, device=DEV)
    lay.route_stats(idx, None, load, None)
    with pytest.raises(moe.MoeError) as ei:
        lay.sync()
    assert ei.value.status == 6


# ------------------------------------------------------------------ a3-a5
PLACEMENTS = [
    (1, [0] * 8),
    (2, [0, 0, 0, 0, 1, 1, 1, 1]),
    (4, [0, 0, 1, 1, 2, 2, 3, 3]),
    (4, [0, 1, 2, 2, 3, 2, 3, 3]),       # ILP-1 balanced, uneven experts per rank
    (4, [3, 3, 3, 3, 3, 3, 1, 1]),       # ranks 0 and 2 host no expert (reading G13)
    (8, [7, 6, 5, 4, 3, 2, 1, 0]),
]


@pytest.mark.parametrize("G,P", PLACEMENTS)
@pytest.mark.parametrize("T", [1000, 130])
def test_dispatch_plan_bit_exact(cuda_ok, G, P, T):
    E, k, H = 8, 2, 64
    inp = Inputs(T, H, 128, E, k, s=1.6, seed=G * 100 + T, with_weights=False)
    lay = make_layer(T, H, 128, E, k, G)
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, k)
    info = lay.dispatch(x, idx, P, info=True)
    dr, rp, ss, cnt = lay.debug_plan()
    ridx, _ = oroute.route(inp.logits.numpy(), k)
    blocks = oplan.token_blocks(T, G)
    pl = oplan.plan([ridx[a:b] for a, b in blocks], np.array(P), G)
    assert np.array_equal(cnt, pl["cnt"])
    for s, (a, b) in enumerate(blocks):
        assert np.array_equal(ss[a:b], pl["slot"][s])
        assert np.array_equal(rp[a:b], pl["recv_pos"][s])
        assert np.array_equal(dr[a:b], np.array(P)[ridx[a:b]])
    assert list(info.recv_counts)[:G] == pl["recv_counts"].tolist()
    # payload: every received row is bit-identical to its source row, in receive order
    rows = lay.debug_recv()
    xb = inp.x.view(torch.int16).numpy().view(np.uint16)
    ref = np.concatenate([xb[[blocks[s][0] + t for (s, t, j, e) in pl["recv"][g]]].reshape(-1, H)
                          for g in range(G)])
    assert np.array_equal(rows, ref)


@pytest.mark.parametrize("G,P", PLACEMENTS)
def test_identity_expert_round_trip_bit_exact(cuda_ok, G, P):
    """dispatch -> identity expert -> combine returns x bit-exactly."""
    T, E, k, H = 999, 8, 2, 256
    inp = Inputs(T, H, 128, E, k, s=1.6, seed=7, with_weights=False)
    lay = make_layer(T, H, 128, E, k, G)
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, k)
    lay.dispatch(x, idx, P)
    lay.identity_ffn()
    out = lay.combine(w)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), x.view(torch.int16))


def test_empty_and_invalid_inputs(cuda_ok):
    moe = _moe()
    lay = make_layer(64, 64, 128, 8, 2, 4)
    x = torch.zeros(0, 64, dtype=torch.bfloat16, device=DEV)
    idx = torch.zeros(0, 2, dtype=torch.int32, device=DEV)
    lay.dispatch(x, idx, [0, 0, 1, 1, 2, 2, 3, 3])
    out = lay.combine(torch.zeros(0, 2, device=DEV))
    assert out.shape == (0, 64)
    lay.dispatch(x, idx, [0, 0, 1, 1, 2, 2, 3, 4])          # placement value >= G: device-validated
    with pytest.raises(moe.MoeError) as ei:
        lay.sync()
    assert ei.value.status == 6 and "expert_to_rank value" in str(ei.value)
    with pytest.raises(moe.MoeError) as ei:
        lay.route(torch.zeros(65, 8, device=DEV), 2)          # T > max_tokens
    assert ei.value.status == 4
    with pytest.raises(moe.MoeError):
        lay.route(torch.zeros(8, 8, device=DEV), 9)           # k > E


# ------------------------------------------------------------------ a6-a8, whole layer
def run_layer(lay, inp, P, G):
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, inp.k)
    lay.dispatch(x, idx, P)
    hosted = list(range(inp.E)) if G > 1 or lay.G > 1 else [e for e in range(inp.E) if P[e] == 0]
    w1, w3, w2 = inp.device_weights(DEV, hosted)
    moe = _moe()
    w13 = moe.pack_w13(w1, w3)
    lay.expert_ffn(w13, w2)
    out = lay.combine(w)
    lay.sync()
    return out, idx, w


@pytest.mark.parametrize("T,H,F,E,k,G,P", [
    (1024, 64, 128, 8, 2, 4, [0, 0, 1, 1, 2, 2, 3, 3]),     # BASELINE configs[0] (tiny, 4 virtual ranks)
    (1024, 64, 128, 8, 2, 4, [0, 1, 2, 2, 3, 2, 3, 3]),
    (2000, 512, 1024, 8, 2, 1, [0] * 8),                   # several M/N/K tiles, ragged M tails
    (1500, 256, 192, 6, 3, 2, [1, 0, 1, 1, 0, 1]),           # F % 128 != 0 -> 128-wide SwiGLU tiles
    (700, 128, 256, 16, 4, 4, [e % 4 for e in range(16)]),
    (600, 128, 128, 64, 8, 8, [e // 8 for e in range(64)]),   # D5 shape family (E64 top-8), 8 virtual ranks
    (333, 64, 64, 5, 5, 1, [0] * 5),                         # k = E, ragged everything, BN = 64 tiles
    (97, 64, 128, 256, 16, 4, [(7 * e) % 4 for e in range(256)]),  # maximum E and k (kMaxExperts, kMaxK)
    (1, 64, 128, 8, 2, 1, [0] * 8),                          # a single token
])
def test_layer_parity(cuda_ok, T, H, F, E, k, G, P):
    inp = Inputs(T, H, F, E, k, s=1.6, seed=11)
    lay = make_layer(T, H, F, E, k, G)
    out, idx, w = run_layer(lay, inp, P, G)
    ref, ridx, rw = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
    assert np.array_equal(idx.cpu().numpy(), ridx)
    assert_close_layer(bf16_to_f64(out), ref)


@pytest.mark.parametrize("cg", ["1", "2"])
def test_both_gemm_tile_modes(cuda_ok, cg, monkeypatch):
    """128-row tiles on one CTA (decode-sized contexts) and 256-row tiles on a
    CTA pair (tcgen05 cta_group::2) are both checked against the oracle at a
    size that spans several tiles of either kind."""
    monkeypatch.setenv("MOE_GEMM_CG", cg)
    T, H, F, E, k, G = 1100, 256, 512, 8, 2, 2
    P = [0, 1, 1, 1, 0, 1, 0, 1]
    inp = Inputs(T, H, F, E, k, s=1.6, seed=17)
    lay = make_layer(T, H, F, E, k, G)
    out, idx, w = run_layer(lay, inp, P, G)
    ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
    assert_close_layer(bf16_to_f64(out), ref)


def test_placement_invariance_bit_exact(cuda_ok):
    """The GEMM is deterministic (fixed K order, no split-K), so the layer output is
    bit-identical across placements and G (SURVEY §8(c) 'Placement invariance')."""
    T, H, F, E, k = 1200, 128, 256, 8, 2
    inp = Inputs(T, H, F, E, k, s=1.6, seed=3)
    outs = []
    for G, P in [(1, [0] * 8), (4, [0, 0, 1, 1, 2, 2, 3, 3]), (4, [0, 1, 2, 2, 3, 2, 3, 3]), (8, list(range(8)))]:
        lay = make_layer(T, H, F, E, k, G)
        out, _, _ = run_layer(lay, inp, P, G)
        outs.append(out.view(torch.int16).cpu())
        lay.close()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def tile_cover_tokens(ridx, E, tile, seed):
    """Tokens such that every M tile of every expert segment holds a checked row.

    The receive layout puts expert e's rows in one segment ordered by (source,
    token) -- i.e. by token, since sources own contiguous token blocks (G7, G9) --
    padded to the GEMM M tile, so routed row i of expert e lies in M tile i // tile.
    A checked output row of token t covers, for each of its k experts, that
    expert's K5 and K6 M tile across every N tile (the row's full h and y).  One
    pseudo-random token per (expert, M tile) plus the first and last token."""
    rng = np.random.default_rng(seed)
    T = ridx.shape[0]
    sel = {0, T - 1}
    for e in range(E):
        toks = np.nonzero((ridx == e).any(1))[0]
        for m0 in range(0, len(toks), tile):
            chunk = toks[m0:m0 + tile]
            sel.add(int(chunk[rng.integers(0, len(chunk))]))
    sel = np.array(sorted(sel))
    for e in range(E):                     # assert the coverage claimed above
        toks = np.nonzero((ridx == e).any(1))[0]
        pos = np.searchsorted(toks, sel[np.isin(sel, toks)])
        assert set((pos // tile).tolist()) == set(range((len(toks) + tile - 1) // tile)), e
    return sel


@pytest.mark.parametrize("G,P,s", [
    (1, [0] * 8, 1.6),                            # the bench's N = 1 workload
    (4, [0, 1, 2, 2, 3, 2, 3, 3], 1.6),           # D3: ILP-1 balanced placement, 4 virtual EP ranks
    (4, [0, 0, 1, 1, 2, 2, 3, 3], 0.0),           # D2: uniform routing, contiguous placement
])
def test_mixtral_layer_full_size_every_tile(cuda_ok, G, P, s):
    """BASELINE configs[1]/[2] shape (E8 k2 H4096 F14336, T = 16384 tokens) at the
    bench's launch configuration, checked against the oracle's direct definition
    on tokens chosen so that every 256-row M tile of every expert segment -- hence
    every K5 and K6 output tile -- holds at least one checked row."""
    T, H, F, E, k = 16384, 4096, 14336, 8, 2
    dev = torch.device(DEV)
    x = synth.hidden_states(T, H, seed=0, device=dev)
    logits = synth.zipf_logits(T, E, s, seed=0, device=dev)
    ws = [synth.expert_weights(e, H, F, 0, device=dev) for e in range(E)]
    moe = _moe()
    lay = make_layer(T, H, F, E, k, G)
    idx, w = lay.route(logits, k)
    lay.dispatch(x, idx, P)
    w13 = moe.pack_w13(torch.stack([q[0] for q in ws]), torch.stack([q[1] for q in ws]))
    w2 = torch.stack([q[2] for q in ws])
    lay.expert_ffn(w13, w2)
    out = lay.combine(w)
    lay.sync()
    gidx = idx.cpu().numpy()
    sel = tile_cover_tokens(gidx, E, 256, seed=G)
    xs = bf16_to_f64(x[sel])
    ls = logits[sel].cpu().numpy()
    cache = {}

    def fn(e, rows):
        if e not in cache:
            cache.clear()
            cache[e] = tuple(bf16_to_f64(m) for m in ws[e])
        from oracle import ffn
        return ffn.swiglu(rows, *cache[e])[1]
    ref, ridx, rw = olayer.layer_direct(xs, ls, k, fn)
    assert np.array_equal(gidx[sel], ridx)
    assert_close_layer(bf16_to_f64(out[sel]), ref)
    lay.close()


def test_e64_layer_full_size_every_tile(cuda_ok):
    """BASELINE configs[4] shape (E64 top-8, H4096, F2048, T = 65536) over 4
    virtual EP ranks with the ILP-1 balanced placement, checked against the
    oracle's direct definition on tokens chosen so that every 256-row M tile of
    every expert segment holds a checked row (tile_cover_tokens; each token
    touches 8 experts)."""
    from paper_2502_06643_b200 import placement
    T, H, F, E, k, G = 65536, 4096, 2048, 64, 8, 4
    dev = torch.device(DEV)
    x = synth.hidden_states(T, H, seed=0, device=dev)
    logits = synth.zipf_logits(T, E, 1.6, seed=0, device=dev)
    ws = [synth.expert_weights(e, H, F, 0, device=dev) for e in range(E)]
    moe = _moe()
    lay = make_layer(T, H, F, E, k, G)
    idx, w = lay.route(logits, k)
    load = np.bincount(idx.cpu().numpy().ravel(), minlength=E)
    P = placement.balanced(load, G)
    lay.dispatch(x, idx, P)
    w13 = moe.pack_w13(torch.stack([q[0] for q in ws]), torch.stack([q[1] for q in ws]))
    w2 = torch.stack([q[2] for q in ws])
    lay.expert_ffn(w13, w2)
    out = lay.combine(w)
    lay.sync()
    sel = tile_cover_tokens(idx.cpu().numpy(), E, 256, seed=5)
    xs = bf16_to_f64(x[sel])
    ls = logits[sel].cpu().numpy()
    cache = {}

    def fn(e, rows):
        if e not in cache:
            cache.clear()                 # layer_direct visits each expert once
            cache[e] = tuple(bf16_to_f64(m) for m in ws[e])
        from oracle import ffn
        return ffn.swiglu(rows, *cache[e])[1]
    ref, ridx, rw = olayer.layer_direct(xs, ls, k, fn)
    assert np.array_equal(idx[sel].cpu().numpy(), ridx)
    assert_close_layer(bf16_to_f64(out[sel]), ref)


def test_cuda_graph_replay_bit_exact(cuda_ok):
    """A whole layer (route .. combine) captured in a CUDA graph replays to the
    eager result bit-exactly (no host round trip on the path; moe.h)."""
    moe = _moe()
    T, H, F, E, k, G = 700, 128, 256, 8, 2, 4
    P = [0, 1, 2, 2, 3, 2, 3, 3]
    inp = Inputs(T, H, F, E, k, s=1.6, seed=29)
    lay = make_layer(T, H, F, E, k, G)
    x, logits = inp.to_device(DEV)
    w1, w3, w2 = inp.device_weights(DEV, list(range(E)))
    w13 = moe.pack_w13(w1, w3)
    idx = torch.empty(T, k, dtype=torch.int32, device=DEV)
    w = torch.empty(T, k, dtype=torch.float32, device=DEV)
    out = torch.empty(T, H, dtype=torch.bfloat16, device=DEV)

    def step():
        lay.route(logits, k, idx, w)
        lay.dispatch(x, idx, P)
        lay.expert_ffn(w13, w2)
        lay.combine(w, out)

    step()
    lay.sync()
    ref = out.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
    lay.sync()


def test_timeline_events_ordered(cuda_ok):
    """moe_timeline_*: 8 events per layer, non-decreasing along the stream order."""
    moe = _moe()
    T, H, F, E, k, G = 500, 128, 256, 8, 2, 2
    inp = Inputs(T, H, F, E, k, s=1.6, seed=31)
    lay = make_layer(T, H, F, E, k, G)
    x, logits = inp.to_device(DEV)
    w1, w3, w2 = inp.device_weights(DEV, list(range(E)))
    w13 = moe.pack_w13(w1, w3)
    lay.timeline(3)
    for _ in range(4):                 # one more layer than records: the extra is not recorded
        idx, w = lay.route(logits, k)
        lay.dispatch(x, idx, [0, 1] * 4)
        lay.expert_ffn(w13, w2)
        lay.combine(w)
    rec = lay.timeline_read()
    assert len(rec) == 3
    for r in rec:
        assert r[0] == 0.0 and all(v >= 0 for v in r)
        main = [r[0], r[1], r[2], r[4], r[5], r[6], r[7]]   # events on the caller's stream
        assert all(b >= a for a, b in zip(main, main[1:]))


@pytest.mark.parametrize("ksplit", ["1", "3", "8"])
def test_decode_splitk(cuda_ok, ksplit, monkeypatch):
    """Decode-sized contexts split K6 over F (fp32 partials, ordered reduction);
    forced slice counts, including slices of a single k-block, against the oracle."""
    monkeypatch.setenv("MOE_GEMM_CG", "1")
    monkeypatch.setenv("MOE_DECODE_SPLITK", ksplit)
    T, H, F, E, k, G = 301, 256, 512, 8, 2, 2
    P = [1, 0, 1, 1, 0, 1, 0, 1]
    inp = Inputs(T, H, F, E, k, s=1.6, seed=37)
    lay = make_layer(T, H, F, E, k, G)
    out, idx, w = run_layer(lay, inp, P, G)
    ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
    assert_close_layer(bf16_to_f64(out), ref)


def test_device_placement_is_validated_on_the_device(cuda_ok):
    """moe_dispatch takes the placement as a device array; a value
    outside [0, G) latches MOE_ERR_DEVICE (and is read as 0, so no buffer index
    leaves its bounds); the next dispatch with a valid map is unaffected."""
    moe = _moe()
    T, H, F, E, k, G = 300, 64, 128, 8, 2, 4
    inp = Inputs(T, H, F, E, k, s=1.6, seed=41)
    lay = make_layer(T, H, F, E, k, G)
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, k)
    bad = torch.tensor([0, 1, 2, 4, 3, 2, 1, 0], dtype=torch.int32, device=DEV)
    lay.dispatch(x, idx, bad)
    with pytest.raises(moe.MoeError) as ei:
        lay.sync()
    assert ei.value.status == 6 and "expert_to_rank value" in str(ei.value)
    good = torch.tensor([0, 1, 2, 3, 3, 2, 1, 0], dtype=torch.int32, device=DEV)
    out, _, _ = run_layer(lay, inp, good, G)
    ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
    assert_close_layer(bf16_to_f64(out), ref)


def test_weight_count_mismatch_is_caught(cuda_ok):
    """moe_expert_ffn's n_w must equal the experts the placement hosts: the host
    cannot see a device placement, so the GEMM checks it (MOE_ERR_DEVICE)."""
    moe = _moe()
    T, H, F, E, k = 200, 64, 128, 8, 2
    inp = Inputs(T, H, F, E, k, s=1.6, seed=43)
    lay = make_layer(T, H, F, E, k, 1)
    x, logits = inp.to_device(DEV)
    idx, w = lay.route(logits, k)
    lay.dispatch(x, idx, [0] * E)
    w1, w3, w2 = inp.device_weights(DEV, list(range(E - 1)))      # one expert short
    lay.expert_ffn(moe.pack_w13(w1, w3), w2)
    lay.combine(w)
    with pytest.raises(moe.MoeError) as ei:
        lay.sync()
    assert ei.value.status == 6 and "n_w" in str(ei.value)
    vl = make_layer(T, H, F, E, k, 2)                                # virtual ranks: n_w == E, host-checked
    vi, vw = vl.route(logits, k)
    vl.dispatch(x, vi, [0, 1] * 4)
    with pytest.raises(moe.MoeError) as ei:
        vl.expert_ffn(moe.pack_w13(w1, w3), w2)
    assert ei.value.status == 1
    vl.close()
    lay.close()


def _chain_home_and_direct(make, inp_list, plans, k, E, dev_ws):
    """Run an L-layer chain twice: home-rank EP (moe_combine, then the next
    moe_dispatch from home) and direct l -> l+1 dispatch (NEXT-4: MOE_OUT_STAY +
    moe_dispatch_from, two contexts alternating).  Returns both final outputs."""
    moe = _moe()
    L = len(plans)
    x0, logits = inp_list
    w13, w2 = dev_ws
    home = make()
    x = x0
    for li in range(L):
        idx, w = home.route(logits[li], k)
        home.dispatch(x, idx, plans[li])
        home.expert_ffn(w13, w2)
        x = home.combine(w)
    home.sync()
    home_out = x
    ctxs = [make(), make()]
    x = x0
    prev = prev_w = None
    for li in range(L):
        c = ctxs[li % 2]
        idx, w = c.route(logits[li], k)
        if prev is None:
            c.dispatch(x, idx, plans[li])
        else:
            c.dispatch_from(prev, prev_w, idx, plans[li])
        c.output_mode("home" if li == L - 1 else "stay")
        c.expert_ffn(w13, w2)
        prev, prev_w = c, w
    out = prev.combine(prev_w)
    prev.sync()
    return home_out, out


@pytest.mark.parametrize("G", [1, 4])
def test_direct_layer_to_layer_dispatch_bit_exact(cuda_ok, G):
    """NEXT-4 (Eq. 8's direct inter-layer traffic): a 3-layer chain with
    per-layer placements run with direct l -> l+1 dispatch equals the home-rank
    chain bit-exactly (the receive rows use the home combine's arithmetic) and the
    oracle's layer-by-layer chain within tolerance (virtual ranks; real ranks in
    tests/test_gpu_group.py)."""
    T, H, F, E, k, L = 700, 128, 256, 8, 2, 3
    inp = Inputs(T, H, F, E, k, s=1.6, seed=51)
    x0 = inp.x.to(DEV)
    logits = [synth.zipf_logits(T, E, 1.6, seed=100 + li).to(DEV) for li in range(L)]
    plans = [[0, 0, 1, 1, 2, 2, 3, 3], [0, 1, 2, 2, 3, 2, 3, 3], [3, 2, 1, 0, 0, 1, 2, 3]]
    plans = [[p % G for p in q] for q in plans]
    w1, w3, w2 = inp.device_weights(DEV, list(range(E)))
    moe = _moe()
    home_out, direct_out = _chain_home_and_direct(lambda: make_layer(T, H, F, E, k, G), (x0, logits), plans, k, E,
                                                  (moe.pack_w13(w1, w3), w2))
    assert torch.equal(home_out.view(torch.int16), direct_out.view(torch.int16))
    xr = bf16_to_f64(inp.x)
    for li in range(L):
        xr, _, _ = olayer.layer_direct(xr, logits[li].cpu().numpy(), k, inp.oracle_expert_fn())
    assert_close_layer(bf16_to_f64(direct_out), xr)


def test_direct_dispatch_argument_checks(cuda_ok):
    """moe_dispatch_from's call discipline (moe.h): prev must be another context of
    the same rank whose last FFN ran with MOE_OUT_STAY on the same T; a
    MOE_OUT_STAY context refuses moe_combine."""
    moe = _moe()
    T, H, F, E, k, G = 300, 64, 128, 8, 2, 2
    inp = Inputs(T, H, F, E, k, s=1.6, seed=81)
    a, b = make_layer(T, H, F, E, k, G), make_layer(T, H, F, E, k, G)
    x, logits = inp.to_device(DEV)
    w1, w3, w2 = inp.device_weights(DEV, list(range(E)))
    w13 = moe.pack_w13(w1, w3)
    P = [0, 1] * 4
    idx, w = a.route(logits, k)
    a.dispatch(x, idx, P)
    with pytest.raises(moe.MoeError) as ei:           # prev is not in MOE_OUT_STAY / has no FFN yet
        b.dispatch_from(a, w, idx, P)
    assert ei.value.status == 1
    a.output_mode("stay")
    a.expert_ffn(w13, w2)
    with pytest.raises(moe.MoeError) as ei:           # the outputs stay: no home combine
        a.combine(w)
    assert ei.value.status == 1
    with pytest.raises(moe.MoeError) as ei:           # prev must be another context
        a.dispatch_from(a, w, idx, P)
    assert ei.value.status == 1
    with pytest.raises(moe.MoeError) as ei:           # T differs from prev's
        b.dispatch_from(a, w[:10].contiguous(), idx[:10].contiguous(), P)
    assert ei.value.status == 1
    b.dispatch_from(a, w, idx, P)                     # valid
    b.expert_ffn(w13, w2)
    out = b.combine(w)
    b.sync()
    assert torch.isfinite(out.float()).all()
    a.close()
    b.close()
