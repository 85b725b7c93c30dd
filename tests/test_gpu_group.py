"""The real multi-rank data plane on ONE GPU: a single-process EP group
(moe_ctx_create_group) of G rank contexts on cuda:0, each rank with its own
streams, buffers and signal block, talking through the same P2P code as G
processes on G GPUs -- the in-kernel count all-gather of k_layout, the
side-stream scatter of the peers' rows, K5's per-tile arrival waits, the fused
(K6 epilogue) and pulled (K8) combines, the TP all-gather fan-out and partial
return -- with the peers' device pointers in the tables instead of CUDA IPC
mappings (an IPC handle cannot be opened by the process that exported it).

Checked against the oracle (the all-to-all before and after the expert FFN,
P:L824; the expert -> GPU map): the plan (count matrix, send slots,
receive positions, destinations) and the received payload bit-exactly, the
identity-expert round trip bit-exactly, the layer output bit-identical to the
virtual-rank run and within 2e-2 of the oracle (G16).  Ranks are issued from
one host thread in rank order; no call blocks on a peer.
"""

import os

import numpy as np
import pytest
import torch

from oracle import layer as olayer
from oracle import plan as oplan
from oracle import route as oroute
from tests._util import Inputs, assert_close_layer, bf16_to_f64

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def _moe():
    from paper_2502_06643_b200 import moe
    return moe


class Group:
    """G rank contexts of one EP group on cuda:0, one stream per rank."""

    def __init__(self, G, T, H, F, E, k, tp=1):
        moe = _moe()
        self.G, self.tp = G, tp
        self.blocks = oplan.token_blocks(T, G)
        tmax = max(max(b - a for a, b in self.blocks), 1)
        self.lays = moe.MoeLayer.group(G, max_tokens=tmax, hidden=H, ffn=F, num_experts=E, max_k=k, tp=tp)
        self.streams = [torch.cuda.Stream(device=DEV) for _ in range(G)]

    def each(self, fn):
        """fn(r, layer) for every rank, issued on rank r's stream; returns the results."""
        res = []
        for r, lay in enumerate(self.lays):
            with torch.cuda.stream(self.streams[r]):
                res.append(fn(r, lay))
        return res

    def sync(self):
        for lay in self.lays:
            lay.sync()
        torch.cuda.synchronize()

    def close(self):
        torch.cuda.synchronize()
        for lay in self.lays:
            lay.close()


def _setup(inp, g, k):
    x_all, logits_all = inp.to_device(DEV)
    xs = [x_all[a:b].contiguous() for a, b in g.blocks]
    ls = [logits_all[a:b].contiguous() for a, b in g.blocks]
    torch.cuda.synchronize()
    return x_all, logits_all, xs, ls


def _virtual_out(inp, P, G, k, tp=1):
    moe = _moe()
    T, H, F, E = inp.T, inp.H, inp.F, inp.E
    vl = moe.MoeLayer(max_tokens=T, hidden=H, ffn=F, num_experts=E, max_k=k, virtual_ranks=G, tp=tp)
    x_all, logits_all = inp.to_device(DEV)
    vi, vw = vl.route(logits_all, k)
    vl.dispatch(x_all, vi, P)
    w1, w3, w2 = inp.device_weights(DEV, list(range(E)))
    vl.expert_ffn(moe.pack_w13(w1, w3), w2)
    out = vl.combine(vw)
    vl.sync()
    vl.close()
    return out


PLACEMENTS = {
    2: [[0, 0, 0, 0, 1, 1, 1, 1], [0, 1, 1, 1, 0, 1, 0, 1], [1] * 6 + [0, 0]],
    4: [[0, 0, 1, 1, 2, 2, 3, 3], [0, 1, 2, 2, 3, 2, 3, 3], [3] * 6 + [0, 0]],   # last: ranks 1, 2 host nothing
}


@pytest.mark.parametrize("dispatch", ["scatter", "gather"])
@pytest.mark.parametrize("fused", ["0", "1"])
@pytest.mark.parametrize("G", [2, 4])
def test_group_plan_payload_and_layer(cuda_ok, G, fused, dispatch, monkeypatch):
    """scatter: every routed row is stored into the hosting rank's receive row by
    the source (NVLink; TMA bulk copies for the peers' rows); gather: every token block is copied once to every peer by
    the copy engines, the source sends only the row -> token map, and the receiver
    expands its rows (k_expand); fused / pulled combine."""
    monkeypatch.setenv("MOE_FUSED_COMBINE", fused)
    monkeypatch.setenv("MOE_DISPATCH", dispatch)
    moe = _moe()
    T, H, F, E, k = 1500, 256, 512, 8, 2
    inp = Inputs(T, H, F, E, k, s=1.6, seed=21 + G)
    g = Group(G, T, H, F, E, k)
    x_all, logits_all, xs, ls = _setup(inp, g, k)
    ridx, _ = oroute.route(inp.logits.numpy(), k)
    ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
    xb = inp.x.view(torch.int16).numpy().view(np.uint16)
    for P in PLACEMENTS[G]:
        P = np.array(P)
        for lay in g.lays:
            lay.placement(P)          # upload the device placement before any rank's layer is issued
        torch.cuda.synchronize()
        rw = g.each(lambda r, lay: lay.route(ls[r], k))
        g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
        pl = oplan.plan([ridx[a:b] for a, b in g.blocks], P, G)
        for r, lay in enumerate(g.lays):
            dr, rp, ss, cnt = lay.debug_plan()
            a, b = g.blocks[r]
            assert np.array_equal(cnt, pl["cnt"]), "count matrix (in-kernel all-gather)"
            assert np.array_equal(ss, pl["slot"][r]), "send slots"
            assert np.array_equal(rp, pl["recv_pos"][r]), "receive positions"
            assert np.array_equal(dr, P[ridx[a:b]]), "destination ranks"
            rows = lay.debug_recv()
            ref_rows = xb[[g.blocks[s][0] + t for (s, t, j, e) in pl["recv"][r]]].reshape(-1, H)
            assert np.array_equal(rows, ref_rows), f"received payload of rank {r}"
        g.each(lambda r, lay: lay.identity_ffn())
        outs = g.each(lambda r, lay: lay.combine(rw[r][1]))
        g.sync()
        for r in range(G):
            assert torch.equal(outs[r].view(torch.int16), xs[r].view(torch.int16)), "identity round trip"
        # the real expert FFN: K5 waits per tile for the peers' rows, K6 returns them
        ws = []
        for r in range(G):
            hosted = [e for e in range(E) if P[e] == r]
            if hosted:
                w1, w3, w2 = inp.device_weights(DEV, hosted)
                ws.append((moe.pack_w13(w1, w3), w2))
            else:
                ws.append((None, None))
        torch.cuda.synchronize()
        g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
        g.each(lambda r, lay: lay.expert_ffn(*ws[r]))
        outs = g.each(lambda r, lay: lay.combine(rw[r][1]))
        g.sync()
        out = torch.cat(outs)
        virt = _virtual_out(inp, P, G, k)
        assert torch.equal(out.view(torch.int16), virt.view(torch.int16)), "cross-mode equality (group vs virtual)"
        assert_close_layer(bf16_to_f64(out), ref)
    g.close()


@pytest.mark.parametrize("G,tp,fused,dispatch", [(2, 2, "0", "scatter"), (2, 2, "1", "gather"),
                                                 (4, 2, "1", "scatter"), (4, 2, "0", "gather"),
                                                 (4, 4, "0", "scatter")])
def test_group_tensor_parallel(cuda_ok, G, tp, fused, dispatch, monkeypatch):
    """EP x TP over G ranks of one GPU (reading G20): the TP all-gather fan-out of
    the dispatch and the bf16 partial return of the combine, against the oracle's
    TP layer and the virtual-rank TP run."""
    monkeypatch.setenv("MOE_FUSED_COMBINE", fused)
    monkeypatch.setenv("MOE_DISPATCH", dispatch)
    moe = _moe()
    T, H, F, E, k = 1100, 256, 512, 8, 2
    n_grp = G // tp
    inp = Inputs(T, H, F, E, k, s=1.6, seed=31 + G + tp)
    g = Group(G, T, H, F, E, k, tp=tp)
    x_all, logits_all, xs, ls = _setup(inp, g, k)
    ridx, _ = oroute.route(inp.logits.numpy(), k)
    w1a, w3a, w2a = inp.device_weights(DEV, list(range(E)))
    xb = inp.x.view(torch.int16).numpy().view(np.uint16)
    for P in ([e * n_grp // E for e in range(E)], [0, 1, 1, 1, 0, 1, 0, 1]):
        P = np.array(P) % n_grp
        ws = []
        for r in range(G):
            hosted = [e for e in range(E) if P[e] == r // tp]
            if hosted:
                sel = torch.tensor(hosted, device=DEV)
                ws.append(moe.tp_slice_weights(w1a[sel], w3a[sel], w2a[sel], tp, r % tp))
            else:
                ws.append((None, None))
            g.lays[r].placement(P)
        torch.cuda.synchronize()
        rw = g.each(lambda r, lay: lay.route(ls[r], k))
        g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
        pl = oplan.plan([ridx[a:b] for a, b in g.blocks], P, n_grp)
        for r, lay in enumerate(g.lays):
            dr, rp, ss, cnt = lay.debug_plan()
            assert np.array_equal(cnt, pl["cnt"])
            assert np.array_equal(ss, pl["slot"][r])
            assert np.array_equal(rp, pl["recv_pos"][r])
            rows = lay.debug_recv()                      # every TP rank of a group holds its rows
            ref_rows = xb[[g.blocks[s][0] + t for (s, t, j, e) in pl["recv"][r // tp]]].reshape(-1, H)
            assert np.array_equal(rows, ref_rows)
        g.each(lambda r, lay: lay.expert_ffn(*ws[r]))
        outs = g.each(lambda r, lay: lay.combine(rw[r][1]))
        g.sync()
        out = torch.cat(outs)
        virt = _virtual_out(inp, P, G, k, tp=tp)
        assert torch.equal(out.view(torch.int16), virt.view(torch.int16)), "cross-mode equality (TP)"
        ref, _, _, _ = olayer.layer_ep_tp(bf16_to_f64(inp.x), inp.logits.numpy(), k, P, n_grp, tp,
                                          inp.oracle_tp_fn(tp))
        assert_close_layer(bf16_to_f64(out), ref)
    g.close()


def test_group_zero_token_ranks_and_per_layer_placements(cuda_ok):
    """Ranks owning 0 tokens (G7) and a different device placement every layer:
    the T = 0 rank's combine waits for every rank's expert outputs, so its next
    dispatch cannot overwrite count rows a peer is still reading (8 layers,
    epochs advance, the placement array changes between layers with no host
    synchronisation)."""
    moe = _moe()
    G, H, F, E, k = 4, 128, 256, 8, 2
    T = 3                                  # ranks 0..2 own 1 token, rank 3 none
    inp = Inputs(64, H, F, E, k, s=1.6, seed=5)
    g = Group(G, T, H, F, E, k)
    x_all, logits_all = inp.to_device(DEV)
    xs = [x_all[:T][a:b].contiguous() for a, b in g.blocks]
    ls = [logits_all[:T][a:b].contiguous() for a, b in g.blocks]
    plans = [np.array(p) for p in ([0, 0, 1, 1, 2, 2, 3, 3], [3, 2, 1, 0, 0, 1, 2, 3], [1] * 8,
                                   [0, 1, 2, 2, 3, 2, 3, 3])]
    w1a, w3a, w2a = inp.device_weights(DEV, list(range(E)))
    wsets = []
    for P in plans:
        row = []
        for r in range(G):
            hosted = [e for e in range(E) if P[e] == r]
            sel = torch.tensor(hosted, device=DEV, dtype=torch.long)
            row.append((moe.pack_w13(w1a[sel], w3a[sel]), w2a[sel].contiguous()) if hosted else (None, None))
            g.lays[r].placement(P)
        wsets.append(row)
    torch.cuda.synchronize()
    outs_all = []
    for layer in range(8):
        li = layer % len(plans)
        P = plans[li]
        rw = g.each(lambda r, lay: lay.route(ls[r], k))
        g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
        g.each(lambda r, lay: lay.expert_ffn(*wsets[li][r]))
        outs_all.append(g.each(lambda r, lay: lay.combine(rw[r][1])))
    g.sync()
    ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x[:T]), inp.logits[:T].numpy(), k, inp.oracle_expert_fn())
    for outs in outs_all:
        assert outs[3].shape == (0, H)
        assert_close_layer(bf16_to_f64(torch.cat(outs)), ref)
        assert torch.equal(torch.cat(outs).view(torch.int16), torch.cat(outs_all[0]).view(torch.int16))
    g.close()


def test_group_graph_capture_per_layer_placements(cuda_ok):
    """Each rank's 4-layer chain -- a different device placement per layer --
    captured into one CUDA graph per rank and replayed (device-side flag epoch,
    device placement arrays: no host synchronisation inside the chain); replays
    are bit-identical to the eager chain."""
    moe = _moe()
    G, T, H, F, E, k, L = 2, 600, 256, 512, 8, 2, 4
    inp = Inputs(T, H, F, E, k, s=1.6, seed=9)
    g = Group(G, T, H, F, E, k)
    x_all, logits_all, xs, ls = _setup(inp, g, k)
    plans = [np.array(p) for p in ([0, 0, 0, 0, 1, 1, 1, 1], [0, 1, 1, 1, 0, 1, 0, 1], [1, 0, 1, 0, 1, 0, 1, 0],
                                   [1, 1, 1, 1, 1, 1, 0, 0])]
    w1a, w3a, w2a = inp.device_weights(DEV, list(range(E)))
    wl, Pd = [], []
    for r in range(G):
        wl.append([])
        Pd.append([])
        for P in plans:
            hosted = [e for e in range(E) if P[e] == r]
            sel = torch.tensor(hosted, device=DEV, dtype=torch.long)
            wl[r].append((moe.pack_w13(w1a[sel], w3a[sel]), w2a[sel].contiguous()) if hosted else (None, None))
            Pd[r].append(g.lays[r].placement(P))
    bufs = [[torch.empty_like(xs[r]) for _ in range(L)] for r in range(G)]
    idx = [torch.empty(xs[r].shape[0], k, dtype=torch.int32, device=DEV) for r in range(G)]
    wts = [torch.empty(xs[r].shape[0], k, dtype=torch.float32, device=DEV) for r in range(G)]
    torch.cuda.synchronize()

    def chain(r, lay):
        xin = xs[r]
        for li in range(L):
            lay.route(ls[r], k, idx[r], wts[r])
            lay.dispatch(xin, idx[r], Pd[r][li])
            lay.expert_ffn(*wl[r][li])
            lay.combine(wts[r], bufs[r][li])
            xin = bufs[r][li]

    # eager (layer by layer across ranks, as a real group would run)
    def eager():
        for li in range(L):
            for r, lay in enumerate(g.lays):
                with torch.cuda.stream(g.streams[r]):
                    xin = xs[r] if li == 0 else bufs[r][li - 1]
                    lay.route(ls[r], k, idx[r], wts[r])
                    lay.dispatch(xin, idx[r], Pd[r][li])
            for r, lay in enumerate(g.lays):
                with torch.cuda.stream(g.streams[r]):
                    lay.expert_ffn(*wl[r][li])
            for r, lay in enumerate(g.lays):
                with torch.cuda.stream(g.streams[r]):
                    lay.combine(wts[r], bufs[r][li])
        g.sync()

    eager()
    ref = [[b.clone() for b in bufs[r]] for r in range(G)]
    graphs = []
    for r, lay in enumerate(g.lays):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=g.streams[r]):
            chain(r, lay)
        graphs.append(gr)
    for rep in range(3):
        for r in range(G):
            for b in bufs[r]:
                b.zero_()
        torch.cuda.synchronize()
        for r in range(G):
            with torch.cuda.stream(g.streams[r]):
                graphs[r].replay()
        g.sync()
        for r in range(G):
            for li in range(L):
                assert torch.equal(bufs[r][li].view(torch.int16), ref[r][li].view(torch.int16)), (rep, r, li)
    ref_l0, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
    assert_close_layer(bf16_to_f64(torch.cat([ref[r][0] for r in range(G)])), ref_l0)
    del graphs
    g.close()


def test_group_detects_mismatched_placements(cuda_ok):
    """Call discipline: ranks dispatching with different maps are
    caught on the device (the placement hash travels with the counts)."""
    moe = _moe()
    G, T, H, F, E, k = 2, 200, 64, 128, 8, 2
    inp = Inputs(T, H, F, E, k, s=1.6, seed=3, with_weights=False)
    g = Group(G, T, H, F, E, k)
    x_all, logits_all, xs, ls = _setup(inp, g, k)
    Ps = [np.array([0, 0, 0, 0, 1, 1, 1, 1]), np.array([1, 1, 1, 1, 0, 0, 0, 0])]
    for r in range(G):
        g.lays[r].placement(Ps[r])
    torch.cuda.synchronize()
    rw = g.each(lambda r, lay: lay.route(ls[r], k))
    g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], Ps[r]))
    for lay in g.lays:
        with pytest.raises(moe.MoeError) as ei:
            lay.sync()
        assert "different expert_to_rank" in str(ei.value)
    g.close()


@pytest.mark.parametrize("dispatch", ["scatter", "gather"])
@pytest.mark.parametrize("G", [2, 4])
def test_group_topk_at_least_ranks(cuda_ok, G, dispatch, monkeypatch):
    """The D5 regime (top-k >= EP ranks: E16 top-4 here, E64 top-8 in the bench),
    where the gather dispatch sends a token once per destination rank; uneven
    experts per rank (G14); plan, payload, layer vs virtual ranks and the oracle."""
    monkeypatch.setenv("MOE_DISPATCH", dispatch)
    moe = _moe()
    T, H, F, E, k = 900, 128, 256, 16, 4
    P = np.array([(3 * e + e // 5) % G for e in range(E)])
    inp = Inputs(T, H, F, E, k, s=1.2, seed=71 + G)
    g = Group(G, T, H, F, E, k)
    x_all, logits_all, xs, ls = _setup(inp, g, k)
    ridx, _ = oroute.route(inp.logits.numpy(), k)
    xb = inp.x.view(torch.int16).numpy().view(np.uint16)
    ws = []
    for r in range(G):
        hosted = [e for e in range(E) if P[e] == r]
        w1, w3, w2 = inp.device_weights(DEV, hosted)
        ws.append((moe.pack_w13(w1, w3), w2) if hosted else (None, None))
        g.lays[r].placement(P)
    torch.cuda.synchronize()
    for rep in range(2):
        rw = g.each(lambda r, lay: lay.route(ls[r], k))
        g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
        if rep == 0:
            pl = oplan.plan([ridx[a:b] for a, b in g.blocks], P, G)
            for r, lay in enumerate(g.lays):
                dr, rp, ss, cnt = lay.debug_plan()
                assert np.array_equal(cnt, pl["cnt"]) and np.array_equal(ss, pl["slot"][r])
                assert np.array_equal(rp, pl["recv_pos"][r])
                ref_rows = xb[[g.blocks[s][0] + t for (s, t, j, e) in pl["recv"][r]]].reshape(-1, H)
                assert np.array_equal(lay.debug_recv(), ref_rows)
        g.each(lambda r, lay: lay.expert_ffn(*ws[r]))
        outs = g.each(lambda r, lay: lay.combine(rw[r][1]))
        g.sync()
        out = torch.cat(outs)
        if rep == 0:
            virt = _virtual_out(inp, P, G, k)
            ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
        assert torch.equal(out.view(torch.int16), virt.view(torch.int16))
        assert_close_layer(bf16_to_f64(out), ref)
    g.close()


@pytest.mark.parametrize("G", [2, 4])
def test_group_direct_layer_to_layer_dispatch(cuda_ok, G):
    """NEXT-4 over real P2P ranks (one GPU): a 4-layer chain with per-layer
    placements, direct l -> l+1 dispatch (each rank's receive rows combined from
    the layer-l outputs where they were computed: local reads for co-located
    experts, peer loads otherwise) vs the home-rank chain -- bit-identical."""
    moe = _moe()
    T, H, F, E, k, L = 800, 128, 256, 8, 2, 4
    inp = Inputs(T, H, F, E, k, s=1.6, seed=61 + G)
    blocks = oplan.token_blocks(T, G)
    tmax = max(b - a for a, b in blocks)
    mk = lambda: moe.MoeLayer.group(G, max_tokens=tmax, hidden=H, ffn=F, num_experts=E, max_k=k)
    home, ca, cb = mk(), mk(), mk()
    streams = [torch.cuda.Stream(device=DEV) for _ in range(G)]
    x_all = inp.x.to(DEV)
    xs = [x_all[a:b].contiguous() for a, b in blocks]
    lg = [synth_logits(T, E, 100 + li) for li in range(L)]
    ls = [[q[a:b].contiguous() for a, b in blocks] for q in lg]
    plans = [np.array(p) % G for p in ([0, 0, 1, 1, 2, 2, 3, 3], [0, 1, 2, 2, 3, 2, 3, 3], [1, 0, 3, 2, 0, 1, 2, 3],
                                       [3, 3, 2, 2, 1, 1, 0, 0])]
    w1a, w3a, w2a = inp.device_weights(DEV, list(range(E)))
    ws = {}
    for li, P in enumerate(plans):
        for r in range(G):
            hosted = [e for e in range(E) if P[e] == r]
            sel = torch.tensor(hosted, device=DEV, dtype=torch.long)
            ws[li, r] = (moe.pack_w13(w1a[sel], w3a[sel]), w2a[sel].contiguous()) if hosted else (None, None)
            for grp_ in (home, ca, cb):
                grp_[r].placement(P)
    torch.cuda.synchronize()

    def each(lays, fn):
        out = []
        for r, lay in enumerate(lays):
            with torch.cuda.stream(streams[r]):
                out.append(fn(r, lay))
        return out

    # home-rank chain
    x = xs
    for li in range(L):
        rw = each(home, lambda r, lay: lay.route(ls[li][r], k))
        each(home, lambda r, lay: lay.dispatch(x[r], rw[r][0], plans[li]))
        each(home, lambda r, lay: lay.expert_ffn(*ws[li, r]))
        x = each(home, lambda r, lay: lay.combine(rw[r][1]))
    torch.cuda.synchronize()
    home_out = torch.cat(x)
    # direct chain: two context groups alternate
    prev = prev_w = None
    for li in range(L):
        cur = (ca, cb)[li % 2]
        rw = each(cur, lambda r, lay: lay.route(ls[li][r], k))
        if prev is None:
            each(cur, lambda r, lay: lay.dispatch(xs[r], rw[r][0], plans[li]))
        else:
            each(cur, lambda r, lay: lay.dispatch_from(prev[r], prev_w[r], rw[r][0], plans[li]))
        each(cur, lambda r, lay: lay.output_mode("home" if li == L - 1 else "stay"))
        each(cur, lambda r, lay: lay.expert_ffn(*ws[li, r]))
        prev, prev_w = cur, [q[1] for q in rw]
    outs = each(prev, lambda r, lay: lay.combine(prev_w[r]))
    for lay in prev:
        lay.sync()
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs).view(torch.int16), home_out.view(torch.int16))
    for grp_ in (home, ca, cb):
        for lay in grp_:
            lay.close()


def synth_logits(T, E, seed):
    import synth
    return synth.zipf_logits(T, E, 1.6, seed=seed).to(DEV)


@pytest.mark.parametrize("P,s,ce", [([0, 1, 2, 2, 3, 2, 3, 3], 1.6, False), ([0, 0, 1, 1, 2, 2, 3, 3], 0.0, False),
                                    ([0, 1, 2, 2, 3, 2, 3, 3], 1.6, True)])
def test_group_mixtral_full_size_every_tile(cuda_ok, P, s, ce, monkeypatch):
    """The bench's 4EP configuration at full size -- Mixtral layer (E8 top-2, H4096,
    F14336), T = 16384 tokens over 4 real P2P ranks on one GPU, ILP-1 balanced
    placement at s = 1.6 (D3) and contiguous at s = 0 (D2) -- checked against the
    oracle on tokens covering every 256-row M tile of every expert segment (on
    each hosting rank, an expert's rows are ordered by source, then token: the
    global token order, as in the virtual-rank layout).  ce: the copy-engine data
    plane (MOE_A2A_CE=1; F = 14336 > 8192, so the rows return by copy engine per
    K6 segment)."""
    if ce:
        monkeypatch.setenv("MOE_A2A_CE", "1")
    import synth
    from tests.test_gpu_parity import tile_cover_tokens
    moe = _moe()
    T, H, F, E, k, G = 16384, 4096, 14336, 8, 2, 4
    P = np.array(P)
    g = Group(G, T, H, F, E, k)
    x_all = synth.hidden_states(T, H, seed=0, device=DEV)
    logits_all = synth.zipf_logits(T, E, s, seed=0, device=DEV)
    xs = [x_all[a:b].contiguous() for a, b in g.blocks]
    ls = [logits_all[a:b].contiguous() for a, b in g.blocks]
    ws_cpu = [synth.expert_weights(e, H, F, 0, device=DEV) for e in range(E)]
    ws = []
    for r in range(G):
        hosted = [e for e in range(E) if P[e] == r]
        w1 = torch.stack([ws_cpu[e][0] for e in hosted])
        w3 = torch.stack([ws_cpu[e][1] for e in hosted])
        ws.append((moe.pack_w13(w1, w3), torch.stack([ws_cpu[e][2] for e in hosted])))
        g.lays[r].placement(P)
    torch.cuda.synchronize()
    rw = g.each(lambda r, lay: lay.route(ls[r], k))
    g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
    g.each(lambda r, lay: lay.expert_ffn(*ws[r]))
    outs = g.each(lambda r, lay: lay.combine(rw[r][1]))
    g.sync()
    if ce:   # the staging buffer exists only when the copy-engine plane ran
        assert g.lays[0].debug_send().shape[0] == rw[0][0].numel()   # rank 0's routed items
    out = torch.cat(outs)
    gidx = torch.cat([q[0] for q in rw]).cpu().numpy()
    sel = tile_cover_tokens(gidx, E, 256, seed=7)
    xsel = bf16_to_f64(x_all[sel])
    cache = {}

    def fn(e, rows):
        if e not in cache:
            cache.clear()
            cache[e] = tuple(bf16_to_f64(m) for m in ws_cpu[e])
        from oracle import ffn
        return ffn.swiglu(rows, *cache[e])[1]
    ref, ridx, _ = olayer.layer_direct(xsel, logits_all[sel].cpu().numpy(), k, fn)
    assert np.array_equal(gidx[sel], ridx)
    assert_close_layer(bf16_to_f64(out[sel]), ref)
    g.close()


RANDOM_CONFIGS = [  # (seed, G, tp, T, H, F, E, k): ragged token splits, uneven and empty ranks
    (1, 2, 1, 257, 64, 128, 4, 1),
    (2, 3, 1, 1031, 128, 256, 6, 2),
    (3, 4, 1, 90, 64, 128, 16, 4),
    (4, 4, 2, 777, 128, 256, 8, 2),
    (5, 6, 1, 2000, 64, 192, 12, 3),
    (6, 8, 1, 513, 64, 128, 64, 8),
    (7, 8, 2, 300, 64, 256, 32, 4),
    (8, 2, 2, 5, 64, 128, 8, 2),
]


@pytest.mark.parametrize("seed,G,tp,T,H,F,E,k", RANDOM_CONFIGS)
def test_group_random_configs_match_virtual(cuda_ok, seed, G, tp, T, H, F, E, k):
    """Seeded random shapes through the real P2P data plane of a single-process
    group on one GPU: a random placement over the G/tp EP groups (some hosting
    nothing), ragged token blocks (some ranks own none when T < G), both dispatch
    forms; the outputs equal the virtual-rank run bit-exactly and the oracle
    within tolerance (the TP oracle when tp > 1)."""
    moe = _moe()
    rng = np.random.default_rng(seed)
    n_grp = G // tp
    P = rng.integers(0, n_grp, E)
    inp = Inputs(T, H, F, E, k, s=float(rng.uniform(0.0, 1.8)), seed=100 + seed)
    g = Group(G, T, H, F, E, k, tp=tp)
    x_all, logits_all, xs, ls = _setup(inp, g, k)
    w1a, w3a, w2a = inp.device_weights(DEV, list(range(E)))
    ws = []
    for r in range(G):
        hosted = [e for e in range(E) if P[e] == r // tp]
        if not hosted:
            ws.append((None, None))
            continue
        sel = torch.tensor(hosted, device=DEV)
        if tp > 1:
            ws.append(moe.tp_slice_weights(w1a[sel], w3a[sel], w2a[sel], tp, r % tp))
        else:
            ws.append((moe.pack_w13(w1a[sel], w3a[sel]), w2a[sel].contiguous()))
    for lay in g.lays:
        lay.placement(P)
    torch.cuda.synchronize()
    virt = _virtual_out(inp, P, G, k, tp=tp)
    if tp == 1:
        ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
    else:
        ref, _, _, _ = olayer.layer_ep_tp(bf16_to_f64(inp.x), inp.logits.numpy(), k, P, n_grp, tp,
                                          inp.oracle_tp_fn(tp))
    for dispatch in ("scatter", "gather"):
        os.environ["MOE_DISPATCH"] = dispatch
        try:
            rw = g.each(lambda r, lay: lay.route(ls[r], k))
            g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
            g.each(lambda r, lay: lay.expert_ffn(*ws[r]))
            outs = g.each(lambda r, lay: lay.combine(rw[r][1]))
            g.sync()
        finally:
            os.environ.pop("MOE_DISPATCH", None)
        out = torch.cat(outs)
        assert torch.equal(out.view(torch.int16), virt.view(torch.int16)), dispatch
        assert_close_layer(bf16_to_f64(out), ref)
    g.close()


@pytest.mark.multigpu
@pytest.mark.parametrize("E,k,tp,fused", [(64, 8, 1, "1"), (8, 2, 2, "0"), (8, 2, 2, "1"), (16, 4, 1, "0"),
                                          (64, 8, 1, "ce"), (16, 4, 1, "ce")])
def test_group_eight_ranks_over_devices(cuda_ok, E, k, tp, fused, monkeypatch):
    """An 8-rank group over the box's GPUs (2 ranks per GPU on 4 GPUs, 4 on 2):
    8EP at E64 top-8 (D5's shape scaled down) and 4EP-2TP (the 8-GPU TP config),
    the P2P data plane crossing NVLink between devices and staying local between
    the ranks of one device; bit-exact with the 8-virtual-rank run, and the
    oracle within tolerance."""
    nd = torch.cuda.device_count()
    if nd < 2:
        pytest.skip("needs >= 2 GPUs")
    nd = 4 if nd >= 4 else 2
    if fused == "ce":                        # copy-engine data plane (256-row GEMM tiles)
        monkeypatch.setenv("MOE_A2A_CE", "1")
        monkeypatch.setenv("MOE_GEMM_CG", "2")
    else:
        monkeypatch.setenv("MOE_FUSED_COMBINE", fused)
    moe = _moe()
    G, T, H, F = 8, 3001, 256, 512
    n_grp = G // tp
    devs = [r * nd // G for r in range(G)]
    inp = Inputs(T, H, F, E, k, s=1.2, seed=77 + E + tp)
    P = np.array([(e * 5 + 3) % n_grp for e in range(E)])       # non-monotone, every group hosts experts
    blocks = oplan.token_blocks(T, G)
    tmax = max(b - a for a, b in blocks)
    lays = moe.MoeLayer.group(G, max_tokens=tmax, hidden=H, ffn=F, num_experts=E, max_k=k, devices=devs, tp=tp)
    streams = [torch.cuda.Stream(device=d) for d in devs]
    w1a, w3a, w2a = inp.device_weights("cpu", list(range(E)))
    xs, ls, ws = [], [], []
    for r, (a, b) in enumerate(blocks):
        d = torch.device("cuda", devs[r])
        xs.append(inp.x[a:b].contiguous().to(d))
        ls.append(inp.logits[a:b].contiguous().to(d))
        hosted = [e for e in range(E) if P[e] == r // tp]
        with torch.cuda.device(d):
            w1, w3, w2 = w1a[hosted].to(d), w3a[hosted].to(d), w2a[hosted].to(d)
            if tp > 1:
                ws.append(moe.tp_slice_weights(w1, w3, w2, tp, r % tp))
            else:
                ws.append((moe.pack_w13(w1, w3), w2.contiguous()))
            lays[r].placement(P)
    for d in range(nd):
        torch.cuda.synchronize(d)

    def each(fn):
        res = []
        for r, lay in enumerate(lays):
            with torch.cuda.device(devs[r]), torch.cuda.stream(streams[r]):
                res.append(fn(r, lay))
        return res

    for _ in range(2):                                   # the second pass reuses the buffers (epochs)
        rw = each(lambda r, lay: lay.route(ls[r], k))
        each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
        each(lambda r, lay: lay.expert_ffn(*ws[r]))
        outs = each(lambda r, lay: lay.combine(rw[r][1]))
        for lay in lays:
            lay.sync()
    out = torch.cat([o.cpu() for o in outs])
    virt = _virtual_out(inp, P, G, k, tp=tp).cpu()
    assert torch.equal(out.view(torch.int16), virt.view(torch.int16)), "8-rank group vs 8 virtual ranks"
    if tp == 1:
        ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
    else:
        ref, _, _, _ = olayer.layer_ep_tp(bf16_to_f64(inp.x), inp.logits.numpy(), k, P, n_grp, tp,
                                          inp.oracle_tp_fn(tp))
    assert_close_layer(bf16_to_f64(out), ref)
    for d in range(nd):
        torch.cuda.synchronize(d)
    for lay in lays:
        lay.close()


@pytest.mark.parametrize("seed,G,tp,T,H,F,E,k", [c for c in RANDOM_CONFIGS if c[2] == 1])
def test_group_copy_engine_data_plane(cuda_ok, seed, G, tp, T, H, F, E, k, monkeypatch):
    """MOE_A2A_CE=1: the peers' rows staged in send order and moved by the copy
    engines (one peer copy per (destination, expert) run, flags by stream memory
    writes), the expert outputs returned per segment as K6 finishes it (stream waits
    on K6's segment counters): bit-exact with the virtual-rank run, the identity
    round trip bit-exact, the received payload in the oracle's order."""
    monkeypatch.setenv("MOE_A2A_CE", "1")
    monkeypatch.setenv("MOE_GEMM_CG", "2")        # the copy-engine plane runs with 256-row tiles
    moe = _moe()
    rng = np.random.default_rng(seed)
    P = rng.integers(0, G, E)
    inp = Inputs(T, H, F, E, k, s=float(rng.uniform(0.0, 1.8)), seed=100 + seed)
    g = Group(G, T, H, F, E, k)
    x_all, logits_all, xs, ls = _setup(inp, g, k)
    ridx, _ = oroute.route(inp.logits.numpy(), k)
    xb = inp.x.view(torch.int16).numpy().view(np.uint16)
    w1a, w3a, w2a = inp.device_weights(DEV, list(range(E)))
    ws = []
    for r in range(G):
        hosted = [e for e in range(E) if P[e] == r]
        if hosted:
            sel = torch.tensor(hosted, device=DEV)
            ws.append((moe.pack_w13(w1a[sel], w3a[sel]), w2a[sel].contiguous()))
        else:
            ws.append((None, None))
    for lay in g.lays:
        lay.placement(P)
    torch.cuda.synchronize()
    pl = oplan.plan([ridx[a:b] for a, b in g.blocks], P, G)
    # identity round trip; the payload is read after the identity FFN (a single-process
    # group queues a rank's dispatch copies in its FFN call, see moe.h)
    rw = g.each(lambda r, lay: lay.route(ls[r], k))
    g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
    g.each(lambda r, lay: lay.identity_ffn())
    for r, lay in enumerate(g.lays):
        rows = lay.debug_recv()
        ref_rows = xb[[g.blocks[s][0] + t for (s, t, j, e) in pl["recv"][r]]].reshape(-1, H)
        assert np.array_equal(rows, ref_rows), f"received payload of rank {r}"
        # the staging buffer the copy engines read: a peer's row at its C3 send slot
        a, b = g.blocks[r]
        send = lay.debug_send()
        sl = pl["slot"][r]
        mine = ridx[a:b]
        remote = [(int(sl[t, j]), t) for t in range(b - a) for j in range(k) if P[mine[t, j]] != r]
        for slot, t in remote:
            assert np.array_equal(send[slot], xb[a + t]), f"staged row (rank {r}, slot {slot})"
    outs = g.each(lambda r, lay: lay.combine(rw[r][1]))
    g.sync()
    for r in range(G):
        assert torch.equal(outs[r].view(torch.int16), xs[r].view(torch.int16)), "identity round trip"
    virt = _virtual_out(inp, P, G, k)
    for rep in range(2):                     # the second layer reuses every buffer
        rw = g.each(lambda r, lay: lay.route(ls[r], k))
        g.each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
        g.each(lambda r, lay: lay.expert_ffn(*ws[r]))
        outs = g.each(lambda r, lay: lay.combine(rw[r][1]))
        g.sync()
        out = torch.cat(outs)
        assert torch.equal(out.view(torch.int16), virt.view(torch.int16)), f"copy-engine plane vs virtual ({rep})"
    g.close()
