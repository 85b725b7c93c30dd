"""Worker for tests/test_multigpu.py (launched with torch.distributed.run, one
process per GPU).  Runs the EP layer over real ranks with NCCL and checks, on
every rank:
  * the plan (dest rank, receive position, send slot, count matrix) is
    bit-exact with the oracle's C3 plan for this source rank;
  * the received payload is bit-identical to the oracle's receive order;
  * the identity-expert round trip returns x bit-exactly;
  * the layer output equals the single-GPU virtual-rank run bit-exactly
    (cross-mode equality) and is within tolerance of the oracle.
Prints "RANK <r> OK" on success.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import layer as olayer  # noqa: E402
from oracle import plan as oplan  # noqa: E402
from oracle import route as oroute  # noqa: E402
from tests._util import Inputs, assert_close_layer, bf16_to_f64  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2502_06643_b200 import moe

    uid = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(moe.get_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    uid = bytes(uid.cpu().numpy().tobytes())

    T, H, F, E, k = 1500, 256, 512, 8, 2
    inp = Inputs(T, H, F, E, k, s=1.6, seed=21)
    blocks = oplan.token_blocks(T, world)
    a, b = blocks[rank]
    Tmax = max(y - x for x, y in blocks)
    lay = moe.MoeLayer(max_tokens=Tmax, hidden=H, ffn=F, num_experts=E, max_k=k, world=world, rank=rank,
                       device=local, uid=uid, a2a=os.environ.get("MOE_TEST_A2A", "nccl"))
    ridx, _ = oroute.route(inp.logits.numpy(), k)
    placements = [np.array([e * world // E for e in range(E)])]
    bal = np.array([0, 1, 2, 2, 3, 2, 3, 3]) % world
    placements.append(bal)
    if world >= 2:
        placements.append(np.array([world - 1] * 6 + [0, 0]))      # ranks 1..w-2 host nothing
    x_all, logits_all = inp.to_device(dev)
    x = x_all[a:b].contiguous()
    logits = logits_all[a:b].contiguous()
    virt_out = None
    for P in placements:
        idx, w = lay.route(logits, k)
        lay.dispatch(x, idx, P)
        dr, rp, ss, cnt = lay.debug_plan()
        pl = oplan.plan([ridx[x0:y0] for x0, y0 in blocks], P, world)
        assert np.array_equal(cnt, pl["cnt"]), "count matrix"
        assert np.array_equal(ss, pl["slot"][rank]), "send slots"
        assert np.array_equal(rp, pl["recv_pos"][rank]), "receive positions"
        assert np.array_equal(dr, P[ridx[a:b]]), "destination ranks"
        xb = inp.x.view(torch.int16).numpy().view(np.uint16)
        if lay.a2a == "nccl":
            # the device's compact send buffer, row by row, in the oracle's C3 send
            # order (G9) restricted to remote destinations
            sl = pl["slot"][rank]
            mine = ridx[a:b]
            items = sorted(((int(sl[t, j]), t) for t in range(b - a) for j in range(k)
                            if P[mine[t, j]] != rank))
            ref_send = xb[[a + t for _, t in items]].reshape(-1, H)
            assert np.array_equal(lay.debug_send(), ref_send), "send buffer order"
        elif os.environ.get("MOE_A2A_CE") == "1":
            # copy-engine plane: the staging buffer holds every remote row at its C3 slot
            sl = pl["slot"][rank]
            mine = ridx[a:b]
            send = lay.debug_send()
            for t in range(b - a):
                for j in range(k):
                    if P[mine[t, j]] != rank:
                        assert np.array_equal(send[int(sl[t, j])], xb[a + t]), "staged send row"
        rows = lay.debug_recv()
        ref_rows = xb[[blocks[s][0] + t for (s, t, j, e) in pl["recv"][rank]]].reshape(-1, H)
        assert np.array_equal(rows, ref_rows), "received payload"
        lay.identity_ffn()
        out = lay.combine(w)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), x.view(torch.int16)), "identity round trip"
        # real expert FFN
        hosted = [e for e in range(E) if P[e] == rank]
        lay.dispatch(x, idx, P)
        if hosted:
            w1, w3, w2 = inp.device_weights(dev, hosted)
            lay.expert_ffn(moe.pack_w13(w1, w3), w2)
        else:
            lay.expert_ffn(None, None)      # collective: a rank hosting no expert still calls it
        out = lay.combine(w)
        lay.sync()
        if virt_out is None:
            # single-GPU virtual-rank run of the same layer (all tokens), for cross-mode equality
            vl = moe.MoeLayer(max_tokens=T, hidden=H, ffn=F, num_experts=E, max_k=k, virtual_ranks=world,
                              device=local)
            vi, vw = vl.route(logits_all, k)
            vl.dispatch(x_all, vi, P)
            w1, w3, w2 = inp.device_weights(dev, list(range(E)))
            vl.expert_ffn(moe.pack_w13(w1, w3), w2)
            virt_out = vl.combine(vw)
            vl.sync()
            vl.close()
            ref, _, _ = olayer.layer_direct(bf16_to_f64(inp.x), inp.logits.numpy(), k, inp.oracle_expert_fn())
        assert torch.equal(out.view(torch.int16), virt_out[a:b].view(torch.int16)), "cross-mode equality"
        assert_close_layer(bf16_to_f64(out), ref[a:b])
    # statistics all-reduce: sum of per-rank loads equals the global load
    load = torch.zeros(E, dtype=torch.int64, device=dev)
    idx, _ = lay.route(logits, k)
    lay.route_stats(idx, None, load, None)
    lay.stats_allreduce(load, None)
    lay.sync()
    assert np.array_equal(load.cpu().numpy(), np.bincount(ridx.ravel(), minlength=E))
    # a multi-layer pass in one collective: per-layer loads and layer-pair co-activation
    L3 = 3
    loads = torch.zeros(L3, E, dtype=torch.int64, device=dev)
    coacts = torch.zeros(L3 - 1, E, E, dtype=torch.int64, device=dev)
    lg = [logits, logits.flip(1).contiguous(), logits.roll(1, 1).contiguous()]
    ids = [lay.route(q, k)[0] for q in lg]
    for li in range(L3):
        lay.route_stats(ids[li], ids[li + 1] if li + 1 < L3 else None, loads[li],
                        coacts[li] if li + 1 < L3 else None)
    lay.stats_allreduce_layers(loads, coacts)
    lay.sync()
    lga = [inp.logits.numpy(), inp.logits.numpy()[:, ::-1].copy(), np.roll(inp.logits.numpy(), 1, 1)]
    rids = [oroute.route(q, k)[0] for q in lga]
    from oracle import stats as ostats
    for li in range(L3):
        assert np.array_equal(loads[li].cpu().numpy(), ostats.load_counts(rids[li], E)), "multi-layer load"
        if li + 1 < L3:
            assert np.array_equal(coacts[li].cpu().numpy(), ostats.coactivation_counts(rids[li], rids[li + 1], E)), \
                "multi-layer co-activation"

    # CUDA-graph capture of a P2P layer: the flags carry a device-side epoch, so
    # replays of the captured layer match the eager result bit-exactly
    if lay.a2a == "p2p":
        P = placements[1]
        hosted = [e for e in range(E) if P[e] == rank]
        w1, w3, w2 = inp.device_weights(dev, hosted) if hosted else (None, None, None)
        w13 = moe.pack_w13(w1, w3) if hosted else None
        idx = torch.empty(b - a, k, dtype=torch.int32, device=dev)
        w = torch.empty(b - a, k, dtype=torch.float32, device=dev)
        out = torch.empty(b - a, H, dtype=torch.bfloat16, device=dev)

        def layer_step():
            lay.route(logits, k, idx, w)
            lay.dispatch(x, idx, P)
            lay.expert_ffn(w13, w2)
            lay.combine(w, out)

        layer_step()
        lay.sync()
        ref = out.clone()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            layer_step()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            layer_step()
        for _ in range(3):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out.view(torch.int16), ref.view(torch.int16)), "graph replay"
        lay.sync()
        del g

    # degenerate split: fewer tokens than ranks, so some ranks own 0 tokens (G7)
    # but still take part in every collective call; repeated layers reuse the
    # buffers (P2P epochs advance)
    Ts = world // 2
    sb = oplan.token_blocks(Ts, world)
    a2, b2 = sb[rank]
    xs = x_all[:Ts][a2:b2].contiguous()
    ls = logits_all[:Ts][a2:b2].contiguous()
    P = placements[0]
    hosted = [e for e in range(E) if P[e] == rank]
    w1, w3, w2 = inp.device_weights(dev, hosted) if hosted else (None, None, None)
    w13 = moe.pack_w13(w1, w3) if hosted else None
    for rep in range(3):
        idx, w = lay.route(ls, k)
        lay.dispatch(xs, idx, P)
        lay.expert_ffn(w13, w2)
        out = lay.combine(w)
        lay.sync()
        assert out.shape == (b2 - a2, H)
        if b2 > a2:
            assert torch.equal(out.view(torch.int16), virt_out[a2:b2].view(torch.int16)), "small-T equality"
    # call discipline: ranks passing different placements to one dispatch are caught
    # (P2P: the placement hash travels with the counts and is checked on the device;
    # NCCL: it is all-gathered with the counts and checked on the host)
    bad = np.array([e * world // E for e in range(E)])
    if rank == world - 1:
        bad = bad[::-1].copy()
    idx, w = lay.route(ls, k) if b2 > a2 else lay.route(logits[:0], k)
    try:
        lay.dispatch(xs if b2 > a2 else x[:0], idx, bad)
        lay.sync()
        raise AssertionError("placement mismatch not detected")
    except moe.MoeError as ex:
        assert "different expert_to_rank" in str(ex), str(ex)
    lay.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"RANK {rank} OK", flush=True)


if __name__ == "__main__":
    main()
