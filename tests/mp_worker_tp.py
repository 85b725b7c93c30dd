"""Worker for tests/test_multigpu.py::test_tp_over_real_ranks (one process per
GPU, torch.distributed.run): tensor parallelism inside the experts over real
ranks (reading G20; the paper's EP x TP layout) with the
P2P transport.  W = WORLD_SIZE ranks form G = W / tp EP groups.  Checks on
every rank:
  * the plan (count matrix over the W sources, send slots, receive positions,
    destination groups) is bit-exact with the oracle's C3 plan;
  * the received payload equals the oracle's receive order of this rank's group
    (every TP rank of a group holds the same rows);
  * the identity-expert round trip returns x bit-exactly;
  * the layer output equals the single-GPU virtual-rank TP run bit-exactly and
    is within tolerance of oracle.layer.layer_ep_tp;
  * ranks owning zero tokens still take part (repeated layers).
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
    tp = int(os.environ.get("MOE_TEST_TP", "2"))
    G = world // tp
    grp, q = rank // tp, rank % tp
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
    inp = Inputs(T, H, F, E, k, s=1.6, seed=31)
    blocks = oplan.token_blocks(T, world)
    a, b = blocks[rank]
    Tmax = max(y - x for x, y in blocks)
    lay = moe.MoeLayer(max_tokens=Tmax, hidden=H, ffn=F, num_experts=E, max_k=k, world=world, rank=rank,
                       device=local, uid=uid, a2a="p2p", tp=tp)
    ridx, _ = oroute.route(inp.logits.numpy(), k)
    placements = [np.array([e * G // E for e in range(E)]), np.array([0, 1, 1, 1, 0, 1, 0, 1]) % G]
    if G >= 2:
        placements.append(np.array([G - 1] * 8))              # groups 0..G-2 host nothing
    x_all, logits_all = inp.to_device(dev)
    x = x_all[a:b].contiguous()
    logits = logits_all[a:b].contiguous()
    w1a, w3a, w2a = inp.device_weights(dev, list(range(E)))
    for P in placements:
        idx, w = lay.route(logits, k)
        lay.dispatch(x, idx, P)
        dr, rp, ss, cnt = lay.debug_plan()
        pl = oplan.plan([ridx[x0:y0] for x0, y0 in blocks], P, G)
        assert np.array_equal(cnt, pl["cnt"]), "count matrix"
        assert np.array_equal(ss, pl["slot"][rank]), "send slots"
        assert np.array_equal(rp, pl["recv_pos"][rank]), "receive positions"
        assert np.array_equal(dr, P[ridx[a:b]]), "destination groups"
        rows = lay.debug_recv()
        xb = inp.x.view(torch.int16).numpy().view(np.uint16)
        ref_rows = xb[[blocks[s][0] + t for (s, t, j, e) in pl["recv"][grp]]].reshape(-1, H)
        assert np.array_equal(rows, ref_rows), "received payload"
        lay.identity_ffn()
        out = lay.combine(w)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), x.view(torch.int16)), "identity round trip"
        # real expert FFN on this rank's FFN slice of its group's experts
        hosted = [e for e in range(E) if P[e] == grp]
        lay.dispatch(x, idx, P)
        if hosted:
            sel = torch.tensor(hosted, device=dev)
            w13q, w2q = moe.tp_slice_weights(w1a[sel], w3a[sel], w2a[sel], tp, q)
            lay.expert_ffn(w13q, w2q)
        else:
            lay.expert_ffn(None, None)
        out = lay.combine(w)
        lay.sync()
        # single-GPU virtual-rank run of the same TP layer (all tokens)
        vl = moe.MoeLayer(max_tokens=T, hidden=H, ffn=F, num_experts=E, max_k=k, virtual_ranks=world,
                          device=local, tp=tp)
        vi, vw = vl.route(logits_all, k)
        vl.dispatch(x_all, vi, P)
        vl.expert_ffn(moe.pack_w13(w1a, w3a), w2a)
        virt_out = vl.combine(vw)
        vl.sync()
        vl.close()
        assert torch.equal(out.view(torch.int16), virt_out[a:b].view(torch.int16)), "cross-mode equality"
        ref, _, _, _ = olayer.layer_ep_tp(bf16_to_f64(inp.x), inp.logits.numpy(), k, P, G, tp,
                                          inp.oracle_tp_fn(tp))
        assert_close_layer(bf16_to_f64(out), ref[a:b])

    # fewer tokens than ranks: some ranks own 0 tokens; repeated layers (epochs advance)
    Ts = world // 2
    sb = oplan.token_blocks(Ts, world)
    a2, b2 = sb[rank]
    xs = x_all[:Ts][a2:b2].contiguous()
    ls = logits_all[:Ts][a2:b2].contiguous()
    P = placements[0]
    hosted = [e for e in range(E) if P[e] == grp]
    sel = torch.tensor(hosted, device=dev)
    w13q, w2q = moe.tp_slice_weights(w1a[sel], w3a[sel], w2a[sel], tp, q) if hosted else (None, None)
    for rep in range(3):
        idx, w = lay.route(ls, k)
        lay.dispatch(xs, idx, P)
        lay.expert_ffn(w13q, w2q)
        out = lay.combine(w)
        lay.sync()
        assert out.shape == (b2 - a2, H)
    lay.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"RANK {rank} OK", flush=True)


if __name__ == "__main__":
    main()
