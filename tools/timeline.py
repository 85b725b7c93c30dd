#!/usr/bin/env python
"""Per-rank layer timeline (moe_timeline_*): where a step's time goes.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/timeline.py --config e64 --placement balanced [--tp T] [--steps 20]

Prints, per rank, the median over steps of each event's time after dispatch
entry (dispatch, layout, scatter_local, scatter_peers, ffn, k5, k6, combine) as
one JSON line per rank.  A profiling tool, not a benchmark.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from bench import CONFIGS, blocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="e64", choices=list(CONFIGS))
    ap.add_argument("--placement", default="balanced", choices=["contiguous", "balanced"])
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--a2a", default="p2p")
    ap.add_argument("--tokens", type=int, default=0, help="override the config's total token count")
    a = ap.parse_args()
    from paper_2502_06643_b200 import moe, placement

    cfg = CONFIGS[a.config]
    E, k, H, F, T = cfg["E"], cfg["k"], cfg["H"], cfg["F"], cfg["T"]
    T = a.tokens or T
    rank = int(os.environ.get("RANK", 0))
    N = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
        u = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            u.copy_(torch.frombuffer(bytearray(moe.get_unique_id()), dtype=torch.uint8))
        dist.broadcast(u, 0)
        uid = bytes(u.cpu().numpy().tobytes())
    tp = a.tp
    G = N // tp
    t0, t1 = blocks(T, N)[rank]
    Tmax = max(y - x for x, y in blocks(T, N))
    lay = moe.MoeLayer(max_tokens=max(Tmax, 1), hidden=H, ffn=F, num_experts=E, max_k=k, world=N, rank=rank,
                       device=local, uid=uid, a2a=a.a2a, tp=tp)
    x = synth.hidden_states(T, H, 0, device=dev)[t0:t1].contiguous()
    logits = synth.zipf_logits(T, E, 1.6, 0, device=dev)[t0:t1].contiguous()
    idx, w = lay.route(logits, k)
    if a.placement == "contiguous":
        P = moe.placement_contiguous(E, G)
    else:
        load = torch.zeros(E, dtype=torch.int64, device=dev)
        lay.route_stats(idx, None, load, None)
        lay.stats_allreduce(load, None)
        lay.sync()
        P = placement.balanced(load.cpu().numpy(), G).astype(np.int32)
    hosted = [e for e in range(E) if P[e] == rank // tp]
    w13 = w2 = None
    if hosted:
        ws = [synth.expert_weights(e, H, F, 0, device=dev) for e in hosted]
        w1, w3, w2 = (torch.stack([q[i] for q in ws]) for i in range(3))
        del ws
        if tp > 1:
            w13, w2 = moe.tp_slice_weights(w1, w3, w2, tp, rank % tp)
        else:
            w13 = moe.pack_w13(w1, w3)
        del w1, w3
    out = torch.empty(t1 - t0, H, dtype=torch.bfloat16, device=dev)

    def step():
        lay.route(logits, k, idx, w)
        lay.dispatch(x, idx, P)
        lay.expert_ffn(w13, w2)
        lay.combine(w, out)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    lay.timeline(a.steps)
    if N > 1:
        dist.barrier()
    for _ in range(a.steps):
        step()
    rec = np.array(lay.timeline_read())
    med = np.median(rec, axis=0)
    err = None
    try:
        lay.sync()
    except moe.MoeError as ex:      # e.g. a P2P flag timeout: report it with the timeline
        err = str(ex)
    print(json.dumps({"rank": rank, "error": err, "config": a.config, "tokens": T, "placement": a.placement, "tp": tp,
                      "env": {kk: v for kk, v in os.environ.items() if kk.startswith("MOE_")},
                      "median_ms": dict(zip(moe.MoeLayer.TIMELINE, [round(float(v), 4) for v in med]))}),
          flush=True)
    lay.close()
    if N > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
