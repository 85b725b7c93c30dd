#!/usr/bin/env python
"""Direct l -> l+1 dispatch over real ranks: a short chain with per-layer
timelines and error checks (a debugging aid for NEXT-4, not a benchmark).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/direct_diag.py [--layers 3] [--tokens 16384]
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
from bench import blocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    a = ap.parse_args()
    from paper_2502_06643_b200 import moe
    E, k, H, F, T, L = 8, 2, a.hidden, a.ffn, a.tokens, a.layers
    rank = int(os.environ.get("RANK", 0))
    N = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)

    def uid():
        u = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            u.copy_(torch.frombuffer(bytearray(moe.get_unique_id()), dtype=torch.uint8))
        dist.broadcast(u, 0)
        return bytes(u.cpu().numpy().tobytes())

    t0, t1 = blocks(T, N)[rank]
    tmax = max(y - x for x, y in blocks(T, N))
    cs = [moe.MoeLayer(max_tokens=tmax, hidden=H, ffn=F, num_experts=E, max_k=k, world=N, rank=rank, device=local,
                       uid=uid(), a2a="p2p") for _ in range(2)]
    x = synth.hidden_states(T, H, 0, device=dev)[t0:t1].contiguous()
    lg = [synth.zipf_logits(T, E, 1.6, 10 + li, device=dev)[t0:t1].contiguous() for li in range(L)]
    P = np.array([e * N // E for e in range(E)], dtype=np.int32)
    hosted = [e for e in range(E) if P[e] == rank]
    q = [synth.expert_weights(e, H, F, 0, device=dev) for e in hosted]
    w1, w3, w2 = (torch.stack([z[i] for z in q]) for i in range(3))
    w13 = moe.pack_w13(w1, w3)
    for c in cs:
        c.placement(P)
        c.timeline(L)
    torch.cuda.synchronize()
    dist.barrier()
    prev = None
    for li in range(L):
        c = cs[li % 2]
        idx, w = c.route(lg[li], k)
        if prev is None:
            c.dispatch(x, idx, P)
        else:
            c.dispatch_from(prev[0], prev[1], idx, P)
        c.output_mode("home" if li == L - 1 else "stay")
        c.expert_ffn(w13, w2)
        prev = (c, w)
    out = prev[0].combine(prev[1])
    errs = []
    for c in cs:
        try:
            c.sync()
        except moe.MoeError as ex:
            errs.append(str(ex))
    tl = [c.timeline_read() for c in cs]
    print(json.dumps({"rank": rank, "errors": errs, "timeline_ctx0": tl[0], "timeline_ctx1": tl[1],
                      "out_finite": bool(torch.isfinite(out.float()).all())}), flush=True)
    for c in cs:
        c.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
