#!/usr/bin/env python
"""NVLink bytes per phase of the EP layer from the GPU's NVLink counters (ncu).

    ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum \\
        -k regex:"k_scatter|k_grouped_gemm|k_combine" --csv \\
        python tools/nvlink_ncu.py --gpus 4 [--config mixtral] [--zipf-s 0] [--placement contiguous]

NVML's NVLink throughput fields return NOT_SUPPORTED on this pool's driver and
`nvidia-smi nvlink -gt d` prints N/A (profiles/r2_nvlink_probe.jsonl), so the
link counters are read through ncu.  ncu profiles one process, so the N EP
ranks run as a single-process group (moe_ctx_create_group) over N devices --
the same P2P data plane as N processes, with peer pointers instead of CUDA IPC.
Under ncu every kernel runs serialised, so a rank's in-kernel flag waits for
its peers time out (MOE_FLAG_TIMEOUT_MS is set low here): the layer's values
are not meaningful under the profiler, but every kernel moves the bytes it
moves in a real run -- k_scatter (peers' rows) is the dispatch, the fused K6
(k_grouped_gemm<..., FUSED>) or k_combine is the combine.  Without ncu the
script runs the layer normally and prints, per rank, the algorithmic bytes the
counters should show (remote routed rows x 2H per direction).
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from bench import CONFIGS, blocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--config", default="mixtral", choices=list(CONFIGS))
    ap.add_argument("--zipf-s", type=float, default=0.0)
    ap.add_argument("--placement", default="contiguous", choices=["contiguous", "balanced"])
    ap.add_argument("--layers", type=int, default=2)
    a = ap.parse_args()
    os.environ.setdefault("MOE_FLAG_TIMEOUT_MS", "200")
    from paper_2502_06643_b200 import moe, placement

    cfg = CONFIGS[a.config]
    E, k, H, F, T = cfg["E"], cfg["k"], cfg["H"], cfg["F"], cfg["T"]
    N = a.gpus
    bl = blocks(T, N)
    tmax = max(y - x for x, y in bl)
    lays = moe.MoeLayer.group(N, max_tokens=tmax, hidden=H, ffn=F, num_experts=E, max_k=k, devices=list(range(N)))
    devs = [torch.device("cuda", r) for r in range(N)]
    streams = [torch.cuda.Stream(device=d) for d in devs]
    logits_all = synth.zipf_logits(T, E, a.zipf_s, 0)
    if a.placement == "contiguous":
        P = moe.placement_contiguous(E, N)
    else:
        from oracle import route as oroute   # host-side load counts for the placement only
        ridx, _ = oroute.route(logits_all.numpy(), k)
        P = placement.balanced(np.bincount(ridx.ravel(), minlength=E), N).astype(np.int32)
    xs, ls, ws = [], [], []
    for r, (t0, t1) in enumerate(bl):
        with torch.cuda.device(devs[r]):
            xs.append(synth.hidden_states(T, H, 0, device=devs[r])[t0:t1].contiguous())
            ls.append(logits_all[t0:t1].to(devs[r]))
            hosted = [e for e in range(E) if P[e] == r]
            if hosted:
                q = [synth.expert_weights(e, H, F, 0, device=devs[r]) for e in hosted]
                w1, w3, w2 = (torch.stack([z[i] for z in q]) for i in range(3))
                ws.append((moe.pack_w13(w1, w3), w2))
            else:
                ws.append((None, None))
            lays[r].placement(P)
    for d in devs:
        torch.cuda.synchronize(d)

    def each(fn):
        out = []
        for r, lay in enumerate(lays):
            with torch.cuda.stream(streams[r]):
                out.append(fn(r, lay))
        return out

    infos = None
    for layer in range(a.layers):
        rw = each(lambda r, lay: lay.route(ls[r], k))
        each(lambda r, lay: lay.dispatch(xs[r], rw[r][0], P))
        each(lambda r, lay: lay.expert_ffn(*ws[r]))
        each(lambda r, lay: lay.combine(rw[r][1]))
        for d in devs:
            torch.cuda.synchronize(d)
    # the split sizes of this routing (host counts, for the algorithmic bytes)
    from oracle import plan as oplan, route as oroute
    ridx, _ = oroute.route(logits_all.numpy(), k)
    pl = oplan.plan([ridx[x:y] for x, y in bl], P, N)
    sc = np.array(pl["send_counts"])          # [source][dest]
    res = {"config": a.config, "gpus": N, "zipf_s": a.zipf_s, "placement": [int(v) for v in P],
           "note": "algorithmic NVLink bytes per rank: dispatch out = rows this rank sends to peers x 2H; "
                   "combine returns the same rows", "ranks": []}
    for r in range(N):
        out_rows = int(sc[r].sum() - sc[r][r])
        in_rows = int(sc[:, r].sum() - sc[r][r])
        res["ranks"].append({"rank": r, "dispatch_tx_bytes": out_rows * 2 * H, "dispatch_rx_bytes": in_rows * 2 * H})
    print(json.dumps(res), flush=True)
    for lay in lays:
        try:
            lay.sync()
        except moe.MoeError as ex:        # flag timeouts under the profiler (see the docstring)
            print(f"rank sync: {ex}", file=sys.stderr)
        lay.close()


if __name__ == "__main__":
    main()
