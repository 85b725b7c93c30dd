"""Small-T (decode-regime) latency of one MoE layer on one GPU (SURVEY §8(f)
NEXT-3): the full hot path (route, stats, dispatch, expert FFN, combine) on
the Mixtral layer shapes for a sweep of token counts, launched eagerly and as
a replayed CUDA graph (no host round trips on this path at N = 1, so the whole
layer captures).  Prints one JSON line per T.

    python tools/small_t_latency.py [--tokens 16,64,256,1024,4096] [--reps 200]
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="16,64,256,1024,4096")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--F", type=int, default=14336)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    a = ap.parse_args()
    from paper_2502_06643_b200 import moe
    dev = torch.device("cuda", 0)
    H, F, E, k = a.H, a.F, a.E, a.k
    Ts = [int(t) for t in a.tokens.split(",")]
    Tmax = max(Ts)
    ws = [synth.expert_weights(e, H, F, 0, device=dev) for e in range(E)]
    w13 = moe.pack_w13(torch.stack([q[0] for q in ws]), torch.stack([q[1] for q in ws]))
    w2 = torch.stack([q[2] for q in ws])
    del ws
    P = [0] * E
    for T in Ts:
        # one context per batch size: contexts whose worst case averages <= 256 rows
        # per expert use 128-row GEMM tiles on one CTA (see moe_ctx_create)
        lay = moe.MoeLayer(max_tokens=T, hidden=H, ffn=F, num_experts=E, max_k=k)
        x = synth.hidden_states(T, H, 1, device=dev)
        logits = synth.zipf_logits(T, E, 1.6, 1, device=dev)
        prev = synth.zipf_logits(T, E, 1.6, 2, device=dev)
        idx_prev, _ = lay.route(prev, k)
        idx = torch.empty(T, k, dtype=torch.int32, device=dev)
        w = torch.empty(T, k, dtype=torch.float32, device=dev)
        out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
        load = torch.zeros(E, dtype=torch.int64, device=dev)
        coact = torch.zeros(E, E, dtype=torch.int64, device=dev)

        def step():
            lay.route(logits, k, idx, w)
            lay.route_stats(idx_prev, idx, load, coact)
            lay.dispatch(x, idx, P)
            lay.expert_ffn(w13, w2)
            lay.combine(w, out)

        def timeit(fn):
            for _ in range(10):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / a.reps

        eager = timeit(step)
        ref = out.clone()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            step()
        graph = timeit(g.replay)
        same = bool(torch.equal(out.view(torch.int16), ref.view(torch.int16)))
        # weight bytes of the experts used must be read at least once (the small-T roofline)
        used = int(torch.unique(idx).numel())
        wbytes_used = used * 3 * H * F * 2
        print(json.dumps({"tokens": T, "gemm_tile_rows": 128 if T * k <= 256 * E else 256,
                          "eager_ms": eager, "graph_ms": graph, "graph_matches_eager": same,
                          "experts_used": used, "weights_GB": wbytes_used / 1e9,
                          "weight_read_GBps_graph": wbytes_used / (graph * 1e-3) / 1e9}), flush=True)
        del g
        lay.close()
    del Tmax


if __name__ == "__main__":
    main()
