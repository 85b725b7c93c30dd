"""Small-T (decode-regime) latency of one MoE layer: the
full hot path (route, stats, dispatch, expert FFN, combine) on the Mixtral
layer shapes for a sweep of token counts, launched eagerly and as a replayed
CUDA graph.  At N = 1 nothing on the path needs the host; at N > 1 (torchrun,
P2P all-to-all, T tokens in total split over the ranks, contiguous placement)
the P2P flags carry a device-side epoch, so the captured layer replays with
fresh flags.  Latency = max over ranks.  Prints one JSON line per T (rank 0).

    python tools/small_t_latency.py [--tokens 16,64,256,1024,4096] [--reps 200]
    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        tools/small_t_latency.py --tokens 64,256
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
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", 0))
    N = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)

    def fresh_uid():  # one NCCL unique id per context
        if N == 1:
            return None
        u = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            u.copy_(torch.frombuffer(bytearray(moe.get_unique_id()), dtype=torch.uint8))
        dist.broadcast(u, 0)
        return bytes(u.cpu().numpy().tobytes())
    H, F, E, k = a.H, a.F, a.E, a.k
    Ts = [int(t) for t in a.tokens.split(",")]
    Tmax = max(Ts)
    P = moe.placement_contiguous(E, N)
    hosted = [e for e in range(E) if P[e] == rank]
    ws = [synth.expert_weights(e, H, F, 0, device=dev) for e in hosted]
    w13 = moe.pack_w13(torch.stack([q[0] for q in ws]), torch.stack([q[1] for q in ws]))
    w2 = torch.stack([q[2] for q in ws])
    del ws
    for T in Ts:
        # one context per batch size: contexts whose worst case averages <= 256 rows
        # per expert use 128-row GEMM tiles on one CTA (see moe_ctx_create)
        t0, t1 = rank * T // N, (rank + 1) * T // N
        Tr = t1 - t0
        lay = moe.MoeLayer(max_tokens=max(T // N + 1, 1), hidden=H, ffn=F, num_experts=E, max_k=k, world=N,
                           rank=rank, device=local, uid=fresh_uid(), a2a="p2p" if N > 1 else "nccl")
        x = synth.hidden_states(T, H, 1, device=dev)[t0:t1].contiguous()
        logits = synth.zipf_logits(T, E, 1.6, 1, device=dev)[t0:t1].contiguous()
        prev = synth.zipf_logits(T, E, 1.6, 2, device=dev)[t0:t1].contiguous()
        idx_prev, _ = lay.route(prev, k)
        idx = torch.empty(Tr, k, dtype=torch.int32, device=dev)
        w = torch.empty(Tr, k, dtype=torch.float32, device=dev)
        out = torch.empty(Tr, H, dtype=torch.bfloat16, device=dev)
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
            if N > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / a.reps], dtype=torch.float64, device=dev)
            if N > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t[0])

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
        same = torch.tensor([int(torch.equal(out.view(torch.int16), ref.view(torch.int16)))], device=dev)
        # weight bytes of the experts used must be read at least once (the small-T roofline)
        used_mask = torch.zeros(E, dtype=torch.int32, device=dev)
        used_mask[torch.unique(idx).long()] = 1
        if N > 1:
            dist.all_reduce(same, op=dist.ReduceOp.MIN)
            dist.all_reduce(used_mask, op=dist.ReduceOp.MAX)
        used = int(used_mask.sum())
        wbytes_used = used * 3 * H * F * 2
        if rank == 0:
            print(json.dumps({"tokens": T, "gpus": N, "a2a": "p2p" if N > 1 else "none",
                              "gemm_tile_rows": 128 if (T // N + 1) * N * k <= 256 * E else 256,
                              "eager_ms": eager, "graph_ms": graph, "graph_matches_eager": bool(same[0]),
                              "experts_used": used, "weights_GB": wbytes_used / 1e9,
                              "weight_read_GBps_graph": wbytes_used / (graph * 1e-3) / 1e9}), flush=True)
        del g
        lay.close()
    del Tmax
    if N > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
