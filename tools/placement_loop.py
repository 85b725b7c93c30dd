#!/usr/bin/env python
"""The paper's profile -> place -> serve loop on the GPU path.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/placement_loop.py [--config mixtral] [--layers 32] [--reps 3] [--graph] [--direct]

1. Profile: route L layers of synthetic multi-layer
   logits (synth.multilayer_logits: per-layer Zipf skew with layer-to-layer
   dependency) and collect P_{e,l} (load) and R_{e1,e2,l} (co-activation) with
   moe_route_stats, summed over ranks with moe_stats_allreduce.
2. Place on the host: ILP 1 per layer (placement.balanced, Eqs. 1-7) and ILP 2
   over the layers (placement.ilp2_dp, Eqs. 8-15 without Eq. 13, whose slack
   is reported), from the GPU-collected statistics.
3. Serve: run the L-layer MoE chain (each layer's output is the next layer's
   input) through moe_route / moe_dispatch / moe_expert_ffn / moe_combine with
   (a) contiguous placement, (b) ILP 1 (cluster c on GPU c), (c) ILP 1 + ILP 2,
   timed on the device (max over ranks).  Every layer's placement is its own
   device array (moe_dispatch reads it on the device), so a chain with per-layer
   placements runs without host synchronisation; --graph captures each plan's
   whole chain in one CUDA graph per rank, checks that the replay is
   bit-identical to the eager chain and times the replays.

In home-rank EP (reading G11) tokens return to their source after every layer,
so ILP 2's objective (inter-layer GPU-pair traffic, Eq. 8) is reported from the
measured R rather than realised as traffic; ILP 1's balance is what moves the
layer time.  --direct also runs every plan as a direct l -> l+1 chain (NEXT-4:
MOE_OUT_STAY + moe_dispatch_from, two contexts alternating): layer l+1's rows
are combined on the ranks hosting its experts from layer l's outputs where they
were computed, so Eq. 8's inter-layer traffic is what crosses NVLink and ILP 2's
co-location shows up in the layer time.  The direct chain's output is checked
bit-identical to the home chain's.  Prints one JSON line (rank 0).  Expert weights are shared by all
layers (synthetic); each layer's placement selects which of them a rank holds.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from bench import CONFIGS, blocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral", choices=list(CONFIGS))
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--zipf-s", type=float, default=1.6)
    ap.add_argument("--dependency", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--graph", action="store_true", help="capture each chain in a CUDA graph and time the replays")
    ap.add_argument("--direct", action="store_true", help="also time direct l -> l+1 dispatch chains (NEXT-4)")
    ap.add_argument("--save-json", default=None, help="write the ILP 1 + ILP 2 placement (SPEC's placement JSON)")
    a = ap.parse_args()
    from paper_2502_06643_b200 import moe, placement

    cfg = CONFIGS[a.config]
    E, k, H, F, T = cfg["E"], cfg["k"], cfg["H"], cfg["F"], cfg["T"]
    L = a.layers
    rank = int(os.environ.get("RANK", 0))
    N = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    def fresh_uid():
        """A new NCCL unique id for each context (one communicator per context)."""
        if N == 1:
            return None
        u = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            u.copy_(torch.frombuffer(bytearray(moe.get_unique_id()), dtype=torch.uint8))
        dist.broadcast(u, 0)
        return bytes(u.cpu().numpy().tobytes())

    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    uid = fresh_uid()
    t0, t1 = blocks(T, N)[rank]
    Tmax = max(y - x for x, y in blocks(T, N))
    lay = moe.MoeLayer(max_tokens=max(Tmax, 1), hidden=H, ffn=F, num_experts=E, max_k=k, world=N, rank=rank,
                       device=local, uid=uid, a2a="p2p" if N > 1 else "nccl")

    # ---- 1. profile on the GPU
    logits = [q[t0:t1].contiguous() for q in
              synth.multilayer_logits(L, T, E, a.zipf_s, a.seed, dependency=a.dependency, device=dev)]
    idx = [torch.empty(t1 - t0, k, dtype=torch.int32, device=dev) for _ in range(L)]
    w = [torch.empty(t1 - t0, k, dtype=torch.float32, device=dev) for _ in range(L)]
    load = torch.zeros(L, E, dtype=torch.int64, device=dev)
    coact = torch.zeros(max(L - 1, 1), E, E, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    for li in range(L):
        lay.route(logits[li], k, idx[li], w[li])
        if li:
            lay.route_stats(idx[li - 1], idx[li], load[li - 1], coact[li - 1])
    lay.route_stats(idx[L - 1], None, load[L - 1], None)
    for li in range(L):
        lay.stats_allreduce(load[li], coact[li] if li < L - 1 else None)
    p1.record()
    lay.sync()
    profile_ms = p0.elapsed_time(p1)
    load_h = load.cpu().numpy()
    coact_h = coact.cpu().numpy()[:L - 1]

    # ---- 2. place on the host
    th = time.perf_counter()
    G = N
    contig = np.stack([placement.contiguous(E, G)] * L)
    ilp1 = np.stack([placement.balanced(load_h[li], G) for li in range(L)]).astype(np.int32)
    C1 = placement.comm_costs(coact_h, ilp1, G)
    goc_id = np.stack([np.arange(G)] * L)
    goc = placement.ilp2_dp(C1, G, L) if G > 1 else goc_id
    ilp12 = placement.expert_to_gpu(ilp1, goc)
    host_s = time.perf_counter() - th
    Cc = placement.comm_costs(coact_h, contig, G)
    plans = {"contiguous": contig, "ilp1": ilp1, "ilp1+ilp2": ilp12}
    if a.save_json and rank == 0:
        with open(a.save_json, "w") as f:
            f.write(placement.to_json(ilp12, goc, objective=placement.objective_o2(C1, goc)))
    o2 = {"contiguous": placement.objective_o2(Cc, goc_id), "ilp1": placement.objective_o2(C1, goc_id),
          "ilp1+ilp2": placement.objective_o2(C1, goc)}

    # ---- 3. serve the L-layer chain
    wcache = {}

    def weights_for(hosted):
        key = tuple(hosted)
        if key not in wcache:
            if not hosted:
                wcache[key] = (None, None)
            else:
                ws = [synth.expert_weights(e, H, F, a.seed, device=dev) for e in hosted]
                w1, w3, w2 = (torch.stack([q[i] for q in ws]) for i in range(3))
                wcache[key] = (moe.pack_w13(w1, w3), w2)
                del ws, w1, w3
        return wcache[key]

    x0 = synth.hidden_states(T, H, a.seed, device=dev)[t0:t1].contiguous()
    bufs = [torch.empty_like(x0), torch.empty_like(x0)]
    wls = {name: [weights_for([e for e in range(E) if plan[li][e] == rank]) for li in range(L)]
           for name, plan in plans.items()}
    # per-layer placements as device arrays (uploaded once; moe_dispatch reads them on the device)
    pdev = {name: [lay.placement(plan[li]) for li in range(L)] for name, plan in plans.items()}

    def chain(plan, wl, name=None):
        xin = x0
        for li in range(L):
            lay.route(logits[li], k, idx[li], w[li])
            lay.dispatch(xin, idx[li], pdev[name][li] if name else plan[li])
            lay.expert_ffn(*wl[li])
            out = bufs[li % 2]
            lay.combine(w[li], out)
            xin = out

    for name, plan in plans.items():      # warm-up (also builds every weight set)
        chain(plan, wls[name], name)
    torch.cuda.synchronize()
    # direct l -> l+1 chain: two more contexts alternate (layer l's outputs stay in one
    # while the other dispatches layer l+1 from them)
    dl = []
    if a.direct:
        dl = [moe.MoeLayer(max_tokens=max(Tmax, 1), hidden=H, ffn=F, num_experts=E, max_k=k, world=N, rank=rank,
                           device=local, uid=fresh_uid(), a2a="p2p" if N > 1 else "nccl") for _ in range(2)]
        for c in dl:
            for name, plan in plans.items():
                for li in range(L):
                    c.placement(plan[li])
        dw = [[torch.empty(t1 - t0, k, dtype=torch.float32, device=dev) for _ in range(L)] for _ in range(2)]
        dout = torch.empty_like(x0)

    def chain_direct(plan, wl, name):
        prev = None
        for li in range(L):
            c = dl[li % 2]
            wt = dw[li % 2][li]
            c.route(logits[li], k, idx[li], wt)
            if prev is None:
                c.dispatch(x0, idx[li], c.placement(plan[li]))
            else:
                c.dispatch_from(prev[0], prev[1], idx[li], c.placement(plan[li]))
            c.output_mode("home" if li == L - 1 else "stay")
            c.expert_ffn(*wl[li])
            prev = (c, wt)
        prev[0].combine(prev[1], dout)

    direct_exact = {}
    if a.direct:
        for name, plan in plans.items():
            if N > 1:
                dist.barrier()
            chain(plan, wls[name], name)
            torch.cuda.synchronize()
            ref = bufs[(L - 1) % 2].clone()
            chain_direct(plan, wls[name], name)
            torch.cuda.synchronize()
            direct_exact[name] = bool(torch.equal(dout.view(torch.int16), ref.view(torch.int16)))
    graphs, replay_exact = {}, {}
    if a.graph:
        eager_out = {}
        for name, plan in plans.items():
            if N > 1:
                dist.barrier()
            chain(plan, wls[name], name)
            torch.cuda.synchronize()
            eager_out[name] = bufs[(L - 1) % 2].clone()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        for name, plan in plans.items():
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=side):
                chain(plan, wls[name], name)
            graphs[name] = gr
        torch.cuda.current_stream().wait_stream(side)
        for name in plans:
            if N > 1:
                dist.barrier()
            bufs[(L - 1) % 2].zero_()
            graphs[name].replay()
            torch.cuda.synchronize()
            replay_exact[name] = bool(torch.equal(bufs[(L - 1) % 2].view(torch.int16),
                                                  eager_out[name].view(torch.int16)))
    # placements interleaved rep by rep, so clock drift under the power cap
    # affects them alike; median over reps of the max over ranks
    times = {name: [] for name in plans}
    dtimes = {name: [] for name in plans}
    for _ in range(a.reps):
        for name, plan in plans.items():
            if a.direct:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if N > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                e0.record()
                chain_direct(plan, wls[name], name)
                e1.record()
                torch.cuda.synchronize()
                dtimes[name].append(e0.elapsed_time(e1))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if N > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0.record()
            if a.graph:
                graphs[name].replay()
            else:
                chain(plan, wls[name], name)
            e1.record()
            torch.cuda.synchronize()
            times[name].append(e0.elapsed_time(e1))
    results = {}
    for name, plan in plans.items():
        t = torch.tensor(times[name], dtype=torch.float64, device=dev)
        if N > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tm = float(t.median())
        rows_max = [int(max(np.bincount(plan[li], weights=load_h[li], minlength=G))) for li in range(L)]
        results[name] = {"ms_per_chain": tm, "ms_per_layer": tm / L, "tokens_per_s": T * L / (tm * 1e-3),
                         "reps_ms": [round(float(v), 3) for v in t.tolist()],
                         "o2_max_pair_tokens_summed": int(o2[name]),
                         "mean_max_gpu_rows": float(np.mean(rows_max)),
                         "balance_slack": placement.balance_slack(plan, G)}
        if a.direct:
            td = torch.tensor(dtimes[name], dtype=torch.float64, device=dev)
            ok = torch.tensor([1 if direct_exact[name] else 0], device=dev)
            if N > 1:
                dist.all_reduce(td, op=dist.ReduceOp.MAX)
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            tdm = float(td.median())
            results[name]["direct"] = {"ms_per_chain": tdm, "ms_per_layer": tdm / L,
                                       "tokens_per_s": T * L / (tdm * 1e-3),
                                       "reps_ms": [round(float(v), 3) for v in td.tolist()],
                                       "bit_identical_to_home_chain_all_ranks": bool(ok.item())}
        if a.graph:
            ok = torch.tensor([1 if replay_exact[name] else 0], device=dev)
            if N > 1:
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            results[name]["graph_replay_bit_exact_all_ranks"] = bool(ok.item())
    if rank == 0:
        print(json.dumps({
            "what": "profile -> ILP 1/ILP 2 -> serve, L-layer chain (tools/placement_loop.py)",
            "config": {"workload": cfg["workload"], "E": E, "k": k, "H": H, "F": F, "T": T, "layers": L,
                       "gpus": N, "zipf_s": a.zipf_s, "dependency": a.dependency},
            "mode": "CUDA graph per rank (one capture of the whole chain)" if a.graph else "eager launches",
            "profile_ms": profile_ms, "profile_us_per_layer": profile_ms * 1e3 / L, "host_placement_s": host_s,
            "results": results,
            "ilp2_gpu_of_cluster_first_layers": goc[:4].tolist()}), flush=True)
    for c in dl:
        c.close()
    lay.close()
    if N > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
