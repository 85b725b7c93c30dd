"""Micro-benchmark of the grouped expert GEMMs (K5 + K6) at the bench workload.

    python tools/gemm_bench.py [--reps 30] [--zipf-s 1.6] [--tokens 16384] [--experts-per-gpu 8]

Builds the N=1 Mixtral layer (all experts on one GPU), dispatches once, then
times moe_expert_ffn with the library's per-call CUDA-event records.  Prints
one JSON line with the mean K5 / K6 time and TFLOP/s.  Used for tuning knobs
(e.g. MOE_GEMM_GROUP_M); not part of the graded bench.
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
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--zipf-s", type=float, default=1.6)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--H", type=int, default=4096)
    ap.add_argument("--F", type=int, default=14336)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--k", type=int, default=2)
    a = ap.parse_args()
    from paper_2502_06643_b200 import moe
    dev = torch.device("cuda", 0)
    T, H, F, E, k = a.tokens, a.H, a.F, a.E, a.k
    lay = moe.MoeLayer(max_tokens=T, hidden=H, ffn=F, num_experts=E, max_k=k)
    x = synth.hidden_states(T, H, 0, device=dev)
    logits = synth.zipf_logits(T, E, a.zipf_s, 0, device=dev)
    ws = [synth.expert_weights(e, H, F, 0, device=dev) for e in range(E)]
    w13 = moe.pack_w13(torch.stack([q[0] for q in ws]), torch.stack([q[1] for q in ws]))
    w2 = torch.stack([q[2] for q in ws])
    del ws
    idx, w = lay.route(logits, k)
    info = lay.dispatch(x, idx, [0] * E, info=True)
    R = info.recv_rows
    for _ in range(3):
        lay.expert_ffn(w13, w2)
    lay.ffn_timing(a.reps)
    for _ in range(a.reps):
        lay.expert_ffn(w13, w2)
    rec = lay.ffn_timing_read()
    k5 = sum(r[0] for r in rec) / len(rec)
    k6 = sum(r[1] for r in rec) / len(rec)
    out = dict(group_m=os.environ.get("MOE_GEMM_GROUP_M", "default"), rows=R, k5_ms=k5, k6_ms=k6,
               k5_tflops=4 * H * F * R / k5 / 1e9, k6_tflops=2 * H * F * R / k6 / 1e9,
               k5_min=min(r[0] for r in rec), k6_min=min(r[1] for r in rec))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
