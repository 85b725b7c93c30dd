#!/usr/bin/env python
"""NVLink bytes per phase of the EP layer, from the GPU's own link counters.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/nvlink_phases.py [--config mixtral] [--zipf-s 0] [--placement contiguous] [--steps 10]

Each step runs dispatch / expert FFN / combine with a device synchronise and a
barrier between the phases, and reads the NVML NVLink data counters
(NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, all links) of this rank's GPU
around every phase, so each phase's transmitted / received bytes and its
device time can be set against the algorithmic bytes (remote routed rows x 2H,
SURVEY §8(d)) and the 900 GB/s per-direction link peak (BASELINE north_star:
"bus GB/s against 900 GB/s per direction for the all-to-all").  The P2P
dispatch's side-stream scatter lands inside the dispatch window; with the fused
combine the return traffic is inside the expert-FFN window (K6's epilogue
stores rows into the sources' return buffers), otherwise inside the combine.
A profiling tool, not a benchmark: the phases are serialised here.
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


class LinkCounters:
    """NVML NVLink data counters (KiB, summed over the GPU's links)."""

    def __init__(self, dev_index):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        h = None
        try:
            p = torch.cuda.get_device_properties(dev_index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
        self.h = h
        self.fields = [pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX]
        self.links = list(range(18))

    def read(self):
        """(tx_bytes, rx_bytes) summed over links."""
        req = [(f, l) for f in self.fields for l in self.links]
        vals = self.nv.nvmlDeviceGetFieldValues(self.h, req)
        tx = rx = 0
        for (f, _), v in zip(req, vals):
            if v.nvmlReturn != 0:
                continue
            x = int(v.value.ullVal)
            if f == self.fields[0]:
                tx += x
            else:
                rx += x
        return tx * 1024, rx * 1024


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral", choices=list(CONFIGS))
    ap.add_argument("--placement", default="contiguous", choices=["contiguous", "balanced"])
    ap.add_argument("--zipf-s", type=float, default=0.0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--fused", default=None, help="MOE_FUSED_COMBINE override (0/1)")
    a = ap.parse_args()
    if a.fused is not None:
        os.environ["MOE_FUSED_COMBINE"] = a.fused
    from paper_2502_06643_b200 import moe, placement

    cfg = CONFIGS[a.config]
    E, k, H, F, T = cfg["E"], cfg["k"], cfg["H"], cfg["F"], cfg["T"]
    rank = int(os.environ.get("RANK", 0))
    N = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    u = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        u.copy_(torch.frombuffer(bytearray(moe.get_unique_id()), dtype=torch.uint8))
    dist.broadcast(u, 0)
    uid = bytes(u.cpu().numpy().tobytes())
    t0, t1 = blocks(T, N)[rank]
    Tmax = max(y - x for x, y in blocks(T, N))
    lay = moe.MoeLayer(max_tokens=Tmax, hidden=H, ffn=F, num_experts=E, max_k=k, world=N, rank=rank,
                       device=local, uid=uid, a2a="p2p")
    x = synth.hidden_states(T, H, 0, device=dev)[t0:t1].contiguous()
    logits = synth.zipf_logits(T, E, a.zipf_s, 0, device=dev)[t0:t1].contiguous()
    idx, w = lay.route(logits, k)
    if a.placement == "contiguous":
        P = moe.placement_contiguous(E, N)
    else:
        load = torch.zeros(E, dtype=torch.int64, device=dev)
        lay.route_stats(idx, None, load, None)
        lay.stats_allreduce(load, None)
        lay.sync()
        P = placement.balanced(load.cpu().numpy(), N).astype(np.int32)
    hosted = [e for e in range(E) if P[e] == rank]
    w13 = w2 = None
    if hosted:
        ws = [synth.expert_weights(e, H, F, 0, device=dev) for e in hosted]
        w1, w3, w2 = (torch.stack([q[i] for q in ws]) for i in range(3))
        del ws
        w13 = moe.pack_w13(w1, w3)
        del w1, w3
    out = torch.empty(t1 - t0, H, dtype=torch.bfloat16, device=dev)
    info = lay.dispatch(x, idx, P, info=True)
    lay.expert_ffn(w13, w2)
    lay.combine(w, out)
    lay.sync()
    sent_rows = sum(int(info.send_counts[g]) for g in range(N) if g != rank)
    recv_rows = int(info.recv_counts[rank]) - int(info.send_counts[rank])
    ctr = LinkCounters(local)
    phases = ["dispatch", "expert_ffn", "combine"]
    tx = np.zeros((a.steps, 3))
    rx = np.zeros((a.steps, 3))
    ms = np.zeros((a.steps, 3))
    for i in range(a.warmup + a.steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        c = []
        dist.barrier()
        torch.cuda.synchronize()
        c.append(ctr.read())
        ev[0].record()
        lay.dispatch(x, idx, P)
        ev[1].record()
        torch.cuda.synchronize()
        dist.barrier()
        c.append(ctr.read())
        torch.cuda.synchronize()
        ev2 = torch.cuda.Event(enable_timing=True)
        ev2.record()
        lay.expert_ffn(w13, w2)
        ev[2].record()
        torch.cuda.synchronize()
        dist.barrier()
        c.append(ctr.read())
        ev3 = torch.cuda.Event(enable_timing=True)
        ev3.record()
        lay.combine(w, out)
        ev[3].record()
        torch.cuda.synchronize()
        dist.barrier()
        c.append(ctr.read())
        if i >= a.warmup:
            j = i - a.warmup
            for p in range(3):
                tx[j, p] = c[p + 1][0] - c[p][0]
                rx[j, p] = c[p + 1][1] - c[p][1]
            ms[j] = [ev[0].elapsed_time(ev[1]), ev2.elapsed_time(ev[2]), ev3.elapsed_time(ev[3])]
    algo = 2 * H * sent_rows     # bytes this rank pushes in dispatch (= pulls/receives back in combine)
    algo_in = 2 * H * recv_rows  # bytes this rank receives in dispatch (= returns in combine)
    res = {"rank": rank, "config": a.config, "zipf_s": a.zipf_s, "placement": [int(v) for v in P],
           "fused_env": os.environ.get("MOE_FUSED_COMBINE"),
           "remote_rows_sent": sent_rows, "remote_rows_received": recv_rows,
           "algorithmic_bytes": {"dispatch_out": algo, "dispatch_in": algo_in},
           "phases": {}}
    for p, name in enumerate(phases):
        mtx, mrx, mms = float(np.median(tx[:, p])), float(np.median(rx[:, p])), float(np.median(ms[:, p]))
        res["phases"][name] = {"ms": mms, "nvlink_tx_bytes": mtx, "nvlink_rx_bytes": mrx,
                               "tx_GBps_over_phase": mtx / (mms * 1e-3) / 1e9 if mms > 0 else None,
                               "rx_GBps_over_phase": mrx / (mms * 1e-3) / 1e9 if mms > 0 else None}
    print(json.dumps(res), flush=True)
    lay.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
