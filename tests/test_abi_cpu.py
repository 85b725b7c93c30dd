"""CPU-only checks of the C ABI: libmoe.so loads, exports every symbol that
include/moe.h declares, validates arguments synchronously without a GPU, and its
host-side layout (the arithmetic NCCL mode posts its send/recv segments with)
agrees with the oracle's plan (C3).  The world-size-2 gloo test covers the
multi-rank host logic: each rank computes its own count row, the rows are
all-gathered, and both ranks must derive the same layout as the oracle."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import plan as oplan
from oracle import route as oroute
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _moe():
    from paper_2502_06643_b200 import build
    build.build()
    from paper_2502_06643_b200 import moe
    return moe


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "moe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(moe_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    moe = _moe()
    lib = moe.lib()
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(moe.EXPORTS) == decl
    assert lib.moe_abi_version() == 3
    assert lib.moe_status_str(4) == b"MOE_ERR_CAPACITY"


def test_contiguous_placement_and_error():
    moe = _moe()
    assert moe.placement_contiguous(8, 4).tolist() == [0, 0, 1, 1, 2, 2, 3, 3]
    with pytest.raises(moe.MoeError) as ei:
        moe.placement_contiguous(6, 4)
    assert ei.value.status == 1


def test_ctx_create_validates_before_touching_the_device():
    moe = _moe()
    bad = [dict(hidden=100), dict(ffn=0), dict(num_experts=0), dict(max_k=9), dict(world=2, rank=2),
           dict(virtual_ranks=4, world=2),
           dict(virtual_ranks=6, tp=4), dict(virtual_ranks=4, tp=16), dict(virtual_ranks=4, tp=4, ffn=128),
           dict(world=2, rank=0, tp=2)]   # tp: must divide the ranks, <= 8, F/tp % 64 == 0; real TP needs P2P
    for b in bad:
        kw = dict(max_tokens=16, hidden=64, ffn=128, num_experts=8, max_k=2, world=1, rank=0, device=0,
                  virtual_ranks=1)
        kw.update(b)
        with pytest.raises(moe.MoeError) as ei:
            moe.MoeLayer(**kw)
        assert ei.value.status in (1, 5), b


def test_null_ctx_calls_fail_cleanly():
    moe = _moe()
    lib = moe.lib()
    assert lib.moe_route(None, None, 1, 8, 2, None, None, None) == 1
    assert lib.moe_dispatch(None, None, None, 1, 2, None, None, None) == 1
    assert lib.moe_expert_ffn(None, None, None, 0, None) == 1
    assert lib.moe_combine(None, None, None, None) == 1


def test_group_create_validates_before_touching_the_device():
    """moe_ctx_create_group (single-process EP group): P2P only, n >= 2, no
    virtual ranks, and every rank's config passes the moe_ctx_create checks."""
    moe = _moe()
    lib = moe.lib()
    base = dict(max_tokens=16, hidden=64, ffn=128, num_experts=8, max_k=2, world=1, rank=0, device=0,
                virtual_ranks=1, a2a_mode=1, tp=1)
    bad = [(dict(), 1), (dict(a2a_mode=0), 4), (dict(virtual_ranks=4), 4), (dict(hidden=96), 4),
           (dict(tp=3), 4), (dict(), 65)]
    for upd, n in bad:
        kw = dict(base)
        kw.update(upd)
        cfg = moe.Config(*[kw[f] for f, _ in moe.Config._fields_])
        hs = (ctypes.c_void_p * max(n, 1))()
        st = lib.moe_ctx_create_group(ctypes.byref(cfg), n, None, hs)
        assert st in (1, 5), (upd, n, st)


def test_group_create_checks_hardware_queues(monkeypatch):
    """s ranks of a single-process group on one device drive 2s streams that spin
    on each other's flags: with fewer hardware queues (CUDA_DEVICE_MAX_CONNECTIONS,
    default 8) two of them alias onto one queue and can deadlock until the flag
    timeout, so creation refuses before touching the device."""
    moe = _moe()
    lib = moe.lib()
    kw = dict(max_tokens=16, hidden=64, ffn=128, num_experts=8, max_k=2, world=1, rank=0, device=0,
              virtual_ranks=1, a2a_mode=1, tp=1)
    cfg = moe.Config(*[kw[f] for f, _ in moe.Config._fields_])
    for conns, n in (("8", 5), (None, 6), ("12", 8)):
        if conns is None:
            monkeypatch.delenv("CUDA_DEVICE_MAX_CONNECTIONS", raising=False)
        else:
            monkeypatch.setenv("CUDA_DEVICE_MAX_CONNECTIONS", conns)
        hs = (ctypes.c_void_p * n)()
        assert lib.moe_ctx_create_group(ctypes.byref(cfg), n, None, hs) == 5
        assert b"CUDA_DEVICE_MAX_CONNECTIONS" in lib.moe_last_error(None)


def _layout_checks(moe, P, cnt, idx_by_source):
    G, E = cnt.shape
    seg, rb, rr, sb = moe.layout_host(P, cnt)
    pl = oplan.plan(idx_by_source, P, G)
    assert np.array_equal(pl["cnt"], cnt)
    assert rr.tolist() == pl["recv_counts"].tolist()
    for g in range(G):
        hosted = [e for e in range(E) if P[e] == g]
        end = 0
        for e in hosted:                         # ascending experts, 128-row aligned, non-overlapping
            assert seg[e] % 128 == 0 and seg[e] >= end
            end = seg[e] + cnt[:, e].sum()
    for s in range(G):
        for e in range(E):
            assert rb[s, e] - seg[e] == cnt[:s, e].sum()
            items = [(t, j) for t in range(len(idx_by_source[s])) for j in range(idx_by_source[s].shape[1])
                     if idx_by_source[s][t, j] == e]
            if items:
                first = pl["slot"][s][items[0]]
                assert sb[s, e] == first                 # C3 slot of the first (s, e) item
                # unpadded receive position of the first item
                off = sum(cnt[:, q].sum() for q in range(E) if P[q] == P[e] and q < e)
                assert pl["recv_pos"][s][items[0]] == off + cnt[:s, e].sum()


@pytest.mark.parametrize("G,P", [(4, [0, 0, 1, 1, 2, 2, 3, 3]), (4, [0, 1, 2, 2, 3, 2, 3, 3]),
                                 (3, [2, 2, 2, 2, 2, 2, 1, 1]), (1, [0] * 8)])
def test_layout_host_matches_oracle_plan(G, P):
    moe = _moe()
    T, E, k = 403, 8, 2
    idx, _ = oroute.route(synth.zipf_logits(T, E, 1.6, seed=G).numpy(), k)
    blocks = oplan.token_blocks(T, G)
    srcs = [idx[a:b] for a, b in blocks]
    cnt = np.stack([np.bincount(s.ravel(), minlength=E) for s in srcs]).astype(np.int32)
    _layout_checks(moe, np.array(P), cnt, srcs)


def _gloo_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import torch
        moe = _moe()
        T, E, k = 517, 8, 2
        P = np.array([0, 1, 1, 1, 0, 1, 0, 1])            # ILP-1 balanced at G=2
        idx, _ = oroute.route(synth.zipf_logits(T, E, 1.6, seed=5).numpy(), k)
        blocks = oplan.token_blocks(T, world)
        a, b = blocks[rank]
        mine = torch.from_numpy(np.bincount(idx[a:b].ravel(), minlength=E).astype(np.int32))
        rows = [torch.zeros(E, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(rows, mine)                       # the count exchange of moe_dispatch
        cnt = torch.stack(rows).numpy()
        seg, rb, rr, sb = moe.layout_host(P, cnt)
        _layout_checks(moe, P, cnt, [idx[x:y] for x, y in blocks])
        allv = [torch.zeros(2 * E + world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allv, torch.from_numpy(np.concatenate([seg, rb[rank], rr]).astype(np.int64)))
        # every rank derives the same segment starts and receive totals
        assert all(torch.equal(v[:E], allv[0][:E]) and torch.equal(v[2 * E:], allv[0][2 * E:]) for v in allv)
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # pragma: no cover - reported to the parent
        q.put((rank, repr(ex)))


def test_two_rank_gloo_count_exchange_and_layout():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
