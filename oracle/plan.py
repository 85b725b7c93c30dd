"""C3 -- placement-aware dispatch plan (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Paper: in expert parallelism "tokens are routed to remote GPUs using all-to-all
communication based on their assigned experts"; the placement is
an expert->GPU map, contiguous blocks for Megatron ("experts 0 and 1
are assigned to GPU 0") or any custom map, possibly with a
different number of experts per GPU (reading G14).

Readings:
  G7  token ownership: source rank s owns a contiguous block of
      floor(T/G) + [s < T mod G] tokens, blocks in rank order.
  G8  experts on a GPU are ordered by ascending global id.
  G9  send order on source s: items (t, j) stably sorted by key (P[e], e);
      receive order on rank g: e ascending over {e : P[e] == g}, then source s
      ascending, then t ascending.
  G13 a rank may host zero experts.
"""

import numpy as np


def token_blocks(T, G):
    """[(start, stop)] of the G source blocks (reading G7)."""
    base, rem = divmod(T, G)
    out, start = [], 0
    for s in range(G):
        n = base + (1 if s < rem else 0)
        out.append((start, start + n))
        start += n
    return out


def validate_placement(P, G):
    P = np.asarray(P)
    if P.ndim != 1 or np.any(P < 0) or np.any(P >= G):
        raise ValueError("placement values must lie in [0, G)")


def plan(idx_by_source, P, G):
    """C3 for S = len(idx_by_source) source ranks and G destination ranks.

    S == G for plain expert parallelism.  With tensor parallelism inside the
    experts (reading G20, `layer.layer_ep_tp`) every one of the S = G * tp ranks
    is a source and the destinations are the G EP groups; every rank of group g
    receives the same rows, in the receive order below.

    idx_by_source[s]: int [T_s][k] expert ids of source s's tokens.
    P: int [E] expert -> rank (EP group).

    Returns a dict with
      slot[s]       int [T_s][k]  position of item (t, j) in source s's send order
      cnt           int [S][E]    cnt[s][e] = items of s routed to e
      send_counts   int [S][G]    send_counts[s][g] = sum_{P[e]=g} cnt[s][e]
      recv_counts   int [G]       rows received by rank g
      recv[g]       list of (s, t, j, e) in rank g's receive order
      recv_pos[s]   int [T_s][k]  position of item (t, j) of s in recv[P[e]]
    """
    P = np.asarray(P, dtype=np.int64)
    E = len(P)
    validate_placement(P, G)
    S = len(idx_by_source)
    cnt = np.zeros((S, E), dtype=np.int64)
    slot = []
    for s in range(S):
        idx = np.asarray(idx_by_source[s])
        T_s, k = idx.shape
        items = [(t, j) for t in range(T_s) for j in range(k)]     # flattened order
        order = sorted(range(len(items)),
                       key=lambda i: (P[idx[items[i]]], idx[items[i]]))  # stable
        sl = np.zeros((T_s, k), dtype=np.int64)
        for pos, i in enumerate(order):
            sl[items[i]] = pos
        slot.append(sl)
        for (t, j) in items:
            cnt[s, idx[t, j]] += 1
    send_counts = np.zeros((S, G), dtype=np.int64)
    for s in range(S):
        for e in range(E):
            send_counts[s, P[e]] += cnt[s, e]
    recv = []
    recv_pos = [np.full(np.asarray(idx_by_source[s]).shape, -1, dtype=np.int64) for s in range(S)]
    for g in range(G):
        rows = []
        for e in range(E):
            if P[e] != g:
                continue
            for s in range(S):
                idx = np.asarray(idx_by_source[s])
                for t in range(idx.shape[0]):
                    for j in range(idx.shape[1]):
                        if idx[t, j] == e:
                            recv_pos[s][t, j] = len(rows)
                            rows.append((s, t, j, e))
        recv.append(rows)
    recv_counts = np.array([len(r) for r in recv], dtype=np.int64)
    return dict(slot=slot, cnt=cnt, send_counts=send_counts,
                recv_counts=recv_counts, recv=recv, recv_pos=recv_pos)
