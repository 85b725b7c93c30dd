"""C4/C6/C7 payload moves and the whole-layer compositions (TEST INFRASTRUCTURE ONLY).

(`layer_ep_tp` adds tensor parallelism inside the experts, reading G20.)

The expert-parallel layer of the paper (Fig. background-ep(b)):
router -> permute -> all-to-all -> expert FFN -> all-to-all -> unpermute.

  layer_ep     follows that algorithm step by step (C1, C3, C4, C5, C6, C7).
  layer_direct is the plain definition the EP algorithm must reproduce (C8):
                 out[t] = bf16( sum_{j<k} w[t][j] * FFN_{idx[t][j]}(x[t]) )
               computed with no permutation at all; it is independent of the
               placement and of G.

C7 (reading G4): the k expert outputs are combined with the float32 gate
weights in float64, j ascending, and rounded once to bf16.

``expert_fn(e, rows) -> y`` lets tests substitute special experts (identity,
zero) for the SwiGLU FFN; the default is oracle.ffn.swiglu with the given
weights.
"""

import numpy as np

from .bf16 import round_to_bf16
from .ffn import swiglu
from .plan import plan, token_blocks
from .route import route


def swiglu_experts(w1, w3, w2):
    """expert_fn for per-expert float64 weight lists w1[e], w3[e], w2[e]."""
    def fn(e, rows):
        return swiglu(rows, w1[e], w3[e], w2[e])[1]
    return fn


def identity_expert(e, rows):
    return rows.copy()


def unpermute(ret_rows, w):
    """C7 for one source: ret_rows[j] float64 [T_s][H] = the returned row of item
    (t, j); w float32 [T_s][k].  out[t] = bf16(sum_j w[t][j] * ret_rows[j][t])."""
    w = np.asarray(w, dtype=np.float32).astype(np.float64)
    acc = np.zeros_like(ret_rows[0])
    for j in range(w.shape[1]):
        acc = acc + w[:, j:j + 1] * ret_rows[j]
    return round_to_bf16(acc)


def layer_ep(x, logits, k, P, G, expert_fn):
    """The EP layer over G ranks, step by step.

    x float64 [T][H] (bf16 values), logits float32 [T][E].  Returns
    (out float64 [T][H], idx, w, the C3 plan, recv payloads per rank).
    """
    T = x.shape[0]
    idx, w = route(logits, k)                                      # C1
    blocks = token_blocks(T, G)
    pl = plan([idx[a:b] for (a, b) in blocks], P, G)               # C3
    H = x.shape[1]
    # C4: dispatch payload -- rank g receives x_s[t] for each item in recv order.
    recv = []
    for g in range(G):
        rows = np.zeros((len(pl["recv"][g]), H))
        for r, (s, t, j, e) in enumerate(pl["recv"][g]):
            rows[r] = x[blocks[s][0] + t]
        recv.append(rows)
    # C5: each rank runs its experts on its received rows (expert-major order).
    y_recv = []
    for g in range(G):
        y = np.zeros_like(recv[g])
        experts = [e for e in range(len(P)) if P[e] == g]
        for e in experts:
            sel = [r for r, item in enumerate(pl["recv"][g]) if item[3] == e]
            if sel:
                y[sel] = expert_fn(e, recv[g][sel])
        y_recv.append(y)
    # C6: combine payload -- back to the source, into send order (ret[slot]).
    out = np.zeros_like(x)
    for s, (a, b) in enumerate(blocks):
        T_s = b - a
        n_items = T_s * k
        ret = np.zeros((n_items, H))
        for g in range(G):
            for r, (s2, t, j, e) in enumerate(pl["recv"][g]):
                if s2 == s:
                    ret[pl["slot"][s][t, j]] = y_recv[g][r]
        ret_rows = [ret[pl["slot"][s][:, j]] for j in range(k)] if T_s else [np.zeros((0, H))] * k
        out[a:b] = unpermute(ret_rows, w[a:b])                     # C7
    return out, idx, w, pl, recv


def layer_direct(x, logits, k, expert_fn):
    """C8: out[t] = bf16(sum_j w[t][j] * FFN_{idx[t][j]}(x[t])), no permutation."""
    idx, w = route(logits, k)
    T, H = x.shape
    E = logits.shape[1]
    acc = np.zeros((T, H))
    w64 = w.astype(np.float64)
    # Evaluate each expert on the tokens that chose it, then accumulate in j order.
    y_of = {}
    for e in range(E):
        toks = np.nonzero((idx == e).any(axis=1))[0]
        if len(toks):
            y_of[e] = (toks, expert_fn(e, x[toks]))
    for j in range(k):
        yj = np.zeros((T, H))
        for e, (toks, y) in y_of.items():
            sel = idx[toks, j] == e
            yj[toks[sel]] = y[sel]
        acc = acc + w64[:, j:j + 1] * yj
    return round_to_bf16(acc), idx, w


# ---------------------------------------------------------------------------
# Tensor parallelism inside the experts (the paper's "4EP-2TP",
# P:L77-79).  Reading G20:
#   * W = G * tp ranks; rank r is TP index r % tp of EP group r // tp; every rank
#     owns a token block (G7 over W ranks) and is a source;
#   * the placement maps experts to EP groups; every rank of group g receives
#     group g's rows (the TP all-gather), in the receive order of C3;
#   * TP slice q of expert e holds the contiguous FFN rows [q F/tp, (q+1) F/tp)
#     of W1_e and W3_e and the matching columns of W2_e (Megatron's column /
#     row-parallel split of the expert MLP);
#   * each rank returns a bf16 partial output (its slice's h times its W2
#     columns, rounded once to bf16 -- the TP reduction operates on bf16
#     activations); the source sums the tp partials (q ascending) and then
#     combines the k experts as in C7.

def swiglu_tp_experts(w1, w3, w2, tp):
    """expert_part_fn(e, rows, q) -> bf16 partial output of TP slice q."""
    def fn(e, rows, q):
        F = w1[e].shape[0]
        f = F // tp
        sl = slice(q * f, (q + 1) * f)
        return swiglu(rows, w1[e][sl], w3[e][sl], w2[e][:, sl])[1]
    return fn


def layer_ep_tp(x, logits, k, P, G, tp, expert_part_fn):
    """The EP layer over G EP groups of tp ranks each, step by step.

    Returns (out float64 [T][H], idx, w, the C3 plan over W = G*tp sources).
    """
    W = G * tp
    T, H = x.shape
    idx, w = route(logits, k)                                      # C1
    blocks = token_blocks(T, W)
    pl = plan([idx[a:b] for (a, b) in blocks], P, G)               # C3 (W sources, G groups)
    # C4: rank (g, q) receives group g's rows
    recv = []
    for g in range(G):
        rows = np.zeros((len(pl["recv"][g]), H))
        for r, (s, t, j, e) in enumerate(pl["recv"][g]):
            rows[r] = x[blocks[s][0] + t]
        recv.append(rows)
    # C5: rank (g, q) computes the partial outputs of its F slice
    y_part = []                                                    # [g][q] -> rows
    for g in range(G):
        parts = []
        for q in range(tp):
            y = np.zeros_like(recv[g])
            for e in [e for e in range(len(P)) if P[e] == g]:
                sel = [r for r, item in enumerate(pl["recv"][g]) if item[3] == e]
                if sel:
                    y[sel] = expert_part_fn(e, recv[g][sel], q)
            parts.append(y)
        y_part.append(parts)
    # C6: every rank of the group returns its partial rows to the source
    # (ret[q][slot]); C7 with the tp partials summed first.
    out = np.zeros_like(x)
    for s, (a, b) in enumerate(blocks):
        n_items = (b - a) * k
        ret = np.zeros((tp, n_items, H))
        for g in range(G):
            for r, (s2, t, j, e) in enumerate(pl["recv"][g]):
                if s2 == s:
                    for q in range(tp):
                        ret[q, pl["slot"][s][t, j]] = y_part[g][q][r]
        y_sum = ret[0].copy()
        for q in range(1, tp):
            y_sum = y_sum + ret[q]
        ret_rows = [y_sum[pl["slot"][s][:, j]] for j in range(k)] if b > a else [np.zeros((0, H))] * k
        out[a:b] = unpermute(ret_rows, w[a:b])                     # C7
    return out, idx, w, pl
