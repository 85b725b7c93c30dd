"""C1 -- top-k gating (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Paper: "Some models, such as Mixtral, employ a top-2 router that routes each
token to the two most relevant experts" (§Background/MoE).  The
paper gives no gate formula; reading G1: the Mixtral gate
G(x) = Softmax(TopK(logits)), i.e. pick the k largest router logits and take a
softmax over those k only.  The router GEMM is not on the path: logits are the
input (BASELINE north_star "moe_route(logits,k)").

Reading G2: ties go to the lower expert id, slot j = 0 holds the largest logit,
and -0.0 compares equal to +0.0.  Reading G3: logits are finite float32.
"""

import math

import numpy as np


def route_row(logits_row, k):
    """Top-k of one token's logits by a full stable sort (the plain definition).

    Returns (experts, weights): experts in descending-logit order (ties: lower
    expert id first); weights = softmax over the k selected logits, computed in
    float64 as exp(l_j - l_0) / sum_j' exp(l_j' - l_0).
    """
    E = len(logits_row)
    if not 1 <= k <= E:
        raise ValueError("top_k must be in [1, E]")
    # +0.0 canonicalises -0.0 (G2); sort key (-logit, e) is descending logit,
    # ascending expert id among equal logits.
    pairs = [(float(logits_row[e]) + 0.0, e) for e in range(E)]
    pairs.sort(key=lambda p: (-p[0], p[1]))
    top = pairs[:k]
    l0 = top[0][0]
    num = [math.exp(l - l0) for (l, _) in top]
    den = sum(num)
    return [e for (_, e) in top], [n / den for n in num]


def route(logits, k):
    """C1 over all tokens.  logits: float32 [T][E].  Returns idx int32 [T][k],
    w float32 [T][k] (the float64 weights stored as float32)."""
    logits = np.asarray(logits, dtype=np.float32)
    T, E = logits.shape
    idx = np.zeros((T, k), dtype=np.int32)
    w = np.zeros((T, k), dtype=np.float32)
    for t in range(T):
        experts, weights = route_row(logits[t], k)
        idx[t] = experts
        w[t] = np.asarray(weights, dtype=np.float64).astype(np.float32)
    return idx, w
