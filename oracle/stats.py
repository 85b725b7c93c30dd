"""C2 -- routing statistics (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Paper: P_{e,l} = "the number of tokens routed to expert e in layer l"
(§ILP 1 Inputs) and R_{e1,e2,l} = "the number of tokens routed between
experts e1 and e2" of layers l and l+1 (§ILP 2 Inputs), collected by
"token routing profiling".

Reading G10: under top-k each token contributes k x k (e1, e2) pairs per layer
step, on the same token rows in both layers; counts are int64.
Reading G12: Eq. (2)'s spurious sum over t is dropped -- P is already a count.
"""

import numpy as np


def load_counts(idx_l, E):
    """P_{.,l}: load[e] = #{(t, j) : idx_l[t][j] == e}.  int64 [E]."""
    idx_l = np.asarray(idx_l)
    load = np.zeros(E, dtype=np.int64)
    T, k = idx_l.shape
    for j in range(k):
        np.add.at(load, idx_l[:, j], 1)
    return load


def coactivation_counts(idx_l, idx_l1, E):
    """R_{.,.,l}: coact[e1][e2] = #{(t, j1, j2) : idx_l[t][j1] == e1 and
    idx_l1[t][j2] == e2}.  int64 [E][E], e1-major."""
    idx_l = np.asarray(idx_l)
    idx_l1 = np.asarray(idx_l1)
    assert idx_l.shape == idx_l1.shape
    coact = np.zeros((E, E), dtype=np.int64)
    T, k = idx_l.shape
    for j1 in range(k):
        for j2 in range(k):
            np.add.at(coact, (idx_l[:, j1], idx_l1[:, j2]), 1)
    return coact


def route_stats(idx_l, idx_l1, E):
    """The per-layer statistics pass: (load of layer l, co-activation l -> l+1)."""
    return load_counts(idx_l, E), coactivation_counts(idx_l, idx_l1, E)
