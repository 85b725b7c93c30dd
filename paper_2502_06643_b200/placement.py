"""Host-side expert placements (the input of the GPU path; not on the GPU).

The paper computes the expert->GPU map offline with two ILPs solved by Gurobi
 and loads it at serving start.  The GPU
path takes that map as an ``int32 expert_to_rank[E]`` input (BASELINE
north_star).  This module provides the two maps the benchmark compares:

* ``contiguous(E, G)`` -- Megatron's baseline: "experts 0 and 1 are assigned
  to GPU 0, experts 2 and 3 to GPU 1, and so on" (§Baseline).
  E not divisible by G is an error.
* ``ilp1_exact(load, G)`` -- ILP 1 (Eqs. (1)-(7)) for one layer,
  solved exactly by enumerating every partition of the E experts into G
  non-empty clusters (Eq. 7), minimising O1 = sum_c |T_c - T_bar| (Eqs. 1-3,
  reading G12 drops Eq. 2's spurious sum over t).  Ties are broken by the
  lexicographically smallest canonical assignment.  Cluster c is
  placed on GPU c: ILP 2 (Eqs. 8-15) has no layer pairs at L = 1, so its
  objective is identically 0 and the identity bijection is optimal.

Harness utility: exhaustive enumeration is meant for E <= 12.
"""

import numpy as np


def contiguous(E, G):
    if G <= 0 or E % G != 0:
        raise ValueError(f"contiguous placement needs E % G == 0 (E={E}, G={G})")
    per = E // G
    return np.array([e // per for e in range(E)], dtype=np.int32)


def _restricted_growth_strings(E, G):
    """All canonical labelings of partitions of range(E) into exactly G blocks
    (restricted growth strings): a[0] = 0, a[i] <= max(a[:i]) + 1."""
    a = [0] * E

    def rec(i, m):
        if E - i < G - (m + 1):      # not enough experts left to open G blocks
            return
        if i == E:
            if m + 1 == G:
                yield tuple(a)
            return
        for c in range(min(m + 2, G)):
            a[i] = c
            yield from rec(i + 1, max(m, c))

    if E == 0:
        return
    yield from rec(1, 0)


def o1_times_G(load, assign, G):
    """G * O1 for one layer, in exact integers: sum_c |G*T_c - sum_e P_e|."""
    load = [int(v) for v in load]
    total = sum(load)
    T = [0] * G
    for e, c in enumerate(assign):
        T[c] += load[e]
    return sum(abs(G * t - total) for t in T)


def ilp1_exact(load, G):
    """Exact ILP-1 clustering of one layer.  Returns (assign int32 [E], O1)."""
    E = len(load)
    if not 1 <= G <= E:
        raise ValueError("ILP 1 needs 1 <= G <= E (Eq. 7)")
    best, best_a = None, None
    for a in _restricted_growth_strings(E, G):
        v = o1_times_G(load, a, G)
        if best is None or v < best or (v == best and a < best_a):
            best, best_a = v, a
    return np.array(best_a, dtype=np.int32), best / G


def _canonical(assign):
    """Relabel clusters canonically: the block holding the lowest unassigned
    expert gets the lowest free id."""
    mapping, out = {}, []
    for c in assign:
        if c not in mapping:
            mapping[c] = len(mapping)
        out.append(mapping[c])
    return out


def ilp1_heuristic(load, G):
    """ILP 1 for instances too large to enumerate: longest-
    processing-time greedy seeding, then single-expert moves and pairwise
    swaps while O1 decreases, never emptying a cluster (Eq. 7)."""
    load = [int(v) for v in load]
    E = len(load)
    if not 1 <= G <= E:
        raise ValueError("ILP 1 needs 1 <= G <= E (Eq. 7)")
    order = sorted(range(E), key=lambda e: (-load[e], e))
    assign = [0] * E
    T = [0] * G
    size = [0] * G
    for i, e in enumerate(order):
        if i < G:
            c = i                       # every cluster gets one expert first
        else:
            c = min(range(G), key=lambda q: (T[q], q))
        assign[e] = c
        T[c] += load[e]
        size[c] += 1
    total = sum(load)

    def obj(Tv):
        return sum(abs(G * t - total) for t in Tv)

    best = obj(T)
    improved = True
    while improved:
        improved = False
        for e in range(E):                      # moves
            a = assign[e]
            if size[a] == 1:
                continue
            for c in range(G):
                if c == a:
                    continue
                T[a] -= load[e]
                T[c] += load[e]
                v = obj(T)
                if v < best:
                    best, assign[e] = v, c
                    size[a] -= 1
                    size[c] += 1
                    improved = True
                    break
                T[a] += load[e]
                T[c] -= load[e]
        for e1 in range(E):                     # swaps
            for e2 in range(e1 + 1, E):
                a, b = assign[e1], assign[e2]
                if a == b:
                    continue
                d = load[e1] - load[e2]
                T[a] -= d
                T[b] += d
                v = obj(T)
                if v < best:
                    best = v
                    assign[e1], assign[e2] = b, a
                    improved = True
                else:
                    T[a] += d
                    T[b] -= d
    return np.array(_canonical(assign), dtype=np.int32), best / G


def stirling2(n, k):
    """Number of partitions of n items into k non-empty blocks."""
    S = [[0] * (k + 1) for _ in range(n + 1)]
    S[0][0] = 1
    for i in range(1, n + 1):
        for j in range(1, min(i, k) + 1):
            S[i][j] = j * S[i - 1][j] + S[i - 1][j - 1]
    return S[n][k]


def balanced(load, G):
    """Placement used for the 'balanced' benchmark arm: ILP-1 cluster c -> GPU c;
    exact enumeration when at most 10^6 partitions, else the heuristic."""
    if stirling2(len(load), G) <= 10 ** 6:
        assign, _ = ilp1_exact(load, G)
    else:
        assign, _ = ilp1_heuristic(load, G)
    return assign.astype(np.int32)


# ---------------------------------------------------------------------------
# ILP 2 (Eqs. 8-15): place each layer's ILP-1 clusters on GPUs.
# Host tooling for the placement-feedback loop: the routing
# statistics come from the GPU (moe_route_stats + moe_stats_allreduce).

def comm_costs(coact, assign, G):
    """Eq. (9): C[l][c1][c2] = sum of R[l][e1][e2] over e1 in cluster c1 of layer l
    and e2 in cluster c2 of layer l+1.  coact: int [L-1][E][E]; assign: int [L][E]."""
    coact = np.asarray(coact, dtype=np.int64)
    assign = np.asarray(assign)
    L1 = coact.shape[0]
    C = np.zeros((L1, G, G), dtype=np.int64)
    for l in range(L1):
        A = np.eye(G, dtype=np.int64)[assign[l]]        # [E][G] one-hot x_{c,e,l}
        B = np.eye(G, dtype=np.int64)[assign[l + 1]]
        C[l] = A.T @ coact[l] @ B
    return C


def _pair_max(Cl, p1, p2, G):
    """max over ordered GPU pairs g1 != g2 of the volume C[c1][c2] moved from GPU
    p1[c1] to GPU p2[c2] (uniform NVSwitch bandwidth: B constant)."""
    V = np.zeros((G, G), dtype=np.int64)
    np.add.at(V, (np.asarray(p1)[:, None].repeat(G, 1), np.asarray(p2)[None, :].repeat(G, 0)), Cl)
    np.fill_diagonal(V, 0)                              # same-GPU traffic costs nothing
    return int(V.max()) if G > 1 else 0


def objective_o2(C, gpu_of_cluster):
    """Eq. (8) read as in SPEC place_opt: sum over layer transitions of the max
    over ordered GPU pairs g1 != g2 of the volume on that pair."""
    C = np.asarray(C)
    G = C.shape[1] if C.ndim == 3 else len(gpu_of_cluster[0])
    return sum(_pair_max(C[l], gpu_of_cluster[l], gpu_of_cluster[l + 1], G) for l in range(C.shape[0]))


def ilp2_dp(C, G, L):
    """Exact minimiser of O2 over per-layer cluster->GPU bijections (Eqs. 14-15)
    by dynamic programming over (layer, permutation) -- the chain structure of
    Eq. (8) makes the relaxation without Eq. (13) exact.  Eq. (13) (equal expert
    counts per GPU over all layers) is not enforced here; `balance_slack`
    reports how far the result is from it.  Ties: lexicographically smallest
    permutation sequence.  Intended for G <= 5 (G! states per layer)."""
    import itertools
    perms = list(itertools.permutations(range(G)))
    P = len(perms)
    if L == 1:
        return np.array([perms[0]], dtype=np.int32)
    # trans[l][i][j] = transition l with layer-l permutation i, layer-(l+1) permutation j;
    # togo[l][i] = the least cost of layers l.. given permutation i at layer l (backward DP)
    trans = [np.array([[_pair_max(C[l], perms[i], perms[j], G) for j in range(P)] for i in range(P)])
             for l in range(L - 1)]
    togo = [None] * L
    togo[L - 1] = np.zeros(P, dtype=np.int64)
    for l in range(L - 2, -1, -1):
        togo[l] = (trans[l] + togo[l + 1][None, :]).min(axis=1)
    # forward: the smallest optimal permutation index at every layer, given the ones
    # chosen before it -- the lexicographically smallest optimal sequence (perms are
    # generated in lexicographic order)
    seq = [int(np.argmin(togo[0]))]
    for l in range(L - 1):
        i = seq[-1]
        seq.append(int(np.argmin(trans[l][i] + togo[l + 1])))   # argmin: first among ties
    return np.array([perms[i] for i in seq], dtype=np.int32)


def expert_to_gpu(assign, gpu_of_cluster):
    """Composite map expert_to_gpu[l][e] = gpu_of_cluster[l][assign[l][e]]."""
    assign = np.asarray(assign)
    gpu_of_cluster = np.asarray(gpu_of_cluster)
    return np.stack([gpu_of_cluster[l][assign[l]] for l in range(assign.shape[0])]).astype(np.int32)


def balance_slack(e2g, G):
    """max_g |#{(l, e): e2g[l][e] == g} - E L / G| (Eq. 13 at slack 0)."""
    e2g = np.asarray(e2g)
    counts = np.bincount(e2g.ravel(), minlength=G)
    return float(np.abs(counts - e2g.size / G).max())


def to_json(expert_to_gpu_, gpu_of_cluster=None, objective=None, balance_slack_=None):
    """The portable placement file of SPEC's External Interfaces,
    {"balance_slack", "objective", "gpu_of_cluster": [[...]], "expert_to_gpu": [[...]]}
    -- what the paper stores as a framework-specific tensor file (§Leveraging ILP
    optimization).  expert_to_gpu: [L][E]; gpu_of_cluster: [L][G] (identity if
    None); the balance slack is computed when not given."""
    import json
    e2g = np.asarray(expert_to_gpu_, dtype=np.int64)
    if e2g.ndim == 1:
        e2g = e2g[None, :]
    G = int(e2g.max()) + 1 if e2g.size else 1
    goc = np.stack([np.arange(G)] * e2g.shape[0]) if gpu_of_cluster is None else np.asarray(gpu_of_cluster)
    return json.dumps({"balance_slack": float(balance_slack(e2g, G) if balance_slack_ is None else balance_slack_),
                       "objective": None if objective is None else float(objective),
                       "gpu_of_cluster": goc.astype(int).tolist(), "expert_to_gpu": e2g.astype(int).tolist()})


def from_json(text):
    """Inverse of to_json: returns (expert_to_gpu int32 [L][E], the parsed dict).
    Each row is one layer's expert_to_rank input of moe_dispatch (as a device
    array per layer).  Rejects ragged or negative maps (S:L296-style errors)."""
    import json
    d = json.loads(text)
    e2g = d.get("expert_to_gpu")
    if not isinstance(e2g, list) or not e2g or not all(isinstance(r, list) for r in e2g):
        raise ValueError("expert_to_gpu must be a non-empty list of per-layer lists")
    if len({len(r) for r in e2g}) != 1:
        raise ValueError("expert_to_gpu rows differ in length")
    arr = np.asarray(e2g, dtype=np.int64)
    if (arr < 0).any():
        raise ValueError("negative GPU id in expert_to_gpu")
    return arr.astype(np.int32), d
