"""Seeded synthetic input generators, shared by the oracle tests, the GPU tests
and the bench.  This module holds none of the method's arithmetic (no top-k,
no permutation, no FFN): it only draws random numbers with fixed seeds.

Recipe:
  x        ~ N(0, 1)                      -> bf16           [T][H]
  W1, W3   ~ N(0, 1/H)                    -> bf16 per expert [F][H]
  W2       ~ N(0, 1/F)                    -> bf16 per expert [H][F]
           seeded per GLOBAL expert id (seed * 1000 + e), so a placement change
           moves identical weights to another rank.
  logits   = log p_s(rank(e)) + Gumbel    fp32 [T][E]
           p_s(r) ~ (r + 1)^-s (Zipf), rank = identity (expert 0 hottest, the
           paper's layer-14 worst case for contiguous placement) or a
           seed permutation per layer.  s = 1.6 gives the paper's 64%
           contiguous GPU-0 share.
  Multi-layer logits (D4) add a cross-layer dependency by mixing each layer's
  Gumbel noise with the previous layer's, through a fixed per-layer expert
  permutation (the "preferred successor" structure of P:L419-426).
"""

import math

import torch


def _gen(seed, device="cpu"):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def hidden_states(T, H, seed, device="cpu"):
    g = _gen(seed * 7919 + 17, device)
    return torch.randn(T, H, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)


def expert_weights(e, H, F, seed, device="cpu"):
    """(W1 [F][H], W3 [F][H], W2 [H][F]) bf16 of global expert e."""
    g = _gen(seed * 1000 + e, device)
    w1 = (torch.randn(F, H, generator=g, device=device) / math.sqrt(H)).to(torch.bfloat16)
    w3 = (torch.randn(F, H, generator=g, device=device) / math.sqrt(H)).to(torch.bfloat16)
    w2 = (torch.randn(H, F, generator=g, device=device) / math.sqrt(F)).to(torch.bfloat16)
    return w1, w3, w2


def zipf_log_probs(E, s, perm=None):
    """log p_s(e), p_s(e) ~ (rank(e)+1)^-s, rank = perm[e] (identity if None)."""
    r = torch.arange(E, dtype=torch.float64) if perm is None else torch.as_tensor(perm, dtype=torch.float64)
    logp = -s * torch.log(r + 1.0)
    logp = logp - torch.logsumexp(logp, 0)
    return logp.to(torch.float32)


def gumbel(T, E, gen, device="cpu"):
    u = torch.rand(T, E, generator=gen, device=device, dtype=torch.float32)
    u = u.clamp_(min=1e-12, max=1.0 - 1e-7)
    return -torch.log(-torch.log(u))


def zipf_logits(T, E, s, seed, perm=None, device="cpu"):
    """Router logits: log p_s(e) + Gumbel noise (Gumbel-top-k sampling of a
    Plackett-Luce Zipf distribution)."""
    g = _gen(seed * 104729 + 3, device)
    return gumbel(T, E, g, device) + zipf_log_probs(E, s, perm).to(device)


def layer_perm(E, seed, layer):
    g = _gen(seed * 31337 + layer, "cpu")
    return torch.randperm(E, generator=g)


def multilayer_logits(L, T, E, s, seed, dependency=0.5, device="cpu"):
    """L layers of logits with a seed-permuted Zipf marginal per layer and a
    cross-layer dependency of strength `dependency` in [0, 1]: layer l+1's noise
    for expert pi_l(e) is sqrt(d) * (layer l's noise for e) + sqrt(1-d) * fresh."""
    g = _gen(seed * 15485863 + 11, device)
    out = []
    prev = None
    for l in range(L):
        fresh = torch.randn(T, E, generator=g, device=device)
        if prev is None:
            z = fresh
        else:
            pi = layer_perm(E, seed, 1000 + l).to(device)
            carried = torch.empty_like(prev)
            carried[:, pi] = prev
            z = math.sqrt(dependency) * carried + math.sqrt(1.0 - dependency) * fresh
        prev = z
        logp = zipf_log_probs(E, s, layer_perm(E, seed, l)).to(device)
        out.append((z * 1.2825 + logp).to(torch.float32))   # 1.2825 = Gumbel std dev
    return out
