"""Shared test helpers: synthetic inputs (via synth/) and tolerance checks.

Tolerance (north_star "within 2e-2 relative (bf16 storage, fp32 accumulate)";
reading G16 in DESIGN.md): elementwise relative error is ill-posed near zero,
so a float tensor passes when BOTH
    max|gpu - ref| / max|ref|                 <= 2e-2
    max_t ||gpu_t - ref_t||_2 / ||ref_t||_2   <= 2e-2
hold; gate weights are compared elementwise (rtol 2e-2; expected ~1e-6).
"""

import numpy as np
import torch

import synth
from oracle import bf16

TOL = 2e-2


def bf16_to_f64(t):
    """torch bf16 tensor (any device) -> float64 numpy with the same values."""
    return bf16.from_bits(t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16))


def assert_close_layer(gpu, ref, tol=TOL):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape
    if ref.size == 0:
        return 0.0, 0.0
    assert np.all(np.isfinite(gpu))
    d = gpu - ref
    scale = np.abs(ref).max()
    maxnorm = np.abs(d).max() / scale if scale > 0 else np.abs(d).max()
    rn = np.linalg.norm(ref, axis=1)
    dn = np.linalg.norm(d, axis=1)
    ok = rn > 0
    row = (dn[ok] / rn[ok]).max() if ok.any() else 0.0
    assert np.all(dn[~ok] == 0) or scale == 0
    assert maxnorm <= tol, f"max-norm relative error {maxnorm:.3e} > {tol}"
    assert row <= tol, f"row-L2 relative error {row:.3e} > {tol}"
    return maxnorm, row


class Inputs:
    """Seeded inputs of one layer configuration (CPU tensors)."""

    def __init__(self, T, H, F, E, k, s=1.6, seed=0, with_weights=True):
        self.T, self.H, self.F, self.E, self.k = T, H, F, E, k
        self.x = synth.hidden_states(T, H, seed)
        self.logits = synth.zipf_logits(T, E, s, seed)
        self.w = [synth.expert_weights(e, H, F, seed) for e in range(E)] if with_weights else None

    def to_device(self, dev):
        x = self.x.to(dev)
        logits = self.logits.to(dev)
        return x, logits

    def device_weights(self, dev, experts):
        """(w1 [n][F][H], w3, w2 [n][H][F]) on the device for the given experts."""
        w1 = torch.stack([self.w[e][0] for e in experts]).to(dev)
        w3 = torch.stack([self.w[e][1] for e in experts]).to(dev)
        w2 = torch.stack([self.w[e][2] for e in experts]).to(dev)
        return w1, w3, w2

    def oracle_expert_fn(self):
        from oracle import ffn
        cache = {}

        def fn(e, rows):
            if e not in cache:
                cache.clear()
                cache[e] = tuple(bf16_to_f64(m) for m in self.w[e])
            w1, w3, w2 = cache[e]
            return ffn.swiglu(rows, w1, w3, w2)[1]
        return fn

    def oracle_tp_fn(self, tp):
        """expert_part_fn(e, rows, q) of oracle.layer.layer_ep_tp for these weights."""
        from oracle import ffn
        cache = {}

        def fn(e, rows, q):
            if e not in cache:
                cache.clear()
                cache[e] = tuple(bf16_to_f64(m) for m in self.w[e])
            w1, w3, w2 = cache[e]
            f = w1.shape[0] // tp
            sl = slice(q * f, (q + 1) * f)
            return ffn.swiglu(rows, w1[sl], w3[sl], w2[:, sl])[1]
        return fn
