"""Pins for oracle.bf16 (round-to-nearest-even to bf16) against torch's own
fp32->bf16 conversion (a library routine) and a brute-force nearest-neighbour
search on the bf16 grid."""

import numpy as np
import torch

from oracle import bf16


def test_matches_torch_on_fp32_values():
    rng = np.random.default_rng(0)
    x32 = np.concatenate([
        rng.standard_normal(20000).astype(np.float32),
        (rng.standard_normal(2000) * 1e-39).astype(np.float32),      # fp32 subnormals
        (rng.standard_normal(2000) * 1e30).astype(np.float32),
        np.array([0.0, -0.0, 1.0, -1.0, 3.0e38, -3.0e38, 1e-45], dtype=np.float32),
    ])
    # exact ties of the bf16 grid: 1 + 2^-8, 1 + 3*2^-8
    x32 = np.concatenate([x32, np.array([1 + 2.0**-8, 1 + 3 * 2.0**-8, -(1 + 2.0**-8)], dtype=np.float32)])
    ref = torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = bf16.to_bits(x32.astype(np.float64))
    assert np.array_equal(ref, got)


def _neighbours(r):
    bits = bf16.to_bits(r).astype(np.int64)
    up = bf16.from_bits(((bits + 1) & 0xFFFF).astype(np.uint16))
    dn = bf16.from_bits(((bits - 1) & 0xFFFF).astype(np.uint16))
    return up, dn


def test_nearest_even_brute_force_on_fp64_values():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(50000) * np.exp(rng.uniform(-20, 20, 50000))
    r = bf16.round_to_bf16(x)
    # representable
    assert np.array_equal(bf16.from_bits(bf16.to_bits(r)), r)
    up, dn = _neighbours(r)
    d = np.abs(x - r)
    assert np.all(d <= np.abs(x - up))
    assert np.all(d <= np.abs(x - dn))


def test_ties_go_to_even_in_fp64():
    # 1 + 2^-8 lies exactly between 1 and 1 + 2^-7 -> even (1.0)
    assert bf16.round_to_bf16(np.array([1 + 2.0**-8]))[0] == 1.0
    # 1 + 3*2^-8 between 1+2^-7 (odd mantissa) and 1+2^-6 (even) -> 1 + 2^-6
    assert bf16.round_to_bf16(np.array([1 + 3 * 2.0**-8]))[0] == 1 + 2.0**-6
    # just above the tie rounds up (no double rounding through fp32)
    assert bf16.round_to_bf16(np.array([1 + 2.0**-8 + 2.0**-40]))[0] == 1 + 2.0**-7
    # overflow past the largest finite bf16 -> inf
    assert np.isinf(bf16.round_to_bf16(np.array([3.4e38]))[0])
