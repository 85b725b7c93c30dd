"""C5 -- SwiGLU expert FFN (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

The paper runs the expert FFN between the two all-to-alls (Fig.
background-ep(b)) but does not describe it; its model is Mixtral-8x7B
(P:L47).  Reading G5: the Mixtral expert is
    FFN_e(x) = W2_e ( silu(W1_e x) * (W3_e x) ),   silu(z) = z / (1 + e^-z),
no bias; W1, W3: [F][H], W2: [H][F] (row-major, nn.Linear layout).
Rounding points: h and y are each rounded once to bf16 (RNE); everything else
is float64 here (bf16 inputs are exact in float64).
"""

import numpy as np

from .bf16 import round_to_bf16


def silu(z):
    with np.errstate(over="ignore"):
        return z / (1.0 + np.exp(-z))


def swiglu(x, w1, w3, w2):
    """x: float64 [n][H] (bf16 values); w1, w3: [F][H]; w2: [H][F].
    Returns (h, y): h = bf16(silu(x W1^T) * (x W3^T)) [n][F],
                    y = bf16(h W2^T) [n][H], both as float64 values."""
    a = x @ w1.T
    u = x @ w3.T
    h = round_to_bf16(silu(a) * u)
    y = round_to_bf16(h @ w2.T)
    return h, y
