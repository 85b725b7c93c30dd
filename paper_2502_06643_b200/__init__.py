"""B200-native (sm_100a) expert-parallel MoE layer of MoETuner (arXiv 2502.06643).

The product is libmoe.so (C ABI, include/moe.h) with hand-written CUDA kernels;
``moe`` is its thin ctypes binding and ``placement`` the host-side placement
inputs (contiguous baseline, exact ILP-1).  Import ``paper_2502_06643_b200.moe``
explicitly: it loads libmoe.so and fails loudly if it is missing.
"""

__all__ = ["moe", "placement", "build"]
