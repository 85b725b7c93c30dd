"""CPU oracle for the MoETuner expert-parallel MoE-layer hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_2502_06643_b200``)
may import, call or execute anything under ``oracle/``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
leg do.  The oracle shares no code with the CUDA path: it is plain numpy in
float64, written step by step from the paper (and, where the paper is silent,
from the readings listed in DESIGN.md §3 / SURVEY.md §8(c)).

Citation key: ``P:Lnnn`` = /root/reference/PAPER.md line nnn, ``S:Lnnn`` =
/root/reference/SPEC.md line nnn.  The reference tree is not read at run time.

Modules (SURVEY §8(c) step ids):
  bf16    -- round-to-nearest-even to bfloat16 (storage rounding points, G5)
  route   -- C1 top-k gating
  stats   -- C2 load / co-activation statistics
  plan    -- C3 placement-aware permutation plan
  ffn     -- C5 SwiGLU expert FFN                   (Mixtral expert)
  layer   -- C4/C6/C7 payload moves, unpermute, and C8 direct definition

Parity status: every function is pinned by ``tests/test_oracle_*.py`` against
values the paper prints, closed forms, library routines or brute force; none is
"parity unpinned".
"""

from . import bf16, route, stats, plan, ffn, layer  # noqa: F401
