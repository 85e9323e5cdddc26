"""CPU ORACLE for the SeCO / SpaCO chunked-attention hot path (arXiv 2505.16710).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call or
execute anything under ``oracle/``.  The product path
(``paper_2505_16710_b200``) never imports it and shares no code with it; the two
meet only at the seeded input generator ``synth/`` (which holds no arithmetic of
the method).

Plain, slow, obviously-correct NumPy in float64 (float32 allowed for timing).
Citations: ``P:n`` = /root/reference/PAPER.md line n (section / equation /
algorithm given alongside); readings of ambiguous passages are the Z-numbered
entries of DESIGN.md §3.

Modules
  attention   O1 full causal GQA forward, O2 its VJP, O3 chunk forward, O4 chunk backward
  chunkwise   O5 SeCO step (Alg. 1), O6 SpaCO step (Alg. 2)
  sampler     O8 splitmix64 index sampler and compensation / seed scales
  expectation O7 exact closed forms of E[SpaCO gradient] + subset enumeration
  multilayer  O9 L-layer RoPE + LoRA attention stack: loss and exact full-sequence gradients

Every function is pinned by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py``
against something other than itself (torch SDPA + autograd on CPU fp64, central
finite differences, closed-form special cases, invariants, published splitmix64
values, exhaustive subset enumeration).  No function is "parity unpinned".
"""
from . import attention, chunkwise, sampler, expectation, multilayer  # noqa: F401
