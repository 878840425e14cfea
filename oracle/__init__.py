"""PackInfer oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the PackInfer hot path
(arXiv 2602.06072) computes, written from the paper (`PAPER.md`, cited as ``P:<line>``)
and the readings recorded in ``DESIGN.md`` §3 (which follow ``SURVEY.md`` §8(c)).

Rules (task ③):
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
    ``--impl reference`` legs may import anything under ``oracle/``.  The product package
    ``paper_2602_06072_b200`` never imports it and has no CPU fallback.
  * The oracle shares no code with the CUDA path: no kernels, headers, helpers, tables or
    constant generators.  Only the seeded input generators in ``synth/`` (which hold none of
    the method's arithmetic) serve both sides.
  * Floating point is fp64 (inputs are upcast exactly from bf16/fp32); planner arithmetic is
    Python integers (unbounded, so int64 overflow cannot hide a bug).

Modules:
  plan       — Alg. 1 Part 1 + Part 2 with prefix-aware L̂, Eq. 1/3/5.
  attention  — per-request causal softmax attention, naive (materialised) softmax, fp64.
  merge      — log-sum-exp merge of partial attention outputs ("lossless ... FlashAttention
               semantics"; equations per DESIGN.md reading R10).
  layout     — expected group-contiguous KV buffers from the copy plan (Alg. 1 Copy lines).

Every function is pinned by ``tests/test_oracle_*.py`` against something other than itself
(paper/SPEC worked examples, closed forms, brute force, an independent library routine).
"""

from . import plan, attention, merge, layout  # noqa: F401
