"""Seeded synthetic workload generators shared by the oracle tests, the GPU parity tests and
bench.py.  Holds NONE of PackInfer's arithmetic: only request lengths, prefix ids, random
tensors and the (shuffled) paged KV-cache placement that stand in for a serving engine's
state.  Recipes: DESIGN.md §4 (from SURVEY.md §8(d) and P:161)."""

from .workloads import (  # noqa: F401
    Batch, CONFIGS, make_batch, make_tensors, toy_prefill, toy_decode, cfg2_prefill,
    cfg3_decode, cfg4_decode, cfg4_prefill, cfg5_mixed, random_batch,
)
