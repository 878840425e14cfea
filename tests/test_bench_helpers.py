"""bench.py's algorithmic work counts (the numerators of every reported TFLOP/s and GB/s): pinned
by brute-force enumeration of the visible (query, key) pairs and by the configs[1] totals the
survey derived from the workload recipe (cfg 2 has 54,702 query tokens,
115,195,757 causal pairs per head, 1.887 TFLOP)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from synth import workloads as W  # noqa: E402


def brute_pairs(kv_len, q_len):
    """Visible (query, key) pairs of the prefill rows, one row at a time (q_len > 1 only: decode
    rows are counted as bytes, not FLOPs)."""
    total = 0
    for L, q in zip(kv_len.tolist(), q_len.tolist()):
        if q <= 1:
            continue
        for t in range(q):
            pos = L - q + t          # causal: keys 0..pos, prefix included (reading R11)
            total += pos + 1
    return total


@pytest.mark.parametrize("seed", range(6))
def test_prefill_flops_match_brute_force(seed):
    b = W.random_batch(seed, n=10, max_len=300, hq=8, hkv=2, d=64)
    flops, _, qo = bench.algorithmic(b, None, b.hkv)
    assert flops == 4 * b.d * b.hq * brute_pairs(b.kv_len, b.q_len)
    n_dec = int((b.q_len == 1).sum())
    assert qo == 2 * n_dec * b.hq * b.d * 2


def test_head_shard_scales_linearly():
    b = W.random_batch(3, n=8, max_len=200, hq=8, hkv=4, d=64)
    f_all, _, _ = bench.algorithmic(b, None, 4)
    f_one, _, _ = bench.algorithmic(b, None, 1)
    assert f_all == 4 * f_one


def test_cfg2_totals_from_survey():
    b = W.cfg2_prefill(0)
    assert int(b.q_len.sum()) == 54702
    pairs = brute_pairs(b.kv_len, b.q_len)
    assert pairs == 115_195_757
    flops, _, _ = bench.algorithmic(b, None, b.hkv)
    assert round(flops / 1e12, 3) == 1.887


def test_both_arms_report_the_same_config():
    b = W.cfg2_prefill(0)
    c = bench.arm_config(b, "group", 1)
    assert c == bench.arm_config(b, "group", 1)
    assert c["workload"].startswith("cfg2") and c["hq"] == 32 and c["hkv"] == 8 and c["head_dim"] == 128
    assert abs(c["algorithmic_tflop"] - 1.887367282688) < 1e-9
