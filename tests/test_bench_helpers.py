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


def test_gpus_n_self_launches_n_ranks():
    """bench.py --gpus 2 outside torchrun re-launches itself under torchrun with 2 ranks (dry-run
    hook: the ranks rendezvous over gloo on 127.0.0.1 and report the world they formed)."""
    import json
    import subprocess
    env = dict(os.environ, PI_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line == {"dryrun": True, "world": 2, "ranks_seen": 2, "kv_head_shards": [[0, 4], [4, 4]]}


def test_gpus_n_without_enough_devices_fails_loudly():
    import subprocess
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "PI_BENCH_DRYRUN", "PI_BENCH_ONE_GPU"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "only" in r.stdout


def test_stratified_oracle_sample_covers_all_strata():
    b = W.cfg2_prefill(0)
    order = bench.stratified_requests(b, 0)
    assert sorted(order) == list(range(b.n))
    # the first 8 picks come from 8 different length strata: shortest and longest requests both appear
    idx = np.argsort(b.kv_len, kind="stable")
    strata = np.array_split(idx, 8)
    first = order[:8]
    assert sorted(next(k for k, s in enumerate(strata) if i in s) for i in first) == list(range(8))
