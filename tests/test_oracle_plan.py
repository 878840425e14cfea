"""Pins for the planner oracle (oracle/plan.py) — CPU only.

Each test pins the oracle to something other than itself: the SPEC hand traces of Alg. 1
(tests/golden/plan_examples.json, each entry cited), hand-derived toy pins, exhaustive
brute force on tiny instances, and layout round-trips against the paged cache."""

import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import plan as P
from oracle import layout as OL
from synth import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "plan_examples.json")))


def _plan(kv, C, q=None, pid=None, plen=(), **kw):
    kv = list(kv)
    q = [1] * len(kv) if q is None else list(q)
    return P.plan(kv, q, pid, list(plen), C, **kw)


@pytest.mark.parametrize("ex", GOLD["greedy"], ids=lambda e: e["cite"])
def test_greedy_hand_traces(ex):
    pl = _plan(ex["kv_len"], ex["capacity"])
    groups = [sorted(pl.pieces[k].request for k in g.members) for g in pl.groups]
    assert groups == ex["groups"]
    assert [g.load for g in pl.groups] == ex["loads"]
    assert len(pl.groups) == ex["G"]
    assert pl.discrepancy() == ex["discrepancy"]


@pytest.mark.parametrize("ex", GOLD["split"], ids=lambda e: e["cite"])
def test_split_rule(ex):
    assert [list(s) for s in P.split_long(ex["L"], ex["capacity"])] == ex["pieces"]
    pl = _plan([ex["L"]], ex["capacity"])
    assert [(p.kv_begin, p.kv_len) for p in pl.pieces] == [tuple(s) for s in ex["pieces"]]
    # pieces of one request land in distinct groups (any two pieces sum to > C)
    assert len({p.group for p in pl.pieces}) == len(pl.pieces)


@pytest.mark.parametrize("ex", GOLD["eta"], ids=lambda e: e["cite"])
def test_eta_eq1(ex):
    assert P.eta_batch(ex["lengths"], ex["G"], ex["T"]) == Fraction(ex["num"], ex["den"])


def test_eq5_dedup_volume():
    ex = GOLD["eq5"][0]
    LP = ex["prefix_len"]
    kv = [LP + s for s in ex["suffixes"]]
    pl = _plan(kv, 8192, pid=[0, 0, 0], plen=[LP])
    assert pl.io_volume() == ex["io"]
    assert sum(kv) == ex["naive"]
    assert len(pl.groups) == 1
    # exactly one prefix copy
    assert sum(1 for c in pl.copies if c.src_kind == 1) == 1
    assert sum(c.length for c in pl.copies) == ex["io"]


@pytest.mark.parametrize("ex", GOLD["consolidate"][:2], ids=lambda e: e["cite"])
def test_consolidate_prefix_example(ex):
    LP = ex["prefix_len"]
    kv = [LP + ex["suffixes"]["r1"], LP + ex["suffixes"]["r2"]]     # request 0 = r1, 1 = r2
    pl = _plan(kv, 8192, pid=[0, 0], plen=[LP], headroom=ex["headroom"])
    off = {pl.pieces[k].request: pl.offsets[k] for k in range(len(pl.pieces))}
    assert list(off[0]) == ex["offsets"]["r1"]
    assert list(off[1]) == ex["offsets"]["r2"]
    assert pl.groups[0].cap == ex["cursor"]


def test_consolidate_single():
    ex = GOLD["consolidate"][2]
    pl = _plan([ex["single_L"]], 8192, headroom=ex["headroom"])
    assert list(pl.offsets[0]) == ex["offsets"]
    assert pl.buffer_tokens == ex["cursor"]


def test_toy_pins():
    a, b = GOLD["toy"]
    pl = _plan(a["kv_len"], a["capacity"], q=a["kv_len"])
    assert len(pl.groups) == a["G"]
    for k, pc in enumerate(pl.pieces):
        assert list(pl.offsets[k]) == a["offsets_by_request"][str(pc.request)]
    pl = _plan(b["kv_len"], b["capacity"], q=b["kv_len"])
    assert pl.G0 == b["G0"]
    assert [g.load for g in pl.groups] == b["loads"]
    for k, pc in enumerate(pl.pieces):
        assert pc.group == b["piece_groups"][f"{pc.request}.{pc.piece}"]
        key = f"{pc.request}.{pc.piece}"
        if key in b["offsets"]:
            assert list(pl.offsets[k]) == b["offsets"][key]


def test_regroup_eq4():
    ex = GOLD["regroup"][0]
    for dL, t_expect in zip(ex["dL"], ex["fires_at"]):
        t = next(t for t in range(1, 10000) if P.should_regroup(t, dL, ex["C"]))
        assert t == t_expect
    assert P.should_regroup(4, 1024, 8192)          # boundary inclusive: 4*1024 == 8192/2
    assert not P.should_regroup(3, 1024, 8192)


def test_validation_errors():
    with pytest.raises(P.PlanError):
        _plan([0], 10)
    with pytest.raises(P.PlanError):
        _plan([10], 10, q=[11])
    with pytest.raises(P.PlanError):
        _plan([10], 10, q=[5], pid=[0], plen=[6])     # prefix would hold query rows
    with pytest.raises(P.PlanError):
        _plan([10], 10, pid=[3], plen=[5])            # prefix id out of range
    pl = _plan([], 10)
    assert pl.pieces == [] and pl.groups == [] and pl.buffer_tokens == 0


# ---------------------------------------------------------------- properties on random inputs
def _random_instance(rng, n, C, with_prefix=True):
    n_prefix = 3 if with_prefix else 0
    plen = [int(x) for x in rng.integers(1, max(2, C // 3), size=n_prefix)]
    kv, q, pid = [], [], []
    for _ in range(n):
        p = int(rng.integers(-1, n_prefix)) if n_prefix else -1
        base = plen[p] if p >= 0 else 0
        L = base + int(rng.integers(1, 2 * C))
        kv.append(L)
        q.append(int(rng.integers(1, L - base + 1)))
        pid.append(p)
    return kv, q, pid, plen


@pytest.mark.parametrize("seed", range(40))
def test_plan_invariants(seed):
    rng = np.random.default_rng(seed)
    C = int(rng.integers(16, 300))
    delta = int(rng.integers(0, 5))
    mem = 0 if seed % 3 else C + delta + int(rng.integers(0, 200))
    kv, q, pid, plen = _random_instance(rng, int(rng.integers(1, 30)), C)
    pl = P.plan(kv, q, pid, plen, C, mem_cap=mem, headroom=delta,
                num_groups=int(rng.integers(0, 4)) if seed % 5 == 0 else 0)
    # partition: each request's pieces cover [0, L) disjointly, in order
    by_req = {}
    for pc in pl.pieces:
        by_req.setdefault(pc.request, []).append((pc.kv_begin, pc.kv_len))
    for i, L in enumerate(kv):
        segs = sorted(by_req[i])
        assert segs[0][0] == 0 and sum(s[1] for s in segs) == L
        assert all(a[0] + a[1] == b[0] for a, b in zip(segs, segs[1:]))
    # every piece assigned exactly once
    assigned = sorted(k for g in pl.groups for k in g.members)
    assert assigned == list(range(len(pl.pieces)))
    # capacity (Eq. 2) and memory terms
    for g in pl.groups:
        assert g.load <= C
        if mem:
            assert g.load + delta * len(g.members) <= mem
        assert g.cap == g.load + delta * len(g.members)
    # G monotonicity
    assert len(pl.groups) >= pl.G0
    # Eq. 5: copy volume == sum of loads; buffers partition [0, buffer_tokens) up to headroom
    assert sum(c.length for c in pl.copies) == pl.io_volume()
    assert pl.buffer_tokens == sum(g.cap for g in pl.groups)
    # eta invariance: depends only on G
    G = len(pl.groups)
    assert P.eta_batch(kv, G, 128) == Fraction(sum(L * L for L in kv), G * 128 * 128)


def _brute_force(lengths, C, G):
    """Exhaustive optimum of Eq. 3 under capacity (no prefixes), and its max load."""
    best = None
    for assign in itertools.product(range(G), repeat=len(lengths)):
        if assign[0] != 0:
            continue
        loads = [0] * G
        for L, g in zip(lengths, assign):
            loads[g] += L
        if max(loads) > C:
            continue
        key = (max(loads) - min(loads), max(loads))
        if best is None or key < best:
            best = key
    return best


@pytest.mark.parametrize("seed", range(60))
def test_greedy_vs_brute_force(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 8))
    C = int(rng.integers(20, 100))
    kv = [int(x) for x in rng.integers(1, C + 1, size=n)]
    pl = _plan(kv, C)
    G = len(pl.groups)
    opt = _brute_force(kv, C, G)
    assert opt is not None
    greedy_disc = pl.discrepancy()
    assert greedy_disc >= opt[0]
    # greedy max load within 4/3 of the brute-force minimum max-load at the same G
    best_max = min(
        max(sum(L for L, g in zip(kv, a) if g == gg) for gg in range(G))
        for a in itertools.product(range(G), repeat=n)
        if all(sum(L for L, g in zip(kv, a) if g == gg) <= C for gg in range(G)))
    assert 3 * max(g.load for g in pl.groups) <= 4 * best_max


@pytest.mark.parametrize("seed", range(12))
def test_layout_round_trip(seed):
    """Part 2 consolidation is lossless: every piece's logical KV is recovered from the group
    buffer through its offset-table entry and equals the paged cache."""
    b = W.random_batch(seed, n=10, max_len=400)
    t = W.make_tensors(b, device="cpu")
    C = int(np.random.default_rng(seed).integers(128, 900))
    pl = P.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, C, headroom=seed % 4)
    buf, valid = OL.expected_buffers(pl.copies, t["k_paged"], t["block_table"], b.n,
                                     b.page_size, pl.buffer_tokens)
    kp = t["k_paged"].view(__import__("torch").int16).numpy()
    bt = t["block_table"].numpy()
    for k, pc in enumerate(pl.pieces):
        dp, lp, ds, lq = pl.offsets[k]
        base = pl.groups[pc.group].base
        got = np.concatenate([buf[:, base + dp:base + dp + lp], buf[:, base + ds:base + ds + lq]], axis=1)
        j = np.arange(pc.kv_begin, pc.kv_begin + pc.kv_len)
        want = kp[bt[pc.request, j // b.page_size], j % b.page_size].transpose(1, 0, 2)
        assert lp + lq == pc.kv_len
        assert np.array_equal(got, want)
    # single-copy prefixes: each prefix copied at most once per group
    seen = set()
    for c in pl.copies:
        if c.src_kind == 1:
            g = next(gi for gi, g in enumerate(pl.groups) if g.base <= c.dst < g.base + g.cap)
            assert (g, c.src_id) not in seen
            seen.add((g, c.src_id))


def test_cfg4_prefix_colocation():
    """The prefix-aware greedy co-locates shared prefixes: far fewer KV tokens than the
    naive per-request sum, and well above the ideal of one copy per prefix."""
    b = W.cfg4_decode()
    pl = P.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, 8192, headroom=32)
    naive = int(b.kv_len.sum())
    ideal = int(b.prefix_len.sum() + (b.kv_len - 2048).sum())
    assert ideal < pl.io_volume() < 0.5 * naive
    assert sum(1 for c in pl.copies if c.src_kind == 1) <= 64
