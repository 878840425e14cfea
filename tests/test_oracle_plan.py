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


# ---------------------------------------------------------------- further pins (round 2)
def test_eta_group_eq1():
    """Eq. 1 left side: eta(S_g) = sum_{i in S_g} L_i^2 / T^2 — SPEC S:131-133's printed
    values (two 64-token requests in one 128-tile group: 0.5; one 128-token request: 1.0) — and the
    right side of the same equation: eta_batch = sum_g eta(S_g) / G for any partition."""
    assert P.eta_group([64, 64], 128) == Fraction(1, 2)
    assert P.eta_group([128], 128) == 1
    assert P.eta_group([], 128) == 0
    rng = np.random.default_rng(5)
    for _ in range(20):
        kv = [int(x) for x in rng.integers(1, 400, size=int(rng.integers(1, 25)))]
        pl = _plan(kv, 500)
        per_group = [P.eta_group([pl.pieces[k].kv_len for k in g.members], 128) for g in pl.groups]
        assert sum(per_group) / len(pl.groups) == P.eta_batch(kv, len(pl.groups), 128)


def test_num_groups_override_hand_traces():
    """Alg. 1 line 1 with G supplied by the caller (num_groups, reading R2); hand traces on
    SPEC's instance [100, 80, 60, 40], C = 150 (natural G0 = 2):
      G = 3: 100 -> S0 (resulting 100 everywhere, lowest g); 80 -> S1 (S0: 180 > 150; S1 = S2 = 80);
             60 -> S2 (S0: 160 > 150; S1 140, S2 60); 40 -> argmin(140, 120, 100) = S2.
             Loads [100, 80, 100].
      G = 1: 100 -> S0; 80 infeasible (180 > 150) -> opens S1; 60 -> S1 (140; S0 would be
             160 > 150); 40 -> S0 (140; S1 would be 180).  Loads [140, 140], G grows 1 -> 2."""
    pl = _plan([100, 80, 60, 40], 150, num_groups=3)
    assert pl.G0 == 3
    assert [sorted(pl.pieces[k].request for k in g.members) for g in pl.groups] == [[0], [1], [2, 3]]
    assert [g.load for g in pl.groups] == [100, 80, 100]
    pl = _plan([100, 80, 60, 40], 150, num_groups=1)
    assert pl.G0 == 1
    assert [sorted(pl.pieces[k].request for k in g.members) for g in pl.groups] == [[0, 3], [1, 2]]
    assert [g.load for g in pl.groups] == [140, 140]
    # with G = 2 supplied the trace is SPEC's own
    pl = _plan([100, 80, 60, 40], 150, num_groups=2)
    assert [g.load for g in pl.groups] == [140, 140]


def test_prefix_argmin_two_group_hand_trace():
    """Reading R1 (argmin of the RESULTING load load_g + L^_i with L^_i = L_i - L^g_shared,i)
    on a batch whose prefix P0 (100 tokens) ends up in two groups.  C = 300, q_len = 1.
      r0 = P0+80 (180), r1 = 170 (no prefix), r2 = P0+60 (160), r3 = P0+20 (120), r4 = P0+90 (190)
      L_dedup = 820 - 3*100 = 520  ->  G0 = 2
      r4 190 -> S0 (tie, lowest g)                                   loads [190, 0]
      r0 180: S0 190+80 = 270, S1 0+180 = 180           -> S1          loads [190, 180]
      r1 170: S0 360 > 300, S1 350 > 300                -> opens S2    loads [190, 180, 170]
      r2 160: S0 190+60 = 250, S1 180+60 = 240, S2 330  -> S1          loads [190, 240, 170]
      r3 120: S0 190+20 = 210, S1 260, S2 290           -> S0          loads [210, 240, 170]
    Part 2 (R7-R9): S0 = [P0 | r4's 90 | r3's 20], S1 = [P0 | r0's 80 | r2's 60], S2 = [r1]."""
    kv = [180, 170, 160, 120, 190]
    pl = _plan(kv, 300, pid=[0, -1, 0, 0, 0], plen=[100])
    assert pl.G0 == 2
    assert [pl.pieces[k].request for k in pl.order] == [4, 0, 1, 2, 3]
    assert [sorted(pl.pieces[k].request for k in g.members) for g in pl.groups] == [[3, 4], [0, 2], [1]]
    assert [g.load for g in pl.groups] == [210, 240, 170]
    assert [g.base for g in pl.groups] == [0, 210, 450] and pl.buffer_tokens == 620
    off = {pl.pieces[k].request: tuple(pl.offsets[k]) for k in range(len(pl.pieces))}
    assert off == {4: (0, 100, 100, 90), 3: (0, 100, 190, 20), 0: (0, 100, 100, 80), 2: (0, 100, 180, 60),
                   1: (0, 0, 0, 170)}
    assert [(c.src_kind, c.src_id, c.src_begin, c.length, c.dst) for c in pl.copies] == [
        (1, 0, 0, 100, 0), (0, 4, 100, 90, 100), (0, 3, 100, 20, 190),
        (1, 0, 0, 100, 210), (0, 0, 100, 80, 310), (0, 2, 100, 60, 390), (0, 1, 0, 170, 450)]
    # Eq. 5: two prefix copies, below the naive per-request sum
    assert pl.io_volume() == 620 < sum(kv)


@pytest.mark.parametrize("seed", range(30))
def test_greedy_step_replay(seed):
    """SPEC S:152 "Greedy step property": replaying the assignment order against the plan's own
    final membership, every piece landed in a group that was feasible for it at that moment and had
    the least resulting load among the feasible groups (lowest index on ties), or opened a new group
    exactly when none was feasible.  The replay rebuilds the intermediate loads from the output
    (groups' member lists + order), not from the oracle's loop."""
    rng = np.random.default_rng(3000 + seed)
    C = int(rng.integers(64, 600))
    delta = int(rng.integers(0, 4))
    mem = 0 if seed % 2 else C + delta + int(rng.integers(0, 300))
    kv, q, pid, plen = _random_instance(rng, int(rng.integers(2, 40)), C)
    G_in = int(rng.integers(1, 5)) if seed % 4 == 0 else 0
    pl = P.plan(kv, q, pid, plen, C, mem_cap=mem, headroom=delta, num_groups=G_in)
    where = {k: g for g, grp in enumerate(pl.groups) for k in grp.members}
    loads = [0] * pl.G0
    members = [0] * pl.G0
    held = [set() for _ in range(pl.G0)]
    for k in pl.order:
        pc = pl.pieces[k]
        contrib = [pc.kv_len - (plen[pc.prefix] if pc.prefix >= 0 and pc.prefix in held[g] else 0)
                   for g in range(len(loads))]
        feas = [g for g in range(len(loads)) if loads[g] + contrib[g] <= C and
                (mem == 0 or loads[g] + contrib[g] + delta * (members[g] + 1) <= mem)]
        g = where[k]
        if feas:
            best = min(feas, key=lambda x: (loads[x] + contrib[x], x))
            assert g == best, (k, g, best)
        else:
            assert g == len(loads)              # a new group, opened at the end
            loads.append(0)
            members.append(0)
            held.append(set())
            contrib.append(pc.kv_len)
        loads[g] += contrib[g]
        members[g] += 1
        if pc.prefix >= 0:
            held[g].add(pc.prefix)
    assert loads == [grp.load for grp in pl.groups]


@pytest.mark.parametrize("seed", range(5))
def test_valid_pairs_count_brute_force(seed):
    """oracle.plan.valid_pairs_count (reading R11: causal within a request, block-diagonal across
    requests) against enumerating every (query, key) pair of tiny batches, plus the closed forms
    L(L+1)/2 (full prefill) and L (one decode row)."""
    rng = np.random.default_rng(seed)
    kv = rng.integers(1, 40, size=6)
    q = np.array([int(rng.integers(1, L + 1)) for L in kv])
    brute = 0
    for L, ql in zip(kv.tolist(), q.tolist()):
        for t in range(ql):
            pos = L - ql + t
            brute += sum(1 for key in range(L) if key <= pos)
    assert P.valid_pairs_count(kv, q) == brute
    assert P.valid_pairs_count([37], [37]) == 37 * 38 // 2
    assert P.valid_pairs_count([37], [1]) == 37
