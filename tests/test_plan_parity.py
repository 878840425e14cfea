"""C++ planner (libpackinfer packinfer_plan) vs the oracle planner — bit-exact, CPU only.

Compared bit-exactly (north star gate "group assignment and offset tables match the oracle"):
pieces (request, piece, kv_begin, kv_len, group), offsets O_g, groups (base, load, members,
cap), the copy plan, G0 and buffer_tokens.  The packed execution domain (work items, rows,
spans, merge map) is implementation-side and is checked by the coverage invariant: over all
work items, the multiset of admitted (row, key) cells equals the oracle's set of causally
visible (request, query position, logical key) pairs, each exactly once."""

import collections

import numpy as np
import pytest

from oracle import plan as OP
from synth import workloads as W

pk = pytest.importorskip("paper_2602_06072_b200.packinfer")


def _both(kv, q, pid, plen, C, delta=0, G=0, mem=0, r=1, chunk=1024):
    cfg = pk.default_config(capacity=C, headroom=delta, num_groups=G, mem_cap=mem, gqa_ratio=r, decode_chunk=chunk)
    hp = pk.packinfer_plan(kv, q, pid, plen, cfg)
    op = OP.plan(list(map(int, kv)), list(map(int, q)), None if pid is None else list(map(int, pid)),
                 list(map(int, plen)), C, num_groups=G, mem_cap=mem, headroom=delta)
    return hp, op


def assert_bit_exact(hp, op):
    c = hp.c
    assert c.n_pieces == len(op.pieces)
    assert c.n_groups == len(op.groups)
    assert c.g0 == op.G0
    assert c.buffer_tokens == op.buffer_tokens
    P = hp.pieces
    for k, pc in enumerate(op.pieces):
        assert tuple(P[k]) == (pc.request, pc.piece, pc.kv_begin, pc.kv_len, pc.group), k
    O = hp.offsets
    for k, o in enumerate(op.offsets):
        assert tuple(O[k]) == tuple(o), k
    Gs = hp.groups
    for g, grp in enumerate(op.groups):
        assert (int(Gs[g]["base"]), int(Gs[g]["load"]), int(Gs[g]["members"]), int(Gs[g]["cap"])) == \
            (grp.base, grp.load, len(grp.members), grp.cap), g
    Cp = hp.copies
    assert c.n_copies == len(op.copies)
    for i, cp in enumerate(op.copies):
        assert tuple(int(x) for x in Cp[i]) == (cp.src_kind, cp.src_id, cp.src_begin, cp.length, cp.dst), i
    assert c.copy_tokens == op.io_volume()
    assert c.discrepancy == op.discrepancy()


def check_coverage(hp, op, kv, q, pid, plen, r):
    """Every causally visible (request, pos, key) pair is computed exactly once."""
    kv = [int(x) for x in kv]
    q = [int(x) for x in q]
    n = len(kv)
    q_off = np.concatenate([[0], np.cumsum(q)])
    # buffer cell -> (kind, id, logical token)
    cell = {}
    for cp in op.copies:
        for t in range(cp.length):
            cell[cp.dst + t] = (cp.src_kind, cp.src_id, cp.src_begin + t)
    rows, spans = hp.rows, hp.spans
    seen = collections.Counter()
    for work, is_dec in ((hp.prefill_work, False), (hp.decode_work, True)):
        for w in work:
            sp = spans[w["span_begin"]:w["span_begin"] + w["span_count"]]
            n_kt = sum(-(-int(s["len"]) // 128) for s in sp)
            assert n_kt == w["n_ktiles"]
            assert 1 <= w["row_count"] <= 128
            for rr in rows[w["row_begin"]:w["row_begin"] + w["row_count"]]:
                tok = int(rr["q_token"])
                i = int(np.searchsorted(q_off, tok, side="right") - 1)
                pos = kv[i] - q[i] + (tok - q_off[i])
                hsub = int(rr["out"]) & 15
                assert is_dec == (q[i] == 1)
                for si, s in enumerate(sp):
                    b, e = int(s["begin"]), int(s["begin"]) + int(s["len"])
                    if si == len(sp) - 1:
                        b, e = max(b, int(rr["lo"])), min(e, int(rr["hi"]))
                    for k in range(b, e):
                        kind, sid, j = cell[k]
                        if kind == 0:
                            assert sid == i, "cross-request key"
                        else:
                            assert pid is not None and int(pid[i]) == sid, "foreign prefix"
                        seen[(i, pos, j, hsub)] += 1
    want = collections.Counter()
    for i in range(n):
        for t in range(q[i]):
            pos = kv[i] - q[i] + t
            for h in (range(r) if q[i] == 1 else [0]):
                for j in range(pos + 1):
                    want[(i, pos, j, h)] += 1
    assert seen == want


def check_merge_map(hp, q, r):
    """Rows with more than one decode item get consecutive private partial slots."""
    slots = collections.defaultdict(set)
    for w in hp.decode_work:
        for rr in hp.rows[w["row_begin"]:w["row_begin"] + w["row_count"]]:
            slot = (int(rr["out"]) >> 4) - 1
            slots[int(rr["q_token"])].add(slot)
    merged = {int(m["q_token"]): (int(m["slot_begin"]), int(m["slot_count"])) for m in hp.merges}
    used = set()
    for tok, s in slots.items():
        if tok in merged:
            b, c = merged[tok]
            assert s == set(range(b, b + c))
            assert not (used & s)
            used |= s
        else:
            assert s == {-1}
    assert len(used) == hp.c.n_partial_slots


@pytest.mark.parametrize("kv,C", [([100, 80, 60, 40], 150), ([100, 100], 100), ([90, 90, 90], 100),
                                  ([200], 150), ([7, 33, 128, 500], 8192), ([7, 33, 128, 500], 128)])
def test_spec_examples_bit_exact(kv, C):
    hp, op = _both(kv, [1] * len(kv), None, [], C)
    assert_bit_exact(hp, op)
    hp, op = _both(kv, kv, None, [], C)
    assert_bit_exact(hp, op)
    check_coverage(hp, op, kv, kv, None, [], 1)


def test_prefix_examples_bit_exact():
    for delta in (0, 8):
        hp, op = _both([60, 70], [1, 1], [0, 0], [50], 8192, delta=delta)
        assert_bit_exact(hp, op)


@pytest.mark.parametrize("name", ["toy_prefill", "toy_decode", "cfg2", "cfg3", "cfg4_decode", "cfg4_prefill", "cfg5"])
@pytest.mark.parametrize("C", [8192, 2048])
def test_configs_bit_exact(name, C):
    b = W.make_batch(name)
    hp, op = _both(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, C, delta=32, r=b.hq // b.hkv)
    assert_bit_exact(hp, op)
    check_merge_map(hp, b.q_len, b.hq // b.hkv)


@pytest.mark.parametrize("name", ["toy_prefill", "toy_decode", "cfg4_decode"])
def test_configs_coverage(name):
    b = W.make_batch(name)
    for C in (8192, 128):
        hp, op = _both(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, C, delta=3, r=b.hq // b.hkv, chunk=256)
        check_coverage(hp, op, b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hq // b.hkv)


@pytest.mark.parametrize("seed", range(300))
def test_random_bit_exact(seed):
    rng = np.random.default_rng(seed)
    C = int(rng.integers(16, 400))
    delta = int(rng.integers(0, 6))
    mem = 0 if seed % 3 else C + delta + int(rng.integers(0, 300))
    n = int(rng.integers(0, 40))
    n_prefix = int(rng.integers(0, 4))
    plen = [int(x) for x in rng.integers(1, max(2, C // 2), size=n_prefix)]
    kv, q, pid = [], [], []
    for _ in range(n):
        p = int(rng.integers(-1, n_prefix)) if n_prefix else -1
        base = plen[p] if p >= 0 else 0
        L = base + int(rng.integers(1, 3 * C))
        kv.append(L)
        q.append(1 if rng.random() < 0.4 else int(rng.integers(1, L - base + 1)))
        pid.append(p)
    G = int(rng.integers(0, 5)) if seed % 7 == 0 else 0
    hp, op = _both(kv, q, pid if n else None, plen, C, delta=delta, G=G, mem=mem, r=int(rng.integers(1, 5)))
    assert_bit_exact(hp, op)


@pytest.mark.parametrize("seed", range(25))
def test_random_coverage(seed):
    rng = np.random.default_rng(500 + seed)
    b = W.random_batch(seed, n=int(rng.integers(1, 12)), max_len=int(rng.integers(20, 400)), hq=4, hkv=2,
                       n_prefix=2, page_size=16)
    C = int(rng.integers(32, 500))
    hp, op = _both(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, C, delta=int(rng.integers(0, 4)), r=2,
                   chunk=128 * int(rng.integers(1, 3)))
    assert_bit_exact(hp, op)
    check_coverage(hp, op, b.kv_len, b.q_len, b.prefix_id, b.prefix_len, 2)
    check_merge_map(hp, b.q_len, 2)


def test_deterministic_bytes():
    b = W.cfg4_prefill()
    a1 = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, pk.default_config(headroom=32))
    a2 = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, pk.default_config(headroom=32))
    assert a1.c.arena_bytes == a2.c.arena_bytes
    assert bytes(a1.arena) == bytes(a2.arena)


@pytest.mark.parametrize("G", [1, 2, 3, 7])
def test_num_groups_override_bit_exact(G):
    """num_groups (Alg. 1 line 1 override) above and below the natural G0, on the hand-traced
    instance of tests/test_oracle_plan.py and on a prefix batch."""
    hp, op = _both([100, 80, 60, 40], [1] * 4, None, [], 150, G=G)
    assert hp.c.g0 == G
    assert_bit_exact(hp, op)
    b = W.random_batch(17, n=30, max_len=900, n_prefix=3)
    hp, op = _both(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, 700, G=G, delta=3)
    assert_bit_exact(hp, op)


def test_prefix_two_group_trace_bit_exact():
    hp, op = _both([180, 170, 160, 120, 190], [1] * 5, [0, -1, 0, 0, 0], [100], 300)
    assert_bit_exact(hp, op)
    assert [int(g["load"]) for g in hp.groups] == [210, 240, 170]


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("flags", [1, 2, 8, 2 | 8])
def test_plan_options_keep_layout_and_coverage(seed, flags):
    """PI_PLAN_NO_QPACK (1), PI_PLAN_DPACK (2) and PI_PLAN_LPT_EXACT (8) change only the execution
    domain: Parts 1-2 stay bit-exact with the oracle and every visible (request, query, key) pair is
    still computed exactly once (packed decode items: per-row intervals inside the hull)."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(3, 14))
    kv = rng.integers(2, 400, size=n).astype(np.int32)
    q = np.where(rng.random(n) < 0.6, 1, np.maximum(1, (kv * rng.random(n)).astype(np.int32))).astype(np.int32)
    pid = np.full(n, -1, np.int32)
    plen = []
    if seed % 2:
        plen = [1, 1]
        for i in range(n):
            if kv[i] - q[i] >= 2 and rng.random() < 0.5:
                pid[i] = int(rng.integers(0, 2))
                plen[pid[i]] = max(plen[pid[i]], 1)
        for p in range(2):
            mem = [i for i in range(n) if pid[i] == p]
            plen[p] = int(min(kv[i] - q[i] for i in mem)) if mem else 1
    C, r, chunk = int(rng.choice([128, 256, 1024])), int(rng.choice([1, 4])), 128
    cfg = pk.default_config(capacity=C, headroom=2, gqa_ratio=r, decode_chunk=chunk, flags=flags)
    hp = pk.packinfer_plan(kv, q, pid, plen, cfg)
    op = OP.plan(list(map(int, kv)), list(map(int, q)), list(map(int, pid)), plen, C, headroom=2)
    assert_bit_exact(hp, op)
    check_coverage(hp, op, kv, q, pid, plen, r)
    check_merge_map(hp, q, r)


@pytest.mark.parametrize("name", ["cfg3", "cfg4_decode"])
def test_default_config_packs_decode_items_within_slice_rows(name):
    """packinfer_default_config packs short decode suffixes (PI_PLAN_DPACK): a packed item - rows of
    several requests with different key intervals - never exceeds 32 rows (the kernel lane-slices
    decode units of <= 32 rows) nor a decode_chunk-long hull, and the layout (Parts 1-2) is the
    same as without the option."""
    b = W.make_batch(name)
    r = b.hq // b.hkv
    cfg = pk.default_config(gqa_ratio=r)
    assert cfg.flags == pk.PI_PLAN_DPACK
    hp = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, cfg)
    h0 = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, pk.default_config(gqa_ratio=r, flags=0))
    for f in ("pieces", "offsets", "groups", "copies"):
        assert np.array_equal(getattr(hp, f), getattr(h0, f)), f
    segs = hp.segs
    packed = 0
    for w in hp.decode_work:
        mine = [sg for sg in segs if w["row_begin"] <= sg["row_begin"] < w["row_begin"] + w["row_count"]]
        intervals = {(int(sg["lo"]), int(sg["hi"])) for sg in mine}
        if len({int(sg["q_token"]) for sg in mine}) > 1 and len(intervals) > 1:   # a packed suffix item
            packed += 1
            assert int(w["row_count"]) <= 32
            assert int(w["span_count"]) == 1 and int(hp.spans[w["span_begin"]]["len"]) <= cfg.decode_chunk
    assert packed > 0
    assert int(hp.c.n_decode_work) < int(h0.c.n_decode_work)


@pytest.mark.parametrize("seed", range(6))
def test_paged_plan_covers_logical_tokens(seed):
    """PI_PLAN_PAGED (NEXT-4 ablation): decode items over each request's logical tokens; every
    (request, GQA sub-head, key) is covered exactly once, chunk boundaries are tile multiples, and the
    block-table row rides in the item's reserved field."""
    rng = np.random.default_rng(950 + seed)
    n = int(rng.integers(2, 12))
    kv = rng.integers(1, 3000, size=n).astype(np.int32)
    q = np.ones(n, np.int32)
    r = 4
    cfg = pk.default_config(capacity=1024, gqa_ratio=r, decode_chunk=512, flags=pk.PI_PLAN_PAGED)
    hp = pk.packinfer_plan(kv, q, None, [], cfg)
    rows, spans = hp.rows, hp.spans
    seen = collections.Counter()
    for w in hp.decode_work:
        i = int(w["reserved"])
        sp = spans[w["span_begin"]]
        assert int(sp["begin"]) % 128 == 0
        for rr in rows[w["row_begin"]:w["row_begin"] + w["row_count"]]:
            assert int(rr["q_token"]) == i
            for k in range(max(int(sp["begin"]), int(rr["lo"])), min(int(sp["begin"]) + int(sp["len"]), int(rr["hi"]))):
                seen[(i, int(rr["out"]) & 15, k)] += 1
    want = collections.Counter({(i, h, k): 1 for i in range(n) for h in range(r) for k in range(int(kv[i]))})
    assert seen == want
    check_merge_map(hp, q, r)
    with pytest.raises(pk.PackInferError):
        pk.packinfer_plan(kv, np.minimum(kv, 2), None, [], cfg)   # prefill rows are rejected
