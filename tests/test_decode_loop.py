"""Decode loop without re-consolidation (NEXT-1; Eq. 4, P:306-309 headroom) — CPU parts.

packinfer_plan_step(appended) must keep the consolidation's layout bit-identical (groups, offsets,
copies) and extend only the execution domain: every decode row sees exactly kv_len + appended keys,
the new tokens living in the suffix headroom slots the plan hands out (append_pos)."""

import collections

import numpy as np
import pytest

from oracle import plan as OP
from synth import workloads as W

pk = pytest.importorskip("paper_2602_06072_b200.packinfer")


def _plans(b, C, delta, appended, r=4, chunk=256):
    cfg = pk.default_config(capacity=C, headroom=delta, gqa_ratio=r, decode_chunk=chunk)
    base = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, cfg)
    step = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, cfg, appended=appended)
    return base, step


def _decode_batch(seed, n=16):
    b = W.random_batch(seed, n=n, max_len=900, hq=8, hkv=2, d=64, n_prefix=2, decode_frac=0.7, page_size=128)
    return b


@pytest.mark.parametrize("seed", range(10))
def test_layout_unchanged_and_slots_in_headroom(seed):
    b = _decode_batch(seed)
    rng = np.random.default_rng(seed)
    delta = 6
    appended = np.where(b.q_len == 1, rng.integers(0, delta + 1, size=b.n), 0).astype(np.int32)
    base, step = _plans(b, int(rng.integers(200, 2000)), delta, appended)
    for name in ("pieces", "offsets", "groups", "copies"):
        assert np.array_equal(getattr(base, name), getattr(step, name)), name
    assert base.c.buffer_tokens == step.c.buffer_tokens
    # append slots: right after the grown suffix, inside its headroom, never a copied cell
    P, O, G = step.pieces, step.offsets, step.groups
    copied = np.zeros(int(step.c.buffer_tokens), bool)
    for c in step.copies:
        copied[int(c["dst"]):int(c["dst"]) + int(c["len"])] = True
    last_piece = {}
    for k, pc in enumerate(P):
        last_piece[int(pc["request"])] = k
    for i in range(b.n):
        pos = int(step.append_pos[i])
        if b.q_len[i] != 1 or appended[i] == delta:
            assert pos == -1
            continue
        k = last_piece[i]
        end = int(G[int(P[k]["group"])]["base"]) + int(O[k]["d_suffix"]) + int(O[k]["l_suffix"])
        assert pos == end + int(appended[i])
        assert end <= pos < end + delta
        assert not copied[pos]


@pytest.mark.parametrize("seed", range(8))
def test_step_coverage(seed):
    """Every (decode row, GQA head) sees exactly its kv_len + appended logical keys once."""
    b = _decode_batch(100 + seed, n=10)
    rng = np.random.default_rng(seed)
    delta, r = 5, 4
    appended = np.where(b.q_len == 1, rng.integers(0, delta + 1, size=b.n), 0).astype(np.int32)
    C = int(rng.integers(150, 1200))
    _, step = _plans(b, C, delta, appended, r=r, chunk=128)
    op = OP.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, C, headroom=delta)
    cell = {}
    for cp in op.copies:
        for t in range(cp.length):
            cell[cp.dst + t] = (cp.src_kind, cp.src_id, cp.src_begin + t)
    for k, pc in enumerate(op.pieces):       # appended tokens sit in the last piece's headroom
        i = pc.request
        if k == max(kk for kk, p2 in enumerate(op.pieces) if p2.request == i):
            end = op.groups[pc.group].base + op.offsets[k][2] + op.offsets[k][3]
            for a in range(int(appended[i])):
                cell[end + a] = (0, i, int(b.kv_len[i]) + a)
    q_off = np.concatenate([[0], np.cumsum(b.q_len)])
    seen = collections.Counter()
    rows, spans = step.rows, step.spans
    for w in step.decode_work:
        sp = spans[w["span_begin"]:w["span_begin"] + w["span_count"]]
        for rr in rows[w["row_begin"]:w["row_begin"] + w["row_count"]]:
            i = int(np.searchsorted(q_off, int(rr["q_token"]), side="right") - 1)
            for s_i, s in enumerate(sp):
                lo, hi = int(s["begin"]), int(s["begin"]) + int(s["len"])
                if s_i == len(sp) - 1:
                    lo, hi = max(lo, int(rr["lo"])), min(hi, int(rr["hi"]))
                for key in range(lo, hi):
                    kind, sid, j = cell[key]
                    assert (kind == 0 and sid == i) or (kind == 1 and sid == int(b.prefix_id[i]))
                    seen[(i, int(rr["out"]) & 15, j)] += 1
    want = collections.Counter()
    for i in range(b.n):
        if b.q_len[i] == 1:
            for h in range(r):
                for j in range(int(b.kv_len[i]) + int(appended[i])):
                    want[(i, h, j)] += 1
    assert seen == want


def test_headroom_exhausted_and_validation():
    b = _decode_batch(3)
    dec = np.where(b.q_len == 1)[0]
    appended = np.zeros(b.n, np.int32)
    appended[dec[0]] = 5
    with pytest.raises(pk.PackInferError) as e:
        _plans(b, 1000, 4, appended)
    assert e.value.status == pk.PI_EREGROUP
    pre = np.where(b.q_len > 1)[0]
    if len(pre):
        bad = np.zeros(b.n, np.int32)
        bad[pre[0]] = 1
        with pytest.raises(pk.PackInferError) as e:
            _plans(b, 1000, 4, bad)
        assert e.value.status == pk.PI_EINVAL


def test_drift_and_eq4_against_oracle():
    """drift = max_g L - min_g L including appended tokens; Eq. 4 helper == oracle."""
    b = _decode_batch(5, n=24)
    delta = 8
    for k in range(0, delta + 1):
        appended = np.where(b.q_len == 1, k, 0).astype(np.int32)
        _, step = _plans(b, 1500, delta, appended)
        loads = [int(g["load"]) for g in step.groups]
        for i in range(b.n):
            if b.q_len[i] == 1:
                last = [kk for kk, pc in enumerate(step.pieces) if int(pc["request"]) == i][-1]
                loads[int(step.pieces[last]["group"])] += k
        assert step.c.drift == max(loads) - min(loads)
    for C in (8192, 4096, 1000):
        for dL in (0, 1, 103, 128, 204, 5000):
            for t in range(0, 60):
                assert pk.packinfer_should_regroup(t, dL, C) == OP.should_regroup(t, dL, C)
