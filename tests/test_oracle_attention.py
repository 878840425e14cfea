"""Pins for the attention and merge oracles (oracle/attention.py, oracle/merge.py) — CPU only.

Pinned against: pure-Python brute force (math.fsum loops), an independent library routine
(torch scaled_dot_product_attention in float64 with an explicit boolean mask), closed forms
(single key, identical keys, q = 0), the bf16-exact mask probe, and the paper's invariants
(permutation, split-then-merge == unsplit, prefix sharing == duplicated KV)."""

import math

import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import merge as OM
from synth import workloads as W


def _brute_row(qv, K, V, scale):
    s = [scale * math.fsum(float(a) * float(b) for a, b in zip(qv, k)) for k in K]
    m = max(s)
    p = [math.exp(x - m) for x in s]
    l = math.fsum(p)
    o = [math.fsum(pj * float(V[j][c]) for j, pj in enumerate(p)) / l for c in range(len(V[0]))]
    return o, m + math.log(l)


def test_brute_force_tiny():
    b = W.random_batch(3, n=4, max_len=20, hq=2, hkv=1, d=8, n_prefix=1, page_size=16)
    t = W.make_tensors(b)
    out, lse = OA.attention(t["q"], t["k_paged"], t["v_paged"], t["block_table"], b.kv_len,
                            b.q_len, b.page_size)
    q = t["q"].double().numpy()
    kp, vp = t["k_paged"].double().numpy(), t["v_paged"].double().numpy()
    bt = t["block_table"].numpy()
    row = 0
    for i in range(b.n):
        L, ql = int(b.kv_len[i]), int(b.q_len[i])
        for tq in range(ql):
            pos = L - ql + tq
            for h in range(b.hq):
                K = [kp[bt[i, j // 16], j % 16, h // 2] for j in range(pos + 1)]
                V = [vp[bt[i, j // 16], j % 16, h // 2] for j in range(pos + 1)]
                o, l = _brute_row(q[row, h], K, V, 1 / math.sqrt(8))
                assert np.allclose(out[row, h], o, rtol=0, atol=1e-12)
                assert abs(lse[h, row] - l) < 1e-12
            row += 1


@pytest.mark.parametrize("seed", range(3))
def test_against_torch_sdpa(seed):
    """Independent library routine: SDPA(float64) with an explicit boolean causal mask."""
    b = W.random_batch(seed, n=6, max_len=300, hq=4, hkv=2, d=32)
    t = W.make_tensors(b)
    out, lse = OA.attention(t["q"], t["k_paged"], t["v_paged"], t["block_table"], b.kv_len,
                            b.q_len, b.page_size)
    bt = t["block_table"]
    kp, vp = t["k_paged"].double(), t["v_paged"].double()
    off = 0
    for i in range(b.n):
        L, ql = int(b.kv_len[i]), int(b.q_len[i])
        j = torch.arange(L)
        K = kp[bt[i, j // b.page_size].long(), j % b.page_size]        # [L, Hkv, d]
        V = vp[bt[i, j // b.page_size].long(), j % b.page_size]
        K = K.repeat_interleave(b.hq // b.hkv, dim=1).transpose(0, 1)  # [Hq, L, d]
        V = V.repeat_interleave(b.hq // b.hkv, dim=1).transpose(0, 1)
        Q = t["q"][off:off + ql].double().transpose(0, 1)              # [Hq, ql, d]
        pos = L - ql + torch.arange(ql)
        mask = torch.arange(L)[None, :] <= pos[:, None]
        ref = torch.nn.functional.scaled_dot_product_attention(Q, K, V, attn_mask=mask)
        assert np.allclose(out[off:off + ql], ref.transpose(0, 1).numpy(), rtol=0, atol=1e-12)
        off += ql


def _single_request_batch(kv, q, d=16, hq=2, hkv=1):
    return W.Batch("t", np.array([kv], np.int32), np.array([q], np.int32), np.array([-1], np.int32),
                   np.zeros(0, np.int32), hq, hkv, d, "fp32", 16, 5)


def test_closed_form_single_key():
    b = _single_request_batch(1, 1)
    t = W.make_tensors(b)
    out, lse = OA.attention(t["q"], t["k_paged"], t["v_paged"], t["block_table"], b.kv_len, b.q_len, 16)
    v0 = t["v_paged"][t["block_table"][0, 0], 0, 0].double().numpy()
    assert np.array_equal(out[0, 0], v0) and np.array_equal(out[0, 1], v0)
    s = float((t["q"][0, 0].double() @ t["k_paged"][t["block_table"][0, 0], 0, 0].double()) / 4.0)
    assert abs(lse[0, 0] - s) < 1e-12


def test_closed_form_identical_keys_and_zero_query():
    b = _single_request_batch(40, 5)
    t = W.make_tensors(b)
    kp = t["k_paged"].clone()
    kp[:] = kp[0, 0, 0]                                   # identical keys -> mean of V
    out, _ = OA.attention(t["q"], kp, t["v_paged"], t["block_table"], b.kv_len, b.q_len, 16)
    q0 = torch.zeros_like(t["q"])                          # q = 0 -> mean of V, lse = ln(n)
    out0, lse0 = OA.attention(q0, t["k_paged"], t["v_paged"], t["block_table"], b.kv_len, b.q_len, 16)
    vp = t["v_paged"].double().numpy()
    bt = t["block_table"].numpy()
    for tq in range(5):
        pos = 35 + tq
        V = np.stack([vp[bt[0, j // 16], j % 16, 0] for j in range(pos + 1)])
        assert np.allclose(out[tq, 0], V.mean(0), atol=1e-12)
        assert np.allclose(out0[tq, 0], V.mean(0), atol=1e-12)
        assert abs(lse0[0, tq] - math.log(pos + 1)) < 1e-12


def test_mask_probe_oracle():
    """q = 0 and V channel 0 = request id (exact in bf16): any cross-request leak changes o[0];
    exp(lse) counts the visible keys exactly (pos + 1)."""
    b = W.random_batch(7, n=8, max_len=300, hq=4, hkv=2, d=16)
    t = W.make_tensors(b)
    q0 = torch.zeros_like(t["q"])
    vp = t["v_paged"].clone()
    bt = t["block_table"].numpy()
    # stamp request ids on each request's own (non-prefix) blocks; prefix blocks get -1
    vp[..., 0] = -1.0
    for i in range(b.n):
        base = int(b.prefix_len[b.prefix_id[i]]) if b.prefix_id[i] >= 0 else 0
        for j in range(base // b.page_size, -(-int(b.kv_len[i]) // b.page_size)):
            vp[bt[i, j], :, :, 0] = float(i)
    out, lse = OA.attention(q0, t["k_paged"], vp, t["block_table"], b.kv_len, b.q_len, b.page_size)
    off = 0
    for i in range(b.n):
        L, ql = int(b.kv_len[i]), int(b.q_len[i])
        base = int(b.prefix_len[b.prefix_id[i]]) if b.prefix_id[i] >= 0 else 0
        for tq in range(ql):
            pos = L - ql + tq
            n_own = pos + 1 - base
            want = (n_own * i + base * -1.0) / (pos + 1)
            assert abs(out[off + tq, 0, 0] - want) < 1e-12
            assert round(math.exp(lse[0, off + tq])) == pos + 1
        off += ql


def test_permutation_invariance():
    b = W.random_batch(11, n=6, max_len=200, hq=2, hkv=1, d=16, n_prefix=0)
    t = W.make_tensors(b)
    out, _ = OA.attention(t["q"], t["k_paged"], t["v_paged"], t["block_table"], b.kv_len, b.q_len, b.page_size)
    perm = np.random.default_rng(0).permutation(b.n)
    qoff = np.concatenate([[0], np.cumsum(b.q_len)])
    qp = torch.cat([t["q"][qoff[i]:qoff[i + 1]] for i in perm])
    out2, _ = OA.attention(qp, t["k_paged"], t["v_paged"], t["block_table"][torch.from_numpy(perm)],
                           b.kv_len[perm], b.q_len[perm], b.page_size)
    pos = 0
    for i in perm:
        n = int(b.q_len[i])
        assert np.array_equal(out2[pos:pos + n], out[qoff[i]:qoff[i] + n])
        pos += n


def test_split_then_merge_equals_unsplit():
    """P:61 lossless split-merge: any contiguous segmentation merged with the LSE rule equals the
    unsplit row (fp64, <= 1e-12)."""
    rng = np.random.default_rng(0)
    for trial in range(60):
        L, d = int(rng.integers(2, 256)), 16
        K = rng.standard_normal((L, d))
        V = rng.standard_normal((L, d))
        qv = rng.standard_normal(d) * (4 if trial % 3 == 0 else 1)
        full = OA.partial_attention(qv, K, V, 0.25)
        cuts = sorted(set(rng.integers(1, L, size=int(rng.integers(1, 8))).tolist()))
        bounds = [0] + cuts + [L]
        parts = [OA.partial_attention(qv, K[a:b], V[a:b], 0.25) for a, b in zip(bounds, bounds[1:])]
        o, l = OM.merge(parts)
        assert np.abs(o - full[0]).max() <= 1e-12 and abs(l - full[1]) <= 1e-12


def test_merge_identity_order_and_adversarial():
    rng = np.random.default_rng(1)
    o = rng.standard_normal(8)
    got = OM.merge([(o, 3.5)])
    assert np.array_equal(got[0], o) and got[1] == 3.5
    parts = [(rng.standard_normal(8), float(x)) for x in rng.uniform(-700, 700, size=3)]
    a = OM.merge2(OM.merge2(parts[0], parts[1]), parts[2])
    b = OM.merge2(parts[0], OM.merge2(parts[1], parts[2]))
    assert np.abs(a[0] - b[0]).max() <= 1e-12 and abs(a[1] - b[1]) <= 1e-9
    assert np.all(np.isfinite(a[0]))
    empty = (np.zeros(8), -math.inf)
    c = OM.merge([empty, parts[0]])
    assert np.array_equal(c[0], parts[0][0]) and c[1] == parts[0][1]
    z = OM.merge([empty, empty])
    assert np.array_equal(z[0], np.zeros(8)) and z[1] == -math.inf


def test_prefix_sharing_equals_duplicated_kv():
    """Prefix pages shared through the block table == every request holding a private copy."""
    b = W.random_batch(5, n=8, max_len=150, hq=2, hkv=1, d=16, prefix_frac=1.0, decode_frac=0.5)
    t = W.make_tensors(b)
    out, lse = OA.attention(t["q"], t["k_paged"], t["v_paged"], t["block_table"], b.kv_len, b.q_len, b.page_size)
    # duplicate: give every request private copies of its prefix blocks
    kp, vp = [t["k_paged"]], [t["v_paged"]]
    bt = t["block_table"].clone()
    nxt = t["k_paged"].shape[0]
    for i in range(b.n):
        p = int(b.prefix_id[i])
        if p < 0:
            continue
        for j in range(int(b.prefix_len[p]) // b.page_size):
            src = int(bt[i, j])
            kp.append(t["k_paged"][src:src + 1])
            vp.append(t["v_paged"][src:src + 1])
            bt[i, j] = nxt
            nxt += 1
    out2, lse2 = OA.attention(t["q"], torch.cat(kp), torch.cat(vp), bt, b.kv_len, b.q_len, b.page_size)
    assert np.array_equal(out, out2) and np.array_equal(lse, lse2)


def test_attention_rows_matches_full():
    b = W.random_batch(9, n=5, max_len=260, hq=4, hkv=2, d=16)
    t = W.make_tensors(b)
    out, lse = OA.attention(t["q"], t["k_paged"], t["v_paged"], t["block_table"], b.kv_len, b.q_len, b.page_size)
    rows = [(i, tq) for i in range(b.n) for tq in range(int(b.q_len[i])) if (i + tq) % 7 == 0]
    o2, l2 = OA.attention_rows(t["q"], t["k_paged"], t["v_paged"], t["block_table"], b.kv_len,
                               b.q_len, b.page_size, rows)
    qoff = np.concatenate([[0], np.cumsum(b.q_len)])
    for n, (i, tq) in enumerate(rows):
        assert np.allclose(o2[n], out[qoff[i] + tq], atol=1e-12)
        assert np.allclose(l2[n], lse[:, qoff[i] + tq], atol=1e-12)
