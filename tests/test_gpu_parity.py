"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Gate (BASELINE.json north star): bf16 inputs / fp32 accumulation within 1e-2 max-abs and 1e-3
mean-abs of the oracle; relayout bitwise; LSE within 1e-3 (fp32 statistics; tf32 toy: 5e-3).
Sizes span several 128-row/128-key tiles, ragged tails, packed short requests, shared
prefixes, split requests (C small) and decode chunks with partials + merge."""

import math

import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import layout as OL
from oracle import plan as OP
from synth import workloads as W

pytestmark = pytest.mark.gpu

H = pytest.importorskip("tests.gpu_helpers")


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("C,delta", [(8192, 0), (300, 5), (128, 0)])
def test_relayout_bitwise(C, delta):
    b = W.random_batch(1, n=12, max_len=500, hq=8, hkv=4, d=128, n_prefix=2)
    t = W.make_tensors(b, device="cuda")
    _, _, pb = H.run_batch(b, t, C=C, delta=delta)
    op = OP.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, C, headroom=delta)
    for buf_gpu, src in ((pb.k_buf, "k_paged"), (pb.v_buf, "v_paged")):
        want, valid = OL.expected_buffers(op.copies, t[src].cpu(), t["block_table"].cpu(), b.n, b.page_size,
                                          op.buffer_tokens)
        got = buf_gpu.cpu().view(torch.int16).numpy()
        assert np.array_equal(got[:, valid], want[:, valid])
        assert (got[:, ~valid] == 0).all()           # headroom zero-filled


def test_relayout_bitwise_full_bf16_range():
    """K and V cells are bitwise copies over the whole finite bf16 range: values far outside fp16
    (|x| up to 3e38, subnormal bf16 down to 1e-40) and signed zeros survive the relayout."""
    b = W.random_batch(3, n=9, max_len=400, hq=4, hkv=2, d=128, n_prefix=1)
    t = W.make_tensors(b, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    for name in ("k_paged", "v_paged"):
        x = t[name].float()
        e = torch.randint(-133, 127, x.shape, generator=g, device="cuda").float()   # exponents incl. subnormal
        t[name] = (x * torch.exp2(e)).to(torch.bfloat16)
        t[name].view(-1)[:7] = torch.tensor([0.0, -0.0, 1e-40, -3e38, 65520.0, 1e5, 6e-8],
                                            device="cuda").to(torch.bfloat16)
    assert torch.isfinite(t["v_paged"].float()).all()
    _, _, pb = H.run_batch(b, t, C=256, delta=3)
    op = OP.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, 256, headroom=3)
    for buf_gpu, src in ((pb.k_buf, "k_paged"), (pb.v_buf, "v_paged")):
        want, valid = OL.expected_buffers(op.copies, t[src].cpu(), t["block_table"].cpu(), b.n, b.page_size,
                                          op.buffer_tokens)
        got = buf_gpu.cpu().view(torch.int16).numpy()
        assert np.array_equal(got[:, valid], want[:, valid])


@pytest.mark.parametrize("k", [17, -20])
def test_v_scale_equivariance(k):
    """Attention is linear in V (o(q, K, c V) = c o(q, K, V), the oracle's definition): scaling V by
    2^k (|v| ~ 1e5 for k = 17, far beyond fp16; ~1e-6 for k = -20, fp16-subnormal) scales every output
    exactly — bf16 P x bf16 V with fp32 accumulation commutes with a power-of-two scale — and the
    scaled outputs meet the gate after dividing by 2^k."""
    b = W.random_batch(13, n=10, max_len=700, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=0.4)
    t = W.make_tensors(b, device="cuda")
    o1, l1, _ = H.run_batch(b, t, C=300, decode_chunk=256, out_f32=True)
    ts = dict(t)
    ts["v_paged"] = (t["v_paged"].float() * 2.0 ** k).to(torch.bfloat16)
    assert torch.equal(ts["v_paged"].float(), t["v_paged"].float() * 2.0 ** k)   # exact in bf16
    o2, l2, _ = H.run_batch(b, ts, C=300, decode_chunk=256, out_f32=True)
    assert torch.equal(o2, o1 * 2.0 ** k)
    assert torch.equal(l2, l1)
    ro, rl = H.oracle_full(b, ts)
    H.compare(o2 * 2.0 ** -k, l2, ro * 2.0 ** -k, rl)


@pytest.mark.parametrize("delta", [0, 5])
def test_relayout_many_copies(delta):
    """~2k copy entries: the relayout's 32-ary copy-entry search takes several rounds, and buffer
    cells sit on every kind of entry boundary (prefix / suffix / headroom / group base)."""
    b = W.random_batch(9, n=2000, max_len=24, hq=4, hkv=2, d=64, n_prefix=3)
    t = W.make_tensors(b, device="cuda")
    _, _, pb = H.run_batch(b, t, C=256, delta=delta)
    op = OP.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, 256, headroom=delta)
    assert len(op.copies) > 1024
    want, valid = OL.expected_buffers(op.copies, t["k_paged"].cpu(), t["block_table"].cpu(), b.n, b.page_size,
                                      op.buffer_tokens)
    got = pb.k_buf.cpu().view(torch.int16).numpy()
    assert np.array_equal(got[:, valid], want[:, valid])
    assert (got[:, ~valid] == 0).all()


def test_relayout_head_slice():
    b = W.random_batch(2, n=6, max_len=300, hq=8, hkv=4, d=64)
    t = W.make_tensors(b, device="cuda")
    _, _, pb = H.run_batch(b, t, hkv_begin=1, hkv_count=2)
    op = OP.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, 8192)
    want, valid = OL.expected_buffers(op.copies, t["k_paged"].cpu(), t["block_table"].cpu(), b.n, b.page_size,
                                      op.buffer_tokens, heads=[1, 2])
    got = pb.k_buf.cpu().view(torch.int16).numpy()
    assert np.array_equal(got[:, valid], want[:, valid])


@pytest.mark.parametrize("C,chunk", [(8192, 1024), (128, 128)])
@pytest.mark.parametrize("maker", [W.toy_prefill, W.toy_decode])
def test_toy_fp32(maker, C, chunk):
    b = maker()
    t = W.make_tensors(b, device="cuda")
    out, lse, _ = H.run_batch(b, t, C=C, decode_chunk=chunk)
    ro, rl = H.oracle_full(b, t)
    H.compare(out, lse, ro, rl, lse_tol=5e-3)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("d", [64, 128])
def test_random_mixed_bf16(seed, d):
    rng = np.random.default_rng(seed)
    hkv = int(rng.choice([1, 2, 4]))
    r = int(rng.choice([1, 4, 8]))
    b = W.random_batch(100 + seed, n=int(rng.integers(3, 14)), max_len=int(rng.integers(40, 900)), hq=hkv * r,
                       hkv=hkv, d=d, n_prefix=2, page_size=128 if seed % 2 else 256)
    C = int(rng.choice([8192, 512, 200]))
    t = W.make_tensors(b, device="cuda")
    out, lse, _ = H.run_batch(b, t, C=C, delta=int(rng.integers(0, 9)), decode_chunk=128 * int(rng.integers(1, 4)))
    ro, rl = H.oracle_full(b, t)
    H.compare(out, lse, ro, rl)


@pytest.mark.parametrize("seed", range(200, 240))
def test_random_sweep_small(seed):
    """Forty more seeded mixed batches (prefill, suffix prefill over shared prefixes, decode, splits
    at small C, headroom, both head dims and GQA ratios), fused launch, element-wise vs the oracle."""
    rng = np.random.default_rng(seed)
    hkv = int(rng.choice([1, 2, 3]))
    r = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([64, 128]))
    b = W.random_batch(seed, n=int(rng.integers(1, 10)), max_len=int(rng.integers(2, 600)), hq=hkv * r, hkv=hkv,
                       d=d, n_prefix=int(rng.integers(0, 3)), decode_frac=float(rng.choice([0.0, 0.3, 1.0])),
                       page_size=int(rng.choice([128, 256])))
    C = int(rng.choice([8192, 384, 130]))
    t = W.make_tensors(b, device="cuda")
    out, lse, _ = H.run_batch(b, t, C=C, delta=int(rng.integers(0, 5)), decode_chunk=128 * int(rng.integers(1, 3)))
    ro, rl = H.oracle_full(b, t)
    H.compare(out, lse, ro, rl)


def test_peaky_queries():
    """q x 4 stresses the max-subtraction / lazy rescale path."""
    b = W.random_batch(77, n=8, max_len=800, hq=8, hkv=2, d=128)
    t = W.make_tensors(b, device="cuda", peaky=4.0)
    ro, rl = H.oracle_full(b, t)
    o32, l32, _ = H.run_batch(b, t, C=300, decode_chunk=256, out_f32=True)
    H.compare(o32, l32, ro, rl)
    o16, l16, _ = H.run_batch(b, t, C=300, decode_chunk=256, out_f32=False)
    H.assert_bf16_is_rne_of_f32(o16, o32)
    assert torch.equal(l16, l32)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_bf16_output_is_rne_of_f32(seed):
    """The bf16-output mode differs from the fp32-output mode only by the final RNE store (prefill
    epilogue, decode epilogue and merge), bit for bit."""
    b = W.random_batch(500 + seed, n=14, max_len=900, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=0.4)
    t = W.make_tensors(b, device="cuda")
    o32, l32, _ = H.run_batch(b, t, C=384, delta=2, decode_chunk=256, out_f32=True)
    o16, l16, _ = H.run_batch(b, t, C=384, delta=2, decode_chunk=256, out_f32=False)
    H.assert_bf16_is_rne_of_f32(o16, o32)
    assert torch.equal(l16, l32)


@pytest.mark.parametrize("seed", [5, 6])
def test_fused_launch_equals_split(seed):
    """NEXT-3: one launch over prefill + decode work items computes, unit for unit, what the two
    separate launches compute (bitwise), and matches the oracle."""
    b = W.random_batch(seed, n=16, max_len=900, hq=8, hkv=2, d=128, decode_frac=0.5)
    assert (b.q_len == 1).any() and (b.q_len > 1).any()
    t = W.make_tensors(b, device="cuda")
    out_f, lse_f, _ = H.run_batch(b, t, C=512, decode_chunk=256, fused=True)
    out_s, lse_s, _ = H.run_batch(b, t, C=512, decode_chunk=256, fused=False)
    assert torch.equal(out_f, out_s)
    dl = (lse_f != lse_s).nonzero()
    assert dl.numel() == 0, (dl[:8].tolist(), lse_f[tuple(dl[:8].T)].tolist(), lse_s[tuple(dl[:8].T)].tolist())
    ro, rl = H.oracle_full(b, t)
    H.compare(out_f, lse_f, ro, rl)
    H.compare(out_s, lse_s, ro, rl)


@pytest.mark.parametrize("hq,hkv", [(6, 2), (2, 1), (5, 1)])
def test_odd_gqa_ratio_mixed_units(hq, hkv):
    """r = 3 (or 5) leaves a single-tile unit beside each head pair in prefill, and the fused launch
    mixes pair and single units on every CTA: the per-region barrier phases must stay in step."""
    b = W.random_batch(40 + hq, n=12, max_len=700, hq=hq, hkv=hkv, d=128, decode_frac=0.4)
    t = W.make_tensors(b, device="cuda")
    out, lse, _ = H.run_batch(b, t, C=384, decode_chunk=256)
    ro, rl = H.oracle_full(b, t)
    H.compare(out, lse, ro, rl)


def test_outlier_keys_late():
    """Keys far above every earlier score appear late in long rows (score jumps of > 128 in log2
    units): the speculative half (exp against the running max, certified by its sum) must detect
    the overflow, including on the FMA-pipe exp2 lanes, and fall back to the exact rescale."""
    b = W.random_batch(91, n=6, max_len=900, hq=8, hkv=2, d=128, n_prefix=0)
    t = W.make_tensors(b, device="cuda")
    t["q"] = (t["q"].float() + 0.5).to(t["q"].dtype)          # positive mean: q . 1 ~ 64
    P = b.page_size
    bt = t["block_table"].cpu().numpy()
    for i in range(b.n):
        L = int(b.kv_len[i])
        for pos in (L // 3, (2 * L) // 3, L - 2):
            if pos <= 0:
                continue
            blk, slot = int(bt[i, pos // P]), pos % P
            t["k_paged"][blk, slot, :, :] = 20.0 * (1 + (pos % 5))   # q . k / sqrt(d) >> 128 / log2(e)
    out, lse, _ = H.run_batch(b, t, C=400, decode_chunk=256, out_f32=True)
    ro, rl = H.oracle_full(b, t)
    H.compare(out, lse, ro, rl)


def test_mask_probe():
    """q = 0, V channel 0 = request id (exact in bf16): any cross-request leak moves o[0]; exp(lse)
    must count exactly the causally visible keys (pos + 1)."""
    b = W.random_batch(55, n=10, max_len=600, hq=4, hkv=2, d=128, n_prefix=0)
    t = W.make_tensors(b, device="cuda")
    t["q"].zero_()
    bt = t["block_table"].cpu().numpy()
    t["v_paged"][..., 0] = -1.0
    for i in range(b.n):
        for j in range(-(-int(b.kv_len[i]) // b.page_size)):
            t["v_paged"][int(bt[i, j]), :, :, 0] = float(i)
    out, lse, _ = H.run_batch(b, t, C=256, decode_chunk=128, out_f32=False)   # integers: exact in bf16
    o = out.float().cpu().numpy()
    l = lse.cpu().numpy()
    off = 0
    for i in range(b.n):
        L, ql = int(b.kv_len[i]), int(b.q_len[i])
        for tq in range(ql):
            assert np.all(o[off + tq, :, 0] == float(i)), (i, tq)
            assert np.all(np.round(np.exp(l[:, off + tq].astype(np.float64))) == L - ql + tq + 1), (i, tq)
        off += ql


def test_head_sharding_bitwise():
    """KV-head sharding: a rank computing heads [h0, h1) gets bitwise the 1-GPU result."""
    b = W.random_batch(9, n=8, max_len=500, hq=8, hkv=4, d=128)
    t = W.make_tensors(b, device="cuda")
    full, full_lse, _ = H.run_batch(b, t, C=300)
    for h0, hc in ((0, 2), (2, 2), (1, 1), (3, 1)):
        part, plse, _ = H.run_batch(b, t, C=300, hkv_begin=h0, hkv_count=hc)
        r = b.hq // b.hkv
        assert torch.equal(part.view(torch.int16), full[:, h0 * r:(h0 + hc) * r].contiguous().view(torch.int16))
        assert torch.equal(plse, full_lse[h0 * r:(h0 + hc) * r])


def test_regroup_invariance():
    """Outputs do not depend on the grouping (C, G): permuting/regrouping is lossless."""
    b = W.random_batch(31, n=10, max_len=700, hq=4, hkv=2, d=128)
    t = W.make_tensors(b, device="cuda")
    ro, rl = H.oracle_full(b, t)
    for C, G in ((8192, 0), (700, 0), (8192, 5), (150, 0)):
        out, lse, _ = H.run_batch(b, t, C=C, num_groups=G, decode_chunk=256)
        H.compare(out, lse, ro, rl)


def test_empty_and_degenerate():
    b = W.Batch("single-token", np.array([1], np.int32), np.array([1], np.int32), np.array([-1], np.int32),
                np.zeros(0, np.int32), 2, 1, 128, "bf16", 128, 4)
    t = W.make_tensors(b, device="cuda")
    out, lse, _ = H.run_batch(b, t)
    v0 = t["v_paged"][int(t["block_table"][0, 0]), 0, 0].float()
    assert torch.equal(out[0, 0].float(), v0) and torch.equal(out[0, 1].float(), v0)   # 1 key -> o = v0
    from paper_2602_06072_b200 import packinfer as pk
    pb = pk.PackedBatch([], [], None, [], 1, 1, 128, torch.bfloat16, "cuda")
    q = torch.empty((0, 1, 128), dtype=torch.bfloat16, device="cuda")
    pb.run(q, t["k_paged"], t["v_paged"], t["block_table"], q.clone())
    torch.cuda.synchronize()


def _sampled_rows(b, rng, per_req=3):
    rows = []
    for i in range(b.n):
        ql = int(b.q_len[i])
        ts = {0, ql - 1} | set(rng.integers(0, ql, size=per_req).tolist())
        rows += [(i, int(x)) for x in sorted(ts)]
    return rows


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4_decode", "cfg4_prefill", "cfg5"])
def test_full_size_sampled(name):
    """BASELINE.json full sizes in bench.py's launch configuration; oracle on sampled rows.
    cfg5 (Llama-3-70B shape) splits each 131,072-token request into 16 pieces across groups
    (prefill rows attend to earlier pieces in other groups' buffers; decode rows merge partials)."""
    b = W.make_batch(name)
    t = W.make_tensors(b, device="cuda")
    out, lse, pb = H.run_batch(b, t, C=8192, delta=32 if "cfg4" in name else 0, out_f32=True)
    rng = np.random.default_rng(0)
    rows = _sampled_rows(b, rng, per_req=1 if name == "cfg5" else 3)
    if name == "cfg5":
        # every piece boundary of the 128k requests (first / last row of each 8192-token piece)
        for i in range(b.n):
            if int(b.q_len[i]) > 8192:
                rows += [(i, a) for a in range(0, int(b.q_len[i]), 8192)]
                rows += [(i, a + 8191) for a in range(0, int(b.q_len[i]), 8192)]
        rows = sorted(set(rows))
    ro, rl = OA.attention_rows(t["q"].cpu(), t["k_paged"].cpu(), t["v_paged"].cpu(), t["block_table"].cpu(),
                               b.kv_len, b.q_len, b.page_size, rows)
    q_off = np.concatenate([[0], np.cumsum(b.q_len)])
    idx = torch.tensor([q_off[i] + tq for i, tq in rows], device="cuda")
    o = out[idx].float().cpu().numpy()
    l = lse[:, idx].cpu().numpy().T
    err = np.abs(o - ro)
    assert err.max() <= H.ATOL_MAX and err.mean() <= H.ATOL_MEAN, (err.max(), err.mean())
    assert np.abs(l - rl).max() <= 1e-3
    # property at any size: every row written (finite) exactly
    assert torch.isfinite(out.float()).all()


def test_decode_loop_append():
    """NEXT-1: decode tokens appended into the suffix headroom (no re-consolidation) for up to
    delta steps, re-planned with packinfer_plan_step; regroup (re-plan + relayout) when the
    headroom is exhausted or Eq. 4 fires.  Every step matches the oracle on kv_len + k keys."""
    from paper_2602_06072_b200 import packinfer as pk
    b = W.random_batch(404, n=12, max_len=700, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=1.0)
    steps, delta, C = 10, 4, 600
    t = W.make_tensors(b, device="cuda", extra_tokens=steps)
    r = b.hq // b.hkv
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    kv0 = b.kv_len.copy()
    mk = lambda kv: pk.PackedBatch(kv, b.q_len, b.prefix_id, b.prefix_len, b.hkv, r, b.d, torch.bfloat16, "cuda",
                                   capacity=C, headroom=delta, decode_chunk=256)
    pb = mk(kv0)
    pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], torch.empty_like(t["q"]))
    bt = t["block_table"].cpu().numpy()
    appended, since, regroups = 0, 0, 0
    for k in range(1, steps + 1):
        # the model produces one new token per request: K/V into the paged cache (engine state, read
        # by the oracle) and into the group buffer's headroom (packinfer_append_kv)
        kn = torch.randn((b.n, b.hkv, b.d), generator=g, device="cuda").to(torch.bfloat16)
        vn = torch.randn((b.n, b.hkv, b.d), generator=g, device="cuda").to(torch.bfloat16)
        for i in range(b.n):
            j = int(b.kv_len[i]) + k - 1
            t["k_paged"][int(bt[i, j // b.page_size]), j % b.page_size] = kn[i]
            t["v_paged"][int(bt[i, j // b.page_size]), j % b.page_size] = vn[i]
        q = torch.randn((b.n, b.hq, b.d), generator=g, device="cuda").to(torch.bfloat16)
        kv_now = b.kv_len + k
        if appended < delta and not pk.packinfer_should_regroup(since, int(pb.plan.c.drift), C):
            pb.append(kn, vn)
            appended += 1
            since += 1
            pb.replan(appended=np.full(b.n, appended, np.int32))
            relayout = False
        else:                                        # regroup: consolidate kv_len + k from the paged cache
            pb = mk(kv_now)
            appended, since, regroups = 0, 0, regroups + 1
            relayout = True
        out = torch.full((b.n, b.hq, b.d), float("nan"), dtype=torch.float32, device="cuda")
        lse = torch.empty((b.hq, b.n), dtype=torch.float32, device="cuda")
        pb.run(q, t["k_paged"], t["v_paged"], t["block_table"], out, lse, relayout=relayout)
        torch.cuda.synchronize()
        ro, rl = OA.attention(q.cpu(), t["k_paged"].cpu(), t["v_paged"].cpu(), t["block_table"].cpu(), kv_now,
                              b.q_len, b.page_size)
        H.compare(out, lse, ro, rl)
    assert regroups >= 1                              # the headroom (4) ran out within 10 steps


def test_graph_step_equals_eager():
    """A decode loop whose device part runs as ONE CUDA graph per step (PackedBatch.graph_run: plan
    upload + relayout + attention + merge captured, replayed with each step's new host tables) is
    bitwise equal to the eager launches, including steps whose plan shape changes (appended tokens
    cross a decode_chunk boundary -> re-capture)."""
    from paper_2602_06072_b200 import packinfer as pk
    b = W.random_batch(405, n=10, max_len=600, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=1.0)
    steps, delta = 5, 6
    t = W.make_tensors(b, device="cuda", extra_tokens=steps)
    r = b.hq // b.hkv
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    mk = lambda: pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, r, b.d, torch.bfloat16,
                                "cuda", capacity=700, headroom=delta, decode_chunk=128)
    pe, pg = mk(), mk()
    qb = torch.empty((b.n, b.hq, b.d), dtype=torch.bfloat16, device="cuda")
    oe = torch.empty((b.n, b.hq, b.d), dtype=torch.bfloat16, device="cuda")
    og, le, lg = torch.empty_like(oe), torch.empty((b.hq, b.n), device="cuda"), torch.empty((b.hq, b.n), device="cuda")
    captures = 0
    for k in range(steps):
        qb.copy_(torch.randn((b.n, b.hq, b.d), generator=g, device="cuda").to(torch.bfloat16))
        if k > 0:
            kn = torch.randn((b.n, b.hkv, b.d), generator=g, device="cuda").to(torch.bfloat16)
            vn = torch.randn((b.n, b.hkv, b.d), generator=g, device="cuda").to(torch.bfloat16)
            pe.append(kn, vn)
            pg.append(kn, vn)
            app = np.full(b.n, k, np.int32)
            pe.replan(appended=app)
            pg.replan(appended=app, upload=False)
        else:
            pg.replan(upload=False)
        pe.run(qb, t["k_paged"], t["v_paged"], t["block_table"], oe, le, relayout=(k == 0))
        pg.graph_run(qb, og, lg, t["k_paged"], t["v_paged"], t["block_table"], relayout=(k == 0))
        captures = pg.graph_captures
        torch.cuda.synchronize()
        assert torch.equal(oe.view(torch.int16), og.view(torch.int16)), k
        assert torch.equal(le, lg), k
    assert captures < steps          # at least one step replayed an existing graph


@pytest.mark.parametrize("world", [2, 3])
def test_decode_group_sharding_one_batch(world):
    """Group sharding of ONE decode batch (shard.RankPlan), the ranks simulated one after the other
    on cuda:0 with every buffer (K/V, partials, out, lse) pre-filled with NaN: each rank
    consolidates only its groups (+ guard zero cells), attends only its items, the cross-rank split
    rows' partials - and nothing else - are exchanged (the SUM / MAX of exchange_split_rows, done
    here with the same torch reductions over the cross range), and each rank's merge then holds the
    oracle's result for every token it owns."""
    from paper_2602_06072_b200 import packinfer as pk, shard
    b = W.random_batch(31, n=24, max_len=1500, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=1.0)
    assert (b.q_len == 1).all()
    t = W.make_tensors(b, device="cuda")
    r = b.hq // b.hkv
    pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, r, b.d, t["q"].dtype, "cuda",
                        capacity=256, decode_chunk=256)
    owner = shard.group_shard(shard.group_costs(pb.plan), world)
    assert len(set(owner)) == world
    nan = float("nan")
    st = []
    for rank in range(world):
        rp = shard.RankPlan(pb, owner, rank)
        kb = torch.full_like(pb.k_buf, nan)
        vb = torch.full_like(pb.v_buf, nan)
        po, pl = torch.full_like(pb.partial_o, nan), torch.full_like(pb.partial_lse, nan)
        out = torch.full((b.total_q, b.hq, b.d), nan, dtype=torch.float32, device="cuda")
        lse = torch.full((b.hq, b.total_q), nan, dtype=torch.float32, device="cuda")
        pk.packinfer_relayout_kv(rp.dp, t["k_paged"], t["v_paged"], t["block_table"], kb, vb, 0, b.hkv)
        shard.neutral_cross_slots(po, pl, rp.n_cross_slots)
        pk.packinfer_attention_decode(rp.dp, t["q"], kb, vb, out, lse, po, pl, r)
        st.append((rp, po, pl, out, lse))
    torch.cuda.synchronize()
    ncs = st[0][0].n_cross_slots
    assert ncs > 0 and all(x[0].n_cross_slots == ncs for x in st)
    xo = torch.stack([x[1][:ncs] for x in st]).sum(0)     # exchange_split_rows: SUM / MAX over ranks
    xl = torch.stack([x[2][:ncs] for x in st]).amax(0)
    ro, rl = H.oracle_full(b, t)
    held = set()
    for rp, po, pl, out, lse in st:
        po[:ncs] = xo
        pl[:ncs] = xl
        pk.packinfer_merge(rp.dp, po, pl, out, lse)
        torch.cuda.synchronize()
        tok = torch.tensor(rp.owned_tokens, device="cuda")
        H.compare(out[tok], lse[:, tok], ro[rp.owned_tokens], rl[:, rp.owned_tokens])
        held |= set(rp.owned_tokens)
        assert rp.exchange_bytes == ncs * b.hq * (b.d + 1) * 4
    assert held == set(range(b.total_q))
    # fewer bytes than exchanging every partial slot
    assert ncs < int(pb.plan.c.n_partial_slots)


def test_replan_grows_partials():
    """Appended decode tokens that cross a decode_chunk boundary add decode items and partial slots
    (plan_step); the batch's partial buffers grow with the plan and the result stays exact."""
    from paper_2602_06072_b200 import packinfer as pk
    chunk, delta = 256, 6
    kv = np.array([chunk - 2, 2 * chunk - 1, 3 * chunk - 3, 40], np.int32)
    b = W.Batch("chunk-edge", kv, np.ones(4, np.int32), np.full(4, -1, np.int32), np.zeros(0, np.int32),
                8, 2, 128, "bf16", 128, 21)
    t = W.make_tensors(b, device="cuda", extra_tokens=delta)
    r = b.hq // b.hkv
    pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, r, b.d, torch.bfloat16, "cuda",
                        capacity=8192, headroom=delta, decode_chunk=chunk)
    pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], torch.empty_like(t["q"]))
    slots0 = int(pb.plan.c.n_partial_slots)
    bt = t["block_table"].cpu().numpy()
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    for k in range(1, delta + 1):
        kn = torch.randn((b.n, b.hkv, b.d), generator=g, device="cuda").to(torch.bfloat16)
        vn = torch.randn((b.n, b.hkv, b.d), generator=g, device="cuda").to(torch.bfloat16)
        for i in range(b.n):
            j = int(b.kv_len[i]) + k - 1
            t["k_paged"][int(bt[i, j // b.page_size]), j % b.page_size] = kn[i]
            t["v_paged"][int(bt[i, j // b.page_size]), j % b.page_size] = vn[i]
        pb.append(kn, vn)
        pb.replan(appended=np.full(b.n, k, np.int32))
        assert pb.partial_o.shape[0] >= int(pb.plan.c.n_partial_slots)
        out = torch.full((b.n, b.hq, b.d), float("nan"), dtype=torch.float32, device="cuda")
        lse = torch.empty((b.hq, b.n), dtype=torch.float32, device="cuda")
        pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out, lse, relayout=False)
        torch.cuda.synchronize()
        ro, rl = OA.attention(t["q"].cpu(), t["k_paged"].cpu(), t["v_paged"].cpu(), t["block_table"].cpu(),
                              b.kv_len + k, b.q_len, b.page_size)
        H.compare(out, lse, ro, rl)
    assert int(pb.plan.c.n_partial_slots) > slots0


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4_decode", "cfg5"])
def test_device_row_expansion_bitwise(name):
    """packinfer_plan_upload expands the planner's row segments on the device: the device row
    table equals the host expansion (packinfer_plan_rows) bit for bit, and every row of every
    work item is inside its item's range."""
    from paper_2602_06072_b200 import packinfer as pk
    b = W.make_batch(name)
    cfg = pk.default_config(capacity=8192, gqa_ratio=b.hq // b.hkv)
    hp = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, cfg, pinned=True)
    c = hp.c
    arena = torch.full((int(c.device_arena_bytes),), 0xAB, dtype=torch.uint8, device="cuda")
    pk.packinfer_plan_upload(hp, arena)
    torch.cuda.synchronize()
    n = int(c.n_rows)
    dev_rows = arena[int(c.rows_offset):int(c.rows_offset) + 16 * n].cpu().numpy().view(pk.ROW_DT)
    host_rows = hp.rows
    assert n > 0 and dev_rows.shape == host_rows.shape
    assert dev_rows.tobytes() == host_rows.tobytes()
    segs = hp.segs
    assert int(segs["count"].sum()) == n


@pytest.mark.parametrize("seed", range(4))
def test_in_kernel_merge_bitwise(seed):
    """NEXT-3 last-arriver merge: packinfer_attention_merge (prefill + decode + LSE merge in ONE
    launch) equals packinfer_attention + packinfer_merge bit for bit (same arithmetic, same slot
    order), passes the oracle gate, and leaves every merge counter at zero (so the next launch
    starts clean); run twice to show the counters are reusable."""
    from paper_2602_06072_b200 import packinfer as pk
    rng = np.random.default_rng(seed)
    b = W.random_batch(400 + seed, n=int(rng.integers(6, 16)), max_len=int(rng.integers(600, 1800)), hq=8, hkv=2,
                       d=128, n_prefix=2, decode_frac=0.6)
    t = W.make_tensors(b, device="cuda")
    r = b.hq // b.hkv
    pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, r, b.d, torch.bfloat16, "cuda",
                        capacity=512, decode_chunk=128)
    assert int(pb.plan.c.n_merges) > 0
    res = {}
    for mode in ("separate", "kernel", "kernel2"):
        for odt in (torch.float32, torch.bfloat16):
            out = torch.full((b.total_q, b.hq, b.d), float("nan"), dtype=odt, device="cuda")
            lse = torch.full((b.hq, b.total_q), float("nan"), dtype=torch.float32, device="cuda")
            pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out, lse, kernel_merge=(mode != "separate"))
            torch.cuda.synchronize()
            res[mode, odt] = (out, lse)
            assert int(pb.merge_counters.abs().sum()) == 0
    for odt in (torch.float32, torch.bfloat16):
        o0, l0 = res["separate", odt]
        for mode in ("kernel", "kernel2"):
            o1, l1 = res[mode, odt]
            assert torch.equal(o0.view(torch.int8), o1.view(torch.int8)), mode
            assert torch.equal(l0, l1)
    ro, rl = H.oracle_full(b, t)
    H.compare(*res["kernel", torch.float32], ro, rl)


@pytest.mark.parametrize("seed", range(3))
def test_packed_decode_items_option(seed):
    """PI_PLAN_DPACK: short decode suffixes of one group packed into one decode item (per-row
    [lo, hi) inside the hull) - same results as the oracle, fewer decode items."""
    from paper_2602_06072_b200 import packinfer as pk
    b = W.random_batch(700 + seed, n=20, max_len=900, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=1.0)
    t = W.make_tensors(b, device="cuda")
    r = b.hq // b.hkv
    res = {}
    for flags in (0, pk.PI_PLAN_DPACK):
        pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, r, b.d, torch.bfloat16, "cuda",
                            capacity=2048, decode_chunk=512, headroom=3, flags=flags)
        out = torch.full((b.total_q, b.hq, b.d), float("nan"), dtype=torch.float32, device="cuda")
        lse = torch.full((b.hq, b.total_q), float("nan"), dtype=torch.float32, device="cuda")
        pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out, lse)
        torch.cuda.synchronize()
        res[flags] = (out, lse, int(pb.plan.c.n_decode_work))
    assert res[pk.PI_PLAN_DPACK][2] < res[0][2]
    ro, rl = H.oracle_full(b, t)
    H.compare(res[pk.PI_PLAN_DPACK][0], res[pk.PI_PLAN_DPACK][1], ro, rl)


@pytest.mark.parametrize("name", ["small", "cfg4_decode"])
def test_paged_decode_ablation(name):
    """NEXT-4 "no packed I/O" ablation: a PI_PLAN_PAGED plan decoded straight from the paged cache
    (packinfer_attention_decode_paged: no relayout, no prefix co-location) matches the oracle, as
    does the packed path on the same batch; the packed plan reads fewer KV tokens when prefixes are
    shared (Eq. 5)."""
    from paper_2602_06072_b200 import packinfer as pk
    if name == "small":
        b = W.random_batch(811, n=14, max_len=2500, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=1.0)
    else:
        b = W.make_batch(name)
    t = W.make_tensors(b, device="cuda")
    r = b.hq // b.hkv
    pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, r, b.d, torch.bfloat16, "cuda",
                        decode_chunk=512, flags=pk.PI_PLAN_PAGED)
    out = torch.full((b.total_q, b.hq, b.d), float("nan"), dtype=torch.float32, device="cuda")
    lse = torch.full((b.hq, b.total_q), float("nan"), dtype=torch.float32, device="cuda")
    pk.packinfer_attention_decode_paged(pb.dp, t["q"], t["k_paged"], t["v_paged"], t["block_table"], out, lse,
                                        pb.partial_o, pb.partial_lse, r)
    pk.packinfer_merge(pb.dp, pb.partial_o, pb.partial_lse, out, lse)
    torch.cuda.synchronize()
    if name == "small":
        ro, rl = H.oracle_full(b, t)
        H.compare(out, lse, ro, rl)
    else:
        rows = [(i, 0) for i in range(b.n)]
        ro, rl = OA.attention_rows(t["q"].cpu(), t["k_paged"].cpu(), t["v_paged"].cpu(), t["block_table"].cpu(),
                                   b.kv_len, b.q_len, b.page_size, rows)
        err = np.abs(out.cpu().numpy() - ro)
        assert err.max() <= H.ATOL_MAX and err.mean() <= H.ATOL_MEAN
        assert np.abs(lse.cpu().numpy().T - rl).max() <= 1e-3
        packed = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, pk.default_config(gqa_ratio=r))
        paged_keys = int(sum(s["len"] for s in pb.plan.spans))
        assert int(packed.c.copy_tokens) < paged_keys == int(b.kv_len.sum())


def test_repeated_launches_bitwise_stable():
    """The dynamic scheduler's counters are zeroed at plan upload and reset by the last CTA of every
    launch, and attention / merge launches are programmatic dependents of the kernel before them:
    many back-to-back launches of different kinds and grid sizes on one device plan (fused with its
    PDL-chained decode half, split prefill / decode, KV-head slices, in-kernel merge) must each
    reproduce their first result bit for bit."""
    from paper_2602_06072_b200 import packinfer as pk
    b = W.random_batch(406, n=16, max_len=900, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=0.5)
    t = W.make_tensors(b, device="cuda")
    r = b.hq // b.hkv
    pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, r, b.d, torch.bfloat16, "cuda",
                        capacity=600, headroom=2, decode_chunk=256)
    pb1 = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, 1, r, b.d, torch.bfloat16, "cuda",
                         capacity=600, headroom=2, decode_chunk=256)
    variants = [("fused", pb, 0, dict(fused=True)), ("split", pb, 0, dict(fused=False)),
                ("merge_in_kernel", pb, 0, dict(fused=True, kernel_merge=True)), ("head1", pb1, 1, dict(fused=True))]
    ref = {}
    for rep in range(6):
        for name, p_, h0, kw in variants:
            hc = p_.hkv
            out = torch.full((b.total_q, hc * r, b.d), float("nan"), dtype=torch.bfloat16, device="cuda")
            lse = torch.full((hc * r, b.total_q), float("nan"), dtype=torch.float32, device="cuda")
            p_.run(t["q"][:, h0 * r:(h0 + hc) * r], t["k_paged"], t["v_paged"], t["block_table"], out, lse,
                   hkv_begin=h0, relayout=(rep == 0), **kw)
            got = (out.view(torch.int16).clone(), lse.view(torch.int32).clone())
            if name not in ref:
                ref[name] = got
            else:
                assert torch.equal(got[0], ref[name][0]) and torch.equal(got[1], ref[name][1]), (rep, name)
    # the three full-head variants agree with each other too
    assert torch.equal(ref["fused"][0], ref["split"][0]) and torch.equal(ref["fused"][0], ref["merge_in_kernel"][0])
    assert torch.equal(ref["head1"][0], ref["fused"][0][:, r:2 * r])
