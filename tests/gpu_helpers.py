"""Shared helpers for the -m gpu parity tests: run the CUDA path through the C ABI and compare
with the oracle on the same seeded inputs."""

from __future__ import annotations

import numpy as np
import torch

from oracle import attention as OA
from oracle import plan as OP
from oracle import layout as OL
from paper_2602_06072_b200 import packinfer as pk

ATOL_MAX = 1e-2   # north star: max-abs <= 1e-2 (BASELINE.json)
ATOL_MEAN = 1e-3  # north star: mean-abs <= 1e-3


def run_batch(b, t, C=8192, delta=0, decode_chunk=1024, num_groups=0, hkv_begin=0, hkv_count=None,
              relayout=True, out_f32=None, fused=True):
    """Runs plan -> upload -> relayout -> attention (one fused launch, or prefill + decode launches)
    -> merge on cuda:0.
    t: tensors on cuda (from synth.make_tensors).  Returns (out, lse, PackedBatch).
    out_f32: True -> fp32 outputs (PI_BF16_OUT_F32), False -> bf16 outputs, None (default) -> both:
    the bf16-output run must be bit-for-bit the RNE of the fp32-output run (the only difference
    between the two modes is the final store, reading R13), and the fp32 outputs are returned for
    the north-star gate."""
    if out_f32 is None and t["q"].dtype == torch.bfloat16:
        o32, l32, _ = run_batch(b, t, C, delta, decode_chunk, num_groups, hkv_begin, hkv_count, relayout, True, fused)
        o16, l16, pb = run_batch(b, t, C, delta, decode_chunk, num_groups, hkv_begin, hkv_count, relayout, False,
                                 fused)
        assert_bf16_is_rne_of_f32(o16, o32)
        assert torch.equal(l16, l32)
        return o32, l32, pb
    r = b.hq // b.hkv
    hkv_count = b.hkv - hkv_begin if hkv_count is None else hkv_count
    dt = t["q"].dtype
    pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, hkv_count, r, b.d, dt, "cuda",
                        capacity=C, headroom=delta, num_groups=num_groups, decode_chunk=decode_chunk)
    q = t["q"][:, hkv_begin * r:(hkv_begin + hkv_count) * r]
    out = torch.full((b.total_q, hkv_count * r, b.d), float("nan"), dtype=torch.float32 if out_f32 else dt,
                     device="cuda")
    lse = torch.full((hkv_count * r, b.total_q), float("nan"), dtype=torch.float32, device="cuda")
    pb.partial_o.fill_(float("nan"))        # every partial slot the merge reads must be written
    pb.partial_lse.fill_(float("nan"))
    pb.run(q, t["k_paged"], t["v_paged"], t["block_table"], out, lse, hkv_begin=hkv_begin, fused=fused)
    torch.cuda.synchronize()
    return out, lse, pb


def oracle_full(b, t):
    return OA.attention(t["q"].cpu(), t["k_paged"].cpu(), t["v_paged"].cpu(), t["block_table"].cpu(),
                        b.kv_len, b.q_len, b.page_size)


def compare(out, lse, ref_out, ref_lse, atol_max=ATOL_MAX, atol_mean=ATOL_MEAN, lse_tol=1e-3):
    """The north-star gate, the same for bf16 and fp32 outputs: |o - ref| <= 1e-2 everywhere,
    mean |o - ref| <= 1e-3, |lse - ref_lse| <= 1e-3 (tf32 toy: 5e-3)."""
    o = out.float().cpu().numpy().astype(np.float64)
    assert np.isfinite(o).all(), "non-finite output (unwritten rows?)"
    err = np.abs(o - ref_out)
    l = lse.cpu().numpy().astype(np.float64)
    lerr = np.abs(l - ref_lse)
    k = int(err.argmax())
    info = dict(max_abs=float(err.max()), mean_abs=float(err.mean()), lse_max=float(lerr.max()),
                at=np.unravel_index(k, err.shape), ref_at=float(ref_out.flat[k]))
    assert err.max() <= atol_max, info
    assert err.mean() <= atol_mean, info
    assert lerr.max() <= lse_tol, info
    return info


def assert_bf16_is_rne_of_f32(out_bf16, out_f32):
    """bf16-output mode stores exactly RNE(fp32-output mode): the kernel arithmetic is the same and
    only the final store rounds (reading R13)."""
    want = out_f32.to(torch.bfloat16).view(torch.int16)
    got = out_bf16.view(torch.int16)
    bad = (want != got).nonzero()
    assert bad.numel() == 0, (bad[:8].tolist(), out_bf16[tuple(bad[:8].T)].tolist(), out_f32[tuple(bad[:8].T)].tolist())
