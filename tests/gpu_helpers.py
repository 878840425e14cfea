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
              relayout=True, out_f32=False, fused=True):
    """Runs plan -> upload -> relayout -> attention (one fused launch, or prefill + decode launches)
    -> merge on cuda:0.
    t: tensors on cuda (from synth.make_tensors).  Returns (out, lse, PackedBatch)."""
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
    """fp32 outputs: |o - ref| <= 1e-2 everywhere, mean <= 1e-3.  bf16 outputs additionally allow the
    unavoidable output rounding, half a bf16 ulp <= 2^-8 |ref| (reading R13)."""
    o = out.float().cpu().numpy().astype(np.float64)
    assert np.isfinite(o).all(), "non-finite output (unwritten rows?)"
    err = np.abs(o - ref_out)
    if out.dtype == torch.bfloat16:
        err = np.maximum(err - np.abs(ref_out) * 2.0 ** -8, 0.0)
    l = lse.cpu().numpy().astype(np.float64)
    lerr = np.abs(l - ref_lse)
    info = dict(max_abs=float(err.max()), mean_abs=float(err.mean()), lse_max=float(lerr.max()))
    assert err.max() <= atol_max, info
    assert err.mean() <= atol_mean, info
    assert lerr.max() <= lse_tol, info
    return info
