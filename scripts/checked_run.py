"""Runs a set of representative batches through the hot path and saves every output (used by
tests/test_gpu_checks.py with the PI_CHECKS=1 library and with the production library: the
device bounds checks must never fire, and the outputs must be bitwise the same).
    PACKINFER_LIB=... python scripts/checked_run.py out.pt"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from synth import workloads as W
from paper_2602_06072_b200 import packinfer as pk

torch.manual_seed(0)
res = []


def run(b, C, delta, chunk, hkv_begin=0, hkv_count=None, fused=True, kernel_merge=False, flags=None, seed=0):
    t = W.make_tensors(b, device="cuda", seed=seed)
    r = b.hq // b.hkv
    hc = b.hkv - hkv_begin if hkv_count is None else hkv_count
    pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, hc, r, b.d, t["q"].dtype, "cuda",
                        capacity=C, headroom=delta, decode_chunk=chunk, flags=flags)
    q = t["q"][:, hkv_begin * r:(hkv_begin + hc) * r]
    out = torch.zeros((b.total_q, hc * r, b.d), dtype=t["q"].dtype, device="cuda")
    lse = torch.zeros((hc * r, b.total_q), dtype=torch.float32, device="cuda")
    pb.run(q, t["k_paged"], t["v_paged"], t["block_table"], out, lse, hkv_begin=hkv_begin, fused=fused,
           kernel_merge=kernel_merge)
    res.append(out.float().cpu())
    res.append(lse.cpu())
    return pb, t, q, out, lse


if len(sys.argv) > 2 and sys.argv[2] == "--corrupt":
    # negative control: one row of the device row table points past the end of Q; the checked
    # library must trap (check 4 / 5) instead of reading out of bounds
    b0 = W.random_batch(3000, n=6, max_len=300, hq=8, hkv=2, d=128, decode_frac=0.0)
    t0 = W.make_tensors(b0, device="cuda", seed=0)
    pb0 = pk.PackedBatch(b0.kv_len, b0.q_len, b0.prefix_id, b0.prefix_len, b0.hkv, 4, b0.d, torch.bfloat16, "cuda")
    rows = pb0.dev_arena[int(pb0.plan.c.rows_offset):].view(torch.int32)
    rows[0] = b0.total_q + 5                          # pi_row.q_token of row 0
    o0 = torch.zeros((b0.total_q, b0.hq, b0.d), dtype=torch.bfloat16, device="cuda")
    pk.packinfer_relayout_kv(pb0.dp, t0["k_paged"], t0["v_paged"], t0["block_table"], pb0.k_buf, pb0.v_buf, 0,
                             b0.hkv)
    pk.packinfer_attention(pb0.dp, t0["q"], pb0.k_buf, pb0.v_buf, o0, None, pb0.partial_o, pb0.partial_lse, 4, 0.0)
    torch.cuda.synchronize()
    print("corrupted row table ran without a trap")
    sys.exit(0)

# prefill + decode + shared prefixes, splits (small C), decode chunks with partials
b1 = W.random_batch(3001, n=14, max_len=900, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=0.5)
run(b1, 600, 3, 256)
run(b1, 600, 3, 256, fused=False)
run(b1, 600, 3, 256, kernel_merge=True)
run(b1, 8192, 0, 1024, flags=0)
run(b1, 600, 3, 256, hkv_begin=1, hkv_count=1)
# decode-only: packed items of 4-32 rows, shared-prefix items, d = 64
b2 = W.random_batch(3002, n=24, max_len=1500, hq=8, hkv=2, d=128, n_prefix=3, decode_frac=1.0)
pb, t, q, out, lse = run(b2, 2048, 8, 512)
for k in range(1, 4):    # decode loop: append + plan_step
    pb.append(torch.randn((b2.n, b2.hkv, b2.d), device="cuda").to(torch.bfloat16),
              torch.randn((b2.n, b2.hkv, b2.d), device="cuda").to(torch.bfloat16))
    pb.replan(appended=np.full(b2.n, k, np.int32))
    pb.run(q, t["k_paged"], t["v_paged"], t["block_table"], out, lse, relayout=False)
    res.append(out.float().cpu())
b3 = W.random_batch(3003, n=10, max_len=700, hq=4, hkv=4, d=64, n_prefix=1, decode_frac=0.5)
run(b3, 512, 2, 128)
# configs[3] decode (full size): packed suffix items + prefix items of up to 128 rows
run(W.cfg4_decode(2), 8192, 0, 1024)
torch.cuda.synchronize()
torch.save(res, sys.argv[1])
print("checked_run ok", len(res))
