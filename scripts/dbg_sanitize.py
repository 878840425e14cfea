"""Small runs of every kernel for compute-sanitizer (scripts/sanitize.sh); checks results against
the oracle too, so a sanitizer-clean run is also a correct one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth import workloads as W  # noqa: E402
from tests import gpu_helpers as H  # noqa: E402
from paper_2602_06072_b200 import packinfer as pk, shard  # noqa: E402

# bf16 mixed batch: prefill pair units, suffix prefill over shared prefixes, decode, splits, merge
b = W.random_batch(5, n=10, max_len=700, hq=8, hkv=2, d=128, decode_frac=0.5)
t = W.make_tensors(b, device="cuda")
ro, rl = H.oracle_full(b, t)
for fused in (True, False):
    out, lse, _ = H.run_batch(b, t, C=384, delta=3, decode_chunk=256, fused=fused)
    H.compare(out, lse, ro, rl)
# head_dim 64, GQA 4
b2 = W.random_batch(6, n=6, max_len=400, hq=8, hkv=2, d=64, decode_frac=0.3)
t2 = W.make_tensors(b2, device="cuda")
out, lse, _ = H.run_batch(b2, t2, C=8192)
H.compare(out, lse, *H.oracle_full(b2, t2))
# fp32 toy (kind::tf32)
for maker in (W.toy_prefill, W.toy_decode):
    bt = maker()
    tt = W.make_tensors(bt, device="cuda")
    out, lse, _ = H.run_batch(bt, tt, C=128, decode_chunk=128)
    H.compare(out, lse, *H.oracle_full(bt, tt), lse_tol=5e-3)
# decode group sharding of one batch (2 simulated ranks)
bd = W.random_batch(31, n=12, max_len=900, hq=8, hkv=2, d=128, decode_frac=1.0)
td = W.make_tensors(bd, device="cuda")
r = bd.hq // bd.hkv
pb = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, bd.hkv, r, bd.d, td["q"].dtype, "cuda",
                    capacity=256, decode_chunk=256)
owner = shard.group_shard(shard.group_costs(pb.plan), 2)
for rank in range(2):
    rp = shard.RankPlan(pb, owner, rank)
    pk.packinfer_relayout_kv(rp.dp, td["k_paged"], td["v_paged"], td["block_table"], pb.k_buf, pb.v_buf, 0, bd.hkv)
# ... its decode attention + merge with the rank's renumbered slot tables (cross range neutral)
for rank in range(2):
    rp = shard.RankPlan(pb, owner, rank)
    shard.neutral_cross_slots(pb.partial_o, pb.partial_lse, rp.n_cross_slots)
    o = torch.zeros((bd.total_q, bd.hq, bd.d), dtype=torch.bfloat16, device="cuda")
    pk.packinfer_attention_decode(rp.dp, td["q"], pb.k_buf, pb.v_buf, o, None, pb.partial_o, pb.partial_lse, r)
    pk.packinfer_merge(rp.dp, pb.partial_o, pb.partial_lse, o, None)
# one launch with the in-kernel LSE merge (merge warp, counters) vs the oracle
bm = W.random_batch(402, n=10, max_len=1200, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=0.6)
tm = W.make_tensors(bm, device="cuda")
pbm = pk.PackedBatch(bm.kv_len, bm.q_len, bm.prefix_id, bm.prefix_len, bm.hkv, 4, bm.d, torch.bfloat16, "cuda",
                     capacity=512, decode_chunk=128)
om = torch.full((bm.total_q, bm.hq, bm.d), float("nan"), dtype=torch.float32, device="cuda")
lm = torch.full((bm.hq, bm.total_q), float("nan"), dtype=torch.float32, device="cuda")
pbm.run(tm["q"], tm["k_paged"], tm["v_paged"], tm["block_table"], om, lm, kernel_merge=True)
H.compare(om, lm, *H.oracle_full(bm, tm))
# paged-KV decode (NEXT-4 ablation)
pbp = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, bd.hkv, r, bd.d, torch.bfloat16, "cuda",
                     decode_chunk=256, flags=pk.PI_PLAN_PAGED)
op = torch.full((bd.total_q, bd.hq, bd.d), float("nan"), dtype=torch.float32, device="cuda")
lp = torch.full((bd.hq, bd.total_q), float("nan"), dtype=torch.float32, device="cuda")
pk.packinfer_attention_decode_paged(pbp.dp, td["q"], td["k_paged"], td["v_paged"], td["block_table"], op, lp,
                                    pbp.partial_o, pbp.partial_lse, r)
pk.packinfer_merge(pbp.dp, pbp.partial_o, pbp.partial_lse, op, lp)
H.compare(op, lp, *H.oracle_full(bd, td))
torch.cuda.synchronize()
print("ok")
