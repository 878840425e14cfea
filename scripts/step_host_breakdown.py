"""Host-side cost of each call in one bench step (configs[1], one KV head per rank = N = 8)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2602_06072_b200 import packinfer as pk

dev = torch.device("cuda", 0)
b = bench.make_workload("cfg2", 0)
r = bench.Runner(b, dev, 0, 1, seed=b.seed)
for i in range(5):
    r.step(i)
torch.cuda.synchronize()
T = {k: [] for k in ("evsync", "plan", "upload", "ensure", "relayout", "attention", "merge", "event")}
pb = r.pbs[0]
kv_len, q_len, prefix_id, prefix_len = pb.args
for it in range(200):
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan = pk.packinfer_plan(kv_len, q_len, prefix_id, prefix_len, pb.cfg, arena=pb._arenas[0])
    t2 = time.perf_counter()
    dp = pk.packinfer_plan_upload(plan, pb.dev_arena, r.stream)
    t3 = time.perf_counter()
    pb._ensure_partials()
    t4 = time.perf_counter()
    pk.packinfer_relayout_kv(dp, r.t["k_paged"], r.t["v_paged"], r.t["block_table"], pb.k_buf, pb.v_buf, 0, 1, r.stream)
    t5 = time.perf_counter()
    pk.packinfer_attention(dp, r.q, pb.k_buf, pb.v_buf, r.out, r.lse, pb.partial_o, pb.partial_lse, r.r, 0.0, r.stream)
    t6 = time.perf_counter()
    pk.packinfer_merge(dp, pb.partial_o, pb.partial_lse, r.out, r.lse, r.stream)
    t7 = time.perf_counter()
    e = torch.cuda.Event(enable_timing=True); e.record(r.stream)
    t8 = time.perf_counter()
    pass
    torch.cuda.synchronize()
    for k, a, bb in (("evsync", t0, t1), ("plan", t1, t2), ("upload", t2, t3), ("ensure", t3, t4), ("relayout", t4, t5),
                     ("attention", t5, t6), ("merge", t6, t7), ("event", t7, t8)):
        T[k].append((bb - a) * 1e6)
print({k: round(statistics.median(v), 1) for k, v in T.items()})
