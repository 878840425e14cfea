"""In-process A/B of library variants on whole decode steps (KV resident: plan + upload + attention
+ merge, eager launches), blocks of 10 steps alternated; median ms per step.
    python scripts/ab_step_inproc.py cfg4_decode cur pdl [--relayout]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2602_06072_b200 import packinfer as pk
import bench

cfg, names = sys.argv[1], [a for a in sys.argv[2:] if not a.startswith("--")]
relayout = "--relayout" in sys.argv
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = {}
for v in names:
    pk._lib = None
    os.environ["PACKINFER_LIB"] = os.path.join(root, "variants", f"libpi_{v}.so")
    libs[v] = pk.lib()
b = bench.make_workload(cfg, 0)
pk._lib = libs[names[0]]
r = bench.Runner(b, "cuda", 0, b.hkv, seed=b.seed)
r.step(0)
pb = r.pbs[0]
res = {v: [] for v in names}
for blk in range(14):
    for v in names:
        pk._lib = libs[v]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(10):
            pb.replan()
            pb.run(r.q, r.t["k_paged"], r.t["v_paged"], r.t["block_table"], r.out, r.lse, relayout=relayout)
        e1.record()
        torch.cuda.synchronize()
        if blk >= 2:
            res[v].append(e0.elapsed_time(e1) / 10)
for v in names:
    print(f"{cfg} {'relayout ' if relayout else ''}{v}: median {np.median(res[v]):.4f} ms/step  min {min(res[v]):.4f}")
