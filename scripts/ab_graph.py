"""Resident decode step, eager launches vs ONE CUDA graph per step (PackedBatch.graph_run),
alternating blocks of 10 steps in one process; prints median ms per step of each mode.
    python scripts/ab_graph.py cfg3|cfg4_decode"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
b = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg3", 0)
r = bench.Runner(b, "cuda", 0, b.hkv, seed=b.seed)
r.step(0)
r.relayout = False
pb = r.pbs[0]
res = {"eager": [], "graph": []}
for blk in range(12):
    for mode in ("eager", "graph"):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(10):
            if mode == "eager":
                pb.replan()
                pb.run(r.q, None, None, None, r.out, r.lse, relayout=False)
            else:
                pb.replan(upload=False)
                pb.graph_run(r.q, r.out, r.lse)
        e1.record()
        torch.cuda.synchronize()
        if blk >= 2:
            res[mode].append(e0.elapsed_time(e1) / 10)
for m, v in res.items():
    print(f"{sys.argv[1]} {m}: median {np.median(v):.4f} ms/step  min {min(v):.4f}  max {max(v):.4f}")
print("graph captures", getattr(pb, "graph_captures", 0))
