"""Kernel timeline (torch.profiler / CUPTI) of a few decode or prefill steps of one BASELINE batch:
kernel durations and the gaps between them (launch latency, memsets) inside the bench's step.
    python scripts/step_timeline.py [cfg4_decode|cfg3|cfg2] [resident]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_decode"
resident = "resident" in sys.argv
graph = "graph" in sys.argv
b = bench.make_workload(name, 0)
heads1 = "h1" in sys.argv   # one KV head (the per-rank share of KV-head sharding at N = 8), pipelined steps
r = bench.Runner(b, "cuda", 0, 1 if heads1 else b.hkv, seed=b.seed, pipeline=heads1)
for i in range(5):
    r.step(i)
torch.cuda.synchronize()
r.relayout = not resident
from torch.profiler import profile, ProfilerActivity
pb = r.pbs[0]
if graph:   # the resident step with its device part as one CUDA graph (PackedBatch.graph_run)
    for _ in range(3):
        pb.replan(upload=False)
        pb.graph_run(r.q, r.out, r.lse)
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(5, 10):
        if graph:
            pb.replan(upload=False)
            pb.graph_run(r.q, r.out, r.lse)
        else:
            r.step(i, time_kernel=True)
    torch.cuda.synchronize()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev = None
for e in ev:
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = (e.time_range.start - prev) if prev is not None else 0
    print(f"{s:9.1f} us  +gap {gap:6.1f}  dur {d:8.1f}  {e.name[:70]}")
    prev = e.time_range.end
if not graph:
    print("event-timed: attention", r.kernel_ms(), "merge", r.merge_ms())
