"""CUPTI timeline of a few decode-loop steps (configs[2], headroom 32: append + plan_step + device
part), eager vs one CUDA graph per step (PackedBatch.graph_run)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import workloads as W
from paper_2602_06072_b200 import packinfer as pk
from torch.profiler import profile, ProfilerActivity
graph = "graph" in sys.argv
bd = W.cfg3_decode(1)
tl = W.make_tensors(bd, device="cuda", seed=bd.seed, extra_tokens=40)
rr = bd.hq // bd.hkv
pbl = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, bd.hkv, rr, bd.d, torch.bfloat16, "cuda", headroom=32)
outl = torch.empty((bd.n, bd.hq, bd.d), dtype=torch.bfloat16, device="cuda")
kn = torch.randn((bd.n, bd.hkv, bd.d), device="cuda").to(torch.bfloat16)
vn = torch.randn_like(kn)
pbl.run(tl["q"], tl["k_paged"], tl["v_paged"], tl["block_table"], outl)
def step(k):
    pbl.append(kn, vn)
    if graph:
        pbl.replan(appended=np.full(bd.n, k, np.int32), upload=False)
        pbl.graph_run(tl["q"], outl, None)
    else:
        pbl.replan(appended=np.full(bd.n, k, np.int32))
        pbl.run(tl["q"], tl["k_paged"], tl["v_paged"], tl["block_table"], outl, relayout=False)
for k in range(1, 8):
    step(k)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(8, 12):
        step(k)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start; prev = None
for e in ev:
    gap = (e.time_range.start - prev) if prev is not None else 0
    print(f"{e.time_range.start - t0:9.1f} us  +gap {gap:6.1f}  dur {e.time_range.end - e.time_range.start:8.1f}  {e.name[:60]}")
    prev = e.time_range.end
