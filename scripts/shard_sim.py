"""Strong-scaling estimate on ONE GPU: the per-rank step of KV-head sharding (hkv_count = 8 / N heads
of configs[1]) timed alone, against the unsharded step: efficiency(N) ~= T(8 heads) / (N * T(8/N
heads)).  (On an 8-GPU box bench.py --gpus N measures the real thing, max over ranks.)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

dev = torch.device("cuda", 0)
b = bench.make_workload("cfg2", 0)
res = {}
for hc in (8, 4, 2, 1):
    r = bench.Runner(b, dev, 0, hc, seed=b.seed, pipeline=True)
    ms = bench.timed_steps(r, 50, 5, False) / 50
    res[hc] = {"step_ms": ms, "kernel_ms": r.kernel_ms()}
    del r
t1 = res[8]["step_ms"]
out = {str(8 // hc): {"heads_per_rank": hc, **v, "efficiency_est": t1 / ((8 // hc) * v["step_ms"]),
                      "kernel_eff_est": res[8]["kernel_ms"] / ((8 // hc) * v["kernel_ms"])}
       for hc, v in res.items()}
print(json.dumps(out, indent=1))
