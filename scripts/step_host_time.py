"""Host enqueue time of one bench step (Python + ctypes + C++ planner + tensor-map encodes) vs the
GPU time of the same step, per KV-head shard size of configs[1].  If the host time reaches the GPU
time the step is host-bound."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

dev = torch.device("cuda", 0)
b = bench.make_workload("cfg2", 0)
out = {}
for hc in (8, 1):
    r = bench.Runner(b, dev, 0, hc, seed=b.seed)
    for i in range(5):
        r.step(i)
    torch.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for i in range(n):
        r.step(10 + i, time_kernel=True)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    lat = r.step_latency()
    # split the step: time the pieces of one step with events on the stream
    pb = r.pbs[0]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    s = r.stream
    ev[0].record(s); pb.replan(s); ev[1].record(s)
    bench_pk = r.pk
    bench_pk.packinfer_relayout_kv(pb.dp, r.t["k_paged"], r.t["v_paged"], r.t["block_table"], pb.k_buf, pb.v_buf, 0, hc, s)
    ev[2].record(s)
    bench_pk.packinfer_attention(pb.dp, r.q, pb.k_buf, pb.v_buf, r.out, r.lse, pb.partial_o, pb.partial_lse, r.r, 0.0, s)
    ev[3].record(s)
    torch.cuda.synchronize()
    out[hc] = {"host_enqueue_ms_per_step": (t1 - t0) * 1e3 / n, "wall_ms_per_step": (t2 - t0) * 1e3 / n,
               "gpu_step_median_ms": lat["median_ms"], "kernel_ms": r.kernel_ms(),
               "piece_ms": {"upload+expand": ev[0].elapsed_time(ev[1]), "relayout": ev[1].elapsed_time(ev[2]),
                            "attention(incl. counter memset)": ev[2].elapsed_time(ev[3])}}
    del r
print(json.dumps(out, indent=1))
