"""In-process A/B of library variants (variants/libpi_<name>.so, optionally with plan flags:
<name>:<flags>) on one batch's attention launch:
the variants are loaded side by side and launched alternately on the same device plan and
buffers, with an L2 flush (256 MB write) before every timed launch, so process-to-process
spread (clocks, allocation placement) cancels.  Prints per-variant median / p10 / p90 ms.
    python scripts/ab_inproc.py cfg4_decode s8 s32 [--reps 40]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("variants", nargs="+")
ap.add_argument("--reps", type=int, default=40)
a = ap.parse_args()
from paper_2602_06072_b200 import packinfer as pk
import bench

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = {}
for v in a.variants:
    name = v.split(":")[0]
    if name not in libs:
        pk._lib = None
        os.environ["PACKINFER_LIB"] = os.path.join(root, "variants", f"libpi_{name}.so")
        libs[name] = pk.lib()
b = bench.make_workload(a.cfg, 0)
runners = {}
for v in a.variants:
    flags = ":".join(v.split(":")[1:]) if ":" in v else "default"
    if flags not in runners:
        if flags.count(":"):   # <lib>:<flags>:<PI_DPACK_ROWS> (planner A/B hook)
            os.environ["PI_DPACK_ROWS"] = flags.split(":")[1]
        pk._lib = libs[v.split(":")[0]]
        if flags == "default":
            os.environ.pop("PI_BENCH_PLAN_FLAGS", None)
        else:
            os.environ["PI_BENCH_PLAN_FLAGS"] = flags.split(":")[0]
        rr = bench.Runner(b, "cuda", 0, b.hkv, seed=b.seed)
        rr.step(0)
        runners[flags] = rr
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
times = {v: [] for v in a.variants}
for rep in range(a.reps + 3):
    for v in a.variants:
        pk._lib = libs[v.split(":")[0]]
        r = runners[":".join(v.split(":")[1:]) if ":" in v else "default"]
        pb = r.pbs[0]
        flush.fill_(rep & 0xff)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        pk.packinfer_attention(pb.dp, r.q, pb.k_buf, pb.v_buf, r.out, r.lse, pb.partial_o, pb.partial_lse,
                               r.r, 0.0, st)
        e1.record(st)
        torch.cuda.synchronize()
        if rep >= 3:
            times[v].append(e0.elapsed_time(e1))
for v in a.variants:
    t = np.array(times[v])
    print(f"{a.cfg} {v:>8s}: median {np.median(t):.4f} ms  p10 {np.percentile(t, 10):.4f}  p90 {np.percentile(t, 90):.4f}")
