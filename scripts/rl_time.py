"""Relayout kernel time (CUDA events, L2 flushed) of configs[1] at 1 / 2 / 8 local KV heads for the
libraries named on the command line (variants/libpi_<name>.so), alternated in one process."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_06072_b200 import packinfer as pk
from synth import workloads as W
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = {}
for v in sys.argv[1:]:
    pk._lib = None
    os.environ["PACKINFER_LIB"] = os.path.join(root, "variants", f"libpi_{v}.so")
    libs[v] = pk.lib()
b = W.cfg2_prefill(0)
t = W.make_tensors(b, device="cuda", seed=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for hc in (1, 2, 8):
    pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, hc, 4, b.d, torch.bfloat16, "cuda")
    res = {v: [] for v in libs}
    for rep in range(23):
        for v, L in libs.items():
            pk._lib = L
            flush.fill_(rep)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pk.packinfer_relayout_kv(pb.dp, t["k_paged"], t["v_paged"], t["block_table"], pb.k_buf, pb.v_buf, 0, hc)
            e1.record()
            torch.cuda.synchronize()
            if rep >= 3:
                res[v].append(e0.elapsed_time(e1) * 1e3)
    print(f"heads {hc}: " + "  ".join(f"{v} {np.median(x):.1f} us" for v, x in res.items()))
