"""Component breakdown on B200 (NEXT-4; the paper's Fig. "breakdown"):
packed compute vs packed I/O, each switched off on its own, same kernels, same inputs.

  * packed compute  — cfg2 prefill (BASELINE.json configs[1]) with and without packing short
    requests into shared 128-row Q tiles (pi_config.flags = PI_PLAN_NO_QPACK).
  * packed I/O      — cfg4 (configs[3], 8 shared 2k-token prompts) decode step and suffix
    prefill with prefix co-location (prefix ids: each prompt stored and streamed once per group,
    Eq. 5) and without (prefix_id = -1: every request carries its own copy, the naive volume).

Prints one JSON object (kernel ms from CUDA events, averaged over reps after warm-up; KV tokens
in the group buffers).  Usage: python scripts/breakdown.py [--reps 10] [--out FILE]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2602_06072_b200 import packinfer as pk
from synth import workloads as W


def measure(b, t, reps, flags=0, drop_prefix=False, capacity=8192):
    r = b.hq // b.hkv
    pid = np.full_like(b.prefix_id, -1) if drop_prefix else b.prefix_id
    plen = np.zeros(0, np.int32) if drop_prefix else b.prefix_len
    pb = pk.PackedBatch(b.kv_len, b.q_len, pid, plen, b.hkv, r, b.d, torch.bfloat16, "cuda", capacity=capacity)
    pb.cfg.flags = flags
    pb.replan()
    out = torch.empty((b.total_q, b.hq, b.d), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((b.hq, b.total_q), dtype=torch.float32, device="cuda")
    ev = lambda: torch.cuda.Event(enable_timing=True)
    times, rtimes = [], []
    for i in range(reps + 2):
        e0, e1, e2 = ev(), ev(), ev()
        e0.record()
        pk.packinfer_relayout_kv(pb.dp, t["k_paged"], t["v_paged"], t["block_table"], pb.k_buf, pb.v_buf, 0, b.hkv)
        e1.record()
        pk.packinfer_attention(pb.dp, t["q"], pb.k_buf, pb.v_buf, out, lse, pb.partial_o, pb.partial_lse, r)
        e2.record()
        pk.packinfer_merge(pb.dp, pb.partial_o, pb.partial_lse, out, lse)
        torch.cuda.synchronize()
        if i >= 2:
            rtimes.append(e0.elapsed_time(e1))
            times.append(e1.elapsed_time(e2))
    c = pb.plan.c
    return {"attention_ms": float(np.mean(times)), "relayout_ms": float(np.mean(rtimes)),
            "buffer_kv_tokens": int(c.copy_tokens), "work_items": int(c.n_prefill_work + c.n_decode_work),
            "key_tiles": int(pb.plan.prefill_work["n_ktiles"].sum() + pb.plan.decode_work["n_ktiles"].sum()),
            "tile_efficiency": float(c.valid_cells / max(1, c.tile_cells)), "groups": int(c.n_groups)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {}
    b = W.cfg2_prefill(0)
    t = W.make_tensors(b, device="cuda")
    res["cfg2_prefill"] = {"packed": measure(b, t, a.reps),
                           "unpacked_compute": measure(b, t, a.reps, flags=pk.PI_PLAN_NO_QPACK)}
    del t
    for name, mk in (("cfg4_decode", W.cfg4_decode), ("cfg4_suffix_prefill", W.cfg4_prefill)):
        b = mk()
        t = W.make_tensors(b, device="cuda")
        res[name] = {"packed_io": measure(b, t, a.reps),
                     "no_prefix_colocation": measure(b, t, a.reps, drop_prefix=True)}
        del t
    for k, v in res.items():
        base = list(v.values())[0]["attention_ms"]
        for kk, vv in v.items():
            vv["attention_vs_packed"] = vv["attention_ms"] / base
    res["gpu"] = torch.cuda.get_device_name(0)
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s)


if __name__ == "__main__":
    main()
