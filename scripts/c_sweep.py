"""Offline capacity sweep on B200 (NEXT-2): for each
BASELINE.json workload and C in {1024 .. 16384}, the hot path (plan, relayout, one fused
attention launch, merge) timed with CUDA events; prints JSON with per-C device ms, groups, key
tiles and the offline choice, and an online-tuner replay that starts from a wrong prior.

Usage: python scripts/c_sweep.py [--reps 5] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2602_06072_b200 import packinfer as pk
from paper_2602_06072_b200.tuning import CapacityTuner, offline_profile
from synth import workloads as W

CANDS = [1024, 2048, 4096, 8192, 16384]


class Sweep:
    def __init__(self, b):
        self.b, self.r = b, b.hq // b.hkv
        self.t = W.make_tensors(b, device="cuda")
        self.out = torch.empty((b.total_q, b.hq, b.d), dtype=torch.bfloat16, device="cuda")
        self.lse = torch.empty((b.hq, b.total_q), dtype=torch.float32, device="cuda")
        self.pbs = {}
        self.info = {}

    def run(self, C):
        b, t = self.b, self.t
        if C not in self.pbs:
            self.pbs[C] = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, self.r, b.d,
                                         torch.bfloat16, "cuda", capacity=C)
        pb = self.pbs[C]
        h0 = time.perf_counter()
        pb.replan()
        host_ms = (time.perf_counter() - h0) * 1e3
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        pk.packinfer_relayout_kv(pb.dp, t["k_paged"], t["v_paged"], t["block_table"], pb.k_buf, pb.v_buf, 0, b.hkv)
        e1.record()
        pk.packinfer_attention(pb.dp, t["q"], pb.k_buf, pb.v_buf, self.out, self.lse, pb.partial_o, pb.partial_lse,
                               self.r)
        pk.packinfer_merge(pb.dp, pb.partial_o, pb.partial_lse, self.out, self.lse)
        e2.record()
        torch.cuda.synchronize()
        c = pb.plan.c
        self.info[C] = {"groups": int(c.n_groups), "work_items": int(c.n_prefill_work + c.n_decode_work),
                        "key_tiles": int(pb.plan.prefill_work["n_ktiles"].sum() + pb.plan.decode_work["n_ktiles"].sum()),
                        "buffer_kv_tokens": int(c.copy_tokens), "partial_slots": int(c.n_partial_slots),
                        "relayout_ms": e0.elapsed_time(e1), "attention_merge_ms": e1.elapsed_time(e2),
                        "host_plan_ms": host_ms}
        return e0.elapsed_time(e2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(0), "candidates": CANDS}
    for name, mk in (("cfg2_prefill", W.cfg2_prefill), ("cfg3_decode", W.cfg3_decode),
                     ("cfg4_decode", W.cfg4_decode)):
        sw = Sweep(mk())
        for C in CANDS:
            sw.run(C)                                  # warm-up (allocation, tensor maps)
        prof = offline_profile(sw.run, CANDS, reps=a.reps)
        best = min(prof, key=prof.get)
        # online replay: start from a deliberately wrong prior (C = 16384 best) and let
        # per-step samples move the choice
        tu = CapacityTuner(CANDS, prior={C: (0.5 if C == 16384 else 1e9) for C in CANDS})
        picks = []
        for _ in range(24):
            C = tu.choose()
            tu.observe(C, sw.run(C))
            picks.append(C)
        res[name] = {"device_ms": prof, "offline_best": best, "detail": sw.info,
                     "online_picks": picks, "online_best": tu.best()}
        del sw
        torch.cuda.empty_cache()
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s)


if __name__ == "__main__":
    main()
