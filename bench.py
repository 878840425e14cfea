#!/usr/bin/env python
"""PackInfer hot-path benchmark (BASELINE.json metric: packed prefill TFLOP/s & decode KV HBM GB/s
vs B200 peak; batch step latency).

One STEP = one pass of the whole hot path over one batch:
    packinfer_plan (host C++) -> plan upload (H2D) -> packinfer_relayout_kv -> packed prefill
    -> packed decode -> LSE merge
Headline workload (N=1): BASELINE.json configs[1], the Llama-3-8B-shaped heterogeneous prefill
batch (64 requests, 16..8192 tokens; 32 Q / 8 KV heads, d=128, bf16).  value = algorithmic
prefill FLOPs / step time (TFLOP/s).  The decode row (configs[2], 256 requests, KV 32..32k) is
reported under "decode" (GB/s of Eq. 5 KV bytes).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--shard group|heads]
Multi-GPU (torchrun, one process per GPU): default --shard group = weak scaling, rank r runs
its own batch (seed 0 + r; groups of independent sub-batches, no collective on the data path);
--shard heads = strong scaling by KV head over one batch.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------- workloads
def make_workload(name: str, seed: int):
    from synth import workloads as W
    if name == "cfg2":
        return W.cfg2_prefill(seed)
    if name == "cfg3":
        return W.cfg3_decode(seed + 1)
    if name == "cfg4_decode":
        return W.cfg4_decode(seed + 2)
    raise ValueError(name)


def algorithmic(b, plan_c, hkv_local):
    """Algorithmic work of one step: prefill FLOPs over visible pairs only; decode
    bytes = Eq. 5 KV volume of the decode requests + their Q and O."""
    r = b.hq // b.hkv
    flops = 0
    for L, q in zip(b.kv_len.tolist(), b.q_len.tolist()):
        if q > 1:
            flops += q * (L - q) + q * (q + 1) // 2
    flops *= 4 * b.d * hkv_local * r
    es = 2 if b.dtype == "bf16" else 4
    dec_tokens = int(plan_c.copy_tokens) if (b.q_len == 1).all() else None
    kv_bytes = None if dec_tokens is None else 2 * dec_tokens * hkv_local * b.d * es
    qo_bytes = 2 * int((b.q_len == 1).sum()) * hkv_local * r * b.d * es
    return flops, kv_bytes, qo_bytes


METRIC = "packed prefill TFLOP/s (cfg2 batch step)"


def arm_config(b, shard, world):
    """The workload both arms (this implementation and --impl reference) report as `config`:
    only what defines the batch, nothing the planner derives (that goes under "plan")."""
    flops, _, _ = algorithmic(b, None, b.hkv)
    return {"workload": b.name + " (BASELINE.json configs[1])", "requests": b.n, "tokens": int(b.kv_len.sum()),
            "hq": b.hq, "hkv": b.hkv, "head_dim": b.d, "capacity": 8192,
            "l2": "inputs larger than L2 (paged KV 224 MB + Q 448 MB per step > 126 MB)",
            "parallelism": f"{shard}-sharded x{world}", "algorithmic_tflop": flops / 1e12}


class Runner:
    """Owns the device state of one batch and runs steps on one stream (double-buffered plans)."""

    def __init__(self, b, device, hkv_begin, hkv_count, capacity=8192, headroom=0, seed=0):
        import torch
        from synth import workloads as W
        from paper_2602_06072_b200 import packinfer as pk
        self.pk, self.torch, self.b = pk, torch, b
        self.r = b.hq // b.hkv
        self.hkv_begin, self.hkv_count = hkv_begin, hkv_count
        self.t = W.make_tensors(b, device=device, seed=seed)
        dt = self.t["q"].dtype
        self.pbs = [pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, hkv_count, self.r, b.d, dt,
                                   device, capacity=capacity, headroom=headroom) for _ in range(2)]
        self.events = [torch.cuda.Event() for _ in range(2)]
        for e in self.events:
            e.record()
        self.q = self.t["q"][:, hkv_begin * self.r:(hkv_begin + hkv_count) * self.r]
        self.out = torch.empty((b.total_q, hkv_count * self.r, b.d), dtype=dt, device=device)
        self.lse = torch.empty((hkv_count * self.r, b.total_q), dtype=torch.float32, device=device)
        self.stream = torch.cuda.current_stream()
        c = self.pbs[0].plan.c
        self.launches_per_step = 1 + (c.n_prefill_work > 0) + (c.n_decode_work > 0) + (c.n_merges > 0)
        self.kernel_events = []
        self.step_events = []

    def step(self, i, time_kernel=False, t=None, out=None):
        """One batch step on this runner's stream; t / out select another (e.g. double-buffered)
        input set / output buffer of the same shapes."""
        pk, torch = self.pk, self.torch
        t = self.t if t is None else t
        q = self.q if t is self.t else t["q"][:, self.hkv_begin * self.r:(self.hkv_begin + self.hkv_count) * self.r]
        out = self.out if out is None else out
        pb = self.pbs[i % 2]
        if time_kernel:
            es = torch.cuda.Event(enable_timing=True)
            es.record(self.stream)
        self.events[i % 2].synchronize()            # host arena of this slot no longer read by H2D
        pb.replan(self.stream)                       # host planner + async upload
        self.events[i % 2].record(self.stream)
        pk.packinfer_relayout_kv(pb.dp, t["k_paged"], t["v_paged"], t["block_table"], pb.k_buf,
                                 pb.v_buf, self.hkv_begin, self.hkv_count, self.stream)
        if time_kernel:
            e0, e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), \
                torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
        pk.packinfer_attention_prefill(pb.dp, q, pb.k_buf, pb.v_buf, out, self.lse, pb.partial_o,
                                       pb.partial_lse, self.r, 0.0, self.stream)
        if time_kernel:
            e1.record(self.stream)
        pk.packinfer_attention_decode(pb.dp, q, pb.k_buf, pb.v_buf, out, self.lse, pb.partial_o,
                                      pb.partial_lse, self.r, 0.0, self.stream)
        if time_kernel:
            e2.record(self.stream)
            self.kernel_events.append((e0, e1, e2))
        pk.packinfer_merge(pb.dp, pb.partial_o, pb.partial_lse, out, self.lse, self.stream)
        if time_kernel:
            ee = torch.cuda.Event(enable_timing=True)
            ee.record(self.stream)
            self.step_events.append((es, ee))

    def step_latency(self):
        """Per-step device latency (first to last op of the step on the stream): median, p90."""
        import numpy as np
        v = np.array([a.elapsed_time(b) for a, b in self.step_events])
        return {"median_ms": float(np.median(v)), "p90_ms": float(np.percentile(v, 90)), "n": int(v.size)}

    def kernel_ms(self):
        pre = [a.elapsed_time(b) for a, b, _ in self.kernel_events]
        dec = [b.elapsed_time(c) for _, b, c in self.kernel_events]
        return (sum(pre) / len(pre) if pre else 0.0), (sum(dec) / len(dec) if dec else 0.0)


def timed_steps(runner, steps, warmup, dist_on):
    import torch
    for i in range(warmup):
        runner.step(i)
    torch.cuda.synchronize()
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    runner.kernel_events.clear()
    runner.step_events.clear()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(steps):
        runner.step(warmup + i, time_kernel=True)
    e.record()
    torch.cuda.synchronize()
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
    return s.elapsed_time(e)


def e2e_steps(b, runner, steps):
    """Same metric through the public API with HOST buffers: every step copies the step's inputs
    H2D from pinned memory, runs the hot path, and reads the output back D2H.  The copies are
    pipelined the way a serving loop would run them: two device input sets and two output
    buffers, H2D of step i+1 on a copy-in stream and D2H of step i-1 on a copy-out stream while
    step i computes (PCIe is full duplex, so the step costs max(H2D, compute, D2H) in steady state).
    Every step still moves all of its own bytes; the timed region runs from the first H2D to the
    last D2H."""
    import torch
    t0 = runner.t
    host = {k: v.cpu().pin_memory() for k, v in t0.items()}
    sets = [t0, {k: torch.empty_like(v) for k, v in t0.items()}]
    outs = [runner.out, torch.empty_like(runner.out)]
    outs_h = [torch.empty(runner.out.shape, dtype=runner.out.dtype).pin_memory() for _ in range(2)]
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    d2h = outs_h[0].numel() * outs_h[0].element_size()
    comp = runner.stream
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    in_ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    out_free = [torch.cuda.Event() for _ in range(2)]
    for e in done + out_free:
        e.record(comp)

    def run(n, base):
        for i in range(n):
            k = i % 2
            s_in.wait_event(done[k])                 # step i-2 no longer reads input set k
            with torch.cuda.stream(s_in):
                for name in host:
                    sets[k][name].copy_(host[name], non_blocking=True)
            in_ready[k].record(s_in)
            comp.wait_event(in_ready[k])
            comp.wait_event(out_free[k])             # D2H of step i-2 no longer reads out[k]
            runner.step(base + i, t=sets[k], out=outs[k])
            done[k].record(comp)
            s_out.wait_event(done[k])
            with torch.cuda.stream(s_out):
                outs_h[k].copy_(outs[k], non_blocking=True)
            out_free[k].record(s_out)
        comp.wait_event(out_free[(n - 1) % 2])
        comp.wait_event(out_free[n % 2])

    run(2, 20_000)                                   # warm-up (streams, pinned transfers)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(comp)
    s_in.wait_event(s)
    run(steps, 10_000)
    e.record(comp)
    torch.cuda.synchronize()
    # the last step's output landed on the host: spot-check it against the device copy
    k = (steps - 1) % 2
    assert torch.equal(outs_h[k][:4].to(outs[k].device), outs[k][:4])
    return s.elapsed_time(e) / steps, h2d, d2h


def decode_group_sharded(dev, rank, world, args, peaks):
    """N > 1 only: ONE configs[2] decode batch (the same on every rank) group-sharded across the
    ranks (shard.RankPlan, SURVEY 8(e) optional group sharding): each rank consolidates and attends
    only its groups; split rows are completed by shard.combine (SUM / MAX all-reduce over NCCL) and
    the batch merge.  Step = relayout (own groups) + decode attention (own items) + combine + merge,
    timed with CUDA events, max over ranks (strong scaling of one batch)."""
    import torch
    import torch.distributed as dist
    from paper_2602_06072_b200 import packinfer as pk, shard
    bd = make_workload("cfg3", 0)
    r = bd.hq // bd.hkv
    t = W_tensors(bd, dev)
    pb = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, bd.hkv, r, bd.d, t["q"].dtype, dev)
    owner = shard.group_shard(shard.group_costs(pb.plan), world)
    rp = shard.RankPlan(pb, owner, rank)
    out = torch.empty((bd.total_q, bd.hq, bd.d), dtype=t["q"].dtype, device=dev)
    st = torch.cuda.current_stream()

    def once():
        pk.packinfer_relayout_kv(rp.dp, t["k_paged"], t["v_paged"], t["block_table"], pb.k_buf, pb.v_buf, 0,
                                 bd.hkv, st)
        shard.init_partials(pb.partial_o, pb.partial_lse, out)
        pk.packinfer_attention_decode(rp.dp, t["q"], pb.k_buf, pb.v_buf, out, None, pb.partial_o,
                                      pb.partial_lse, r, 0.0, st)
        shard.combine(pb.partial_o, pb.partial_lse, out)
        pk.packinfer_merge(pb.dp, pb.partial_o, pb.partial_lse, out, None, st)

    for _ in range(args.warmup):
        once()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(3, args.steps)
    e0.record(st)
    for _ in range(n):
        once()
    e1.record(st)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / n], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    kv_bytes = 2 * int(pb.plan.c.copy_tokens) * bd.hkv * bd.d * 2
    return {"workload": bd.name + " (BASELINE.json configs[2]), one batch over all ranks",
            "ms_per_step": float(ms[0]), "step_gbs": kv_bytes / (float(ms[0]) * 1e-3) / 1e9,
            "rank_cells": rp.cells, "rank_work_items": rp.n_work, "groups": int(pb.plan.c.n_groups),
            "scaling": "strong", "note": "relayout + decode attention of this rank's groups, SUM/MAX "
                                         "all-reduce of partials and direct rows, merge"}


def W_tensors(b, dev):
    from synth import workloads as W
    return W.make_tensors(b, device=dev, seed=b.seed)


def mixed_section(dev, h0, hc, rank, args, peaks, dist_on):
    """BASELINE.json configs[4]: Llama-3-70B-shaped mixed batch (2 x 128k-token prefills split
    across groups + 30 short prefills + 224 decodes up to 32k), ONE fused attention launch over
    prefill and decode work items (NEXT-3) + LSE merge; the split form (one launch per kind) is
    timed beside it on the same plan."""
    import torch
    from synth import workloads as W
    from paper_2602_06072_b200 import packinfer as pk
    bm = W.cfg5_mixed(3 + (0 if args.shard == "heads" else rank))
    r = bm.hq // bm.hkv
    tm = W.make_tensors(bm, device=dev, seed=bm.seed)
    pbm = pk.PackedBatch(bm.kv_len, bm.q_len, bm.prefix_id, bm.prefix_len, hc, r, bm.d, torch.bfloat16, dev)
    qm = tm["q"][:, h0 * r:(h0 + hc) * r]
    outm = torch.empty((bm.total_q, hc * r, bm.d), dtype=torch.bfloat16, device=dev)
    lsem = torch.empty((hc * r, bm.total_q), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def once(fused, times):
        pbm.replan(st)
        pk.packinfer_relayout_kv(pbm.dp, tm["k_paged"], tm["v_paged"], tm["block_table"], pbm.k_buf, pbm.v_buf,
                                 h0, hc, st)
        a, m, e = ev(), ev(), ev()
        a.record(st)
        if fused:
            pk.packinfer_attention(pbm.dp, qm, pbm.k_buf, pbm.v_buf, outm, lsem, pbm.partial_o, pbm.partial_lse,
                                   r, 0.0, st)
            m.record(st)
        else:
            pk.packinfer_attention_prefill(pbm.dp, qm, pbm.k_buf, pbm.v_buf, outm, lsem, pbm.partial_o,
                                           pbm.partial_lse, r, 0.0, st)
            m.record(st)
            pk.packinfer_attention_decode(pbm.dp, qm, pbm.k_buf, pbm.v_buf, outm, lsem, pbm.partial_o,
                                          pbm.partial_lse, r, 0.0, st)
        e.record(st)
        pk.packinfer_merge(pbm.dp, pbm.partial_o, pbm.partial_lse, outm, lsem, st)
        times.append((a, m, e))

    steps = 2
    for fused in (True, False):
        once(fused, [])
    torch.cuda.synchronize()
    res = {}
    for fused in (True, False):
        times = []
        s0, s1 = ev(), ev()
        s0.record(st)
        for _ in range(steps):
            once(fused, times)
        s1.record(st)
        torch.cuda.synchronize()
        res[fused] = (s0.elapsed_time(s1) / steps, sum(a.elapsed_time(e) for a, _, e in times) / steps,
                      sum(a.elapsed_time(m) for a, m, _ in times) / steps)
    step_ms, fused_ms, _ = res[True]
    _, split_ms, split_pre_ms = res[False]
    flops = 4 * bm.d * hc * r * sum(q * (L - q) + q * (q + 1) // 2
                                    for L, q in zip(bm.kv_len.tolist(), bm.q_len.tolist()) if q > 1)
    c = pbm.plan.c
    out = {"workload": bm.name + " (BASELINE.json configs[4])", "requests": bm.n,
           "prefill_tokens": int(bm.q_len[bm.q_len > 1].sum()), "decode_requests": int((bm.q_len == 1).sum()),
           "hq": bm.hq, "hkv": bm.hkv, "groups": int(c.n_groups), "prefill_items": int(c.n_prefill_work),
           "decode_items": int(c.n_decode_work), "partial_slots": int(c.n_partial_slots),
           "prefill_tflop": flops / 1e12, "ms_per_step": step_ms,
           "fused_attention_ms": fused_ms, "split_attention_ms": split_ms, "split_prefill_ms": split_pre_ms,
           "tflops_fused": flops / (fused_ms * 1e-3) / 1e12,
           "frac_fused": flops / (fused_ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
           "note": "tflops_fused counts prefill FLOPs only over the fused (prefill + decode) kernel time",
           "gpu_launches": 4 * steps}
    del tm, pbm
    return out


# ------------------------------------------------------------------------------- oracle timing
def oracle_sample(b, budget_s: float, seed: int):
    """Times the oracle (as it stands) on a bounded sample of the workload's requests on this
    host.  Returns (algorithmic FLOP/s or KV bytes/s, seconds, description, cores)."""
    import torch
    from oracle import attention as OA
    from synth import workloads as W
    cores = len(os.sched_getaffinity(0))
    t = W.make_tensors(b, device="cpu", seed=seed)
    order = np.argsort(b.kv_len)                      # short requests first, then longer ones
    done, flops, kv_bytes, t0 = [], 0, 0, time.time()
    for i in order:
        if time.time() - t0 > budget_s:
            break
        OA.attention(t["q"], t["k_paged"], t["v_paged"], t["block_table"], b.kv_len, b.q_len, b.page_size,
                     requests=[int(i)])
        L, q = int(b.kv_len[i]), int(b.q_len[i])
        flops += 4 * b.d * b.hq * (q * (L - q) + q * (q + 1) // 2)
        kv_bytes += 2 * L * b.hkv * b.d * 2
        done.append(int(i))
    dt = time.time() - t0
    desc = (f"{len(done)}/{b.n} requests of {b.name} (shortest first, {int(b.kv_len[done].sum())} KV tokens), "
            f"fp64 numpy, {dt:.1f}s")
    return flops, kv_bytes, dt, desc, cores


def run_reference(args, cfg_name):
    """--impl reference: the oracle timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    b = make_workload(cfg_name, 0)
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(b, per_step, 0)
    vals, secs = [], []
    desc, cores = "", 1
    for _ in range(args.steps):
        f, kvb, dt, desc, cores = oracle_sample(b, per_step, 0)
        vals.append(f / dt / 1e12)
        secs.append(dt)
    v = sum(vals) / len(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * sum(secs) / len(secs), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(b, args.shard, args.gpus),
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="packinfer", choices=["packinfer", "reference"])
    ap.add_argument("--shard", default="group", choices=["group", "heads"])
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-loop", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-mixed", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args, "cfg2")
        return

    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: PI_BENCH_ONE_GPU=1 puts every rank on cuda:0 with gloo (exercises the N > 1 code
    # path on a one-GPU box; never used for a reported number)
    one_gpu = os.environ.get("PI_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist_on = world > 1
    if dist_on:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peak_src = load_peaks()
    dev = torch.device("cuda", local)

    b = make_workload("cfg2", 0 if args.shard == "heads" else rank)
    if args.shard == "heads" and world > 1:
        from paper_2602_06072_b200 import shard
        h0, hc = shard.kv_head_shard(b.hkv, rank, world)
    else:
        h0, hc = 0, b.hkv
    runner = Runner(b, dev, h0, hc, seed=b.seed)
    flops, _, _ = algorithmic(b, runner.pbs[0].plan.c, hc)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    total_ms = timed_steps(runner, args.steps, args.warmup, dist_on)
    clocks = sampler.stop()
    ms_step = total_ms / args.steps
    pre_ms, _ = runner.kernel_ms()
    units_total = flops
    if dist_on:
        import torch.distributed as dist
        tt = torch.tensor([ms_step, pre_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)           # step time = slowest rank
        ms_step, pre_ms = float(tt[0]), float(tt[1])
        ft = torch.tensor([float(flops)], device=dev, dtype=torch.float64)
        dist.all_reduce(ft, op=dist.ReduceOp.SUM)           # work of every rank's shard / batch
        units_total = float(ft[0])
    value = units_total / (ms_step * 1e-3) / 1e12
    pc = runner.pbs[0].plan.c
    achieved = flops / (pre_ms * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get("prefill_attention_dram_bytes")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["bf16_tflops"], "traffic": traffic,
                "kernel": "packed_attention_kernel<128,bf16> (prefill)", "kernel_ms": pre_ms,
                "peak_source": peak_src + " bf16 burst", "frac_of_sustained": achieved / peaks.get(
                    "bf16_tflops_sustained", peaks["bf16_tflops"]),
                "tile_efficiency": pc.valid_cells / max(1, pc.tile_cells)}
    # The softmax's exponentials have their own ceiling: one exp2 per visible
    # (query, key) pair and query head, 16 per clock per SM on MUFU (measured,
    # profiles/r01d/mufu_bench.txt); the kernel moves 2 of 8 pairs to the FMA pipe.
    n_exp = flops / (4 * b.d)                                   # = Hq_local * visible pairs
    sm_hz = peaks.get("sm_max_mhz", 1965.0) * 1e6
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    roofline["exp_ceiling"] = {"exps": n_exp, "mufu_only_ms_at_max_clock": n_exp / (16 * nsm * sm_hz) * 1e3,
                               "tensor_only_ms_at_max_clock": flops / (8192 * nsm * sm_hz) * 1e3,
                               "note": "dense bf16 tcgen05 = 8192 FLOP/clk/SM; MUFU ex2 = 16/clk/SM"}

    result = {"metric": METRIC, "value": value, "unit": "TFLOP/s",
              "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
              "higher_is_better": True, "scaling": "weak" if args.shard == "group" else "strong",
              "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
              "config": arm_config(b, args.shard, world),
              "plan": {"groups": int(pc.n_groups), "work_items": int(pc.n_prefill_work),
                       "step": "plan+upload+relayout+prefill(+decode+merge)",
                       "algorithmic_tflop_per_rank": flops / 1e12},
              "roofline": roofline, "clocks": clocks, "step_latency": runner.step_latency(),
              "gpu_launches": runner.launches_per_step * args.steps}

    if dist_on and args.shard == "heads":
        # Full O on every rank (only for callers that need it; not part of the timed step): one
        # NCCL all-gather of the head-sharded outputs over NVLink.
        from paper_2602_06072_b200 import shard
        import torch.distributed as dist
        shard.gather_heads(runner.out, world, b.hkv, runner.r)
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        g0.record()
        for _ in range(reps):
            full = shard.gather_heads(runner.out, world, b.hkv, runner.r)
        g1.record()
        torch.cuda.synchronize()
        gt = torch.tensor([g0.elapsed_time(g1) / reps], device=dev)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gbytes = full.numel() * full.element_size()
        result["gather"] = {"ms": float(gt[0]), "bytes_out": gbytes,
                            "step_ms_with_gather": ms_step + float(gt[0]),
                            "note": "NCCL all_gather_into_tensor of head-major O slabs + layout copy"}
        del full

    if not args.no_decode:
        bd = make_workload("cfg3", 0 if args.shard == "heads" else rank)
        rd = Runner(bd, dev, h0, hc, seed=bd.seed)
        _, kvb, qob = algorithmic(bd, rd.pbs[0].plan.c, hc)
        dms = timed_steps(rd, max(3, args.steps), args.warmup, dist_on) / max(3, args.steps)
        _, dec_ms = rd.kernel_ms()
        ach = (kvb + qob) / (dec_ms * 1e-3) / 1e9
        dtraffic = None
        if os.path.exists(tf):
            dtraffic = json.load(open(tf)).get("decode_attention_dram_bytes")
        result["decode"] = {"workload": bd.name + " (BASELINE.json configs[2])", "ms_per_step": dms, "traffic": dtraffic,
                            "kernel_ms": dec_ms, "kv_bytes": kvb, "achieved_gbs": ach, "peak_gbs": peaks["hbm_gbs"],
                            "frac": ach / peaks["hbm_gbs"], "bound": "hbm",
                            "step_gbs": (kvb + qob) / (dms * 1e-3) / 1e9,
                            "work_items": int(rd.pbs[0].plan.c.n_decode_work),
                            "partial_slots": int(rd.pbs[0].plan.c.n_partial_slots),
                            "step_latency": rd.step_latency()}
        result["decode"]["gpu_launches"] = rd.launches_per_step * max(3, args.steps)
        del rd

    if dist_on and not args.no_decode:
        result["decode_group_sharded"] = decode_group_sharded(dev, rank, world, args, peaks)

    if not args.no_decode and not args.no_loop:
        # Decode loop (NEXT-1): consolidate once with headroom delta = 32
        # (= max new tokens), then each step appends one token per request into its headroom,
        # re-plans the execution domain on the host (packinfer_plan_step) and runs decode + merge.
        import torch
        bd = make_workload("cfg3", 0 if args.shard == "heads" else rank)
        from synth import workloads as W
        from paper_2602_06072_b200 import packinfer as pk
        loop_steps, delta = 32, 32
        tl = W.make_tensors(bd, device=dev, seed=bd.seed, extra_tokens=loop_steps)
        rr = bd.hq // bd.hkv
        pbl = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, hc, rr, bd.d, torch.bfloat16, dev,
                             headroom=delta)
        ql = tl["q"][:, h0 * rr:(h0 + hc) * rr]
        outl = torch.empty((bd.n, hc * rr, bd.d), dtype=torch.bfloat16, device=dev)
        kn = torch.randn((bd.n, bd.hkv, bd.d), device=dev).to(torch.bfloat16)
        vn = torch.randn_like(kn)
        def loop_once():
            pbl.replan()
            pbl.run(ql, tl["k_paged"], tl["v_paged"], tl["block_table"], outl, hkv_begin=h0)   # consolidation
            for k in range(1, loop_steps):
                pbl.append(kn, vn, hkv_begin=h0)
                pbl.replan(appended=np.full(bd.n, k, np.int32))
                pbl.run(ql, tl["k_paged"], tl["v_paged"], tl["block_table"], outl, hkv_begin=h0, relayout=False)
        loop_once()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        loop_once()
        e1.record()
        torch.cuda.synchronize()
        lms = e0.elapsed_time(e1) / loop_steps
        kv_tokens = sum(int(bd.kv_len.sum()) + k * bd.n for k in range(loop_steps)) / loop_steps
        lbytes = 2 * kv_tokens * hc * bd.d * 2 + 2 * bd.n * hc * rr * bd.d * 2
        result.setdefault("decode", {})["loop"] = {
            "steps": loop_steps, "headroom": delta, "ms_per_step_amortized": lms,
            "step_gbs_amortized": lbytes / (lms * 1e-3) / 1e9,
            "note": "consolidation (relayout) once per 32 steps; per step: append + plan_step + upload + "
                    "decode attention + merge"}
        del tl, pbl

    if not args.no_mixed:
        result["mixed"] = mixed_section(dev, h0, hc, rank, args, peaks, dist_on)

    if not args.no_e2e:
        e_ms, h2d, d2h = e2e_steps(b, runner, max(2, min(args.steps, 10)))
        if dist_on:
            import torch.distributed as dist
            et = torch.tensor([e_ms], device=dev)
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
            e_ms = float(et[0])
        result["e2e"] = {"value": units_total / (e_ms * 1e-3) / 1e12,
                         "unit": "TFLOP/s", "ms_per_step": e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                         "note": "pinned host buffers; H2D of step i+1 and D2H of step i-1 overlap step i "
                                 "(double-buffered device inputs/outputs, copy-in / copy-out streams)"}

    if rank == 0 and world == 1 and not args.no_cpu:
        f, kvb, dt, desc, cores = oracle_sample(b, args.cpu_budget, b.seed)
        result["cpu_baseline"] = {"value": f / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                                  "sample": desc}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist_on:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
