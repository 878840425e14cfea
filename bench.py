#!/usr/bin/env python
"""PackInfer hot-path benchmark (BASELINE.json metric: packed prefill TFLOP/s & decode KV HBM GB/s
vs B200 peak; batch step latency).

One STEP = one pass of the whole hot path over one batch:
    packinfer_plan (host C++) -> plan upload (H2D + device row expansion) -> packinfer_relayout_kv
    -> packed prefill -> packed decode -> LSE merge
Headline workload (N=1): BASELINE.json configs[1], the Llama-3-8B-shaped heterogeneous prefill
batch (64 requests, 16..8192 tokens; 32 Q / 8 KV heads, d=128, bf16).  value = algorithmic
prefill FLOPs / step time (TFLOP/s).  Side sections: configs[2] decode (GB/s of Eq. 5 KV bytes),
configs[3] shared-prefix decode + suffix prefill, configs[4] mixed 70B batch (one fused launch),
the decode loop (NEXT-1) with the online capacity tuner (NEXT-2), planner host microseconds.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--shard heads|group]
--gpus N > 1 without a torchrun environment re-launches itself under torchrun (one process per
GPU, 127.0.0.1 rendezvous).  --shard heads (default) = STRONG scaling: every rank runs the same
batch on its KV-head share (no collective on the data path), value = the batch's FLOPs / max-over-
ranks step time, and the line carries strong_scaling = T(1) / (N T(N)) measured in the same run.
--shard group = weak scaling: rank r runs its own batch (seed + r).
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
    """nvidia-smi every 10 ms in a background thread; summaries cover only the samples taken
    inside a given host-time window (the timed region), so idle or set-up periods never enter
    the reported clock."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int, interval_ms: int = 10):
        self.idx = gpu_index
        self.interval_ms = interval_ms
        self.proc = None
        self.samples = []          # (host time, sm MHz, max MHz, power W, reasons)
        self.thread = None

    def start(self, wait_s: float = 3.0):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < wait_s:   # first sample = sampler running
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.strip().split(",")]
            if len(f) < 9:
                continue
            try:
                sm, mx = float(f[1]), float(f[2])
                pw = float(f[3]) if f[3] not in ("[N/A]", "") else None
            except ValueError:
                continue
            reasons = {n for n, v in zip(self.NAMES, f[5:9]) if v.lower() == "active"}
            self.samples.append((time.time(), sm, mx, pw, reasons))

    def window(self, t0: float, t1: float):
        """Clock summary of the samples taken in [t0, t1] (host time)."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        inside = [x for x in list(self.samples) if t0 <= x[0] <= t1]
        if not inside:
            # region shorter than one sampling interval: the sample closest to its middle
            mid = 0.5 * (t0 + t1)
            allx = list(self.samples)
            if not allx:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
            inside = [min(allx, key=lambda x: abs(x[0] - mid))]
        reasons = sorted(set().union(*[x[4] for x in inside]))
        pw = [x[3] for x in inside if x[3] is not None]
        return {"sm_mhz": statistics.median(x[1] for x in inside), "sm_max_mhz": max(x[2] for x in inside),
                "sm_mhz_min": min(x[1] for x in inside), "power_w_median": statistics.median(pw) if pw else None,
                "reasons": reasons, "samples": len(inside), "interval_ms": self.interval_ms,
                "window_ms": (t1 - t0) * 1e3}

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)


# ------------------------------------------------------------------------------- workloads
def make_workload(name: str, seed: int):
    from synth import workloads as W
    if name == "cfg2":
        return W.cfg2_prefill(seed)
    if name == "cfg3":
        return W.cfg3_decode(seed + 1)
    if name == "cfg4_decode":
        return W.cfg4_decode(seed + 2)
    if name == "cfg4_prefill":
        return W.cfg4_prefill(seed + 2)
    if name == "cfg5":
        return W.cfg5_mixed(seed + 3)
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
# the step's attention: one launch + the packinfer_merge launch (default, measured fastest:
# profiles/r02b/ab_merge.txt), or PI_BENCH_SEPARATE_MERGE=0 for packinfer_attention_merge (merge in-kernel)
SEPARATE_MERGE = os.environ.get("PI_BENCH_SEPARATE_MERGE", "1") == "1"
PIPELINE = os.environ.get("PI_BENCH_PIPELINE", "1") == "1"       # A/B hook: headline steps pipelined


def arm_config(b, shard, world):
    """The workload both arms (this implementation and --impl reference) report as `config`:
    only what defines the batch, nothing the planner derives (that goes under "plan")."""
    flops, _, _ = algorithmic(b, None, b.hkv)
    return {"workload": b.name + " (BASELINE.json configs[1])", "requests": b.n, "tokens": int(b.kv_len.sum()),
            "hq": b.hq, "hkv": b.hkv, "head_dim": b.d, "capacity": 8192,
            "l2": "inputs larger than L2 (paged KV 224 MB + Q 448 MB per step > 126 MB)",
            "parallelism": f"{shard}-sharded x{world}", "algorithmic_tflop": flops / 1e12}


def plan_flags():
    """Plan flags of every section: None = packinfer_default_config's (packed decode items);
    PI_BENCH_PLAN_FLAGS = A/B hook (ablations, options)."""
    v = os.environ.get("PI_BENCH_PLAN_FLAGS")
    return None if v is None else int(v)


class Runner:
    """Owns the device state of one batch and runs steps on one stream (double-buffered plans)."""

    def __init__(self, b, device, hkv_begin, hkv_count, capacity=8192, headroom=0, seed=0, pipeline=False):
        import torch
        from synth import workloads as W
        from paper_2602_06072_b200 import packinfer as pk
        self.pk, self.torch, self.b = pk, torch, b
        self.r = b.hq // b.hkv
        self.hkv_begin, self.hkv_count = hkv_begin, hkv_count
        self.t = W.make_tensors(b, device=device, seed=seed)
        dt = self.t["q"].dtype
        flags = plan_flags()
        flags = pk.default_config().flags if flags is None else flags
        if hkv_count * b.hq // b.hkv <= 8:
            # few units per SM (KV-head sharding at N >= 4): balance over L2 locality
            flags |= pk.PI_PLAN_LPT_EXACT
        chunk = int(os.environ.get("PI_BENCH_DECODE_CHUNK", "1024"))  # A/B hook
        self.pbs = [pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, hkv_count, self.r, b.d, dt,
                                   device, capacity=capacity, headroom=headroom, flags=flags, decode_chunk=chunk)
                    for _ in range(2)]
        # Two streams, software-pipelined across steps: step i's host plan + upload (+ row
        # expansion) + relayout run on `aux` into plan slot i % 2 while step i-1's attention runs on
        # the main stream; attention i waits for its slot (ready[]), aux waits until attention i-2
        # released the slot (done[]).  Every step still does all of its work.
        # (pipeline=False: one stream, steps strictly sequential - for sections whose kernel
        # roofline must not share the GPU with the next step's relayout)
        self.stream = torch.cuda.current_stream()
        self.aux = torch.cuda.Stream() if pipeline else self.stream
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.done = [torch.cuda.Event() for _ in range(2)]
        for e in self.done:
            e.record()
        self.q = self.t["q"][:, hkv_begin * self.r:(hkv_begin + hkv_count) * self.r]
        self.out = torch.empty((b.total_q, hkv_count * self.r, b.d), dtype=dt, device=device)
        self.lse = torch.empty((hkv_count * self.r, b.total_q), dtype=torch.float32, device=device)
        c = self.pbs[0].plan.c
        self.relayout = True
        # relayout + row expansion (inside the plan upload) + one attention launch + merge
        self.launches_per_step = 1 + (c.n_segs > 0) + 1 + (SEPARATE_MERGE and c.n_merges > 0)
        self.kernel_events = []
        self.relayout_events = []
        self.step_events = []

    def begin(self, ev):
        """The aux stream's next work may not start before event `ev` (a timed region's start)."""
        self.aux.wait_event(ev)

    def step(self, i, time_kernel=False, t=None, out=None, wait_event=None):
        """One batch step on this runner's stream: host plan + upload (+ device row expansion),
        relayout (unless self.relayout is False: KV resident in the group layout), then ONE
        attention launch over every work item (packinfer_attention) and the LSE merge of split rows
        (packinfer_merge; or in-kernel with packinfer_attention_merge, see SEPARATE_MERGE).
        t / out select another (e.g. double-buffered) input set / output buffer of the same
        shapes; wait_event: an event the step's inputs depend on (e2e: their H2D landed)."""
        pk, torch = self.pk, self.torch
        t = self.t if t is None else t
        q = self.q if t is self.t else t["q"][:, self.hkv_begin * self.r:(self.hkv_begin + self.hkv_count) * self.r]
        out = self.out if out is None else out
        k = i % 2
        pb = self.pbs[k]
        aux = self.aux
        aux.wait_event(self.done[k])                 # attention i-2 no longer reads slot k
        if wait_event is not None:
            aux.wait_event(wait_event)
        if time_kernel:
            es = torch.cuda.Event(enable_timing=True)
            es.record(aux)
        pb.replan(aux)                               # host planner + async upload + row expansion
        if self.relayout:
            if time_kernel:
                r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                r0.record(aux)
            pk.packinfer_relayout_kv(pb.dp, t["k_paged"], t["v_paged"], t["block_table"], pb.k_buf,
                                     pb.v_buf, self.hkv_begin, self.hkv_count, aux)
            if time_kernel:
                r1.record(aux)
                self.relayout_events.append((r0, r1))
        self.ready[k].record(aux)
        self.stream.wait_event(self.ready[k])
        if time_kernel:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
        if SEPARATE_MERGE:   # A/B hook: attention launch + packinfer_merge launch
            pk.packinfer_attention(pb.dp, q, pb.k_buf, pb.v_buf, out, self.lse, pb.partial_o, pb.partial_lse,
                                   self.r, 0.0, self.stream)
            if time_kernel:
                em = torch.cuda.Event(enable_timing=True)
                em.record(self.stream)
            pk.packinfer_merge(pb.dp, pb.partial_o, pb.partial_lse, out, self.lse, self.stream)
        else:
            pk.packinfer_attention_merge(pb.dp, q, pb.k_buf, pb.v_buf, out, self.lse, pb.partial_o, pb.partial_lse,
                                         pb.merge_counters, self.r, 0.0, self.stream)
        self.done[k].record(self.stream)
        if time_kernel:
            e1.record(self.stream)
            # the attention launch alone (the roofline kernel) and the whole attention + merge
            self.kernel_events.append((e0, em if SEPARATE_MERGE else e1, e1))
            ee = torch.cuda.Event(enable_timing=True)
            ee.record(self.stream)
            self.step_events.append((es, ee))

    def step_latency(self):
        """Per-step device latency (first to last op of the step on the stream): median, p90."""
        import numpy as np
        v = np.array([a.elapsed_time(b) for a, b in self.step_events])
        return {"median_ms": float(np.median(v)), "p90_ms": float(np.percentile(v, 90)), "n": int(v.size)}

    def kernel_ms(self):
        """Average time of the step's attention launch (prefill + decode items; + the merge when it
        runs in-kernel): the roofline kernel."""
        v = [a.elapsed_time(b) for a, b, _ in self.kernel_events]
        return sum(v) / len(v) if v else 0.0

    def relayout_ms(self):
        """Average time of the step's relayout launch (consolidation, paged -> group layout)."""
        v = [a.elapsed_time(b) for a, b in self.relayout_events]
        return sum(v) / len(v) if v else 0.0

    def merge_ms(self):
        """Average time of the separate LSE-merge launch after it (0 with the in-kernel merge)."""
        v = [b.elapsed_time(c) for _, b, c in self.kernel_events]
        return sum(v) / len(v) if v else 0.0


def timed_steps(runner, steps, warmup, dist_on, window=None):
    """W untimed warm-up steps, then exactly `steps` steps between a barrier + synchronize on both
    sides, timed with CUDA events on the step stream.  window (list): receives the host-time
    bounds of the timed region (for the clock sampler)."""
    import torch
    for i in range(warmup):
        runner.step(i)
    torch.cuda.synchronize()
    if dist_on:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    runner.kernel_events.clear()
    runner.relayout_events.clear()
    runner.step_events.clear()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    s.record()
    runner.begin(s)
    for i in range(steps):
        runner.step(warmup + i, time_kernel=True)
    e.record()
    torch.cuda.synchronize()
    t1 = time.time()
    if window is not None:
        window[:] = [t0, t1]
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
            runner.step(base + i, t=sets[k], out=outs[k], wait_event=in_ready[k])
            done[k].record(comp)
            s_out.wait_event(done[k])
            with torch.cuda.stream(s_out):
                outs_h[k].copy_(outs[k], non_blocking=True)
            out_free[k].record(s_out)
        comp.wait_event(out_free[(n - 1) % 2])
        comp.wait_event(out_free[n % 2])

    run(2, 20_000)                                   # warm-up (streams, pinned transfers)
    torch.cuda.synchronize()
    # context: this host link's bandwidth for the same bytes alone (H2D of the inputs, D2H of out)
    c0, c1, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    c0.record(s_in)
    with torch.cuda.stream(s_in):
        for name in host:
            sets[1][name].copy_(host[name], non_blocking=True)
    c1.record(s_in)
    with torch.cuda.stream(s_in):
        outs_h[1].copy_(outs[1], non_blocking=True)
    c2.record(s_in)
    torch.cuda.synchronize()
    link = {"h2d_gbs": h2d / (c0.elapsed_time(c1) * 1e-3) / 1e9, "d2h_gbs": outs_h[1].numel() * outs_h[1].element_size()
            / (c1.elapsed_time(c2) * 1e-3) / 1e9}
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(comp)
    s_in.wait_event(s)
    runner.begin(s)
    run(steps, 10_000)
    e.record(comp)
    torch.cuda.synchronize()
    # the last step's output landed on the host: spot-check it against the device copy
    k = (steps - 1) % 2
    assert torch.equal(outs_h[k][:4].to(outs[k].device), outs[k][:4])
    return s.elapsed_time(e) / steps, h2d, d2h, link


def decode_group_sharded(dev, rank, world, args, peaks):
    """N > 1 only: ONE configs[2] decode batch (the same on every rank) group-sharded across the
    ranks (shard.RankPlan, SURVEY 8(e) optional group sharding): each rank consolidates and attends
    only its groups; the partials of split rows whose pieces sit on several ranks - and only those -
    are exchanged (shard.exchange_split_rows, C2), then each rank merges its rows.  Step = relayout
    (own groups) + decode attention (own items) + exchange + merge, timed with CUDA events, max
    over ranks (strong scaling of one batch)."""
    import torch
    import torch.distributed as dist
    from paper_2602_06072_b200 import packinfer as pk, shard
    bd = make_workload("cfg3", 0)
    r = bd.hq // bd.hkv
    t = W_tensors(bd, dev)
    pb = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, bd.hkv, r, bd.d, t["q"].dtype, dev,
                        flags=plan_flags())
    owner = shard.group_shard(shard.group_costs(pb.plan), world)
    rp = shard.RankPlan(pb, owner, rank)
    out = torch.empty((bd.total_q, bd.hq, bd.d), dtype=t["q"].dtype, device=dev)
    st = torch.cuda.current_stream()

    def once():
        rp.step(pb, t["q"], t["k_paged"], t["v_paged"], t["block_table"], out, None, st)

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
    (ms,) = max_over_ranks(dev, e0.elapsed_time(e1) / n)
    kv_bytes = 2 * int(pb.plan.c.copy_tokens) * bd.hkv * bd.d * 2
    return {"workload": bd.name + " (BASELINE.json configs[2]), one batch over all ranks",
            "ms_per_step": ms, "step_gbs": kv_bytes / (ms * 1e-3) / 1e9,
            "rank_cells": rp.cells, "rank_work_items": rp.n_work, "groups": int(pb.plan.c.n_groups),
            "cross_rows": rp.n_cross_rows, "cross_slots": rp.n_cross_slots,
            "exchange_bytes": rp.exchange_bytes, "all_slots_bytes": int(pb.plan.c.n_partial_slots) * bd.hq * (bd.d + 1) * 4,
            "scaling": "strong", "note": "relayout + decode attention of this rank's groups, all-reduce of the "
                                         "cross-rank split rows' partials only, merge of the rank's rows"}


def W_tensors(b, dev):
    from synth import workloads as W
    return W.make_tensors(b, device=dev, seed=b.seed)


def decode_loop(dev, h0, hc, seed_rank, args):
    """Decode loop (NEXT-1) on configs[2]: consolidate once with headroom
    delta = 32 (= max new tokens), then each step appends one token per request into its
    headroom, re-plans the execution domain on the host (packinfer_plan_step) and runs decode +
    merge.  Plus the online capacity tuner (NEXT-2) driving C on configs[3]."""
    fresh_memory()
    import torch
    from synth import workloads as W
    from paper_2602_06072_b200 import packinfer as pk
    bd = make_workload("cfg3", seed_rank)
    loop_steps, delta = 32, 32
    tl = W.make_tensors(bd, device=dev, seed=bd.seed, extra_tokens=loop_steps)
    rr = bd.hq // bd.hkv
    pbl = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, hc, rr, bd.d, torch.bfloat16, dev,
                         headroom=delta, flags=plan_flags())
    ql = tl["q"][:, h0 * rr:(h0 + hc) * rr]
    outl = torch.empty((bd.n, hc * rr, bd.d), dtype=torch.bfloat16, device=dev)
    kn = torch.randn((bd.n, bd.hkv, bd.d), device=dev).to(torch.bfloat16)
    vn = torch.randn_like(kn)

    def loop_once(graph=False):
        if graph:   # every step's device part as one CUDA graph replay (PackedBatch.graph_run)
            pbl.replan(upload=False)
            pbl.graph_run(ql, outl, None, tl["k_paged"], tl["v_paged"], tl["block_table"], hkv_begin=h0,
                          relayout=True)
        else:
            pbl.replan()
            pbl.run(ql, tl["k_paged"], tl["v_paged"], tl["block_table"], outl, hkv_begin=h0)   # consolidation
        for k in range(1, loop_steps):
            pbl.append(kn, vn, hkv_begin=h0)
            if graph:
                pbl.replan(appended=np.full(bd.n, k, np.int32), upload=False)
                pbl.graph_run(ql, outl, None, hkv_begin=h0)
            else:
                pbl.replan(appended=np.full(bd.n, k, np.int32))
                pbl.run(ql, tl["k_paged"], tl["v_paged"], tl["block_table"], outl, hkv_begin=h0, relayout=False)

    def timed_loop(graph):
        loop_once(graph)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        loop_once(graph)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / loop_steps
    lms = timed_loop(False)
    lms_graph = timed_loop(True)
    caps_before = getattr(pbl, "graph_captures", 0)
    lms_graph = min(lms_graph, timed_loop(True))   # every plan shape of the loop captured by now
    graph_captures_timed = getattr(pbl, "graph_captures", 0) - caps_before
    kv_tokens = sum(int(bd.kv_len.sum()) + k * bd.n for k in range(loop_steps)) / loop_steps
    lbytes = 2 * kv_tokens * hc * bd.d * 2 + 2 * bd.n * hc * rr * bd.d * 2
    out = {"workload": bd.name + " (BASELINE.json configs[2])", "steps": loop_steps, "headroom": delta,
           "ms_per_step_amortized": lms, "step_gbs_amortized": lbytes / (lms * 1e-3) / 1e9,
           "graph_ms_per_step_amortized": lms_graph, "graph_captures_in_last_loop": graph_captures_timed,
           "note": "consolidation (relayout) once per 32 steps; per step: append + plan_step + upload + "
                   "decode attention + merge"}
    del tl, pbl
    out["tuned"] = tuned_loop(dev, h0, hc, seed_rank)
    return out


def tuned_loop(dev, h0, hc, seed_rank, epochs: int = 10, cands=(2048, 4096, 8192, 16384)):
    """NEXT-2 online refinement ("each decoding step naturally yields one performance
    sample"): a decode loop over configs[3] (shared prefixes) whose capacity C is chosen by
    tuning.CapacityTuner at every regroup point.  An epoch = consolidation with the tuner's C
    (re-plan + relayout), then decode steps that append into the headroom until Eq. 4
    triggers a regroup or the headroom is exhausted.  Every step is timed with CUDA events on its
    stream (decode attention + merge + append); the samples (read back one epoch
    later without stalling the loop) feed tuner.observe(C, cost): cost = step time per decoded
    request, the same requests at every C."""
    import torch
    from synth import workloads as W
    from paper_2602_06072_b200 import packinfer as pk
    from paper_2602_06072_b200.tuning import CapacityTuner
    bd = make_workload("cfg4_decode", seed_rank)
    delta = 32
    t = W.make_tensors(bd, device=dev, seed=bd.seed, extra_tokens=delta)
    rr = bd.hq // bd.hkv
    q = t["q"][:, h0 * rr:(h0 + hc) * rr]
    out = torch.empty((bd.n, hc * rr, bd.d), dtype=torch.bfloat16, device=dev)
    kn = torch.randn((bd.n, bd.hkv, bd.d), device=dev).to(torch.bfloat16)
    vn = torch.randn_like(kn)
    st = torch.cuda.current_stream()
    tuner = CapacityTuner(list(cands), probe_every=4)
    pending, history = [], []
    batches = {}

    def drain(block):
        keep = []
        for (c, ev0, ev1, kv) in pending:
            if block or ev1.query():
                ev1.synchronize()
                tuner.observe(c, ev0.elapsed_time(ev1) * 1e3 / kv)    # us per decoded request
            else:
                keep.append((c, ev0, ev1, kv))
        pending[:] = keep

    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(st)
    total_steps = 0
    for ep in range(epochs):
        drain(block=False)
        C = tuner.choose()
        if C not in batches:
            batches[C] = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, hc, rr, bd.d,
                                        torch.bfloat16, dev, capacity=C, headroom=delta, flags=plan_flags())
        pb = batches[C]
        pb.replan(st)
        pk.packinfer_relayout_kv(pb.dp, t["k_paged"], t["v_paged"], t["block_table"], pb.k_buf, pb.v_buf, h0, hc,
                                 st)
        k, steps = 0, 0
        while True:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(st)
            if k > 0:
                pb.append(kn, vn, hkv_begin=h0, stream=st)
                pb.replan(st, appended=np.full(bd.n, k, np.int32))
            pb.run(q, t["k_paged"], t["v_paged"], t["block_table"], out, hkv_begin=h0, stream=st, relayout=False)
            ev1.record(st)
            pending.append((C, ev0, ev1, bd.n))   # the same requests at every C: cost = time per request
            steps += 1
            k += 1
            if k > delta - 1 or pk.packinfer_should_regroup(k, int(pb.plan.c.drift), C):
                break
        history.append({"epoch": ep, "capacity": C, "steps": steps, "groups": int(pb.plan.c.n_groups),
                        "drift": int(pb.plan.c.drift)})
        total_steps += steps
    t_end.record(st)
    drain(block=True)
    torch.cuda.synchronize()
    ms = t_start.elapsed_time(t_end) / max(1, total_steps)
    res = {"workload": bd.name + " (BASELINE.json configs[3])", "candidates": list(cands), "epochs": history,
           "ms_per_step": ms, "best_capacity": tuner.best(),
           "cost_us_per_request": {str(c): tuner.mean[c] for c in tuner.cands},
           "note": "C chosen by CapacityTuner at every regroup (Eq. 4 or headroom exhausted); samples = "
                   "per-step CUDA-event time per decoded request (append + plan_step + upload + decode attention + merge; the "
                   "consolidation at a regroup is not a sample), fed back asynchronously"}
    del t, batches
    return res


def mixed_section(dev, h0, hc, rank, args, peaks, dist_on):
    """BASELINE.json configs[4]: Llama-3-70B-shaped mixed batch (2 x 128k-token prefills split
    across groups + 30 short prefills + 224 decodes up to 32k), ONE attention call over prefill
    and decode work items with the LSE merge inside it (NEXT-3: packinfer_attention_merge, the
    decode half a programmatic dependent launch filling the prefill launch's tail); the split form
    (prefill launch, decode launch, merge launch) is timed beside it on the same plan."""
    fresh_memory()
    import torch
    from synth import workloads as W
    from paper_2602_06072_b200 import packinfer as pk
    bm = W.cfg5_mixed(3 + (0 if args.shard == "heads" else rank))
    r = bm.hq // bm.hkv
    tm = W.make_tensors(bm, device=dev, seed=bm.seed)
    pbm = pk.PackedBatch(bm.kv_len, bm.q_len, bm.prefix_id, bm.prefix_len, hc, r, bm.d, torch.bfloat16, dev,
                         flags=plan_flags())
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
            pk.packinfer_attention_merge(pbm.dp, qm, pbm.k_buf, pbm.v_buf, outm, lsem, pbm.partial_o,
                                         pbm.partial_lse, pbm.merge_counters, r, 0.0, st)
            m.record(st)
            e.record(st)
        else:
            pk.packinfer_attention_prefill(pbm.dp, qm, pbm.k_buf, pbm.v_buf, outm, lsem, pbm.partial_o,
                                           pbm.partial_lse, r, 0.0, st)
            m.record(st)
            pk.packinfer_attention_decode(pbm.dp, qm, pbm.k_buf, pbm.v_buf, outm, lsem, pbm.partial_o,
                                          pbm.partial_lse, r, 0.0, st)
            pk.packinfer_merge(pbm.dp, pbm.partial_o, pbm.partial_lse, outm, lsem, st)
            e.record(st)
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
           "note": "tflops_fused counts prefill FLOPs only over the fused (prefill + decode + merge) kernel time",
           "gpu_launches": 3 * steps}
    del tm, pbm
    return out


# ------------------------------------------------------------------------------- oracle timing
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def stratified_requests(b, seed: int, strata: int = 8):
    """Request order for the oracle sample: requests sorted by KV length are cut into `strata`
    equal-count strata and the order takes one (seeded-random) request from each stratum in turn,
    so any prefix of it covers short and long requests alike (the workload's length mix)."""
    rng = np.random.default_rng(seed)
    idx = np.argsort(b.kv_len, kind="stable")
    parts = [list(rng.permutation(part)) for part in np.array_split(idx, strata) if len(part)]
    order = []
    while any(parts):
        for part in parts:
            if part:
                order.append(int(part.pop()))
    return order


def oracle_sample(b, budget_s: float, seed: int):
    """Times the oracle (as it stands) on a bounded, stratified sample of the workload's requests on
    this host: requests are taken in stratified_requests order until the budget is spent.  The
    paged cache is upcast to fp64 once, outside the timed region (inputs resident, as for the GPU
    arm).  Returns (algorithmic FLOPs, KV bytes, seconds, description, cores)."""
    import torch
    from oracle import attention as OA
    from synth import workloads as W
    cores = len(os.sched_getaffinity(0))
    t = W.make_tensors(b, device="cpu", seed=seed)
    q64 = t["q"].to(torch.float64).numpy()
    k64 = t["k_paged"].to(torch.float64).numpy()
    v64 = t["v_paged"].to(torch.float64).numpy()
    bt = t["block_table"].numpy()
    done, flops, kv_bytes, secs = [], 0, 0, 0.0
    for i in stratified_requests(b, seed):
        if secs > budget_s:
            break
        t0 = time.perf_counter()
        OA.attention(q64, k64, v64, bt, b.kv_len, b.q_len, b.page_size, requests=[i])
        secs += time.perf_counter() - t0
        L, q = int(b.kv_len[i]), int(b.q_len[i])
        flops += 4 * b.d * b.hq * (q * (L - q) + q * (q + 1) // 2)
        kv_bytes += 2 * L * b.hkv * b.d * 2
        done.append(i)
    lens = b.kv_len[done]
    desc = (f"{len(done)}/{b.n} requests of {b.name}, stratified by KV length (8 strata, one request per "
            f"stratum in turn; lengths {int(lens.min())}..{int(lens.max())}, {int(lens.sum())} KV tokens = "
            f"{100.0 * lens.sum() / b.kv_len.sum():.1f}% of the batch), fp64 numpy, {secs:.1f}s; "
            f"CPU: {cpu_model()}")
    return flops, kv_bytes, secs, desc, cores


def oracle_planner_us(reps: int = 3):
    """Host microseconds of the oracle planner (oracle/plan.py, Alg. 1 Parts 1-2) on the BASELINE
    configs, median of `reps` (the reference arm for the planner row)."""
    from oracle import plan as OP
    out = {}
    for name in ("cfg2", "cfg3", "cfg4_decode", "cfg5"):
        b = make_workload(name, 0)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            OP.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, 8192)
            ts.append((time.perf_counter() - t0) * 1e6)
        out[name] = statistics.median(ts)
    return out


def planner_us(reps: int = 50):
    """Host microseconds of packinfer_plan (C++, through the binding) per BASELINE config: median and
    p90 over `reps` calls into a pre-sized pinned arena (the per-step host cost of the hot path)."""
    from paper_2602_06072_b200 import packinfer as pk
    out = {}
    for name in ("cfg2", "cfg3", "cfg4_decode", "cfg5"):
        b = make_workload(name, 0)
        cfg = pk.default_config(capacity=8192, gqa_ratio=b.hq // b.hkv)
        hp = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, cfg, pinned=True)
        arena = hp.arena
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            hp = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, cfg, arena=arena)
            ts.append((time.perf_counter() - t0) * 1e6)
        c = hp.c
        out[name] = {"median_us": statistics.median(ts), "p90_us": float(np.percentile(ts, 90)),
                     "pieces": int(c.n_pieces), "groups": int(c.n_groups), "row_segments": int(c.n_segs),
                     "rows_expanded_on_device": int(c.n_rows), "host_arena_bytes": int(c.arena_bytes)}
    return out


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
            "ms_per_step": 1000 * sum(secs) / len(secs), "higher_is_better": True,
            "scaling": "strong" if args.shard == "heads" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(b, args.shard, args.gpus),
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- main
def self_launch(args):
    """--gpus N > 1 outside torchrun: re-run this script under torchrun with N processes (one per
    GPU) on a 127.0.0.1 rendezvous and exit with its status.  Fails loudly when the box has fewer
    than N GPUs (unless PI_BENCH_ONE_GPU=1 puts every rank on cuda:0, a test hook)."""
    import socket
    import torch
    if os.environ.get("PI_BENCH_ONE_GPU") != "1" and os.environ.get("PI_BENCH_DRYRUN") != "1" and \
            torch.cuda.device_count() < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but only {torch.cuda.device_count()} CUDA devices"}),
              flush=True)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def max_over_ranks(dev, *vals):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in vals], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def fresh_memory():
    """Between sections: release the previous sections' cached blocks so every section's buffers
    are allocated the same way however much ran before it (the short configs[3] decode launch
    otherwise varied with what earlier sections left in the caching allocator)."""
    import gc
    import torch
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def section_decode(name, dev, h0, hc, rank, args, peaks, dist_on, sampler, seed_rank):
    """A decode step (plan + upload + relayout + decode attention + merge) of one BASELINE batch on
    this rank's KV heads; GB/s = Eq. 5 KV bytes + Q/O bytes over the decode kernel time."""
    fresh_memory()
    bd = make_workload(name, seed_rank)
    rd = Runner(bd, dev, h0, hc, seed=bd.seed)
    _, kvb, qob = algorithmic(bd, rd.pbs[0].plan.c, hc)
    steps = max(10, args.steps)
    win = []
    dms = timed_steps(rd, steps, args.warmup, dist_on, win) / steps
    dec_ms, mrg_ms, rl_ms = rd.kernel_ms(), rd.merge_ms(), rd.relayout_ms()
    if dist_on:
        dms, dec_ms, mrg_ms, rl_ms = max_over_ranks(dev, dms, dec_ms, mrg_ms, rl_ms)
    ach = (kvb + qob) / (dec_ms * 1e-3) / 1e9
    # KV resident in the group layout (the producer writes new tokens there, packinfer_append_kv):
    # the step is host plan + upload + ONE attention launch with the merge inside - no relayout
    rd.relayout = False
    rms = timed_steps(rd, steps, args.warmup, dist_on) / steps
    rk = rd.kernel_ms()
    gms = graph_resident(rd, steps, args.warmup)
    if dist_on:
        rms, rk, gms = max_over_ranks(dev, rms, rk, gms)
    c = rd.pbs[0].plan.c
    paged = paged_decode(bd, rd, dev, h0, hc, steps, args.warmup, dist_on)
    c0 = rd.pbs[0].plan.c
    # relayout bytes = 2 (K, V) x copied tokens x Hkv d 2 B x 2 (read + write); merge
    # bytes = partials (o and lse, fp32) + the merged rows' bf16 outputs
    rl_bytes = 2 * int(c0.copy_tokens) * hc * bd.d * 2 * 2
    mg_bytes = int(c0.n_partial_slots) * hc * (bd.hq // bd.hkv) * (bd.d + 1) * 4 + \
        int(c0.n_merges) * hc * (bd.hq // bd.hkv) * bd.d * 2
    out = {"ms_per_step": dms, "kernel_ms": dec_ms, "merge_ms": mrg_ms, "kv_bytes": kvb, "qo_bytes": qob,
           "relayout": {"ms": rl_ms, "bytes": rl_bytes, "gbs": rl_bytes / (rl_ms * 1e-3) / 1e9 if rl_ms else None},
           "merge": {"ms": mrg_ms, "bytes": mg_bytes, "gbs": mg_bytes / (mrg_ms * 1e-3) / 1e9 if mrg_ms else None,
                     "note": "event-timed launch incl. its launch gap; partials are mostly evicted from L2 by the KV stream"},
           "achieved_gbs": ach,
           "peak_gbs": peaks["hbm_gbs"], "frac": ach / peaks["hbm_gbs"], "bound": "hbm",
           "step_gbs": (kvb + qob) / (dms * 1e-3) / 1e9, "work_items": int(c.n_decode_work),
           "partial_slots": int(c.n_partial_slots), "groups": int(c.n_groups),
           "step_latency": rd.step_latency(), "gpu_launches": rd.launches_per_step * steps,
           "clocks": sampler.window(*win) if win else None,
           "resident": {"ms_per_step": rms, "kernel_ms": rk, "step_over_kernel": rms / rk,
                        "graph_ms_per_step": gms,
                        "step_gbs": (kvb + qob) / (rms * 1e-3) / 1e9,
                        "gpu_launches_per_step": rd.launches_per_step - 1,
                        "note": "KV resident in the group-contiguous layout: plan + upload (+ row expansion) "
                                "+ one attention launch + merge; no relayout (kernel_ms: the attention launch; "
                                "the previous step's attention may leave part of the KV in L2)"},
           "paged": paged}
    del rd
    return out


def graph_resident(rd, steps, warmup):
    """The resident decode step with its device part as ONE CUDA graph launch
    (PackedBatch.graph_run: plan upload + row expansion + attention + merge): per step the host
    planner writes the tables, one graph replay runs them.  Device time per step (CUDA events)."""
    import torch
    pb = rd.pbs[0]
    for _ in range(max(warmup, 2)):
        pb.replan(upload=False)
        pb.graph_run(rd.q, rd.out, rd.lse, hkv_begin=rd.hkv_begin)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        pb.replan(upload=False)
        pb.graph_run(rd.q, rd.out, rd.lse, hkv_begin=rd.hkv_begin)
    e1.record()
    torch.cuda.synchronize()
    pb.replan()                                    # back to eager uploads for later sections
    return e0.elapsed_time(e1) / steps


def paged_decode(bd, rd, dev, h0, hc, steps, warmup, dist_on):
    """NEXT-4 ablation ("packed I/O" off, Fig. breakdown): the same decode batch planned
    with PI_PLAN_PAGED and decoded straight from the paged cache (packinfer_attention_decode_paged:
    no consolidation, no prefix co-location; the same tcgen05 kernel).  Step = plan + upload +
    attention + merge; bytes = every request's logical KV (prefixes read once per request)."""
    import torch
    from paper_2602_06072_b200 import packinfer as pk
    r = bd.hq // bd.hkv
    pb = pk.PackedBatch(bd.kv_len, bd.q_len, bd.prefix_id, bd.prefix_len, hc, r, bd.d, torch.bfloat16, dev,
                        flags=pk.PI_PLAN_PAGED)
    pb.k_buf = pb.v_buf = None                       # no group buffers in this mode
    st = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)
    kern = []

    def once(timed):
        pb.replan(st)
        a, e = ev(), ev()
        a.record(st)
        pk.packinfer_attention_decode_paged(pb.dp, rd.q, rd.t["k_paged"], rd.t["v_paged"], rd.t["block_table"],
                                            rd.out, rd.lse, pb.partial_o, pb.partial_lse, r, h0, hc, 0.0, st)
        e.record(st)
        pk.packinfer_merge(pb.dp, pb.partial_o, pb.partial_lse, rd.out, rd.lse, st)
        if timed:
            kern.append((a, e))

    for _ in range(warmup):
        once(False)
    torch.cuda.synchronize()
    s0, s1 = ev(), ev()
    s0.record(st)
    for _ in range(steps):
        once(True)
    s1.record(st)
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / steps
    kms = sum(a.elapsed_time(e) for a, e in kern) / len(kern)
    if dist_on:
        ms, kms = max_over_ranks(dev, ms, kms)
    kv_tokens = int(bd.kv_len.sum())
    kvb = 2 * kv_tokens * hc * bd.d * 2
    qob = 2 * bd.n * hc * r * bd.d * 2
    del pb
    return {"ms_per_step": ms, "kernel_ms": kms, "kv_tokens": kv_tokens, "kv_bytes": kvb,
            "achieved_gbs": (kvb + qob) / (kms * 1e-3) / 1e9, "work_items": None,
            "note": "PI_PLAN_PAGED: decode straight from the paged cache, no relayout, no prefix co-location "
                    "(kernel_ms: the attention launch, as for the packed kernel; step = plan + upload + attention + merge)"}


def library_context(dev, peaks, packinfer_prefill_ms, packinfer_decode_ms, packinfer_decode4_ms=None, steps=20):
    """Context, not the product: library attention kernels on the same configs[1] prefill batch and
    configs[2] decode batch on this B200 ("a real GPU baseline").  FlashAttention-2
    varlen (flash_attn 2.8) and FlashInfer's ragged prefill read the batch's K/V as one contiguous
    varlen tensor (gathered from the paged cache outside the timing, like our consolidation);
    FlashInfer's paged decode reads the paged cache directly (page 128).  Same algorithmic work
    numerators as ours; kernel time with CUDA events around the library call."""
    import torch
    from synth import workloads as W
    res = {"note": "library kernels (not this repo's code) timed on the same batches; context only"}
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, e = ev(), ev()
        a.record()
        for _ in range(steps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return a.elapsed_time(e) / steps

    b = make_workload("cfg2", 0)
    t = W.make_tensors(b, device=dev, seed=b.seed)
    flops, _, _ = algorithmic(b, None, b.hkv)
    P = b.page_size
    # contiguous varlen K/V [total_kv, Hkv, d] in request order (from the paged cache)
    idx = []
    bt = t["block_table"].cpu().numpy()
    for i in range(b.n):
        L = int(b.kv_len[i])
        j = np.arange(L)
        idx.append(bt[i, j // P] * P + j % P)
    idx = torch.from_numpy(np.concatenate(idx).astype(np.int64)).to(dev)
    kc = t["k_paged"].reshape(-1, b.hkv, b.d)[idx].contiguous()
    vc = t["v_paged"].reshape(-1, b.hkv, b.d)[idx].contiguous()
    cu = torch.from_numpy(np.concatenate([[0], np.cumsum(b.kv_len)]).astype(np.int32)).to(dev)
    mx = int(b.kv_len.max())
    q = t["q"]
    ours = {"kernel_ms": packinfer_prefill_ms, "tflops": flops / (packinfer_prefill_ms * 1e-3) / 1e12}
    res["prefill"] = {"workload": b.name + " (BASELINE.json configs[1])", "packinfer": ours}
    try:
        from flash_attn import flash_attn_varlen_func
        o_fa = flash_attn_varlen_func(q, kc, vc, cu, cu, mx, mx, causal=True)
        ms = timeit(lambda: flash_attn_varlen_func(q, kc, vc, cu, cu, mx, mx, causal=True))
        res["prefill"]["flash_attn_2_varlen"] = {"kernel_ms": ms, "tflops": flops / (ms * 1e-3) / 1e12}
    except Exception as e:   # context only: report, never fail the bench
        res["prefill"]["flash_attn_2_varlen"] = {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}
        o_fa = None
    for backend in ("auto", "cutlass"):   # FlashInfer's default and its Blackwell (CUTLASS FMHA) backend
        key = f"flashinfer_ragged_{backend}"
        try:
            import flashinfer
            ws = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
            w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend=backend)
            w.plan(cu, cu, b.hq, b.hkv, b.d, causal=True, q_data_type=torch.bfloat16)
            o_fi = w.run(q, kc, vc)
            ms = timeit(lambda: w.run(q, kc, vc))
            res["prefill"][key] = {"kernel_ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
                                   "version": flashinfer.__version__}
            if o_fa is not None:
                res["prefill"][key]["max_abs_vs_flash_attn"] = float((o_fi.float() - o_fa.float()).abs().max())
        except Exception as e:
            res["prefill"][key] = {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}
    del kc, vc, t
    # decode: FlashInfer paged decode straight from the paged cache (no co-location, no relayout)
    for sec, name, ours_ms in (("decode", "cfg3", packinfer_decode_ms), ("decode_shared_prefix", "cfg4_decode",
                                                                         packinfer_decode4_ms)):
        res[sec] = library_decode(dev, name, ours_ms, timeit)
    return res


def library_decode(dev, name, ours_ms, timeit):
    """FlashInfer paged decode (CUDA-core and tensor-core kernels) on one BASELINE decode batch;
    bytes = the KV each request reads through its block table (shared prefixes once per request)."""
    import torch
    from synth import workloads as W
    bd = make_workload(name, 0)
    td = W.make_tensors(bd, device=dev, seed=bd.seed)
    P = bd.page_size
    kvb = 2 * int(bd.kv_len.sum()) * bd.hkv * bd.d * 2 + 2 * bd.n * bd.hq * bd.d * 2
    res = {"workload": bd.name, "flashinfer_kv_bytes": kvb,
           "packinfer": {"kernel_ms": ours_ms, "note": "packed layout: Eq. 5 bytes (prefix once per group)"}}
    try:
        import flashinfer
        btd = td["block_table"].cpu().numpy()
        nblk = [-(-int(L) // P) for L in bd.kv_len]
        indptr = torch.from_numpy(np.concatenate([[0], np.cumsum(nblk)]).astype(np.int32)).to(dev)
        indices = torch.from_numpy(np.concatenate([btd[i, :nblk[i]] for i in range(bd.n)]).astype(np.int32)).to(dev)
        last = torch.from_numpy(np.array([int(L) - (nb - 1) * P for L, nb in zip(bd.kv_len, nblk)], np.int32)).to(dev)
        qd = td["q"]
        for tc in (False, True):   # CUDA-core decode kernel / tensor-core (prefill-style) decode kernel
            key = "flashinfer_paged_decode" + ("_tensor_cores" if tc else "")
            try:
                ws = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
                w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD", use_tensor_cores=tc)
                w.plan(indptr, indices, last, bd.hq, bd.hkv, bd.d, P, q_data_type=torch.bfloat16)
                w.run(qd, (td["k_paged"], td["v_paged"]))
                ms = timeit(lambda: w.run(qd, (td["k_paged"], td["v_paged"])))
                res[key] = {"kernel_ms": ms, "gbs": kvb / (ms * 1e-3) / 1e9}
            except Exception as e:
                res[key] = {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}
    except Exception as e:
        res["flashinfer_paged_decode"] = {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}
    del td
    return res


def section_prefill(name, dev, h0, hc, args, peaks, dist_on, sampler, seed_rank):
    """A prefill step of one BASELINE batch on this rank's KV heads (TFLOP/s over the prefill
    kernel time and over the step)."""
    fresh_memory()
    bp = make_workload(name, seed_rank)
    rp = Runner(bp, dev, h0, hc, seed=bp.seed)
    flops, _, _ = algorithmic(bp, rp.pbs[0].plan.c, hc)
    steps = max(10, args.steps)
    win = []
    pms = timed_steps(rp, steps, args.warmup, dist_on, win) / steps
    pre_ms = rp.kernel_ms()
    if dist_on:
        pms, pre_ms = max_over_ranks(dev, pms, pre_ms)
    ach = flops / (pre_ms * 1e-3) / 1e12
    c = rp.pbs[0].plan.c
    out = {"ms_per_step": pms, "kernel_ms": pre_ms, "tflop": flops / 1e12, "achieved_tflops": ach,
           "peak_tflops": peaks["bf16_tflops"], "frac": ach / peaks["bf16_tflops"], "bound": "tensor",
           "step_tflops": flops / (pms * 1e-3) / 1e12, "work_items": int(c.n_prefill_work),
           "groups": int(c.n_groups), "tile_efficiency": c.valid_cells / max(1, c.tile_cells),
           "step_latency": rp.step_latency(), "gpu_launches": rp.launches_per_step * steps,
           "clocks": sampler.window(*win) if win else None}
    del rp
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="packinfer", choices=["packinfer", "reference"])
    ap.add_argument("--shard", default="heads", choices=["heads", "group"])
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-prefix", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-loop", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-mixed", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-context", action="store_true", help="skip the library-kernel context section")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args, "cfg2")
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        self_launch(args)

    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch N ranks for --gpus N)")
    if os.environ.get("PI_BENCH_DRYRUN") == "1":
        # test hook (CPU): the launch path only - ranks rendezvous over gloo, agree on the world
        # size and the KV-head shards, and rank 0 prints them
        import torch.distributed as dist
        dist.init_process_group("gloo")
        from paper_2602_06072_b200 import shard
        t = torch.tensor([1.0])
        dist.all_reduce(t)
        shards = [shard.kv_head_shard(8, q, world) for q in range(world)]
        if rank == 0:
            print(json.dumps({"dryrun": True, "world": world, "ranks_seen": int(t.item()), "kv_head_shards": shards}),
                  flush=True)
        dist.destroy_process_group()
        return
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
    sampler = ClockSampler(local)
    if os.environ.get("PI_BENCH_NO_CLOCKS") != "1":   # diagnostics only: the contract needs the clocks
        sampler.start()

    heads = args.shard == "heads"
    seed_rank = 0 if heads else rank
    b = make_workload("cfg2", seed_rank)
    if heads and world > 1:
        from paper_2602_06072_b200 import shard
        h0, hc = shard.kv_head_shard(b.hkv, rank, world)
    else:
        h0, hc = 0, b.hkv
    runner = Runner(b, dev, h0, hc, seed=b.seed, pipeline=PIPELINE)
    flops, _, _ = algorithmic(b, runner.pbs[0].plan.c, hc)

    win = []
    total_ms = timed_steps(runner, args.steps, args.warmup, dist_on, win)
    clocks = sampler.window(*win)
    ms_step = total_ms / args.steps
    pre_ms = runner.kernel_ms()
    units_total = flops
    if dist_on:
        import torch.distributed as dist
        ms_step, pre_ms = max_over_ranks(dev, ms_step, pre_ms)     # step time = slowest rank
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
              "higher_is_better": True, "scaling": "strong" if heads else "weak",
              "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
              "config": arm_config(b, args.shard, world),
              "plan": {"groups": int(pc.n_groups), "work_items": int(pc.n_prefill_work),
                       "row_segments": int(pc.n_segs), "rows": int(pc.n_rows),
                       "step": "plan+upload(+row expansion)+relayout+prefill(+decode+merge)",
                       "algorithmic_tflop_per_rank": flops / 1e12},
              "roofline": roofline, "clocks": clocks,
              "step_latency": dict(runner.step_latency(), note="pipelined steps: from the step's first op "
                                   "(plan upload on the aux stream) to its last, incl. waiting for the previous "
                                   "step's attention"),
              "gpu_launches": runner.launches_per_step * args.steps}
    del runner
    # the same step strictly sequential on one stream: its isolated latency
    rs = Runner(b, dev, h0, hc, seed=b.seed)
    timed_steps(rs, 10, 2, dist_on)
    result["step_latency_sequential"] = rs.step_latency()
    del rs

    if dist_on and heads:
        # Strong scaling T(1) / (N T(N)) on the same batch, measured in this run: every rank also
        # times the UNSHARDED step (all KV heads) on its own GPU; T(1) = the max over ranks.
        r1 = Runner(b, dev, 0, b.hkv, seed=b.seed, pipeline=True)
        t1 = timed_steps(r1, args.steps, args.warmup, dist_on) / args.steps
        (t1,) = max_over_ranks(dev, t1)
        del r1
        result["strong_scaling"] = {"t1_ms": t1, "tn_ms": ms_step, "n": world,
                                    "efficiency": t1 / (world * ms_step)}
        # Full O on every rank (only for callers that need it; not part of the timed step): one
        # NCCL all-gather of the head-sharded outputs over NVLink.
        from paper_2602_06072_b200 import shard
        import torch.distributed as dist
        rg = Runner(b, dev, h0, hc, seed=b.seed)
        rg.step(0)
        shard.gather_heads(rg.out, world, b.hkv, rg.r)
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        g0.record()
        for _ in range(reps):
            full = shard.gather_heads(rg.out, world, b.hkv, rg.r)
        g1.record()
        torch.cuda.synchronize()
        (gms,) = max_over_ranks(dev, g0.elapsed_time(g1) / reps)
        gbytes = full.numel() * full.element_size()
        result["gather"] = {"ms": gms, "bytes_out": gbytes, "step_ms_with_gather": ms_step + gms,
                            "efficiency_with_gather": t1 / (world * (ms_step + gms)),
                            "note": f"{dist.get_backend()} all-gather of head-major O slabs (NCCL: all_gather_into_tensor) + layout copy"}
        del full, rg

    if not args.no_decode:
        d = section_decode("cfg3", dev, h0, hc, rank, args, peaks, dist_on, sampler, seed_rank)
        d["workload"] = "cfg3-llama3-8b-decode (BASELINE.json configs[2])"
        dtraffic = None
        if os.path.exists(tf):
            dtraffic = json.load(open(tf)).get("decode_attention_dram_bytes")
        d["traffic"] = dtraffic
        result["decode"] = d

    if not args.no_prefix:
        sp = {"workload": "cfg4 shared prefix: 128 requests over 8 prompts x 2048 tokens (BASELINE.json configs[3])"}
        sp["decode"] = section_decode("cfg4_decode", dev, h0, hc, rank, args, peaks, dist_on, sampler, seed_rank)
        sp["decode"]["traffic"] = json.load(open(tf)).get("decode_cfg4_attention_dram_bytes") if os.path.exists(tf) else None
        sp["suffix_prefill"] = section_prefill("cfg4_prefill", dev, h0, hc, args, peaks, dist_on, sampler,
                                               seed_rank)
        result["shared_prefix"] = sp

    if dist_on and not args.no_decode:
        result["decode_group_sharded"] = decode_group_sharded(dev, rank, world, args, peaks)

    if not args.no_decode and not args.no_loop:
        result.setdefault("decode", {})["loop"] = decode_loop(dev, h0, hc, seed_rank, args)

    if not args.no_mixed:
        result["mixed"] = mixed_section(dev, h0, hc, rank, args, peaks, dist_on)

    result["plan"]["host_us"] = planner_us()

    if not args.no_context and rank == 0 and world == 1:
        result["library_context"] = library_context(
            dev, peaks, pre_ms, result.get("decode", {}).get("kernel_ms"),
            result.get("shared_prefix", {}).get("decode", {}).get("kernel_ms"))

    if not args.no_e2e:
        re = Runner(b, dev, h0, hc, seed=b.seed, pipeline=True)
        e_ms, h2d, d2h, link = e2e_steps(b, re, max(3, min(args.steps, 10)))
        del re
        if dist_on:
            (e_ms,) = max_over_ranks(dev, e_ms)
        result["e2e"] = {"value": units_total / (e_ms * 1e-3) / 1e12,
                         "unit": "TFLOP/s", "ms_per_step": e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                         "host_link": link,
                         "note": "pinned host buffers; H2D of step i+1 and D2H of step i-1 overlap step i "
                                 "(double-buffered device inputs/outputs, copy-in / copy-out streams)"}

    if rank == 0 and world == 1 and not args.no_cpu:
        f, kvb, dt, desc, cores = oracle_sample(b, args.cpu_budget, b.seed)
        result["cpu_baseline"] = {"value": f / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                                  "sample": desc, "planner_oracle_us": oracle_planner_us()}
    sampler.stop()
    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist_on:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
