"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host path:
ranks plan identically without communicating, KV-head shards partition the heads, group shards
(LPT) agree across ranks and balance the load, and the bench's max-over-ranks timing reduction."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_06072_b200 import shard
from synth import workloads as W

pk = pytest.importorskip("paper_2602_06072_b200.packinfer")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for name in ("cfg2", "cfg4_decode", "cfg5"):
            b = W.make_batch(name)
            hp = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len,
                                   pk.default_config(headroom=32, gqa_ratio=b.hq // b.hkv))
            dg = shard.plan_digest(hp)
            allg = [None] * world
            dist.all_gather_object(allg, dg)
            res[name + "_digest_equal"] = len(set(allg)) == 1
            owner = shard.group_shard(shard.group_costs(hp), world)
            allo = [None] * world
            dist.all_gather_object(allo, owner)
            res[name + "_owner_equal"] = all(o == owner for o in allo)
            costs = shard.group_costs(hp)
            loads = [sum(c for c, o in zip(costs, owner) if o == r) for r in range(world)]
            # LPT bound: max load <= mean + largest group
            res[name + "_balance"] = max(loads) <= sum(loads) / world + max(costs)
        # output all-gather of KV-head shards (hkv = 5 does not divide evenly: padded slabs)
        g = torch.Generator().manual_seed(3)
        full = torch.randn((37, 5 * 4, 16), generator=g)
        b0, c0 = shard.kv_head_shard(5, rank, world)
        got = shard.gather_heads(full[:, b0 * 4:(b0 + c0) * 4].contiguous(), world, 5, 4)
        res["gather_equal"] = bool(torch.equal(got, full))
        hb, hc = shard.kv_head_shard(8, rank, world)
        heads = [None] * world
        dist.all_gather_object(heads, list(range(hb, hb + hc)))
        res["heads"] = sorted(h for hs in heads for h in hs)
        # bench.py's max-over-ranks step time
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res["tmax"] = float(t)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        res = out[r]
        for name in ("cfg2", "cfg4_decode", "cfg5"):
            assert res[name + "_digest_equal"], name
            assert res[name + "_owner_equal"], name
            assert res[name + "_balance"], name
        assert res["heads"] == list(range(8))
        assert res["gather_equal"]
        assert res["tmax"] == 2.0


def test_kv_head_shard_partition():
    for hkv in (1, 4, 8, 7):
        for world in (1, 2, 4, 8):
            ranges = [shard.kv_head_shard(hkv, r, world) for r in range(world)]
            heads = [h for b, c in ranges for h in range(b, b + c)]
            assert heads == list(range(hkv))
            counts = [c for _, c in ranges]
            assert max(counts) - min(counts) <= 1


def test_group_shard_lpt_bound():
    rng = np.random.default_rng(0)
    for _ in range(50):
        costs = rng.integers(1, 9000, size=int(rng.integers(1, 200))).tolist()
        for world in (2, 4, 8):
            owner = shard.group_shard(costs, world)
            loads = [sum(c for c, o in zip(costs, owner) if o == r) for r in range(world)]
            # LPT guarantee: max load <= mean + max item
            assert max(loads) <= sum(costs) / world + max(costs)
