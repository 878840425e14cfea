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
        # group sharding of one batch: shard.combine assembles slots / rows owned by one rank each
        g2 = torch.Generator().manual_seed(11)
        po_full = torch.randn((6, 4, 8), generator=g2)
        pl_full = torch.randn((6, 4), generator=g2)
        out_full = torch.randn((5, 4, 8), generator=g2)
        po, pl, o, l = torch.empty(6, 4, 8), torch.empty(6, 4), torch.empty(5, 4, 8), torch.empty(4, 5)
        shard.init_partials(po, pl, o, l)
        for sl in range(6):
            if sl % world == rank:
                po[sl], pl[sl] = po_full[sl], pl_full[sl]
        for row in range(5):
            if row % world == rank:
                o[row] = out_full[row]
                l[:, row] = float(row)
        shard.combine(po, pl, o, l)
        res["combine_equal"] = bool(torch.equal(po, po_full) and torch.equal(pl, pl_full)
                                    and torch.equal(o, out_full)
                                    and torch.equal(l, torch.arange(5.0).expand(4, 5)))
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
        assert res["combine_equal"]
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


def test_rank_plan_partitions_decode_batch():
    """Group sharding of one decode batch (shard.RankPlan host logic): every decode work item and
    every copy entry belongs to exactly one rank, the ranks' buffer cells add up to the batch's, and
    each rank's copy subsequence keeps the batch cell prefix's per-entry extents."""
    import numpy as np
    from synth import workloads as W
    from paper_2602_06072_b200 import packinfer as pk, shard
    b = W.random_batch(31, n=24, max_len=1500, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=1.0)
    cfg = pk.default_config(capacity=256, decode_chunk=256, gqa_ratio=4)
    hp = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, cfg)
    cg = shard.copy_groups(hp)
    bases = np.asarray(hp.groups["base"])
    caps = np.asarray(hp.groups["cap"])
    dst = np.asarray(hp.copies["dst"])
    assert ((dst >= bases[cg]) & (dst < bases[cg] + caps[cg])).all()
    prefix = np.asarray(hp.copy_prefix)
    assert prefix[-1] == hp.c.buffer_tokens
    for world in (1, 2, 3, 5):
        owner = np.asarray(shard.group_shard(shard.group_costs(hp), world))
        w_rank = owner[np.asarray(hp.decode_work["group"])]
        c_rank = owner[cg]
        assert np.bincount(w_rank, minlength=world).sum() == hp.c.n_decode_work
        cells = [int((prefix[1:] - prefix[:-1])[c_rank == r].sum()) for r in range(world)]
        assert sum(cells) == hp.c.buffer_tokens
        # LPT balance: no rank above the mean by more than the largest group
        load = np.bincount(owner, weights=shard.group_costs(hp), minlength=world)
        assert load.max() - load.mean() <= max(shard.group_costs(hp))
