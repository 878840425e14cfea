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
        # group sharding of one batch: exchange_split_rows assembles the cross slots, each written
        # by one rank (the rest of the partial buffer is never exchanged)
        g2 = torch.Generator().manual_seed(11)
        po_full = torch.randn((6, 4, 8), generator=g2)
        pl_full = torch.randn((6, 4), generator=g2)
        n_cross = 4
        po, pl = torch.full((6, 4, 8), float("nan")), torch.full((6, 4), float("nan"))
        shard.neutral_cross_slots(po, pl, n_cross)
        for sl in range(6):
            if sl % world == rank:
                po[sl], pl[sl] = po_full[sl], pl_full[sl]
        shard.exchange_split_rows(po, pl, n_cross)
        res["exchange_equal"] = bool(torch.equal(po[:n_cross], po_full[:n_cross])
                                     and torch.equal(pl[:n_cross], pl_full[:n_cross]))
        # slots past the cross range stay local (not exchanged): NaN where this rank did not write
        res["local_untouched"] = all(bool(torch.isnan(po[sl]).all()) == (sl % world != rank)
                                     for sl in range(n_cross, 6))
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
        assert res["exchange_equal"]
        assert res["local_untouched"]
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


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_rank_tables_split_row_exchange(world):
    """shard.rank_tables (decode group sharding of one batch, C2): every slot is written by exactly
    one rank; the cross rows' slots form the contiguous front range and are the only exchanged ones
    (bytes = cross slots x Hq x (d+1) x 4); each rank merges the cross rows and exactly its own local
    split rows; every decode token is held by its owner after the merge; guard zero-fill cells never
    overlap cells another entry of the same rank writes, and sit past an owned group's end."""
    from synth import workloads as W
    from paper_2602_06072_b200 import packinfer as pk, shard
    b = W.random_batch(31, n=24, max_len=1500, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=1.0)
    cfg = pk.default_config(capacity=256, decode_chunk=256, gqa_ratio=4)
    hp = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, cfg)
    owner = np.asarray(shard.group_shard(shard.group_costs(hp), world))
    tabs = [shard.rank_tables(hp, owner, r) for r in range(world)]
    n_slots = int(hp.c.n_partial_slots)
    writers = np.zeros(n_slots, np.int64)
    for r, tb in enumerate(tabs):
        for w in tb["work"]:
            rr = tb["rows"][w["row_begin"]:w["row_begin"] + w["row_count"]]
            sl = (rr["out"] >> 4) - 1
            np.add.at(writers, np.unique(sl[sl >= 0]), 1)
    assert (writers == 1).all()
    ncs = tabs[0]["n_cross_slots"]
    assert all(tb["n_cross_slots"] == ncs for tb in tabs)
    if world == 1:
        assert ncs == 0
    cross_tokens = set()
    for tb in tabs:
        m = tb["merges"]
        cross = m[m["slot_begin"] < ncs]
        assert (cross["slot_begin"] + cross["slot_count"] <= ncs).all()
        cross_tokens |= set(cross["q_token"].tolist())
    assert all(set(tb["merges"]["q_token"][tb["merges"]["slot_begin"] < ncs].tolist()) == cross_tokens for tb in tabs)
    held = [set(tb["owned_tokens"]) for tb in tabs]
    assert set().union(*held) == set(range(b.total_q))
    for r in range(world):
        for r2 in range(r + 1, world):
            assert held[r] & held[r2] <= cross_tokens
    merged_local = sum(int((tb["merges"]["slot_begin"] >= ncs).sum()) for tb in tabs)
    assert merged_local + len(cross_tokens) == int(hp.c.n_merges)
    bases, caps = np.asarray(hp.groups["base"]), np.asarray(hp.groups["cap"])
    for r, tb in enumerate(tabs):
        cells = []
        pre = tb["prefix"]
        for k, cp in enumerate(tb["copies"]):
            cells.append((int(cp["dst"]), int(cp["dst"]) + int(pre[k + 1] - pre[k]), int(cp["len"]) == 0))
        cells.sort()
        assert all(a[1] <= b2[0] for a, b2 in zip(cells, cells[1:])), "overlapping cells on one rank"
        for lo, hi, guard in cells:
            if guard:
                g = int(np.searchsorted(bases, lo, side="right")) - 1
                assert owner[g] != r or lo == bases[g]  # inside a group another rank owns
                assert hi - lo <= 128


def test_rank_tables_report_plain_ints():
    """The per-rank figures bench.py prints (cross slots, exchange bytes, owned tokens) are plain
    Python ints (JSON-serialisable), not numpy scalars."""
    import json
    from synth import workloads as W
    from paper_2602_06072_b200 import packinfer as pk, shard
    b = W.random_batch(31, n=24, max_len=1500, hq=8, hkv=2, d=128, n_prefix=2, decode_frac=1.0)
    hp = pk.packinfer_plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len,
                           pk.default_config(capacity=256, decode_chunk=256, gqa_ratio=4))
    owner = shard.group_shard(shard.group_costs(hp), 2)
    tb = shard.rank_tables(hp, owner, 0)
    json.dumps({"n_cross_slots": tb["n_cross_slots"], "n_cross_rows": tb["n_cross_rows"],
                "owned": tb["owned_tokens"], "copy_tokens": tb["copy_tokens"]})
