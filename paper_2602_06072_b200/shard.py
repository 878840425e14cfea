"""Multi-GPU partitioning of the hot path — host logic only.

The path shards without communication:
  * KV-head sharding: rank r of N owns KV heads [r*Hkv/N, (r+1)*Hkv/N) and their GQA query heads;
    every rank computes the same plan (the planner is deterministic) and runs relayout/attention
    with hkv_begin/hkv_count.  Outputs are bitwise equal to the single-GPU run.
  * Group sharding: groups (Alg. 1 S_g) are assigned to ranks by LPT on their cost, so each rank
    consolidates and attends only its groups' KV: independent batches per rank (weak scaling), or
    ONE decode batch (`RankPlan`): split rows whose pieces sit on several ranks are completed by
    one SUM / MAX all-reduce of the partial slots and direct outputs (`combine`) + the merge.
Apart from that exchange no collective is on the data path; `plan_digest` lets ranks assert they
planned identically.
A caller that needs the full O on every rank gathers the head shards once per step
(`gather_heads`: one all-gather over NCCL / NVLink).
"""

from __future__ import annotations

import hashlib
from typing import List, Sequence, Tuple


def kv_head_shard(hkv: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous KV-head range (begin, count) of `rank`; balanced when world does not divide hkv.
    Ranks beyond hkv get an empty range."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(hkv, world)
    begin = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return begin, count


def group_shard(costs: Sequence[int], world: int) -> List[int]:
    """LPT assignment of groups to ranks: groups in descending cost (ties: lower index first) go to
    the least-loaded rank (ties: lower rank).  Deterministic on every rank."""
    if world < 1:
        raise ValueError("world must be >= 1")
    owner = [0] * len(costs)
    load = [0] * world
    for g in sorted(range(len(costs)), key=lambda g: (-int(costs[g]), g)):
        r = min(range(world), key=lambda r: (load[r], r))
        owner[g] = r
        load[r] += int(costs[g])
    return owner


def group_costs(host_plan) -> List[int]:
    """Cost of each group for sharding: its prefix-deduplicated load L(S_g) (Eq. 2/5 tokens)."""
    return [int(g["load"]) for g in host_plan.groups]


def plan_digest(host_plan) -> str:
    """SHA-256 of the plan's host arena (byte-identical plans <=> identical digests)."""
    c = host_plan.c
    arena = host_plan.arena
    raw = bytes(arena.numpy().tobytes() if hasattr(arena, "numpy") else bytes(arena))
    return hashlib.sha256(raw[: int(c.arena_bytes)]).hexdigest()


def gather_heads(out_local, world: int, hkv_total: int, gqa_ratio: int, group=None):
    """All-gather of KV-head-sharded outputs (SURVEY 8(e) "gather outputs where a caller needs
    them").  out_local: [T, count_r * gqa_ratio, d] of this rank (kv_head_shard order); returns
    the full [T, hkv_total * gqa_ratio, d] on every rank.  Shards travel as head-major slabs
    [heads, T, d] padded to the largest shard, so one all_gather_into_tensor (NCCL) moves them."""
    import torch
    import torch.distributed as dist
    counts = [kv_head_shard(hkv_total, q, world)[1] for q in range(world)]
    hmax = max(counts) * gqa_ratio
    T, hl, d = out_local.shape
    slab = out_local.new_zeros((hmax, T, d))
    if hl:
        slab[:hl] = out_local.transpose(0, 1)
    gathered = out_local.new_empty((world, hmax, T, d))
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(gathered, slab, group=group)
    else:
        dist.all_gather(list(gathered.unbind(0)), slab, group=group)
    parts = [gathered[q, :counts[q] * gqa_ratio] for q in range(world)]
    return torch.cat(parts, 0).transpose(0, 1).contiguous()


# ------------------------------------------------------------------ group sharding of ONE batch
def copy_groups(host_plan):
    """Group of every copy-plan entry (its destination lies in that group's buffer B_g)."""
    import numpy as np
    bases = np.asarray(host_plan.groups["base"], dtype=np.int64)
    return np.searchsorted(bases, np.asarray(host_plan.copies["dst"], dtype=np.int64), side="right") - 1


class RankPlan:
    """Decode group sharding of one batch (SURVEY 8(e) "optional: group sharding"): `rank` owns
    the groups `owner[g] == rank` (group_shard, LPT on group cost), consolidates only their copy
    entries and attends only their decode work items.  The result is a device plan with the same
    tables as the batch plan except the copy list (+ its cell prefix) and the decode work list,
    which are this rank's subsequences (LPT order kept); buffers stay in batch coordinates.

    Split rows whose pieces land on several ranks are completed by `combine` (one all-reduce of
    the partial slots and of the direct outputs) followed by packinfer_merge on the batch plan.
    Prefill items are not sharded this way: a split request's piece a reads the KV of pieces
    0..a-1, which other ranks would own (KV-head sharding covers prefill)."""

    def __init__(self, batch, owner, rank: int):
        import numpy as np
        import torch
        from . import packinfer as pk
        hp = batch.plan
        c = hp.c
        if int(c.n_prefill_work) > 0:
            raise ValueError("group sharding of one batch covers decode-only batches")
        owner = np.asarray(owner, dtype=np.int64)
        work = np.array(hp.decode_work, copy=True)
        keep_w = owner[work["group"]] == rank
        copies = np.array(hp.copies, copy=True)
        prefix = np.asarray(hp.copy_prefix, dtype=np.int64)
        keep_c = owner[copy_groups(hp)] == rank
        ext = (prefix[1:] - prefix[:-1])[keep_c]
        my_prefix = np.concatenate([[0], np.cumsum(ext)]).astype(np.int64)
        dev = batch.device
        to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(dev)
        self.work = to_dev(work[keep_w]) if keep_w.any() else torch.zeros(64, dtype=torch.uint8, device=dev)
        self.copies = to_dev(copies[keep_c]) if keep_c.any() else torch.zeros(64, dtype=torch.uint8, device=dev)
        self.prefix = to_dev(my_prefix)
        dp = pk.pi_device_plan.from_buffer_copy(batch.dp)
        dp.decode_work = self.work.data_ptr()
        dp.n_decode_work = int(keep_w.sum())
        dp.copies = self.copies.data_ptr()
        dp.copy_prefix = self.prefix.data_ptr()
        dp.n_copies = int(keep_c.sum())
        dp.copy_tokens = int(copies["len"][keep_c].sum())
        dp.buffer_tokens = int(c.buffer_tokens)      # batch coordinates (dst is absolute)
        self.dp = dp
        self.cells = int(my_prefix[-1])              # buffer cells this rank consolidates
        self.n_work = int(keep_w.sum())
        self.ktiles = int(work["n_ktiles"][keep_w].sum())

    def relayout_cells(self) -> int:
        return self.cells


def init_partials(partial_o, partial_lse, out, lse=None):
    """Neutral elements of `combine`: o = 0, lse = -inf (an empty partial, DESIGN R10)."""
    partial_o.zero_()
    partial_lse.fill_(float("-inf"))
    out.zero_()
    if lse is not None:
        lse.fill_(float("-inf"))


def combine(partial_o, partial_lse, out, lse=None, group=None):
    """Every partial slot and every directly written output row is produced by exactly one rank
    and holds the neutral element elsewhere (init_partials), so a SUM all-reduce of o / out and a
    MAX all-reduce of the lse's assemble them exactly on every rank (x + 0 = x, max(x, -inf) = x);
    packinfer_merge on the batch plan then finishes the split rows."""
    import torch.distributed as dist
    dist.all_reduce(partial_o, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(partial_lse, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    if lse is not None:
        dist.all_reduce(lse, op=dist.ReduceOp.MAX, group=group)
