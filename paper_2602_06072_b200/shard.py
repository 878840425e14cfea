"""Multi-GPU partitioning of the hot path — host logic only.

The path shards without communication:
  * KV-head sharding: rank r of N owns KV heads [r*Hkv/N, (r+1)*Hkv/N) and their GQA query heads;
    every rank computes the same plan (the planner is deterministic) and runs relayout/attention
    with hkv_begin/hkv_count.  Outputs are bitwise equal to the single-GPU run.
  * Group sharding: groups (Alg. 1 S_g) are assigned to ranks by LPT on their cost, so each rank
    consolidates and attends only its groups' KV (weak scaling over independent groups/batches).
No collective is on the data path; `plan_digest` lets ranks assert they planned identically.
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
