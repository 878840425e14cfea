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


def rank_tables(host_plan, owner, rank: int):
    """Host tables of rank `rank` under decode group sharding of one batch (SURVEY 8(e) optional
    group sharding; C2 "partial exchange of split rows only").  Pure integer host logic:

    * work: the decode items of the rank's groups (LPT order kept);
    * copies / prefix: the rank's copy entries (+ cell prefix) and, after every owned group whose
      successor is not owned, one GUARD entry that zero-fills up to 128 cells past the group end
      (clamped at the next owned group and the buffer end): a 128-key tile that runs past a span's
      end reads those cells, and masked keys meet P = 0, which must never multiply stale NaN;
    * slots: the partial slots of split rows renumbered so that the CROSS rows - merge rows whose
      slots are written by >= 2 ranks - come first, contiguous ([0, n_cross_slots)); only that
      range is exchanged (exchange_split_rows), local split rows stay local;
    * rows: the batch row table with every decode row's slot remapped;
    * merges: the cross rows (every rank merges them after the exchange) + the rank's local split
      rows; owned_tokens: the q tokens whose out/lse this rank holds after the merge."""
    import numpy as np
    from . import packinfer as pk
    c = host_plan.c
    owner = np.asarray(owner, dtype=np.int64)
    work_all = np.array(host_plan.decode_work, copy=True)
    rows = np.array(host_plan.rows, copy=True)
    merges = np.array(host_plan.merges, copy=True)
    n_slots = int(c.n_partial_slots)
    # owner rank of every slot and of every direct row: the group of the decode item writing it
    slot_rank = np.full(n_slots, -1, np.int64)
    tok_rank = {}
    for w in work_all:
        rr = rows[w["row_begin"]:w["row_begin"] + w["row_count"]]
        slot = (rr["out"] >> 4) - 1
        g_rank = owner[w["group"]]
        slot_rank[slot[slot >= 0]] = g_rank
        for tk in rr["q_token"][slot < 0].tolist():
            tok_rank[tk] = g_rank
    assert (slot_rank >= 0).all(), "every partial slot is written by some decode item"
    cross, local = [], []
    for m in merges:
        ranks = set(slot_rank[m["slot_begin"]:m["slot_begin"] + m["slot_count"]].tolist())
        (cross if len(ranks) > 1 else local).append((m, ranks))
    remap = np.full(n_slots, -1, np.int64)
    nxt = 0
    new_merges = []
    for m, _ in cross:
        remap[m["slot_begin"]:m["slot_begin"] + m["slot_count"]] = np.arange(nxt, nxt + m["slot_count"])
        new_merges.append((m["q_token"], nxt, m["slot_count"], 0))
        nxt += m["slot_count"]
    n_cross_slots = nxt
    for m, ranks in local:
        remap[m["slot_begin"]:m["slot_begin"] + m["slot_count"]] = np.arange(nxt, nxt + m["slot_count"])
        if ranks == {rank}:
            new_merges.append((m["q_token"], nxt, m["slot_count"], 0))
        nxt += m["slot_count"]
    is_dec = np.zeros(len(rows), bool)
    for w in work_all:
        is_dec[w["row_begin"]:w["row_begin"] + w["row_count"]] = True
    slot = (rows["out"] >> 4) - 1
    sel = is_dec & (slot >= 0)
    rows["out"][sel] = ((remap[slot[sel]] + 1) << 4) | (rows["out"][sel] & 15)
    merges_r = np.array(new_merges, dtype=pk.MERGE_DT) if new_merges else np.zeros(0, pk.MERGE_DT)
    # copies of owned groups + guard zero-fill entries
    copies = np.array(host_plan.copies, copy=True)
    prefix = np.asarray(host_plan.copy_prefix, dtype=np.int64)
    ext = prefix[1:] - prefix[:-1]
    cg = copy_groups(host_plan)
    bases = np.asarray(host_plan.groups["base"], dtype=np.int64)
    caps = np.asarray(host_plan.groups["cap"], dtype=np.int64)
    G, bt = len(bases), int(c.buffer_tokens)
    out_c, out_ext = [], []
    owned = [g for g in range(G) if owner[g] == rank]
    for g in owned:
        sel_c = np.nonzero(cg == g)[0]
        out_c.append(copies[sel_c])
        out_ext.append(ext[sel_c])
        end = int(bases[g] + caps[g])
        if g + 1 < G and owner[g + 1] != rank and end < bt:
            later = [h for h in owned if h > g]
            stop = min(end + 128, bt, int(bases[later[0]]) if later else bt)
            if stop > end:
                gc = np.zeros(1, pk.COPY_DT)
                gc["dst"] = end                      # len 0: every cell is zero-filled
                out_c.append(gc)
                out_ext.append(np.array([stop - end], np.int64))
    my_copies = np.concatenate(out_c) if out_c else np.zeros(0, pk.COPY_DT)
    my_ext = np.concatenate(out_ext) if out_ext else np.zeros(0, np.int64)
    keep_w = owner[work_all["group"]] == rank
    owned_tokens = sorted([tk for tk, rk in tok_rank.items() if rk == rank] +
                          [int(m["q_token"]) for m, rk in cross] +
                          [int(m["q_token"]) for m, rk in local if rk == {rank}])
    return {"work": work_all[keep_w], "copies": my_copies,
            "prefix": np.concatenate([[0], np.cumsum(my_ext)]).astype(np.int64),
            "copy_tokens": int(my_copies["len"].sum()) if len(my_copies) else 0,
            "rows": rows, "merges": merges_r, "n_cross_slots": int(n_cross_slots),
            "n_cross_rows": len(cross), "owned_tokens": [int(x) for x in owned_tokens]}


class RankPlan:
    """Decode group sharding of one batch (SURVEY 8(e) "optional: group sharding"): `rank` owns
    the groups `owner[g] == rank` (group_shard, LPT on group cost), consolidates only their copy
    entries (+ guard cells, rank_tables) and attends only their decode work items; buffers stay in
    batch coordinates.  Per step (`step` below): relayout -> neutral cross slots -> decode attention
    -> exchange of the cross-rank split rows' partials only (exchange_split_rows) -> merge of the
    rank's rows.  Prefill items are not sharded this way: a split request's piece a reads the KV of
    pieces 0..a-1, which other ranks would own (KV-head sharding covers prefill)."""

    def __init__(self, batch, owner, rank: int):
        import numpy as np
        import torch
        from . import packinfer as pk
        hp = batch.plan
        c = hp.c
        if int(c.n_prefill_work) > 0:
            raise ValueError("group sharding of one batch covers decode-only batches")
        tb = rank_tables(hp, owner, rank)
        dev = batch.device
        to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(dev) if len(a) \
            else torch.zeros(64, dtype=torch.uint8, device=dev)
        self.work, self.copies, self.prefix = to_dev(tb["work"]), to_dev(tb["copies"]), to_dev(tb["prefix"])
        self.rows, self.merges = to_dev(tb["rows"]), to_dev(tb["merges"])
        dp = pk.pi_device_plan.from_buffer_copy(batch.dp)
        dp.decode_work = self.work.data_ptr()
        dp.n_decode_work = len(tb["work"])
        dp.copies = self.copies.data_ptr()
        dp.copy_prefix = self.prefix.data_ptr()
        dp.n_copies = len(tb["copies"])
        dp.copy_tokens = tb["copy_tokens"]
        dp.rows = self.rows.data_ptr()
        dp.merges = self.merges.data_ptr()
        dp.n_merges = len(tb["merges"])
        dp.slot_merge = None                         # slots are renumbered: merge after the exchange
        dp.buffer_tokens = int(c.buffer_tokens)      # batch coordinates (dst is absolute)
        self.dp = dp
        self.n_cross_slots = tb["n_cross_slots"]
        self.n_cross_rows = tb["n_cross_rows"]
        self.owned_tokens = tb["owned_tokens"]
        self.cells = int(tb["prefix"][-1])           # buffer cells this rank writes (incl. guards)
        self.n_work = len(tb["work"])
        self.ktiles = int(tb["work"]["n_ktiles"].sum()) if len(tb["work"]) else 0
        hq, d = batch.hkv * batch.r, batch.d
        self.exchange_bytes = int(self.n_cross_slots * hq * (d + 1) * 4)

    def relayout_cells(self) -> int:
        return self.cells

    def step(self, batch, q, k_paged, v_paged, block_table, out, lse=None, stream=None, group=None,
             exchange=True):
        """One decode step of this rank (see the class docstring); `exchange=False` leaves the
        cross slots to the caller (single-process simulation of several ranks)."""
        from . import packinfer as pk
        pk.packinfer_relayout_kv(self.dp, k_paged, v_paged, block_table, batch.k_buf, batch.v_buf, 0, batch.hkv,
                                 stream)
        neutral_cross_slots(batch.partial_o, batch.partial_lse, self.n_cross_slots)
        pk.packinfer_attention_decode(self.dp, q, batch.k_buf, batch.v_buf, out, lse, batch.partial_o,
                                      batch.partial_lse, batch.r, 0.0, stream)
        if exchange:
            exchange_split_rows(batch.partial_o, batch.partial_lse, self.n_cross_slots, group)
        pk.packinfer_merge(self.dp, batch.partial_o, batch.partial_lse, out, lse, stream)


def neutral_cross_slots(partial_o, partial_lse, n_cross_slots: int):
    """Neutral elements of the exchange in the cross-slot range: o = 0, lse = -inf (an empty
    partial, DESIGN R10); the rank's attention then overwrites the slots it owns."""
    if n_cross_slots:
        partial_o[:n_cross_slots].zero_()
        partial_lse[:n_cross_slots].fill_(float("-inf"))


def exchange_split_rows(partial_o, partial_lse, n_cross_slots: int, group=None):
    """C2: the partials of split rows whose pieces sit on several ranks, and only those, travel:
    every cross slot is written by exactly one rank and holds the neutral element elsewhere
    (neutral_cross_slots), so one SUM all-reduce of o and one MAX all-reduce of lse over the
    contiguous cross range [0, n_cross_slots) give every rank all of them exactly (x + 0 = x,
    max(x, -inf) = x).  Bytes per rank buffer: n_cross_slots x Hq x (d + 1) x 4."""
    import torch.distributed as dist
    if n_cross_slots == 0:
        return
    dist.all_reduce(partial_o[:n_cross_slots], op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(partial_lse[:n_cross_slots], op=dist.ReduceOp.MAX, group=group)
