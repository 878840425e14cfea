"""Planner oracle — Alg. 1 of PackInfer (arXiv 2602.06072), integers only.  TEST INFRASTRUCTURE.

Follows the paper step by step, in its order and notation:

  Part 1 "Inter-group Workload Balancing"  (Alg. 1; prose P:261-262)
    line 1   L_total <- sum L_i ;  G <- ceil(L_total / C)
             with L_total deduplicated over shared prefixes ("deducting the redundant
             prefix lengths")                                         [reading R2]
    line 3   sort R in descending order of effective length [R3]
    line 4-9 assign to the least-loaded group if Phi holds, else open a new group
             with the prefix-aware contribution  L^_i = L_i - L^g_shared,i [R1, R4]
             and Phi = (sum L <= C) and (M(S_g) <= M_max)                    (Eq. 2) [R6]
    long requests are "partitioned across multiple groups": pieces of exactly C
    tokens except the last                                                    [R5]

  Part 2 "Packed I/O Layout Preparation"   (Alg. 1)
    TriePartition(S_g) in prefix-id form: a prefix entry exists iff >= 2 members of the
    group share the prefix id                                                 [R7]
    Copy(P_k -> B_g); Delta_prefix <- Delta; Delta += L_Pk
    for each suffix: Copy(Q_i -> B_g); O_g[i] <- (Delta_prefix, L_P, Delta, L_Q);
                     Delta += L_Q (+ headroom delta) [R8, R9]

  Reported quantities
    Eq. 1  eta_batch = sum L_i^2 / (G T^2)   as an exact Fraction
    Eq. 3  discrepancy = max_g L(S_g) - min_g L(S_g)
    Eq. 5  M(S_g) = sum_k (L_Pk + sum_i L_Qi,k)

The readings R1..R9 are listed in DESIGN.md §3 (they follow SURVEY.md §8(c) Q1..Q9).
Outputs (pieces' groups, offsets, groups, copies) are compared BIT-EXACTLY with the C++
planner in tests/test_plan_parity.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from typing import List, Optional, Sequence


class PlanError(ValueError):
    """Invalid planner input (the C ABI returns PI_EINVAL for the same conditions)."""


@dataclass
class Piece:
    request: int
    piece: int
    kv_begin: int
    kv_len: int
    prefix: int          # prefix id carried by the piece (-1 = none; dropped for split requests)
    group: int = -1


@dataclass
class Group:
    load: int = 0                                   # L(S_g), prefix-deduplicated tokens
    members: List[int] = field(default_factory=list)  # piece indices in assignment order
    held: set = field(default_factory=set)          # prefix ids already present in the group
    base: int = 0
    cap: int = 0


@dataclass
class Copy:
    src_kind: int   # 0 = request block table, 1 = prefix block table
    src_id: int
    src_begin: int  # first logical token of the source
    length: int
    dst: int        # global buffer token (base_g + Delta)


@dataclass
class Plan:
    pieces: List[Piece]
    offsets: List[tuple]          # indexed like pieces: (d_prefix, l_prefix, d_suffix, l_suffix)
    groups: List[Group]
    copies: List[Copy]
    G0: int
    buffer_tokens: int
    order: List[int]              # assignment order (piece indices)

    # -- reported quantities -------------------------------------------------------
    def discrepancy(self) -> int:
        """Eq. 3: max_g L(S_g) - min_g L(S_g); 0 for an empty plan."""
        if not self.groups:
            return 0
        loads = [g.load for g in self.groups]
        return max(loads) - min(loads)

    def io_volume(self) -> int:
        """Eq. 5 summed over groups: tokens fetched once per group."""
        return sum(g.load for g in self.groups)


def eta_batch(lengths: Sequence[int], G: int, T: int) -> Fraction:
    """Eq. 1: eta_batch = sum_i L_i^2 / (G * T^2), exact rational.

    Reading R-eta: the literal formula is reported even though it is not bounded
    by 1."""
    if G <= 0:
        raise PlanError("G must be positive")
    return Fraction(sum(int(L) * int(L) for L in lengths), G * T * T)


def eta_group(lengths: Sequence[int], T: int) -> Fraction:
    """Eq. 1 left side: eta(S_g) = sum_{i in S_g} L_i^2 / T^2."""
    return Fraction(sum(int(L) * int(L) for L in lengths), T * T)


def should_regroup(t: int, dL: int, C: int) -> bool:
    """Eq. 4: regroup when t * dL >= C / 2 (inclusive, exact rational compare)."""
    return 2 * t * dL >= C


def split_long(L: int, C: int) -> List[tuple]:
    """Reading R5: ceil(L/C) contiguous pieces of exactly C tokens except the
    last, in token order.  Returns [(begin, length), ...]; a request with L <= C is one piece."""
    if L <= C:
        return [(0, L)]
    out = []
    b = 0
    while b < L:
        out.append((b, min(C, L - b)))
        b += C
    return out


def validate(kv_len, q_len, prefix_id, prefix_len, C, mem_cap, headroom, num_groups):
    n = len(kv_len)
    if len(q_len) != n or len(prefix_id) != n:
        raise PlanError("length mismatch")
    if C < 1:
        raise PlanError("capacity must be >= 1")
    if headroom < 0 or num_groups < 0 or mem_cap < 0:
        raise PlanError("negative config value")
    if mem_cap > 0 and mem_cap < C + headroom:
        raise PlanError("mem_cap must be 0 or >= capacity + headroom")
    for i in range(n):
        L, q, p = int(kv_len[i]), int(q_len[i]), int(prefix_id[i])
        if L < 1:
            raise PlanError(f"kv_len[{i}] < 1")
        if q < 1 or q > L:
            raise PlanError(f"q_len[{i}] not in [1, kv_len]")
        if p < -1 or p >= len(prefix_len):
            raise PlanError(f"prefix_id[{i}] out of range")
        if p >= 0 and (int(prefix_len[p]) < 1 or int(prefix_len[p]) > L - q):
            # a shared prefix must be fully cached and hold no query rows
            raise PlanError(f"prefix_len[{p}] must be in [1, kv_len-q_len] for request {i}")


def plan(kv_len: Sequence[int], q_len: Sequence[int], prefix_id: Optional[Sequence[int]],
         prefix_len: Sequence[int], capacity: int, num_groups: int = 0, mem_cap: int = 0,
         headroom: int = 0) -> Plan:
    """Alg. 1 Parts 1 and 2 with readings R1-R9."""
    n = len(kv_len)
    if prefix_id is None:
        prefix_id = [-1] * n
    C = int(capacity)
    delta = int(headroom)
    validate(kv_len, q_len, prefix_id, prefix_len, C, mem_cap, delta, num_groups)

    # ---- pieces (R5: long requests partitioned across groups) ----------------------
    pieces: List[Piece] = []
    for i in range(n):
        L = int(kv_len[i])
        segs = split_long(L, C)
        pid = int(prefix_id[i]) if len(segs) == 1 else -1   # split requests drop the prefix
        for a, (b, ln) in enumerate(segs):
            pieces.append(Piece(i, a, b, ln, pid))
    if n == 0:
        return Plan([], [], [], [], 0, 0, [])

    # ---- Alg. 1 line 1: G <- ceil(L_total / C), L_total prefix-deduplicated (R2) --
    L_total = sum(p.kv_len for p in pieces)
    n_p = {}
    for p in pieces:
        if p.prefix >= 0:
            n_p[p.prefix] = n_p.get(p.prefix, 0) + 1
    for pid, cnt in n_p.items():
        L_total -= (cnt - 1) * int(prefix_len[pid])
    G0 = int(num_groups) if num_groups > 0 else max(1, -(-L_total // C))

    # ---- Alg. 1 line 2: initialise G empty groups ----------------------------------------
    groups = [Group() for _ in range(G0)]

    # ---- Alg. 1 line 3: sort descending by effective length (R3: ties request, piece) ----
    order = sorted(range(len(pieces)),
                   key=lambda k: (-pieces[k].kv_len, pieces[k].request, pieces[k].piece))

    # ---- Alg. 1 lines 4-9: least-loaded feasible group, else open a new group ------------
    for k in order:
        pc = pieces[k]
        best = None
        for g, grp in enumerate(groups):
            # L^_i = L_i - L^g_shared,i
            shared = int(prefix_len[pc.prefix]) if (pc.prefix >= 0 and pc.prefix in grp.held) else 0
            c = pc.kv_len - shared
            # Phi (Eq. 2), boundary inclusive (R6)
            if grp.load + c > C:
                continue
            if mem_cap > 0 and grp.load + c + delta * (len(grp.members) + 1) > mem_cap:
                continue
            key = (grp.load + c, g)        # R1: argmin of the resulting load, lowest g on ties
            if best is None or key < best[0]:
                best = (key, g, c)
        if best is None:                   # Phi fails everywhere: S_{G+1} <- {i}
            groups.append(Group())
            g, c = len(groups) - 1, pc.kv_len
        else:
            _, g, c = best
        grp = groups[g]
        grp.load += c
        grp.members.append(k)
        if pc.prefix >= 0:
            grp.held.add(pc.prefix)
        pc.group = g

    # ---- Alg. 1 Part 2: TriePartition + consolidation + offset table ---------------------
    offsets: List[Optional[tuple]] = [None] * len(pieces)
    copies: List[Copy] = []
    base = 0
    for g, grp in enumerate(groups):
        grp.base = base
        cnt = {}
        for k in grp.members:
            p = pieces[k].prefix
            if p >= 0:
                cnt[p] = cnt.get(p, 0) + 1
        delta_cur = 0                       # "Delta <- 0"
        emitted = set()
        for k in grp.members:              # entries in assignment order (R8)
            pc = pieces[k]
            p = pc.prefix
            if p >= 0 and cnt[p] >= 2:     # shared prefix entry (R7)
                if p in emitted:
                    continue               # its suffixes were emitted with the prefix entry
                emitted.add(p)
                LP = int(prefix_len[p])
                copies.append(Copy(1, p, 0, LP, base + delta_cur))     # Copy(P_k -> B_g)
                d_prefix = delta_cur
                delta_cur += LP
                for k2 in grp.members:     # its suffixes, in assignment order
                    pc2 = pieces[k2]
                    if pc2.prefix != p:
                        continue
                    LQ = pc2.kv_len - LP
                    copies.append(Copy(0, pc2.request, pc2.kv_begin + LP, LQ, base + delta_cur))
                    offsets[k2] = (d_prefix, LP, delta_cur, LQ)        # O_g[i]
                    delta_cur += LQ + delta                             # M(Q_i) = L_Q + delta
            else:                          # singleton entry: L_P = 0, whole piece is the suffix
                copies.append(Copy(0, pc.request, pc.kv_begin, pc.kv_len, base + delta_cur))
                offsets[k] = (delta_cur, 0, delta_cur, pc.kv_len)
                delta_cur += pc.kv_len + delta
        grp.cap = delta_cur
        base += delta_cur
    return Plan(pieces, offsets, groups, copies, G0, base, order)


def valid_pairs_count(kv_len: Sequence[int], q_len: Sequence[int]) -> int:
    """Number of causally visible (query, key) pairs: sum_i q_i (kv_i - q_i) + q_i (q_i + 1) / 2.
    (Reading R11: causal within a request, block-diagonal across requests.)"""
    tot = 0
    for L, q in zip(kv_len, q_len):
        L, q = int(L), int(q)
        tot += q * (L - q) + q * (q + 1) // 2
    return tot
