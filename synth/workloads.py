"""Seeded synthetic workloads shaped like the paper's.

Length recipes:
  cfg1 toy      {7, 33, 128, 500}; Hq = Hkv = 4, d = 64, fp32.  prefill (q = L) and one decode
                step (kv = L + 1, q = 1)                                (BASELINE.json configs[0])
  cfg2 prefill  64 requests, seed 0: 38 uniform-int [16,128) + 26 log-uniform-int [128,8192],
                max forced to 8192, shuffled (">60% shorter than 128 tokens");
                Llama-3-8B GQA: Hq 32, Hkv 8, d 128, bf16            (configs[1])
  cfg3 decode   256 requests, seed 1: kv log-uniform-int [32, 32768], max forced; q = 1
                                                                       (configs[2])
  cfg4 prefix   128 requests, seed 2: 8 prompts x 2048 tokens, prefix id = permutation of
                i mod 8, suffix uniform-int [16, 1024]; decode step or suffix prefill
                                                                       (configs[3])
  cfg5 mixed    Llama-3-70B: Hq 64, Hkv 8, d 128.  prefill: 2 x 131072 + 30 log-uniform
                [16, 4096] (seed 3); decode: 224 log-uniform [32, 32768], max forced
                                                                       (configs[4])
Tensor values: N(0,1) fp32 cast to bf16 (RNE) (or kept fp32 for the toy), from a seeded torch
generator on the requested device.  Paged KV: page 128, physical blocks randomly
permuted to model fragmentation; shared prefixes occupy shared physical pages that
every member's block table maps (prefix lengths are page multiples).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class Batch:
    name: str
    kv_len: np.ndarray            # int32 [n]
    q_len: np.ndarray             # int32 [n]
    prefix_id: np.ndarray         # int32 [n], -1 = none
    prefix_len: np.ndarray        # int32 [n_prefix]
    hq: int
    hkv: int
    d: int
    dtype: str = "bf16"           # "bf16" or "fp32"
    page_size: int = 128
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.kv_len.shape[0])

    @property
    def total_q(self) -> int:
        return int(self.q_len.sum())

    def prefill_flops(self) -> int:
        """4*d*Hq*sum_i [q_i (kv_i - q_i) + q_i (q_i + 1)/2] over q_len > 1 requests."""
        tot = 0
        for L, q in zip(self.kv_len.tolist(), self.q_len.tolist()):
            if q > 1:
                tot += q * (L - q) + q * (q + 1) // 2
        return 4 * self.d * self.hq * tot


def _loguniform_int(rng, lo, hi, size):
    x = np.exp(rng.uniform(math.log(lo), math.log(hi + 1), size=size))
    return np.clip(np.floor(x).astype(np.int64), lo, hi)


def toy_prefill() -> Batch:
    L = np.array([7, 33, 128, 500], dtype=np.int32)
    return Batch("cfg1-toy-prefill", L, L.copy(), np.full(4, -1, np.int32),
                 np.zeros(0, np.int32), 4, 4, 64, "fp32", 128, 11)


def toy_decode() -> Batch:
    L = np.array([7, 33, 128, 500], dtype=np.int32) + 1
    return Batch("cfg1-toy-decode", L, np.ones(4, np.int32), np.full(4, -1, np.int32),
                 np.zeros(0, np.int32), 4, 4, 64, "fp32", 128, 12)


def cfg2_prefill(seed: int = 0) -> Batch:
    rng = np.random.default_rng(seed)
    short = rng.integers(16, 128, size=38)
    long = _loguniform_int(rng, 128, 8192, 26)
    long[np.argmax(long)] = 8192
    L = np.concatenate([short, long]).astype(np.int32)
    L = L[rng.permutation(L.shape[0])]
    return Batch("cfg2-llama3-8b-prefill", L, L.copy(), np.full(L.shape[0], -1, np.int32),
                 np.zeros(0, np.int32), 32, 8, 128, "bf16", 128, seed)


def cfg3_decode(seed: int = 1, n: int = 256) -> Batch:
    rng = np.random.default_rng(seed)
    L = _loguniform_int(rng, 32, 32768, n)
    L[np.argmax(L)] = 32768
    L = L.astype(np.int32)
    return Batch("cfg3-llama3-8b-decode", L, np.ones(n, np.int32), np.full(n, -1, np.int32),
                 np.zeros(0, np.int32), 32, 8, 128, "bf16", 128, seed)


def _cfg4(seed: int, decode: bool) -> Batch:
    rng = np.random.default_rng(seed)
    n, n_prefix, plen = 128, 8, 2048
    pid = (np.arange(n) % n_prefix)[rng.permutation(n)].astype(np.int32)
    suf = rng.integers(16, 1025, size=n).astype(np.int32)
    L = (plen + suf).astype(np.int32)
    q = np.ones(n, np.int32) if decode else suf.copy()
    name = "cfg4-shared-prefix-" + ("decode" if decode else "suffix-prefill")
    return Batch(name, L, q, pid, np.full(n_prefix, plen, np.int32), 32, 8, 128, "bf16", 128, seed)


def cfg4_decode(seed: int = 2) -> Batch:
    return _cfg4(seed, True)


def cfg4_prefill(seed: int = 2) -> Batch:
    return _cfg4(seed, False)


def cfg5_mixed(seed: int = 3, long_len: int = 131072, n_short: int = 30, n_dec: int = 224) -> Batch:
    rng = np.random.default_rng(seed)
    pre = np.concatenate([[long_len, long_len], _loguniform_int(rng, 16, 4096, n_short)])
    dec = _loguniform_int(rng, 32, 32768, n_dec)
    dec[np.argmax(dec)] = 32768
    L = np.concatenate([pre, dec]).astype(np.int32)
    q = np.concatenate([pre, np.ones(n_dec, np.int64)]).astype(np.int32)
    n = L.shape[0]
    return Batch("cfg5-llama3-70b-mixed", L, q, np.full(n, -1, np.int32), np.zeros(0, np.int32),
                 64, 8, 128, "bf16", 128, seed)


def random_batch(seed: int, n: int = 12, max_len: int = 700, hq: int = 4, hkv: int = 2, d: int = 64,
                 dtype: str = "bf16", n_prefix: int = 2, decode_frac: float = 0.3,
                 prefix_frac: float = 0.5, page_size: int = 128) -> Batch:
    """Small mixed batch for parity sweeps: heterogeneous lengths, some decode rows, some
    shared prefixes (prefix lengths are page multiples), some suffix prefills."""
    rng = np.random.default_rng(seed)
    plen = (rng.integers(1, 3, size=n_prefix) * page_size).astype(np.int32)
    kv, q, pid = [], [], []
    for i in range(n):
        use_p = n_prefix > 0 and rng.random() < prefix_frac
        p = int(rng.integers(0, n_prefix)) if use_p else -1
        base = int(plen[p]) if p >= 0 else 0
        L = base + int(_loguniform_int(rng, 1, max_len, 1)[0])
        if rng.random() < decode_frac:
            ql = 1
        elif p >= 0:
            ql = L - base                          # suffix prefill over the cached prefix
        else:
            ql = L if rng.random() < 0.7 else int(rng.integers(1, L + 1))
        if p >= 0 and ql > L - base:
            ql = L - base
        kv.append(L)
        q.append(max(1, ql))
        pid.append(p)
    return Batch(f"random-{seed}", np.array(kv, np.int32), np.array(q, np.int32),
                 np.array(pid, np.int32), plen, hq, hkv, d, dtype, page_size, seed)


CONFIGS = {
    "toy_prefill": toy_prefill, "toy_decode": toy_decode, "cfg2": cfg2_prefill,
    "cfg3": cfg3_decode, "cfg4_decode": cfg4_decode, "cfg4_prefill": cfg4_prefill,
    "cfg5": cfg5_mixed,
}


def make_batch(name: str, **kw) -> Batch:
    return CONFIGS[name](**kw)


def make_tensors(b: Batch, device="cpu", seed: Optional[int] = None, peaky: float = 1.0, extra_tokens: int = 0):
    """Seeded tensors for a batch.

    Returns dict with
      q            [total_q, Hq, d]            (bf16 or fp32)
      k_paged      [num_blocks, page, Hkv, d]
      v_paged      [num_blocks, page, Hkv, d]
      block_table  [n + n_prefix, max_blocks] int32  (rows >= n are the prefixes' tables)
    Every request's table covers its whole logical sequence (+ extra_tokens of room for decode
    appends); a member of a shared prefix maps the prefix's physical blocks first.  Physical blocks
    are randomly permuted."""
    import torch
    seed = b.seed if seed is None else seed
    P = b.page_size
    rng = np.random.default_rng(seed + 7919)
    n, n_prefix = b.n, int(b.prefix_len.shape[0])
    for p in range(n_prefix):
        assert int(b.prefix_len[p]) % P == 0, "prefix lengths must be page multiples"
    pref_blocks = [int(b.prefix_len[p]) // P for p in range(n_prefix)]
    own_blocks = []
    for i in range(n):
        base = int(b.prefix_len[b.prefix_id[i]]) if b.prefix_id[i] >= 0 else 0
        own_blocks.append(-(-(int(b.kv_len[i]) + extra_tokens - base) // P))   # room for decode appends
    nb = sum(pref_blocks) + sum(own_blocks)
    perm = rng.permutation(max(nb, 1)).astype(np.int32)
    cur = 0
    pref_tab = []
    for p in range(n_prefix):
        pref_tab.append(perm[cur:cur + pref_blocks[p]])
        cur += pref_blocks[p]
    rows = []
    for i in range(n):
        own = perm[cur:cur + own_blocks[i]]
        cur += own_blocks[i]
        rows.append(np.concatenate([pref_tab[b.prefix_id[i]], own]) if b.prefix_id[i] >= 0 else own)
    rows += pref_tab
    max_blocks = max([len(r) for r in rows] + [1])
    bt = np.zeros((n + n_prefix, max_blocks), np.int32)
    for k, r in enumerate(rows):
        bt[k, :len(r)] = r
    dt = torch.bfloat16 if b.dtype == "bf16" else torch.float32
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    q = (torch.randn((b.total_q, b.hq, b.d), generator=g, device=device) * peaky).to(dt)
    k = torch.randn((max(nb, 1), P, b.hkv, b.d), generator=g, device=device).to(dt)
    v = torch.randn((max(nb, 1), P, b.hkv, b.d), generator=g, device=device).to(dt)
    return {"q": q, "k_paged": k, "v_paged": v,
            "block_table": torch.from_numpy(bt).to(device)}
