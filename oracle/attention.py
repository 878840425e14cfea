"""Attention oracle — plain causal softmax attention, request by request, fp64.  TEST INFRASTRUCTURE.

PackInfer's packing, splitting, merging and relayout are lossless ("merged in a lossless
manner consistent with FlashAttention semantics"; "preserving lossless attention
semantics"; "preserving lossless attention semantics").  The method therefore reaches,
up to rounding order, plain per-request attention, and this oracle is that definition written
out with no packing, no tiling and no online softmax:

  for request i, query head h (KV head h // r, reading R11), query t in [0, q_len_i):
      pos = kv_len_i - q_len_i + t                      (reading R12: kv_len includes the
                                                          token(s) being computed)
      keys j in [0, pos] are the request's logical KV tokens, read through its block table
      (prefix tokens live in the prefix's shared pages; the table maps them — D6)
      s_j = (q . k_j) * scale,  scale = 1/sqrt(d)         (reading R11)
      m = max_j s_j ;  p_j = exp(s_j - m) ;  l = sum_j p_j  (materialised score row)
      o = (sum_j p_j v_j) / l ;  lse = m + ln l            (natural log, reading R10)

Inputs are the same bf16/fp32 tensors the GPU consumes, upcast exactly to fp64.
"""

from __future__ import annotations

import math
from typing import Iterable, Optional, Sequence, Tuple

import numpy as np


def _np64(x) -> np.ndarray:
    """Exact upcast to float64 (bf16/fp32 -> fp64 is exact).  Accepts torch tensors or arrays."""
    if hasattr(x, "detach"):
        import torch
        return x.detach().to("cpu", torch.float64).numpy()
    return np.asarray(x, dtype=np.float64)


def gather_request_kv(k_paged: np.ndarray, block_table: np.ndarray, row: int, n_tokens: int,
                      page_size: int, first: int = 0) -> np.ndarray:
    """Logical tokens [first, first+n_tokens) of block-table row `row` -> [n_tokens, Hkv, d].

    Paged cache layout [num_blocks, page, Hkv, d] (vLLM-style, D6: P:676 page 128/256)."""
    j = np.arange(first, first + n_tokens)
    blk = block_table[row, j // page_size]
    return k_paged[blk, j % page_size]


def attention(q, k_paged, v_paged, block_table, kv_len: Sequence[int], q_len: Sequence[int],
              page_size: int, scale: Optional[float] = None,
              requests: Optional[Iterable[int]] = None,
              row_block: int = 512) -> Tuple[np.ndarray, np.ndarray]:
    """Full oracle.  q: [total_q, Hq, d] in caller varlen order (request order, q_len rows each).

    Returns out [total_q, Hq, d] fp64 and lse [Hq, total_q] fp64 (NaN where not computed)."""
    q = _np64(q)
    kp = _np64(k_paged)
    vp = _np64(v_paged)
    bt = np.asarray(block_table.cpu() if hasattr(block_table, "cpu") else block_table)
    total_q, Hq, d = q.shape
    Hkv = kp.shape[2]
    r = Hq // Hkv
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    out = np.full((total_q, Hq, d), np.nan)
    lse = np.full((Hq, total_q), np.nan)
    q_off = np.concatenate([[0], np.cumsum(np.asarray(q_len, dtype=np.int64))])
    reqs = range(len(kv_len)) if requests is None else requests
    for i in reqs:
        L, ql = int(kv_len[i]), int(q_len[i])
        K = gather_request_kv(kp, bt, i, L, page_size)          # [L, Hkv, d]
        V = gather_request_kv(vp, bt, i, L, page_size)
        for t0 in range(0, ql, row_block):
            t1 = min(ql, t0 + row_block)
            pos = L - ql + np.arange(t0, t1)                    # [rows]
            n_keys = int(pos[-1]) + 1
            mask = np.arange(n_keys)[None, :] <= pos[:, None]   # causal within the request
            for h in range(Hq):
                hk = h // r
                Q = q[q_off[i] + t0:q_off[i] + t1, h, :]        # [rows, d]
                s = (Q @ K[:n_keys, hk, :].T) * scale           # materialised score rows
                s = np.where(mask, s, -np.inf)
                m = s.max(axis=1, keepdims=True)
                p = np.exp(s - m)
                l = p.sum(axis=1, keepdims=True)
                out[q_off[i] + t0:q_off[i] + t1, h, :] = (p @ V[:n_keys, hk, :]) / l
                lse[h, q_off[i] + t0:q_off[i] + t1] = (m + np.log(l))[:, 0]
    return out, lse


def attention_rows(q, k_paged, v_paged, block_table, kv_len, q_len, page_size,
                   rows: Sequence[Tuple[int, int]], scale: Optional[float] = None):
    """Oracle on selected (request, t) query rows only (all heads): for sampled full-size parity.

    Returns out [len(rows), Hq, d], lse [len(rows), Hq] (fp64)."""
    qn = _np64(q)
    kp = _np64(k_paged)
    vp = _np64(v_paged)
    bt = np.asarray(block_table.cpu() if hasattr(block_table, "cpu") else block_table)
    _, Hq, d = qn.shape
    Hkv = kp.shape[2]
    r = Hq // Hkv
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    q_off = np.concatenate([[0], np.cumsum(np.asarray(q_len, dtype=np.int64))])
    out = np.zeros((len(rows), Hq, d))
    lse = np.zeros((len(rows), Hq))
    cache = {}
    for n, (i, t) in enumerate(rows):
        L, ql = int(kv_len[i]), int(q_len[i])
        pos = L - ql + int(t)
        if i not in cache:
            cache.clear()
            cache[i] = (gather_request_kv(kp, bt, i, L, page_size),
                        gather_request_kv(vp, bt, i, L, page_size))
        K, V = cache[i]
        for h in range(Hq):
            hk = h // r
            s = (K[:pos + 1, hk, :] @ qn[q_off[i] + t, h, :]) * scale
            m = s.max()
            p = np.exp(s - m)
            l = p.sum()
            out[n, h] = (p @ V[:pos + 1, hk, :]) / l
            lse[n, h] = m + math.log(l)
    return out, lse


def partial_attention(qvec: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float):
    """Attention of one query over a key segment (no mask): returns (o normalised, lse).
    An empty segment is the merge identity (0, -inf) (reading R10)."""
    if K.shape[0] == 0:
        return np.zeros(V.shape[1]), -np.inf
    s = (K @ qvec) * scale
    m = s.max()
    p = np.exp(s - m)
    l = p.sum()
    return (p @ V) / l, m + math.log(l)
