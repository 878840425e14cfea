"""Layout oracle — the group-contiguous KV buffers Alg. 1 Part 2 produces.  TEST INFRASTRUCTURE.

Alg. 1 lines "Copy(M_paged[P_k] -> B_g)" and "Copy(M_paged[Q_i] -> B_g)" gather
the valid tokens of the paged cache into contiguous group buffers (§3.2 "copying only valid
token states").  Reading R-layout: all groups' buffers are laid end to end
(base_g = sum of earlier capacities), per KV head: buf[h][base_g + Delta + t].

expected_buffers() evaluates that definition from the ORACLE's copy plan and the paged cache;
headroom cells are unspecified and reported through the `valid` mask.
"""

from __future__ import annotations

import numpy as np


def expected_buffers(copies, k_paged, block_table, n_requests: int, page_size: int,
                     buffer_tokens: int, heads=None):
    """Returns (buf [H, buffer_tokens, d] same dtype as k_paged (numpy), valid [buffer_tokens])."""
    kp = k_paged
    if hasattr(kp, "detach"):
        import torch
        kp = kp.detach().cpu()
        if kp.dtype == torch.bfloat16:          # keep the exact bits: view as int16
            kp = kp.view(torch.int16)
        kp = kp.numpy()
    bt = np.asarray(block_table.cpu() if hasattr(block_table, "cpu") else block_table)
    Hkv, d = kp.shape[2], kp.shape[3]
    heads = list(range(Hkv)) if heads is None else list(heads)
    buf = np.zeros((len(heads), buffer_tokens, d), dtype=kp.dtype)
    valid = np.zeros(buffer_tokens, dtype=bool)
    for c in copies:
        row = c.src_id if c.src_kind == 0 else n_requests + c.src_id
        j = np.arange(c.src_begin, c.src_begin + c.length)
        blk = bt[row, j // page_size]
        for hi, h in enumerate(heads):
            buf[hi, c.dst:c.dst + c.length] = kp[blk, j % page_size, h]
        if valid[c.dst:c.dst + c.length].any():
            raise AssertionError("copy destinations overlap")
        valid[c.dst:c.dst + c.length] = True
    return buf, valid
