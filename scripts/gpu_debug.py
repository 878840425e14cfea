"""First-contact GPU diagnostics: runs each hot-path stage on small inputs and prints errors vs the
oracle (no asserts, so one failing stage does not hide the others)."""
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from synth import workloads as W
from oracle import plan as OP, layout as OL, attention as OA
from paper_2602_06072_b200 import packinfer as pk
from tests import gpu_helpers as H


def stage(name, fn):
    t0 = time.time()
    try:
        res = fn()
        print(f"[OK]   {name}: {res}  ({time.time()-t0:.1f}s)", flush=True)
    except Exception as e:  # noqa
        print(f"[FAIL] {name}: {e!r}  ({time.time()-t0:.1f}s)", flush=True)
        traceback.print_exc()


def relayout_check(b, C=8192, delta=3):
    t = W.make_tensors(b, device="cuda")
    out, lse, pb = H.run_batch(b, t, C=C, delta=delta)
    op = OP.plan(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, C, headroom=delta)
    buf, valid = OL.expected_buffers(op.copies, t["k_paged"].cpu(), t["block_table"].cpu(), b.n, b.page_size,
                                     op.buffer_tokens)
    kb = pb.k_buf.cpu()
    kb = (kb.view(torch.int16) if kb.dtype == torch.bfloat16 else kb).numpy()
    ok = np.array_equal(kb[:, valid], buf[:, valid])
    zero = bool((kb[:, ~valid] == 0).all())
    return dict(bitwise=ok, headroom_zero=zero, cells=int(valid.sum()))


def attn_check(b, C=8192, delta=0, chunk=1024):
    t = W.make_tensors(b, device="cuda")
    out, lse, pb = H.run_batch(b, t, C=C, delta=delta, decode_chunk=chunk)
    ro, rl = H.oracle_full(b, t)
    o = out.float().cpu().numpy()
    err = np.abs(o - ro)
    l = lse.cpu().numpy()
    lerr = np.abs(l - rl)
    bad_rows = np.unique(np.where(~np.isfinite(o) | (err > 1e-2))[0])
    return dict(max_abs=float(np.nanmax(err)), mean_abs=float(np.nanmean(err)), nonfinite=int((~np.isfinite(o)).sum()),
                lse_max=float(np.nanmax(lerr)), bad_rows=bad_rows[:10].tolist(), n_bad=len(bad_rows),
                work=(pb.plan.c.n_prefill_work, pb.plan.c.n_decode_work, pb.plan.c.n_partial_slots))


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0), pk.version(), flush=True)
    stage("relayout bf16 random", lambda: relayout_check(W.random_batch(1, n=8, max_len=300, hq=4, hkv=2, d=128)))
    stage("relayout fp32 toy", lambda: relayout_check(W.toy_prefill()))
    stage("toy prefill fp32 C=8192", lambda: attn_check(W.toy_prefill()))
    stage("toy prefill fp32 C=128", lambda: attn_check(W.toy_prefill(), C=128))
    stage("toy decode fp32 C=8192", lambda: attn_check(W.toy_decode()))
    stage("toy decode fp32 C=128", lambda: attn_check(W.toy_decode(), C=128, chunk=128))
    one = W.Batch("one", np.array([128], np.int32), np.array([128], np.int32), np.array([-1], np.int32),
                  np.zeros(0, np.int32), 1, 1, 128, "bf16", 128, 3)
    stage("single 128 bf16 d128", lambda: attn_check(one))
    stage("random bf16 d128 gqa2", lambda: attn_check(W.random_batch(2, n=10, max_len=600, hq=4, hkv=2, d=128)))
    stage("random bf16 d64 gqa2", lambda: attn_check(W.random_batch(3, n=10, max_len=600, hq=4, hkv=2, d=64)))
    stage("random bf16 d128 C=256 split", lambda: attn_check(W.random_batch(4, n=10, max_len=900, hq=8, hkv=2, d=128),
                                                             C=256, chunk=256))
