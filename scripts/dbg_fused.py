"""Debug: fused vs split attention launches on random mixed batches (bitwise), repeated."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from synth import workloads as W
from tests import gpu_helpers as H
for rep in range(3):
    for seed in (5, 6, 7, 8):
        b = W.random_batch(seed, n=16, max_len=900, hq=8, hkv=2, d=128, decode_frac=0.5)
        t = W.make_tensors(b, device="cuda")
        res = []
        for fused in (True, False, True, False):
            o, l, _ = H.run_batch(b, t, C=512, decode_chunk=256, fused=fused)
            res.append((o.cpu(), l.cpu().numpy()))
        for k in range(1, 4):
            lf, ls = res[0][1], res[k][1]
            d = ~((lf == ls) | (np.isnan(lf) & np.isnan(ls)))
            oeq = torch.equal(res[0][0], res[k][0])
            if d.sum() or not oeq:
                qoff = np.concatenate([[0], np.cumsum(b.q_len)])
                print("rep", rep, "seed", seed, "run", k, "lse diffs", int(d.sum()), "out equal", oeq)
                for h, r in np.argwhere(d)[:6]:
                    req = np.searchsorted(qoff, r, side="right") - 1
                    print("   h", h, "row", r, "req", req, "q_len", b.q_len[req], "kv", b.kv_len[req], lf[h, r], ls[h, r])
print("done")
