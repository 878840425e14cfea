"""CTA-0 timeline of the packed attention kernel on the cfg2 prefill batch (debug hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import workloads as W
from paper_2602_06072_b200 import packinfer as pk

b = W.cfg2_prefill(0)
t = W.make_tensors(b, device="cuda")
pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, b.hq // b.hkv, b.d, torch.bfloat16, "cuda")
out = torch.empty((b.total_q, b.hq, b.d), dtype=torch.bfloat16, device="cuda")
pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out)
tr = torch.zeros(64 * 24 + 64 * 8, dtype=torch.int64, device="cuda")
L = pk.lib()
L.packinfer_debug_trace.argtypes = [ctypes.c_void_p]
L.packinfer_debug_trace(tr.data_ptr())
pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out)
torch.cuda.synchronize()
L.packinfer_debug_trace(None)
A = tr.cpu().numpy().astype(np.int64)
a = A[:64 * 24].reshape(64, 24)
U = A[64 * 24:].reshape(64, 8)
t0 = a[a > 0].min()
names = ["mA_wait", "mA_got", "mA_iss", "mB_wait", "mB_got", "mB_iss",
         "sA_wS", "sA_gotS", "sA_p1", "sA_arrP", "sB_wS", "sB_gotS", "sB_p1", "sB_arrP"]
print("tile " + " ".join(f"{n:>8s}" for n in names))
for i in range(40):
    row = a[i]
    print(f"{i:4d} " + " ".join(f"{(v - t0 if v else -1):8d}" for v in row[:14]))
# per-tile durations
d = lambda x, y: a[:40, y] - a[:40, x]
print("median sA: waitS", np.median(d(6, 7)), "pass1", np.median(d(7, 8)), "pass2+", np.median(d(8, 9)))
print("median sB: waitS", np.median(d(10, 11)), "pass1", np.median(d(11, 12)), "pass2+", np.median(d(12, 13)))
print("median mma: waitPA", np.median(d(0, 1)), "issueA", np.median(d(1, 2)), "waitPB", np.median(d(3, 4)), "issueB", np.median(d(4, 5)))
print("median A: waitV", np.median(d(1, 16)), "PVissue", np.median(d(16, 14)), "waitK", np.median(d(14, 18)), "Sissue", np.median(d(18, 2)))
print("median B: waitV", np.median(d(4, 17)), "PVissue", np.median(d(17, 15)), "waitK", np.median(d(15, 19)), "Sissue", np.median(d(19, 5)))
print("softmax A phases: gotS->ld0", np.median(d(7, 20)), "h0 compute", np.median(d(20, 21)), "->ld1", np.median(d(21, 22)), "h1 compute", np.median(d(22, 23)), "->end", np.median(d(23, 8)))
print("tile period (A arrive->arrive)", np.median(np.diff(a[:40, 9])))

u0 = U[U > 0].min()
print("unit  mma_waitQ  mma_gotQ  mma_gotK  mma_done  ql_waitF  ql_gotF  ql_done   (n_ktiles)")
w = pb.plan.prefill_work
for i in range(48):
    r = U[i]
    item = (0 + i * 148) // 16
    print(f"{i:4d} " + " ".join(f"{(v - u0 if v else -1):9d}" for v in r[:7]), int(w[item]["n_ktiles"]) if item < len(w) else -1)
