"""CTA-0 timeline of the packed attention kernel on a decode batch (debug hook).
    python scripts/trace_decode.py [cfg3|cfg4_decode]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# the trace hooks are compiled in only with -DPI_TRACE=1: build that variant and load it
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_LIB = os.path.join(_ROOT, "variants", "libpi_trace.so")
if "PACKINFER_LIB" not in os.environ:
    from paper_2602_06072_b200 import build as _B
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    _B.build(True, False, _LIB, ("PI_TRACE=1",))
    os.environ["PACKINFER_LIB"] = _LIB
import numpy as np, torch
from synth import workloads as W
from paper_2602_06072_b200 import packinfer as pk

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
b = W.make_batch(name)
t = W.make_tensors(b, device="cuda")
pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, b.hq // b.hkv, b.d, torch.bfloat16, "cuda",
                    headroom=32 if "cfg4" in name else 0)
out = torch.empty((b.total_q, b.hq, b.d), dtype=torch.bfloat16, device="cuda")
pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out)
TT = 128   # TRACE_TILES in attention.cu
tr = torch.zeros(TT * 32 + 64 * 16 + 4 * 1024, dtype=torch.int64, device="cuda")
L = pk.lib()
L.packinfer_debug_trace.argtypes = [ctypes.c_void_p]
L.packinfer_debug_trace(tr.data_ptr())
pk.packinfer_attention_decode(pb.dp, t["q"], pb.k_buf, pb.v_buf, out, None, pb.partial_o, pb.partial_lse, 4)
torch.cuda.synchronize()
L.packinfer_debug_trace(None)
A = tr.cpu().numpy().astype(np.int64)
a = A[:TT * 32].reshape(TT, 32)
U = A[TT * 32:TT * 32 + 64 * 16].reshape(64, 16)
u0 = U[U > 0].min()
w = pb.plan.decode_work
print("unit  mma_waitQ  mma_gotQ  mma_gotK  mma_done  ql_waitF  ql_gotF  ql_done  sm_start sm_gotS0 sm_epi  sm_Oread sm_epidone (n_ktiles rows)")
for i in range(30):
    r = U[i]
    # snake order: CTA 0 takes unit k*148 (even k) / k*148+147 (odd k)
    item = ((i * 148) if i % 2 == 0 else (i * 148 + 147)) // b.hkv
    print(f"{i:4d} " + " ".join(f"{(v - u0 if v else -1):9d}" for v in r[:12]),
          int(w[item]["n_ktiles"]) if item < len(w) else -1, int(w[item]["row_count"]) if item < len(w) else -1)
t0 = a[a > 0].min() if (a > 0).any() else 0
print("softmax A per tile (gotS -> arriveP half 1):", [int(x) for x in (a[:30, 9] - a[:30, 7])])
print("softmax A wait S:", [int(x) for x in (a[:30, 7] - a[:30, 6])])

# per-tile softmax / MMA events (warpgroup A = key half 0 of single units), relative to "before wait S"
names = {30: "smA_exact", 31: "smA_rescl", 24: "pr_wKF", 25: "pr_Kiss", 26: "pr_Viss", 27: "mma_S", 28: "mma_gV", 29: "mma_gOF", 0: "mma_wPH", 1: "mma_gPH", 6: "smA_wS", 7: "smA_gS", 20: "smA_ldS", 22: "smA_exp", 8: "smA_P0", 9: "smA_P1",
         10: "smB_wS", 11: "smB_gS", 12: "smB_P0", 13: "smB_P1", 14: "mma_PV1"}
last = max(i for i in range(TT) if a[i, 6] > 0) if (a[:, 6] > 0).any() else -1
print("tile " + " ".join(f"{v:>8s}" for v in names.values()))
for i in list(range(0, 20)) + list(range(max(20, last - 14), last + 1)):
    base = a[i, 6]
    print(f"{i:4d} " + " ".join(f"{(a[i, e] - base if a[i, e] else -1):8d}" for e in names))

# per-CTA entry / exit (%globaltimer, ns) and units taken: load balance and tail of the traced launch
C0 = TT * 32 + 64 * 16
cta = tr.cpu().numpy()[C0:].reshape(-1, 4)
cta = cta[cta[:, 0] > 0]
if len(cta):
    g0 = cta[:, 0].min()
    st, en = (cta[:, 0] - g0) / 1e3, (cta[:, 1] - g0) / 1e3
    print(f"CTAs {len(cta)}: entry us max {st.max():.2f}; exit us min {en.min():.2f} median {np.median(en):.2f} "
          f"p90 {np.percentile(en, 90):.2f} max {en.max():.2f}; units/CTA min {cta[:, 2].min()} max {cta[:, 2].max()}")
    print("  busy fraction (sum of CTA spans / (CTAs x launch span)):", round(float((en - st).sum() / (len(cta) * en.max())), 3))

# sliced-unit epilogue phases (softmax warp 4, per unit): O landed -> xch merge -> barrier ->
# stage 0 (quarters 2, 3 store) -> stage 1 (quarters 0, 1 add) -> final sum + stores
print("unit  Olanded->xch  ->bar  ->stage0  ->stage1  ->stored   (cycles)")
for i in range(40):
    r = U[i]
    if r[12] > 0:
        print(f"{i:4d} {r[12] - r[9]:12d} {r[13] - r[12]:6d} {r[14] - r[13]:8d} {r[15] - r[14]:8d} {r[10] - r[15]:8d}")
