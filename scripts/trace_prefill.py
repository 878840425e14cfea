"""CTA-0 timeline of the packed attention kernel on the cfg2 prefill batch (debug hook)."""
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

b = W.cfg2_prefill(0)
t = W.make_tensors(b, device="cuda")
pb = pk.PackedBatch(b.kv_len, b.q_len, b.prefix_id, b.prefix_len, b.hkv, b.hq // b.hkv, b.d, torch.bfloat16, "cuda")
out = torch.empty((b.total_q, b.hq, b.d), dtype=torch.bfloat16, device="cuda")
pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out)
TT = 128   # TRACE_TILES in attention.cu
tr = torch.zeros(TT * 32 + 64 * 16 + 4 * 1024, dtype=torch.int64, device="cuda")
L = pk.lib()
L.packinfer_debug_trace.argtypes = [ctypes.c_void_p]
L.packinfer_debug_trace(tr.data_ptr())
pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out)
torch.cuda.synchronize()
L.packinfer_debug_trace(None)
A = tr.cpu().numpy().astype(np.int64)
a = A[:TT * 32].reshape(TT, 32)
U = A[TT * 32:TT * 32 + 64 * 16].reshape(64, 16)
t0 = a[a > 0].min()
names = ["mA_wP", "mA_gotP", "mA_S+", "mB_wP", "mB_gotP", "mB_S+",
         "sA_wS0", "sA_gS0", "sA_PH", "sA_PF", "sB_wS0", "sB_gS0", "sB_PH", "sB_PF", "mA_PV1", "mB_PV1",
         "sA_gS1", "sA_-", "sB_gS1"]
print("tile " + " ".join(f"{n:>7s}" for n in names))
for i in range(40):
    row = a[i]
    print(f"{i:4d} " + " ".join(f"{(v - t0 if v else -1):7d}" for v in row[:19]))
d = lambda x, y: a[2:40, y] - a[2:40, x]
med = lambda x, y: float(np.median(d(x, y)))
for X, nm in ((0, "A"), (1, "B")):
    o = 4 * X
    print(f"softmax {nm}: waitS0 {med(6+o, 7+o):.0f}  h0 {med(7+o, 8+o):.0f}  waitS1 {med(8+o, 16+2*X):.0f}  "
          f"h1 {med(16+2*X, 9+o):.0f}  period {float(np.median(np.diff(a[2:40, 9+o]))):.0f}")
    print(f"mma {nm}: PHALF->got {med(0+3*X, 1+3*X):.0f}  got->PV1 issued {med(1+3*X, 14+X):.0f}  PV1->S+ {med(14+X, 2+3*X):.0f}")
print("S(j+1) issued -> softmax got S0(j+1) A:", float(np.median(a[3:40, 7] - a[2:39, 2])), " B:", float(np.median(a[3:40, 11] - a[2:39, 5])))
print("PFULL(j) -> S(j+1) issued A:", float(np.median(a[2:40, 2] - a[2:40, 9])), " B:", float(np.median(a[2:40, 5] - a[2:40, 13])))

u0 = U[U > 0].min()
nu = int((U[:, 3] > 0).sum())
ev = torch.cuda.Event(enable_timing=True); ev2 = torch.cuda.Event(enable_timing=True)
ev.record(); pb.run(t["q"], t["k_paged"], t["v_paged"], t["block_table"], out); ev2.record(); torch.cuda.synchronize()
print("CTA0 units traced", nu, "cycles first->last", int(U[nu - 1, 3] - u0), "step ms", ev.elapsed_time(ev2))
for X, nm in ((0, "A"), (1, "B")):
    o = 4 * X
    print(f"softmax {nm} detail: ld h0 {med(7+o, 20+X):.0f}  exp h0 {med(20+X, 22+X):.0f}  store+ {med(22+X, 16+2*X):.0f}  "
          f"ldS1+arrive {med(16+2*X, 8+o):.0f}  h1 {med(8+o, 9+o):.0f}")
    fl = a[2:40, 17 + 2 * X]
    print(f"  spec flags (bit0 h0 spec, bit1 h1 spec): {np.bincount((fl & 3).astype(int), minlength=4).tolist()}")

# producer / K-arrival view (events 24 = producer waits K slot, 25 = K TMA issued, 26 = V TMA issued,
# 27 = issuer saw K(j+1) land; all relative to softmax A's S(j) arrival of the same tile)
print("tile  Kwait  Kissue  Vissue  K(j+1)seen  mA_PV1  mA_S+   (relative to sA_gS0 of tile j)")
for i in range(4, 20):
    r0 = a[i, 7]
    print(f"{i:4d} " + " ".join(f"{(a[i, c] - r0 if a[i, c] else -1):7d}" for c in (24, 25, 26, 27, 14, 2)))

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

# per-unit timeline of CTA 0 (cycles relative to the first event): MMA issuer unit start, Q landed,
# K landed, last MMA committed; Q gather waits QFREE / got it / issued; softmax warp 4 unit start,
# first S landed, O landed (epilogue start), O read + stored, epilogue done
print("unit  mma_start  mma_gotQ  mma_gotK  mma_done  ql_waitF  ql_gotF  ql_done  sm_start sm_gotS0  sm_epi  sm_Oread sm_epidone  | gotQ-prev_done  epi(cycles)")
prev_done = None
for i in range(min(nu, 40)):
    r = U[i]
    gap = (r[1] - prev_done) if prev_done else 0
    print(f"{i:4d} " + " ".join(f"{(v - u0 if v else -1):9d}" for v in r[:12]) + f"  | {gap:8d} {r[11] - r[9]:8d}")
    prev_done = r[3]
