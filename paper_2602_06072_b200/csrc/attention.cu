// Packed attention over the union of valid query-key regions (PackInfer §3.1): ONE
// persistent launch per call covers every work item of every group (reading R17).
//
// Work item = <= 128 query rows (prefill: tokens of one or more packed requests; decode:
// (request, GQA sub-head) rows) and a list of key spans in the group-contiguous KV
// buffers (Alg. 1 Part 2).  Every span but the last is visible to every row; in the last span row
// r sees keys [lo_r, hi_r) (causal own-suffix / decode chunk).
//
// Launch unit = (work item, KV head, Q-tile pair).  Prefill units carry TWO Q tiles — two query
// heads of the same GQA group — which share every K/V tile and every mask, so one TMA stream feeds
// two tensor-core pipelines.  Decode units carry one tile (its rows already span the GQA group).
//
// Per CTA (one per SM, 384 threads, warp-specialised, setmaxnreg 56 / 216):
//   warp 0    TMA producer: K/V tiles (128 keys x d, SWIZZLE_128B) into a 2-stage ring
//   warp 1    TMEM allocator + converged tcgen05.mma issuer (elect.sync), FA4-style ping-pong:
//               S_X = Q_X K^T -> TMEM S_X     (SS, M=128 N=128 K=d, one chain)
//               O_X += P_X V  -> TMEM O_X     (TS: P_X read from TMEM where it overwrote S_X,
//                                              in two 64-key halves as the softmax releases them)
//             per K tile j: PV_A(j) half 0 | half 1, S_A(j+1) | PV_B(j) half 0 | half 1, S_B(j+1)
//             (single-tile decode units: S regions alternate per tile, the two warpgroups split
//             the keys of every tile into O_0 / O_1, LSE-merged in the epilogue)
//   warp 2    Q gather for both tiles through the plan's row table (TMA tile::gather4)
//   warp 3    fp32 operands only: stages V^T (K-major) for kind::tf32
//   warps 4-7 softmax / correction / epilogue of tile A; warps 8-11 of tile B.  Thread i owns
//             row i (= TMEM lane i), so row max / sum need no shuffles.  One streaming pass per
//             64-column half (each S element read from TMEM once); once the running max is set an
//             unmasked half is exponentiated speculatively against it and certified by its sum;
//             the O rescale is lazy (only when the running max grows by > 2^8) and happens in TMEM.
//             exp2: MUFU for 6 of every 8 pairs, a minimax cubic on the FMA pipe for the rest.
// bf16 operands run kind::f16, fp32 operands kind::tf32; accumulation fp32 (reading R13).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdint>
#include <type_traits>

#include <cuda_bf16.h>

#include "device_common.h"
#include "packinfer.h"
#include "sm100.cuh"

#ifndef PI_P_ROUNDED_SUM
#define PI_P_ROUNDED_SUM 2   // O normalised by the row sum of the bf16-rounded P: 1 = FHADD.BF16, 2 = PRMT + FADD2; 0 = exact sum
#endif
#ifndef PI_DYN_SCHED
#define PI_DYN_SCHED 1   // dynamic LPT list scheduling of units (0: static snake order, A/B)
#endif
#ifndef PI_SINGLE_S128
#define PI_SINGLE_S128 1   // single-tile units' S: 0 two N = 64 halves, 1 one N = 128 chain,
#endif                     // 2 N = 128 for the first two tiles only, 3 N = 128 when n_ktiles <= 4
#ifndef PI_SYNCCHECK_PVH
#define PI_SYNCCHECK_PVH 0   // 1: wait every PVH phase (synccheck-clean variant, 1-2 % slower)
#endif
#ifndef PI_MERGE_ATOM
#define PI_MERGE_ATOM 0   // merge counters: 0 atom.release, 1 atom.acq_rel, 2 one fence per unit + relaxed, 3 relaxed (A/B)
#endif
#ifndef PI_MERGE_WARP
#define PI_MERGE_WARP 1   // A/B: 0 = no merge warp code, 2 = merge warp handshake only (timing, wrong results)
#endif
#ifndef PI_POLY_SAT
#define PI_POLY_SAT 1
#endif
#ifndef PI_POLY_PAIRS
#define PI_POLY_PAIRS 2   // of every 8 score pairs, this many take exp2 on the FMA pipe (A/B: scripts/ab_poly.sh)
#endif

// Debug build (-DPI_CHECKS=1, tests/test_gpu_checks.py): device-side bounds checks on every plan
// table entry the kernel dereferences (work items, spans, rows, partial slots, heads); a failed
// check prints its id and traps.  compute-sanitizer is not available on every GPU pool; these
// checks cover the indices it would.
#ifndef PI_CHECKS
#define PI_CHECKS 0
#endif
#define PI_CHECK(cond, id)                                                                             \
  do {                                                                                                 \
    if (PI_CHECKS && !(cond)) {                                                                        \
      printf("packinfer device check %d failed: block %d thread %d\n", (int)(id), (int)blockIdx.x,       \
             (int)threadIdx.x);                                                                        \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)

namespace pi {

using namespace sm100;

constexpr float NEG_INF_F = -INFINITY;

struct AttnParams {
  const pi_work* work_p;   // prefill work items (units [0, total_p))
  const pi_work* work_d;   // decode work items (units [total_p, total_p + n_work_d * units_d))
  const pi_row* rows;
  const pi_span* spans;
  int32_t n_work_p, n_work_d;
  int32_t units_p;    // launch units per prefill item: hkv * ceil(r / tiles_per_unit)
  int32_t units_d;    // launch units per decode item: hkv
  int32_t total_p;    // n_work_p * units_p
  int32_t r;          // GQA ratio
  const uint8_t* q;
  int64_t q_row_stride;    // elements
  uint8_t* out;
  int64_t out_row_stride;  // elements
  float* lse;
  int32_t total_q;
  int32_t hq_count;
  float* partial_o;
  float* partial_lse;
  float scale_log2;        // softmax_scale * log2(e)
  int32_t out_f32;         // 1: write out as fp32 (bf16 operands, fp32 output mode)
  const uint8_t* v_buf;    // fp32 path only: V staged transposed by warp 3
  int64_t buffer_tokens;
  unsigned long long* trace;  // debug only (packinfer_debug_trace): CTA-0 clock64 timeline
  int32_t q_heads_stride;  // q_row_stride / head_dim: rows of the 2D (token*stride + head, d) Q view
  int32_t tiles_per_unit;  // prefill: 2 (GQA head pairs; bf16) or 1 (fp32 operands)
  // in-kernel LSE merge (packinfer_attention_merge; NULL merge_ctr = separate packinfer_merge)
  const pi_merge* merges;
  const int32_t* slot_merge;
  uint32_t* merge_ctr;     // [n_merges * hq_count], zero on entry and on exit
  // paged mode (packinfer_attention_decode_paged): K/V tiles straight from the paged cache
  const int32_t* block_table;   // NULL = group-contiguous buffers
  int32_t max_blocks, page, kv_head0;
  uint32_t* sched;              // [0] dynamic unit counter, [1] CTAs exited; zero on entry and on exit
  int32_t n_partial_slots;      // (PI_CHECKS bounds)
  int32_t pdl_wait;             // launched as a programmatic dependent: griddepcontrol.wait after set-up
};

// One paged-mode tile: logical keys [k0, k0 + 128) of block-table row `row` = 128 consecutive slots
// of one page (k0 a multiple of 128, page a multiple of 128); returns the token coordinate of the
// paged tensor map.
__device__ __forceinline__ int paged_token(const AttnParams& p, int row, int k0) {
  const int blk = __ldg(&p.block_table[(int64_t)row * p.max_blocks + k0 / p.page]);
  return blk * p.page + k0 % p.page;
}

// Debug timeline: trace[(tile * 32 + event)], first TRACE_TILES tiles of CTA 0.
constexpr int TRACE_TILES = 128;
// Compiled in only with -DPI_TRACE=1 (scripts/trace_*.py build such a variant): the hot loops of
// the production build carry no trace checks.
#ifndef PI_TRACE
#define PI_TRACE 0
#endif
__device__ __forceinline__ void trace_ev(const AttnParams& p, uint32_t tile, int ev) {
  if (PI_TRACE && p.trace != nullptr && blockIdx.x == 0 && tile < (uint32_t)TRACE_TILES)
    p.trace[tile * 32 + ev] = clock64();
}
// Per-unit events: trace[TRACE_TILES * 32 + unit * 16 + ev], first 64 units of CTA 0 (0-3 MMA issuer, 4-6 Q
// gather, 7-11 softmax warp 4: unit start, first S landed, epilogue start (O landed), O read,
// epilogue done).
__device__ __forceinline__ void trace_unit(const AttnParams& p, uint32_t unit, int ev) {
  if (PI_TRACE && p.trace != nullptr && blockIdx.x == 0 && unit < 64u) p.trace[TRACE_TILES * 32 + unit * 16 + ev] = clock64();
}
// Per-CTA %globaltimer (ns) at entry / exit and units processed: trace[TRACE_TILES * 32 + 64 * 16 + 4 * cta + {0, 1, 2}]
// (load balance / tail of a launch; every CTA)
constexpr int TRACE_CTA_BASE = TRACE_TILES * 32 + 64 * 16;
__device__ __forceinline__ void trace_cta(const AttnParams& p, int ev, unsigned long long v) {
  if (PI_TRACE && p.trace != nullptr) p.trace[TRACE_CTA_BASE + 4 * blockIdx.x + ev] = v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

#ifndef PI_DEC_SLICE
#define PI_DEC_SLICE 1   // lane-sliced single-tile units (<= kSliceRows rows): see unit_sliced()
#endif
#ifndef PI_SLICE_ROWS
#define PI_SLICE_ROWS 32   // lane-sliced single-tile units: up to this many rows (one lane quarter)
#endif
#ifndef PI_FUSED_PDL
#define PI_FUSED_PDL 1   // packinfer_attention(_merge) over both kinds: two specialised launches chained by PDL
#endif
#ifndef PI_STEP_PDL
#define PI_STEP_PDL 1   // attention / merge launches as programmatic dependents (set-up overlaps the previous kernel)
#endif
#ifndef PI_Q_BOX
#define PI_Q_BOX 1   // Q tiles of consecutive tokens as 3D TMA boxes (else every tile via gather4)
#endif
#ifndef PI_DEC_NSV
#define PI_DEC_NSV 3   // V stages of decode-only (single-tile) launches: V is held until P.V
#endif

template <int D, bool F32, int UK = 3>
struct AttnCfg {
  static constexpr int ES = F32 ? 4 : 2;
  static constexpr int ROW_BYTES = D * ES;            // one Q/K/V row
  static constexpr int ATOMS = ROW_BYTES / 128;       // 128-byte swizzle atoms per row
  static constexpr int ATOM_ELEMS = 128 / ES;
  static constexpr int ATOM_BYTES = 128 * 128;        // one atom column of 128 rows
  static constexpr int TILE_BYTES = 128 * ROW_BYTES;  // 128 rows
  // K / V pipeline stages.  V tiles live until their P.V, K tiles only until S: decode-only
  // launches (one Q tile) spend the second Q tile's space on a third V stage, so the producer runs
  // one more tile ahead across unit boundaries.
  static constexpr int NQ = UK == 2 ? 1 : 2;          // Q tiles resident
  static constexpr int NSK = 2;
  static constexpr int NSV = (UK == 2 && !F32) ? PI_DEC_NSV : 2;
  static constexpr int QK_STEPS = ROW_BYTES / 32;     // MMAs per S tile (32 bytes of K each)
  static constexpr int PV_STEPS = 128 * ES / 32;      // MMAs per O update (32 bytes of keys each)
  static constexpr int KEYS_PER_PV_STEP = 32 / ES;
  static constexpr int OFF_Q = 0;                     // Q_A, Q_B
  static constexpr int OFF_K = NQ * TILE_BYTES;
  static constexpr int OFF_V = OFF_K + NSK * TILE_BYTES;
  static constexpr int OFF_BAR = OFF_V + NSV * TILE_BYTES;
  static constexpr int OFF_XCH = OFF_BAR + 512;       // single units: (m, l, l_rounded) of both warpgroups
  // lane-sliced single units: the four lane quarters' O partials of <= kSliceRows rows (padded rows)
  // (two quarter-pair sums, [2][PI_SLICE_ROWS][OBUF_STRIDE] fp32), aliasing XCH: the epilogue
  // reads XCH into registers and passes a barrier before the buffer is written
  static constexpr int OBUF_STRIDE = D + 4;
  static constexpr int XCH_BYTES = 2 * 128 * 16;
  static constexpr int OFF_OBUF = OFF_XCH;
  // (or, for units of <= 8 rows, the eight raw partials [8][8][OBUF_STRIDE] + their (m, l, l_r))
  static constexpr int OBUF_ROWS = 2 * PI_SLICE_ROWS > 64 ? 2 * PI_SLICE_ROWS : 64;
  static constexpr int OBUF_BYTES = ((UK & 2) && !F32) ? OBUF_ROWS * OBUF_STRIDE * 4 : 0;
  static constexpr int SMEM = OFF_XCH + (OBUF_BYTES > XCH_BYTES ? OBUF_BYTES : XCH_BYTES) + 1024;  // + alignment slack
  // single units: warpgroup B writes P of keys 64..127 over the S columns it has read itself
  // (bf16: 32 packed columns at 96..127; fp32: 64 columns at 64..127), never over warpgroup A's
  static constexpr uint32_t P1_SINGLE = F32 ? 64u : 96u;
  static constexpr uint32_t FMT = F32 ? 2u : 1u;
  static constexpr uint32_t IDESC_QK = idesc_make(FMT, 128, 64, 0, 0);   // decode: S in two N=64 halves
  static constexpr uint32_t IDESC_QK128 = idesc_make(FMT, 128, 128, 0, 0);  // pair units: one N=128 S
  // bf16: V is the MN-major B operand straight from TMA.  fp32 (kind::tf32): MN-major tf32 needs
  // the 32B-atom swizzle, so warp 3 stages V^T (K-major, SWIZZLE_128B) instead.
  // P is rounded to bf16 (P <= 2^8 by the lazy rescale) and V is the bitwise bf16 copy in the group
  // buffers: P.V is kind::f16 with bf16 x bf16, V the MN-major B operand (reading R13).
  static constexpr uint32_t IDESC_PV = F32 ? idesc_make(FMT, 128, D, 0, 0) : idesc_make2(1, 1, 128, D, 0, 1);
  // (a_fmt = f16 against b_fmt = bf16 - fp16 P with the bf16 V - is an illegal instruction on
  // sm_100a: kind::f16 needs both operands of one type, profiles/r03a)
  static constexpr int VT_ATOM_BYTES = D * 128;       // fp32 V^T: D rows x 32 keys
  static constexpr uint32_t TM_S0 = 0, TM_S1 = 128, TM_O0 = 256, TM_O1 = 384;
  // warps 0..ROLE-1: TMA producer, MMA issuer, Q gather (+ V^T staging for fp32); then two softmax
  // warpgroups of 4 warps.  A softmax warp may only touch TMEM lane quarter (warp % 4), and warps
  // ROLE..ROLE+3 / ROLE+4..ROLE+7 each cover all four quarters.  Fewer role warps leave more
  // registers per thread (65536 / THREADS) for the 128-column score row.
  static constexpr int ROLE = 4;
  static constexpr int THREADS = 32 * (ROLE + 8);
  static constexpr int REG_ROLE = 56, REG_SOFTMAX = 216;
  // setmaxnreg.inc blocks until the CTA's pool holds the registers: the pool is the launch
  // allocation (65536 / THREADS rounded down to 8 per thread = 168), not the register file
  static_assert(128 * REG_ROLE + 256 * REG_SOFTMAX <= (65536 / (32 * (ROLE + 8)) / 8 * 8) * 32 * (ROLE + 8),
                "setmaxnreg budget exceeds the launch allocation (the increase would never complete)");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// S/P regions b = 0/1 complete per half-tile: SF[b][h] (S columns 64h..64h+63 landed), PHALF[b]
// (P for keys 0..63 written), PFULL[b] (P for keys 64..127 written).  PVH[X] (pair units): the
// first half of P.V into O slot X landed.  Committed every tile, waited only by a rare mid-tile
// rescale (compute-sanitizer synccheck reports its unwaited phases; the waiter computes the parity
// of the phase it needs, which cannot be overtaken: PV(j+1) needs this warpgroup's P(j+1)).
enum BarId {
  B_QFULL = 0, B_QFREE, B_KFULL0, B_KFREE0 = B_KFULL0 + 2, B_VFULL0 = B_KFREE0 + 2, B_VFREE0 = B_VFULL0 + 3,
  B_SF00 = B_VFREE0 + 3, B_SF01, B_SF10, B_SF11, B_PHALF0, B_PHALF1, B_PFULL0, B_PFULL1, B_PVH0, B_PVH1,
  B_OFULL0, B_OFULL1, B_OFREE0, B_OFREE1, B_EFULL0, B_EFREE0 = B_EFULL0 + 4, B_UFULL0 = B_EFREE0 + 4,
  B_UFREE0 = B_UFULL0 + 8, B_COUNT = B_UFREE0 + 8
};

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int N>
__device__ __forceinline__ void reg_dealloc() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
__device__ __forceinline__ void reg_alloc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }

// Makes the compiler treat r[] as produced after the preceding tcgen05.wait::ld.
template <int N>
__device__ __forceinline__ void reg_fence(uint32_t (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}

struct Unit {
  pi_work wk;
  int kvh;
  int head0;   // Q head of tile A (tile B = head0 + 1); decode rows add their h_sub
  bool has_b;
};

// Dynamic LPT schedule: units are sorted by cost (descending); CTA b starts with unit b and then
// takes the next unsorted unit from one global counter whenever its producer warp starts a unit
// (list scheduling of an LPT-sorted list: within ~1-8 % of the mean per-CTA load even when a KV-head
// shard leaves only ~6 units per CTA, where a static snake order left up to 53 %).  The producer
// publishes the sequence through an 8-deep smem ring (full / free mbarriers) that every other role
// warp reads in order; -1 ends it.
constexpr int kUnitRing = 8;
constexpr int kUnitConsumers = 11;   // MMA issuer, Q gather, warp 3, 8 softmax warps (one arrive each)

__device__ __forceinline__ int ring_get(const int* ring, uint64_t* bar, int k) {
  mbar_wait(&bar[B_UFULL0 + (k & (kUnitRing - 1))], (k / kUnitRing) & 1);
  return ring[k & (kUnitRing - 1)];
}
__device__ __forceinline__ void ring_release(uint64_t* bar, int k, int lane) {
  if (lane == 0) mbar_arrive(&bar[B_UFREE0 + (k & (kUnitRing - 1))]);
}

// Unit w: prefill units first (each list is sorted by cost, descending), then decode units, so
// the cheap decode units fill the tail of the one persistent launch (NEXT-3).
// UK (unit kinds a kernel instance handles): 1 = pair units only (prefill launch, even r),
// 2 = single-tile units only (decode launch, fp32 operands), 3 = both.  With one kind the
// compiler drops the other kind's code from every role loop.
// Lane-sliced single-tile units.  A decode unit of r rows (one request's GQA group: 4 for
// Llama-3-8B) leaves 124 of 128 TMEM lanes idle, and only the two softmax warps owning lane quarter
// 0 would work: each exponentiates 64 columns per tile while the other six wait, so short units are
// bound by that one warp's latency (profiles/r02k/decode_cfg4_trace.md).  With <= kSliceRows rows
// the Q gather replicates the rows into all four lane quarters (lanes 32q + i, q = 0..3), so every
// quarter computes the same S rows, and warp (X, q) takes only keys [64X + 16q, 64X + 16q + 16) of
// every tile: its own running max / sums and P (zero outside its 16 keys) into O_X at its lanes.
// The eight partials of a row (2 key halves x 4 quarters) are LSE-merged in the epilogue exactly
// as the two split-K halves are (reading R10), the quarters summed in a fixed order through smem.
constexpr int kSliceRows = PI_SLICE_ROWS;
constexpr int kSliceFast = 8;   // sliced units of <= 8 rows: one-barrier epilogue (8 raw partials in smem)
static_assert(kSliceRows % 8 == 0 && kSliceRows <= 32, "sliced rows fit one lane quarter, 8 per store pass");
template <int UK, bool F32>
__device__ __forceinline__ bool unit_sliced(const Unit& u) {
  return PI_DEC_SLICE && (UK & 2) && !F32 && !u.has_b && u.wk.row_count <= kSliceRows;
}

template <int UK>
__device__ __forceinline__ Unit get_unit(const AttnParams& p, int w) {
  Unit u;
  if (w >= p.total_p) {
    w -= p.total_p;
    u.wk = p.work_d[w / p.units_d];
    const int k = w % p.units_d;
    u.kvh = k;
    u.head0 = k * p.r;
    u.has_b = false;
  } else {
    u.wk = p.work_p[w / p.units_p];
    const int k = w % p.units_p;
    const int tpu = p.tiles_per_unit;
    const int pairs = (p.r + tpu - 1) / tpu;
    u.kvh = k / pairs;
    const int hp = k % pairs;
    u.head0 = u.kvh * p.r + tpu * hp;
    u.has_b = tpu == 2 && 2 * hp + 1 < p.r;
  }
  if (UK == 1) u.has_b = true;
  if (UK == 2) u.has_b = false;
  PI_CHECK(u.wk.row_count >= 1 && u.wk.row_count <= 128 && u.wk.span_count >= 1 && u.wk.n_ktiles >= 1, 1);
  PI_CHECK(u.head0 >= 0 && u.head0 + (u.has_b ? 1 : 0) < p.hq_count, 2);
  return u;
}

template <int D, bool F32, int UK>
__global__ void __launch_bounds__(AttnCfg<D, F32, UK>::THREADS, 1)
    packed_attention_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmK,
                            const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmQ,
                            const __grid_constant__ CUtensorMap tmQB) {
  using C = AttnCfg<D, F32, UK>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + 8 * B_COUNT);
  int* uring = reinterpret_cast<int*>(smem + C::OFF_BAR + 8 * B_COUNT + 16);   // unit ring (kUnitRing)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (PI_TRACE && threadIdx.x == 0) trace_cta(p, 0, globaltimer());
  if (threadIdx.x == 0) {
    mbar_init(&bar[B_QFULL], 1);
    mbar_init(&bar[B_QFREE], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar[B_KFULL0 + s], 1);
      mbar_init(&bar[B_KFREE0 + s], 1);
      mbar_init(&bar[B_SF00 + 2 * s], 1);
      mbar_init(&bar[B_SF00 + 2 * s + 1], 1);
      mbar_init(&bar[B_PHALF0 + s], 128);
      mbar_init(&bar[B_PFULL0 + s], 128);
      mbar_init(&bar[B_PVH0 + s], 1);
      mbar_init(&bar[B_OFULL0 + s], 1);
      mbar_init(&bar[B_OFREE0 + s], 128);
    }
    for (int s = 0; s < 3; ++s) {   // V stages (up to 3)
      mbar_init(&bar[B_VFULL0 + s], F32 ? 32 : 1);
      mbar_init(&bar[B_VFREE0 + s], 1);
    }
    for (int s = 0; s < kUnitRing; ++s) {   // unit ring: producer -> every consumer warp
      mbar_init(&bar[B_UFULL0 + s], 1);
      mbar_init(&bar[B_UFREE0 + s], kUnitConsumers);
    }
    for (int s = 0; s < 4; ++s) {   // merge hand-off ring (4 deep)
      mbar_init(&bar[B_EFULL0 + s], 256);   // all softmax threads stored a single unit's partials
      mbar_init(&bar[B_EFREE0 + s], 1);     // the merge warp took them
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmQB);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // launched as a programmatic dependent of the previous kernel on the stream (relayout, or the
  // previous step's merge): the set-up above overlapped its tail; nothing it writes is read or
  // written before this point
  if (p.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int total = p.total_p + p.n_work_d * p.units_d;
  // Register budget per warpgroup (setmaxnreg, at the top of each role's branch): the role warps
  // need few registers, the softmax warps hold a whole 128-column S row.

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    reg_dealloc<C::REG_ROLE>();
    // The whole warp walks the schedule (uniform values); one elected lane issues each copy.
    uint32_t t = 0;
    // next unit's work item + first span loaded one unit ahead (as in the softmax warps)
    // publish unit k of this CTA into the ring (waits until every consumer read slot k - ring)
    auto ring_put = [&](int k, int wv) {
      mbar_wait(&bar[B_UFREE0 + (k & (kUnitRing - 1))], ((k / kUnitRing) & 1) ^ 1);
      if (lane == 0) {
        uring[k & (kUnitRing - 1)] = wv;
        mbar_arrive(&bar[B_UFULL0 + (k & (kUnitRing - 1))]);
      }
      __syncwarp();
    };
    int w = blockIdx.x;   // grid <= total units
    ring_put(0, w);
    Unit nu = get_unit<UK>(p, w);
    pi_span nsp = p.spans[nu.wk.span_begin];
    for (int k = 0; w >= 0; ++k) {
      const Unit u = nu;
      const pi_span span0 = nsp;
      int wn = 0;
      if (PI_DYN_SCHED) {
        if (lane == 0) wn = (int)atomicAdd(p.sched, 1u) + (int)gridDim.x;
        wn = __shfl_sync(0xffffffffu, wn, 0);
      } else {   // A/B: static "snake" order (round k: k G + b, or k G + G - 1 - b on odd rounds)
        const int r = k + 1;
        wn = r * (int)gridDim.x + ((r & 1) ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x);
      }
      if (wn >= total) wn = -1;
      // no unit left to start here: a programmatic dependent launch may take the SMs that free up
      if (wn < 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      ring_put(k + 1, wn);
      if (wn >= 0) {
        nu = get_unit<UK>(p, wn);
        nsp = p.spans[nu.wk.span_begin];
      }
      for (int s = 0; s < u.wk.span_count; ++s) {
        const pi_span sp = s == 0 ? span0 : p.spans[u.wk.span_begin + s];
        PI_CHECK(sp.begin >= 0 && sp.len >= 0 && (p.block_table != nullptr || sp.begin + sp.len <= p.buffer_tokens), 3);
        for (int k0 = sp.begin; k0 < sp.begin + sp.len; k0 += 128, ++t) {
          const int st = t % C::NSK, sv = t % C::NSV;
          const uint32_t ph = (t / C::NSK) & 1, phv = (t / C::NSV) & 1;
          // coordinates: buffers (d, token, kv head); paged cache (d, kv head, page slot)
          int c1 = k0, c2 = u.kvh;
          if (p.block_table != nullptr) {
            c1 = p.kv_head0 + u.kvh;
            c2 = paged_token(p, u.wk.reserved, k0);
          }
          if (lane == 0) trace_ev(p, t, 24);
          mbar_wait(&bar[B_KFREE0 + st], ph ^ 1);
          if (lane == 0) trace_ev(p, t, 25);
          if (elect_one()) {
            mbar_arrive_expect_tx(&bar[B_KFULL0 + st], C::TILE_BYTES);
#pragma unroll
            for (int a = 0; a < C::ATOMS; ++a)
              tma_load_3d(smem + C::OFF_K + st * C::TILE_BYTES + a * C::ATOM_BYTES, &tmK, &bar[B_KFULL0 + st],
                          a * C::ATOM_ELEMS, c1, c2);
          }
          __syncwarp();
          if constexpr (!F32) {
            mbar_wait(&bar[B_VFREE0 + sv], phv ^ 1);
            if (lane == 0) trace_ev(p, t, 26);
            if (elect_one()) {
              mbar_arrive_expect_tx(&bar[B_VFULL0 + sv], C::TILE_BYTES);
#pragma unroll
              for (int a = 0; a < C::ATOMS; ++a)
                tma_load_3d(smem + C::OFF_V + sv * C::TILE_BYTES + a * C::ATOM_BYTES, &tmV, &bar[B_VFULL0 + sv],
                            a * C::ATOM_ELEMS, c1, c2);
            }
            __syncwarp();
          }
        }
      }
      w = wn;
      if (PI_TRACE && lane == 0) trace_cta(p, 2, (unsigned long long)(k + 1));   // units taken
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    reg_dealloc<C::REG_ROLE>();
    // The whole warp walks the schedule with warp-uniform values (uniform registers); each batch of
    // tcgen05.mma / commit is issued by one elected lane (no per-MMA waterfall loops).
    {
      uint32_t t = 0, item = 0;
      // completions so far of SFULL/PFULL of region 0 / 1 and of OFULL/OFREE (both slots alike).
      // Scalars, not arrays: a runtime region index would put an array in local memory
      uint32_t cntA = 0, cntB = 0, ix = 0;
      auto cnt = [&](int x) { return x ? cntB : cntA; };
      // Descriptors are built once; each k-step adds a compile-time offset to the 14-bit start
      // address field (all smem offsets < 256 KB, so the field never carries).
      const uint64_t dq = sdesc_sw128(sbase + C::OFF_Q, 16, 1024);
      const uint64_t dk = sdesc_sw128(sbase + C::OFF_K, 16, 1024);
      const uint64_t dv = F32 ? sdesc_sw128(sbase + C::OFF_V, 16, 1024)
                              : sdesc_sw128(sbase + C::OFF_V, C::ATOM_BYTES, 1024);
      constexpr uint64_t TILE16 = C::TILE_BYTES >> 4;
      // S(X) = Q_X K(tt)^T into S/P region b, as two N = 64 halves (keys 0..63 / 64..127) so the
      // softmax can start on the first half while the second is computed.
      auto issue_s = [&](int X, int b, uint32_t tt, bool s128) {
        const uint64_t aq = dq + X * TILE16;
        const uint64_t bk = dk + (tt % C::NSK) * TILE16;
        const uint32_t d_tmem = tmem + (b ? C::TM_S1 : C::TM_S0);
        if (elect_one()) {
          if (s128) {
            // one N = 128 chain (an N = 64 SS MMA is shared-memory-port bound: two halves cost
            // 768 instead of 512 cycles); both halves' barriers complete with it
#pragma unroll
            for (int kk = 0; kk < C::QK_STEPS; ++kk) {
              const uint64_t off = (uint64_t)(((kk >> 2) * C::ATOM_BYTES + (kk & 3) * 32) >> 4);
              mma_ss<F32>(d_tmem, aq + off, bk + off, C::IDESC_QK128, kk > 0 ? 1u : 0u);
            }
            mma_commit(&bar[B_SF00 + 2 * b]);
            mma_commit(&bar[B_SF00 + 2 * b + 1]);
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
              for (int kk = 0; kk < C::QK_STEPS; ++kk) {
                const uint64_t off = (uint64_t)(((kk >> 2) * C::ATOM_BYTES + (kk & 3) * 32) >> 4);
                mma_ss<F32>(d_tmem + h * 64, aq + off, bk + off + h * (8192 >> 4), C::IDESC_QK, kk > 0 ? 1u : 0u);
              }
              mma_commit(&bar[B_SF00 + 2 * b + h]);
            }
          }
        }
        __syncwarp();
      };
      // S(X) = Q_X K(tt)^T as one N = 128 chain into S/P region X; commits SF[X][0]
      auto issue_s_full = [&](int X, uint32_t tt) {
        const uint64_t aq = dq + X * TILE16;
        const uint64_t bk = dk + (tt % C::NSK) * TILE16;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < C::QK_STEPS; ++kk) {
            const uint64_t off = (uint64_t)(((kk >> 2) * C::ATOM_BYTES + (kk & 3) * 32) >> 4);
            mma_ss<F32>(tmem + (X ? C::TM_S1 : C::TM_S0), aq + off, bk + off, C::IDESC_QK128, kk > 0 ? 1u : 0u);
          }
          mma_commit(&bar[B_SF00 + 2 * X]);
        }
        __syncwarp();
      };
      auto commit = [&](int id) {
        if (elect_one()) mma_commit(&bar[id]);
        __syncwarp();
      };
      // O_X += P_h V(tt)[keys 64h .. 64h+63]; P_h (this half's P) starts at TMEM column p_col;
      // first: overwrite O_X instead of accumulating
      auto issue_pv = [&](int X, uint32_t p_col, uint32_t tt, bool first, int h) {
        const uint64_t bv = dv + (tt % C::NSV) * TILE16;
        const uint32_t p_tmem = tmem + p_col;
        const uint32_t d_tmem = tmem + (X ? C::TM_O1 : C::TM_O0);
        if (elect_one()) {
#pragma unroll
          for (int q = 0; q < C::PV_STEPS / 2; ++q) {
            const int kk = h * (C::PV_STEPS / 2) + q;
            const uint64_t off = F32 ? (uint64_t)(((kk >> 2) * C::VT_ATOM_BYTES + (kk & 3) * 32) >> 4)
                                     : (uint64_t)((kk * C::KEYS_PER_PV_STEP * 128) >> 4);
            mma_ts<F32>(d_tmem, p_tmem + q * 8, bv + off, C::IDESC_PV, (first && q == 0) ? 0u : 1u);
          }
        }
        __syncwarp();
      };
      int w = ring_get(uring, bar, 0);
      Unit nu = get_unit<UK>(p, w);
      for (int k = 0; w >= 0; ++k) {
        const Unit u = nu;   // loaded one unit ahead
        const int wn = ring_get(uring, bar, k + 1);
        ring_release(bar, k, lane);
        if (wn >= 0) nu = get_unit<UK>(p, wn);
        const int n = u.wk.n_ktiles;
        trace_unit(p, item, 0);
        mbar_wait(&bar[B_QFULL], item & 1);
        trace_unit(p, item, 1);
        mbar_wait(&bar[B_KFULL0 + (t % C::NSK)], (t / C::NSK) & 1);
        trace_unit(p, item, 2);
        tc_fence_after();
        if (u.has_b) {
          // ---- pair unit: slot X keeps S/P region X; ping-pong between the two tiles.  S is one
          // N = 128 chain (an N = 64 SS MMA is bound by the 128 B/clk shared-memory port: 48 instead
          // of 32 cycles), P overwrites S's first 64 columns, S(j+1) follows P(j).V in the in-order pipe.
          issue_s_full(0, t);
          issue_s_full(1, t);
          commit(B_KFREE0 + (t % C::NSK));
          if (n == 1) commit(B_QFREE);
          for (int j = 0; j < n; ++j) {
            const uint32_t tt = t + j;
            for (int X = 0; X < 2; ++X) {
              trace_ev(p, tt, 0 + 3 * X);
              mbar_wait(&bar[B_PHALF0 + X], (cnt(X) + j) & 1);
              trace_ev(p, tt, 1 + 3 * X);
              if (X == 0) mbar_wait(&bar[B_VFULL0 + (tt % C::NSV)], (tt / C::NSV) & 1);
              if (j == 0) mbar_wait(&bar[B_OFREE0 + X], (ix & 1) ^ 1);
              tc_fence_after();
              issue_pv(X, X ? C::TM_S1 : C::TM_S0, tt, j == 0, 0);
              commit(B_PVH0 + X);
              mbar_wait(&bar[B_PFULL0 + X], (cnt(X) + j) & 1);
              tc_fence_after();
              issue_pv(X, (X ? C::TM_S1 : C::TM_S0) + 32, tt, false, 1);
              trace_ev(p, tt, 14 + X);
              if (X == 1) commit(B_VFREE0 + (tt % C::NSV));
              if (j == n - 1) {
                commit(B_OFULL0 + X);
              } else {
                if (X == 0) {
                  mbar_wait(&bar[B_KFULL0 + ((tt + 1) % C::NSK)], ((tt + 1) / C::NSK) & 1);
                  tc_fence_after();
                  trace_ev(p, tt, 27);   // pair units: K(j+1) landed as seen by the issuer
                }
                issue_s_full(X, tt + 1);
                trace_ev(p, tt, 2 + 3 * X);
                if (X == 1) {
                  commit(B_KFREE0 + ((tt + 1) % C::NSK));
                  if (j + 1 == n - 1) commit(B_QFREE);
                }
              }
            }
          }
          cntA += n;
          cntB += n;
          ix += 1;
        } else {
          // ---- single-tile unit: S/P regions alternate per tile so S(j+1) overlaps softmax(j)
          const bool s128_pro = PI_SINGLE_S128 == 1 || PI_SINGLE_S128 == 2 || (PI_SINGLE_S128 == 3 && n <= 4);
          const bool s128_body = PI_SINGLE_S128 == 1 || (PI_SINGLE_S128 == 3 && n <= 4);
          issue_s(0, 0, t, s128_pro);
          trace_ev(p, t, 27);
          commit(B_KFREE0 + (t % C::NSK));
          if (n > 1) {
            mbar_wait(&bar[B_KFULL0 + ((t + 1) % C::NSK)], ((t + 1) / C::NSK) & 1);
            tc_fence_after();
            issue_s(0, 1, t + 1, s128_pro);
            trace_ev(p, t + 1, 27);
            commit(B_KFREE0 + ((t + 1) % C::NSK));
          }
          if (n <= 2) commit(B_QFREE);
          for (int j = 0; j < n; ++j) {
            const uint32_t tt = t + j;
            const int b = j & 1;
            trace_ev(p, tt, 0);
            mbar_wait(&bar[B_PHALF0 + b], (cnt(b) + (j >> 1)) & 1);
            trace_ev(p, tt, 1);
            mbar_wait(&bar[B_VFULL0 + (tt % C::NSV)], (tt / C::NSV) & 1);
            trace_ev(p, tt, 28);
            if (j == 0) {
              mbar_wait(&bar[B_OFREE0], (ix & 1) ^ 1);
              mbar_wait(&bar[B_OFREE1], (ix & 1) ^ 1);
            }
            trace_ev(p, tt, 29);
            tc_fence_after();
            // split-K inside the CTA: keys 0..63 of every tile -> O_0 (softmax warpgroup A),
            // keys 64..127 -> O_1 (warpgroup B); the epilogue merges the two (LSE)
            issue_pv(0, b ? C::TM_S1 : C::TM_S0, tt, j == 0, 0);
            mbar_wait(&bar[B_PFULL0 + b], (cnt(b) + (j >> 1)) & 1);
            tc_fence_after();
            issue_pv(1, (b ? C::TM_S1 : C::TM_S0) + C::P1_SINGLE, tt, j == 0, 1);
            commit(B_VFREE0 + (tt % C::NSV));
            if (j == n - 1) {
              commit(B_OFULL0);
              commit(B_OFULL1);
            }
            if (j + 2 < n) {
              mbar_wait(&bar[B_KFULL0 + ((tt + 2) % C::NSK)], ((tt + 2) / C::NSK) & 1);
              tc_fence_after();
              issue_s(0, b, tt + 2, s128_body);
              trace_ev(p, tt + 2, 27);
              commit(B_KFREE0 + ((tt + 2) % C::NSK));
              if (j + 2 == n - 1) commit(B_QFREE);
            }
          }
          cntA += (n + 1) >> 1;
          cntB += n >> 1;
          ix += 1;
        }
        trace_unit(p, item, 3);
        t += n;
        ++item;
        w = wn;
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ------------------------------------------------------------------ Q gather (TMA tile::gather4)
    reg_dealloc<C::REG_ROLE>();
    // Q rows are addressed through the plan's row table: lane g gathers rows 4g..4g+3 of each tile
    // (one gather4 per 128-byte atom column) straight into the SWIZZLE_128B K-major operand layout.
    uint32_t item = 0;
    for (int k = 0, w = ring_get(uring, bar, 0); w >= 0; ++k, w = ring_get(uring, bar, k)) {
      ring_release(bar, k, lane);
      const Unit u = get_unit<UK>(p, w);
      const int nt = u.has_b ? 2 : 1;
      trace_unit(p, item, 4);
      mbar_wait(&bar[B_QFREE], (item & 1) ^ 1);
      trace_unit(p, item, 5);
      const int rows = u.wk.row_count;
      // lane-sliced units: the rows again at the start of every lane quarter (row groups 8q + g)
      const bool sl = unit_sliced<UK, F32>(u);
      const int gpq = (rows + 3) >> 2;
      const int groups = sl ? 4 * gpq : gpq;
      const int gi = sl ? lane % gpq : lane;
      int32_t ri[4];
      bool run = true;   // this lane's rows are tokens tok0 + row index (one contiguous run of Q)
      int tok0 = 0;
      {
        const int32_t t0 = p.rows[u.wk.row_begin].q_token;
        tok0 = t0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const pi_row row = p.rows[u.wk.row_begin + min(4 * gi + e, rows - 1)];
          ri[e] = row.q_token * p.q_heads_stride + u.head0 + (row.out & 15);
          if (lane < groups && 4 * gi + e < rows) run = run && row.q_token == t0 + 4 * gi + e && (row.out & 15) == 0;
          PI_CHECK(row.q_token >= 0 && row.q_token < p.total_q && u.head0 + (row.out & 15) + (nt - 1) < p.hq_count, 5);
        }
      }
      // A tile whose rows are consecutive tokens of Q (a long request's 128 query positions, or
      // adjacent short ones) is ONE 3D box per 128-byte atom column (tmQB: d x head x token, 128
      // tokens; rows past the tile's row_count are computed and discarded, past the end of Q
      // zero-filled); other tiles gather 4 rows per TMA op.  A gather4 op takes ~120 issue cycles,
      // so a 2-tile gather (128 ops) kept the next unit's S waiting ~8k cycles at every unit start.
      const bool box = PI_Q_BOX && !sl && __all_sync(0xffffffffu, run);
      if (lane == 0)
        mbar_arrive_expect_tx(&bar[B_QFULL], box ? (uint32_t)(nt * C::TILE_BYTES) : (uint32_t)(nt * groups * C::ATOMS * 512));
      __syncwarp();
      if (box) {
        if (lane == 0) {
          for (int X = 0; X < nt; ++X)
#pragma unroll
            for (int a = 0; a < C::ATOMS; ++a)
              tma_load_3d(smem + C::OFF_Q + X * C::TILE_BYTES + a * C::ATOM_BYTES, &tmQB, &bar[B_QFULL],
                          a * C::ATOM_ELEMS, u.head0 + X, tok0);
        }
      } else if (lane < groups) {
        const int dst_group = sl ? 8 * (lane / gpq) + gi : lane;
        for (int X = 0; X < nt; ++X) {
          uint8_t* dst = smem + C::OFF_Q + X * C::TILE_BYTES + dst_group * 512;
#pragma unroll
          for (int a = 0; a < C::ATOMS; ++a)
            tma_gather4(dst + a * C::ATOM_BYTES, &tmQ, &bar[B_QFULL], a * C::ATOM_ELEMS, ri[0] + X, ri[1] + X,
                        ri[2] + X, ri[3] + X);
        }
      }
      if (lane == 0) trace_unit(p, item, 6);
      ++item;
    }
  } else if (warp < C::ROLE) {
    // ------------------------------------------------------------------ warp 3
    reg_dealloc<C::REG_ROLE>();
    if (!F32 && (UK & 2) && PI_MERGE_WARP && p.merge_ctr != nullptr) {
      // bf16: in-kernel LSE merge of split rows (packinfer_attention_merge; reading R10), off the
      // softmax warps' path.  Per single-tile unit, after the softmax threads have stored its
      // partials (EFULL ring), each lane takes rows of the unit with a partial slot and adds one
      // to the (merge row, head) counter with acq_rel at GPU scope: CTA-scope acquire of the
      // stores + the release of the atomic make them visible with it (cumulativity, as in a
      // barrier-then-release split-K semaphore).  The lane completing the count owns the merge:
      // the whole warp then merges it with lanes over channels - packinfer_merge's arithmetic in
      // the same order, so outputs are bitwise equal to the separate merge - and re-zeroes the
      // counter for the next launch.
      uint32_t epi = 0;
      for (int k = 0, w = ring_get(uring, bar, 0); w >= 0; ++k, w = ring_get(uring, bar, k)) {
        ring_release(bar, k, lane);
        const Unit u = get_unit<UK>(p, w);
        if (u.has_b) continue;
        const uint32_t e = epi & 3;
        mbar_wait(&bar[B_EFULL0 + e], (epi >> 2) & 1);
        if (PI_MERGE_ATOM == 2) __threadfence();
        for (int r0 = 0; r0 < u.wk.row_count; r0 += 32) {
          const int rr = r0 + lane;
          int mm = -1, head = 0, qtok = 0;
          if (rr < u.wk.row_count) {
            const pi_row row = p.rows[u.wk.row_begin + rr];
            const int slot = (row.out >> 4) - 1;
            if (slot >= 0 && (PI_MERGE_WARP == 1 || PI_MERGE_WARP == 3)) {
              const int m = p.slot_merge[slot];
              head = u.head0 + (row.out & 15);
              qtok = row.q_token;
              uint32_t* ctr = p.merge_ctr + (int64_t)m * p.hq_count + head;
              uint32_t old;
              if (PI_MERGE_ATOM == 0)
                asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
              else if (PI_MERGE_ATOM == 1)
                asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
              else
                asm volatile("atom.add.relaxed.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
              if (old + 1u == (uint32_t)p.merges[m].slot_count) {
                *ctr = 0u;
                mm = PI_MERGE_WARP == 3 ? -1 : m;   // 3: A/B, counters only
              }
            }
          }
          uint32_t todo = __ballot_sync(0xffffffffu, mm >= 0);
          while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int m = __shfl_sync(0xffffffffu, mm, src);
            const int h = __shfl_sync(0xffffffffu, head, src);
            const pi_merge mg = p.merges[m];
            float M = NEG_INF_F;
            for (int bb = lane; bb < mg.slot_count; bb += 32)
              M = fmaxf(M, __ldcg(&p.partial_lse[(int64_t)(mg.slot_begin + bb) * p.hq_count + h]));
#pragma unroll
            for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            constexpr int V = D / 32;
            float acc[V];
#pragma unroll
            for (int i = 0; i < V; ++i) acc[i] = 0.f;
            float W = 0.f;
            if (M != NEG_INF_F) {
              // slots in batches of MB: every load of a batch is in flight at once (a long split
              // row has up to 32 slots), then the batch is accumulated in slot order
              constexpr int MB = 4;
              for (int b0 = 0; b0 < mg.slot_count; b0 += MB) {
                float lw[MB], x[MB][V];
#pragma unroll
                for (int q = 0; q < MB; ++q) {
                  if (b0 + q < mg.slot_count) {
                    const int64_t sl = mg.slot_begin + b0 + q;
                    lw[q] = __ldcg(&p.partial_lse[sl * p.hq_count + h]);
                    const float* srcp = p.partial_o + (sl * p.hq_count + h) * D;
#pragma unroll
                    for (int i = 0; i < V; ++i) x[q][i] = __ldcg(srcp + lane + 32 * i);
                  }
                }
#pragma unroll
                for (int q = 0; q < MB; ++q) {
                  if (b0 + q < mg.slot_count) {
                    const float wgt = expf(lw[q] - M);
                    W += wgt;
#pragma unroll
                    for (int i = 0; i < V; ++i) acc[i] += wgt * x[q][i];
                  }
                }
              }
            }
            const float inv = W > 0.f ? 1.f / W : 0.f;
            const int64_t o_el = (int64_t)mg.q_token * p.out_row_stride + (int64_t)h * D;
            if (p.out_f32) {
#pragma unroll
              for (int i = 0; i < V; ++i) reinterpret_cast<float*>(p.out)[o_el + lane + 32 * i] = acc[i] * inv;
            } else {
#pragma unroll
              for (int i = 0; i < V; ++i)
                reinterpret_cast<__nv_bfloat16*>(p.out)[o_el + lane + 32 * i] = __float2bfloat16_rn(acc[i] * inv);
            }
            if (p.lse && lane == 0) p.lse[(int64_t)h * p.total_q + mg.q_token] = W > 0.f ? M + logf(W) : NEG_INF_F;
            (void)qtok;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar[B_EFREE0 + e]);
        ++epi;
      }
    }
    else if constexpr (F32) {
      uint32_t t = 0;
      for (int k = 0, w = ring_get(uring, bar, 0); w >= 0; ++k, w = ring_get(uring, bar, k)) {
        ring_release(bar, k, lane);
        const Unit u = get_unit<UK>(p, w);
        const float* vsrc = reinterpret_cast<const float*>(p.v_buf) + (int64_t)u.kvh * p.buffer_tokens * D;
        for (int s = 0; s < u.wk.span_count; ++s) {
          const pi_span sp = p.spans[u.wk.span_begin + s];
          for (int k0 = sp.begin; k0 < sp.begin + sp.len; k0 += 128, ++t) {
            const int st = t % C::NSV;
            mbar_wait(&bar[B_VFREE0 + st], ((t / C::NSV) & 1) ^ 1);
            uint8_t* vt = smem + C::OFF_V + st * C::TILE_BYTES;
            for (int idx = lane; idx < 128 * (D / 4); idx += 32) {
              const int key = idx / (D / 4), c4 = idx % (D / 4);
              float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
              if (k0 + key < p.buffer_tokens)
                v = *reinterpret_cast<const float4*>(vsrc + (int64_t)(k0 + key) * D + c4 * 4);
              const float ve[4] = {v.x, v.y, v.z, v.w};
              const int a = key >> 5, jj = (key & 31) >> 2, wb = (key & 3) * 4;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int dch = c4 * 4 + e;
                *reinterpret_cast<float*>(vt + a * C::VT_ATOM_BYTES + dch * 128 + ((jj ^ (dch & 7)) << 4) + wb) =
                    ve[e];
              }
            }
            fence_proxy_async_smem();
            mbar_arrive(&bar[B_VFULL0 + st]);
          }
        }
      }
    } else {
      // nothing to do for this launch: still consume the unit ring (one reader per slot expected)
      for (int k = 0, w = ring_get(uring, bar, 0); w >= 0; ++k, w = ring_get(uring, bar, k)) ring_release(bar, k, lane);
    }
  } else {
    // ------------------------------------------------------------------ softmax / epilogue
    reg_alloc<C::REG_SOFTMAX>();
    const int X = (warp - C::ROLE) >> 2;   // tile slot: 0 = A, 1 = B
    const int wq = warp & 3;               // the TMEM lane quarter this warp may access
    const int row_id = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t o_tm = tmem + lane_base + (X ? C::TM_O1 : C::TM_O0);
    // completions so far of SF[b][0] / P of region b (scalars: see the MMA issuer)
    uint32_t cntA = 0, cntB = 0, ix = 0, t = 0;
    auto cnt = [&](int x) { return x ? cntB : cntA; };
    // completions so far of SF[b][1] (S half 1 of region b): only single-tile units compute S in
    // two halves; pair units' one N = 128 chain completes SF[X][0] alone
    uint32_t cnt1A = 0, cnt1B = 0;
    auto cnt1 = [&](int x) { return x ? cnt1B : cnt1A; };
    uint32_t pvh = 0;                       // completions so far of PVH[X] (this slot's P.V halves)
    uint32_t epi = 0;                       // units handed to the merge warp so far
    const float NEG_INF = -INFINITY;
    const float sl2 = p.scale_log2;
    // O_X *= alpha, all columns (lazy rescale; rare)
    auto rescale_o = [&](float alpha) {
#pragma unroll
      for (int c4 = 0; c4 < D / 32; ++c4) {
        uint32_t o32[32];
        tmem_ld32(o_tm + c4 * 32, o32);
        tmem_wait_ld();
        reg_fence(o32);
#pragma unroll
        for (int i = 0; i < 32; ++i) o32[i] = __float_as_uint(__uint_as_float(o32[i]) * alpha);
        tmem_st32(o_tm + c4 * 32, o32);
      }
    };
    // The next unit's descriptor (work item, this thread's row, first key span) is loaded one unit
    // ahead: its global-load latency (~2 dependent L2 round trips) hides behind the current unit
    // instead of opening every unit (a 1-tile decode unit is otherwise mostly that latency).
    Unit nu;
    pi_row nrow = {0, 0, 0, 0};
    pi_span nsp = {0, 0};
    auto prefetch = [&](int wn) {
      nu = get_unit<UK>(p, wn);
      const int ri = unit_sliced<UK, F32>(nu) ? lane : row_id;   // sliced: row `lane` in every quarter
      nrow = ri < nu.wk.row_count ? p.rows[nu.wk.row_begin + ri] : pi_row{0, 0, 0, 0};
      PI_CHECK(ri >= nu.wk.row_count || (nrow.q_token >= 0 && nrow.q_token < p.total_q && nrow.lo <= nrow.hi &&
                                         (nrow.out >> 4) - 1 < p.n_partial_slots && (nrow.out >> 4) >= 0),
               4);
      nsp = p.spans[nu.wk.span_begin];
    };
    int w = ring_get(uring, bar, 0);
    prefetch(w);
    for (int k = 0; w >= 0; ++k) {
      const Unit u = nu;
      const pi_row row_pf = nrow;
      const pi_span span0 = nsp;
      const int wn = ring_get(uring, bar, k + 1);
      ring_release(bar, k, lane);
      if (wn >= 0) prefetch(wn);
      const pi_work& wk = u.wk;
      const int n = wk.n_ktiles;
      // pair units: warpgroup X owns tile X (both key halves); single-tile units: warpgroup X owns
      // key half X of every tile (split-K inside the CTA, merged in the epilogue)
      const int h_lo = u.has_b ? 0 : X, h_hi = u.has_b ? 2 : X + 1;
      const bool sl = unit_sliced<UK, F32>(u);
      const bool valid = (sl ? lane : row_id) < wk.row_count;
      const bool warp_any = wq * 32 < wk.row_count;
      const pi_row row = row_pf;
      float m_ref = NEG_INF, l = 0.f, lr = 0.f;   // running max (log2 units), exact / rounded-P sums
      uint32_t j = 0;
      if (warp == C::ROLE && lane == 0) trace_unit(p, ix, 7);
      for (int s = 0; s < wk.span_count; ++s) {
        const pi_span sp = s == 0 ? span0 : p.spans[wk.span_begin + s];
        const bool last = (s == wk.span_count - 1);
        const int se = sp.begin + sp.len;
        for (int k0 = sp.begin; k0 < se; k0 += 128, ++j) {
          const int b = u.has_b ? X : (int)(j & 1);          // S/P region of this tile
          const uint32_t kb = u.has_b ? j : (j >> 1);        // use index of region b in this unit
          const uint32_t region = tmem + lane_base + (b ? C::TM_S1 : C::TM_S0);
          // visible key columns of this row in this tile: [c_lo, c_hi).  Rows past row_count take
          // the full-tile path (their results are discarded) so a warp never diverges on them.
          int c_lo = 0, c_hi = 128;
          if (valid) {
            int lo_k = k0, hi_k = min(k0 + 128, se);
            if (last) {
              lo_k = max(lo_k, row.lo);
              hi_k = min(hi_k, row.hi);
            }
            c_lo = lo_k - k0;
            c_hi = hi_k - k0;
          }
          const bool full = (c_lo == 0 && c_hi == 128);
          float ps[4] = {0.f, 0.f, 0.f, 0.f};   // exact row sum of this tile's P (LSE)
          float rs[4] = {0.f, 0.f, 0.f, 0.f};   // row sum of the bf16-rounded P (O normalisation)
          // Streaming single pass over two 64-column halves, each released to the tensor core as
          // soon as it is written: each S element is read from TMEM once; the running max is lazy
          // (updated only when it grows by > 2^8).  A jump in the first half rescales O before any
          // P of this tile is used; a jump in the second half rescales O after the first half's
          // P.V has landed (O then holds it, so one rescale covers both).
          uint32_t r[64];
          auto load_s = [&](uint32_t col) {
            tmem_ld32(col, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
            tmem_ld32(col + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          };
          if (row_id == 0) trace_ev(p, t + j, 6 + 4 * X);
          if (u.has_b || X == 0)
            mbar_wait(&bar[B_SF00 + 2 * b], (cnt(b) + kb) & 1);   // pair units: the whole N = 128 S
          else
            mbar_wait(&bar[B_SF00 + 2 * b + 1], (cnt1(b) + kb) & 1);
          tc_fence_after();
          if (row_id == 0) trace_ev(p, t + j, 7 + 4 * X);
          if (j == 0 && warp == C::ROLE && lane == 0) trace_unit(p, ix, 8);
          if constexpr ((UK & 2) && !F32) {
            if (sl) {
              // lane-sliced unit: this warp's 16 keys [cs, cs + 16) of the tile (unit_sliced())
              const int cs = 64 * X + 16 * wq;
              uint32_t s16[16];
              tmem_ld16(region + cs, s16);
              tmem_wait_ld();
              reg_fence(s16);
              const int lo = max(c_lo - cs, 0), hi = min(c_hi - cs, 16);
              const bool sfull = lo == 0 && hi == 16;
              uint32_t p8[8];
              float e_sum = 0.f, r_sum = 0.f;   // exact / bf16-rounded sums of this slice's P
              // P = exp2(s * scale_log2 + nm) (MUFU), packed bf16 into p8, both row sums
              auto exp16 = [&](float nm) {
                const uint64_t SL2 = f2(sl2, sl2), NM = f2(nm, nm);
                uint64_t acc = f2(0.f, 0.f), racc = f2(0.f, 0.f);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const uint64_t x = f2_fma(f2(__uint_as_float(s16[2 * i]), __uint_as_float(s16[2 * i + 1])), SL2, NM);
                  const uint64_t e = f2(ex2(f2_lo(x)), ex2(f2_hi(x)));
                  acc = f2_add(acc, e);
                  p8[i] = pack_bf16(f2_lo(e), f2_hi(e));
                  uint32_t rl, rh;
                  asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(rl) : "r"(p8[i]));
                  asm("prmt.b32 %0, %1, 0, 0x3244;" : "=r"(rh) : "r"(p8[i]));
                  racc = f2_add(racc, f2(__uint_as_float(rl), __uint_as_float(rh)));
                }
                e_sum = f2_lo(acc) + f2_hi(acc);
                r_sum = f2_lo(racc) + f2_hi(racc);
              };
              bool done = false;
              // speculative slice against the running max, certified by its sum (as above)
              if (__all_sync(0xffffffffu, !valid || (sfull && m_ref != NEG_INF))) {
                exp16(-m_ref);
                done = !__any_sync(0xffffffffu, valid && !(e_sum <= 256.0f));
              }
              if (!done) {
                if (!sfull) {
#pragma unroll
                  for (int i = 0; i < 16; ++i)
                    if (!(i >= lo && i < hi)) s16[i] = __float_as_uint(NEG_INF);
                }
                float mx = NEG_INF;
#pragma unroll
                for (int i = 0; i < 16; ++i) mx = fmaxf(mx, __uint_as_float(s16[i]));
                const float m_new = fmaxf(m_ref, mx * sl2);
                const bool need = valid && (m_ref != NEG_INF) && (m_new > m_ref + 8.0f);
                if (__any_sync(0xffffffffu, need)) {
                  const float alpha = need ? ex2(m_ref - m_new) : 1.0f;
                  if (j > 0) {
                    const uint32_t tp = t + j - 1;   // P.V(j-1) must have landed in O
                    mbar_wait(&bar[B_VFREE0 + (tp % C::NSV)], (tp / C::NSV) & 1);
                    tc_fence_after();
                    rescale_o(alpha);
                  }
                  if (need) {
                    l *= alpha;
                    lr *= alpha;
                    m_ref = m_new;
                  }
                }
                if (m_ref == NEG_INF) m_ref = m_new;
                exp16(m_ref != NEG_INF ? -m_ref : NEG_INF);
              }
              // P of this warpgroup's key half: this warp's 8 packed columns, zeros for the others
              const uint32_t p_base = region + (X ? C::P1_SINGLE : 0u);
              const uint32_t z8[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
              tmem_st8(p_base + 8u * wq, p8);
              tmem_st8(p_base + 8u * ((wq + 1) & 3), z8);
              tmem_st8(p_base + 8u * ((wq + 2) & 3), z8);
              tmem_st8(p_base + 8u * ((wq + 3) & 3), z8);
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(&bar[(X == 0 ? B_PHALF0 : B_PFULL0) + b]);
              if (valid) {
                l += e_sum;
                lr += r_sum;
              }
              continue;
            }
          }
          if (warp_any) {
            load_s(region + 64u * h_lo);
            tmem_wait_ld();
            reg_fence(r);
          }
          if (row_id == 0) trace_ev(p, t + j, 20 + X);
          uint32_t spec_bits = 0;
          // exp2 of the 64 scores in r, packed in place (bf16 pairs into r[0..31]; fp32 stays put)
          // (use_poly: PI_POLY_PAIRS of 8 pairs on the FMA pipe; clamp: x unbounded, see ex2_poly2)
          // The exact fp32 sum of P (acc0/acc1, FADD2) gives the LSE, certifies the speculative half
          // and normalises O (reading R13).  PI_P_ROUNDED_SUM=1 keeps a second sum of the ROUNDED bf16
          // P that P.V multiplies (racc, FHADD.BF16) to normalise O instead: 7 % slower, same error
          // class against the oracle (profiles/r02a/ab_rowsum.txt, ab_precision.txt).
          auto exp_body = [&](auto use_poly, auto clamp, uint64_t SL2, uint64_t NM, uint64_t& acc0, uint64_t& acc1,
                              float (&racc)[4]) {
#if PI_POLY_SAT
            // poly pairs take the argument saturated (ex2_poly_sat): A = scale / 252, B = (125 - m) / 252
            const float PA = f2_lo(SL2) * (1.0f / 252.0f), PB = (f2_lo(NM) + 125.0f) * (1.0f / 252.0f);
#endif
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const uint64_t x = f2_fma(f2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), SL2, NM);
              uint64_t e;
              if (decltype(use_poly)::value && (i & 7) >= 8 - PI_POLY_PAIRS)
#if PI_POLY_SAT
                e = ex2_poly_sat(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]), PA, PB);
#else
                e = ex2_poly2<decltype(clamp)::value>(x);
#endif
              else
                e = f2(ex2(f2_lo(x)), ex2(f2_hi(x)));
              if (i & 1) acc1 = f2_add(acc1, e); else acc0 = f2_add(acc0, e);
              if constexpr (!F32) {
                r[i] = pack_bf16(f2_lo(e), f2_hi(e));     // in place: i <= 2i
                if (PI_P_ROUNDED_SUM == 1) {
                  add_bf16x2(racc[2 * (i & 1)], racc[2 * (i & 1) + 1], r[i]);
                } else if (PI_P_ROUNDED_SUM == 2) {
                  // the two rounded values as fp32 (bf16 = the high half of an fp32) by byte
                  // permutes on the integer pipe, summed by one FADD2
                  uint32_t lo, hi;
                  asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(lo) : "r"(r[i]));
                  asm("prmt.b32 %0, %1, 0, 0x3244;" : "=r"(hi) : "r"(r[i]));
                  const uint64_t sum = f2_add(f2(racc[2 * (i & 1)], racc[2 * (i & 1) + 1]),
                                              f2(__uint_as_float(lo), __uint_as_float(hi)));
                  racc[2 * (i & 1)] = f2_lo(sum);
                  racc[2 * (i & 1) + 1] = f2_hi(sum);
                }
              } else {
                r[2 * i] = __float_as_uint(f2_lo(e));
                r[2 * i + 1] = __float_as_uint(f2_hi(e));
              }
            }
          };
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h < h_lo || h >= h_hi) continue;
            // the first half this warpgroup handles in this tile (single units: its only one)
            const bool first_half = !u.has_b || h == 0;
            // sanitizer build: wait every PVH phase (the production build waits it only before a
            // rare mid-tile rescale, which compute-sanitizer synccheck reports as a missing wait)
            if (PI_SYNCCHECK_PVH && u.has_b && h == 1) {
              mbar_wait(&bar[B_PVH0 + X], (pvh + j) & 1);
              tc_fence_after();
            }
            if (warp_any) {
              // Speculative half (unmasked tiles once the running max is set): exponentiate against
              // m_ref without computing the half's max.  Every P <= 2^8 (the lazy-max invariant)
              // exactly when no score exceeds m_ref + 8, which the half's sum <= 2^8 certifies;
              // otherwise (rare) reload S from TMEM and take the exact path below.
              bool spec_done = false;
              if constexpr (!F32) {
                // warp-uniform, decided by the valid rows only: rows past row_count hold stale Q
                // rows of an earlier unit (their results are discarded) and must not steer it
                if (__all_sync(0xffffffffu, !valid || (full && m_ref != NEG_INF))) {
                  uint64_t a0 = 0, a1 = 0;
                  float ra[4] = {0.f, 0.f, 0.f, 0.f};
                  exp_body(std::true_type{}, std::true_type{}, f2(sl2, sl2), f2(-m_ref, -m_ref), a0, a1, ra);
                  const uint64_t hs = f2_add(a0, a1);
                  const float half_sum = f2_lo(hs) + f2_hi(hs);
                  if (!__any_sync(0xffffffffu, valid && !(half_sum <= 256.0f))) {
                    ps[0] += f2_lo(a0);
                    ps[1] += f2_hi(a0);
                    ps[2] += f2_lo(a1);
                    ps[3] += f2_hi(a1);
#pragma unroll
                    for (int q = 0; q < 4; ++q) rs[q] += ra[q];
                    spec_done = true;
                  } else {
                    load_s(region + 64u * h);
                    tmem_wait_ld();
                    reg_fence(r);
                  }
                }
              }
              if (!spec_done) {
              if (row_id == 0 && X == 0) trace_ev(p, t + j, 30);
              if (!full) {
#pragma unroll
                for (int i = 0; i < 64; ++i) {
                  const int c = h * 64 + i;
                  if (!(c >= c_lo && c < c_hi)) r[i] = __float_as_uint(NEG_INF);
                }
              }
              float mx[4] = {NEG_INF, NEG_INF, NEG_INF, NEG_INF};
#pragma unroll
              for (int i = 0; i < 64; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(r[i]));
              const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
              const float m_new = fmaxf(m_ref, mt * sl2);
              const bool need = valid && (m_ref != NEG_INF) && (m_new > m_ref + 8.0f);
              if (__any_sync(0xffffffffu, need)) {
                if (row_id == 0 && X == 0) trace_ev(p, t + j, 31);
                const float alpha = need ? ex2(m_ref - m_new) : 1.0f;
                if (first_half) {
                  if (j > 0) {
                    // P.V(j-1) must have landed in O: pair units issue S(j) behind it (in-order
                    // tcgen05 pipe); single-tile units issue it after S(j), so wait
                    if (!u.has_b) {
                      const uint32_t tp = t + j - 1;
                      mbar_wait(&bar[B_VFREE0 + (tp % C::NSV)], (tp / C::NSV) & 1);
                      tc_fence_after();
                    }
                    rescale_o(alpha);
                  }
                } else {
                  // the first half's P.V (issued with the old max) must have landed in O
                  if (!PI_SYNCCHECK_PVH) mbar_wait(&bar[B_PVH0 + X], (pvh + j) & 1);
                  tc_fence_after();
                  rescale_o(alpha);
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    ps[q] *= alpha;
                    rs[q] *= alpha;
                  }
                }
                if (need) {
                  l *= alpha;
                  lr *= alpha;
                  m_ref = m_new;
                }
              }
              if (m_ref == NEG_INF) m_ref = m_new;
              // P = exp2(s * scale_log2 - m_ref): FFMA2 for the argument, PI_POLY_PAIRS of 8 pairs on
              // the FMA pipe (ex2_poly2), the rest on MUFU; masked columns hold -inf -> 0
              const bool live = m_ref != NEG_INF;
              const float nm = live ? -m_ref : NEG_INF;
              const uint64_t SL2 = f2(sl2, sl2), NM = f2(nm, nm);
              uint64_t acc0 = f2(ps[0], ps[1]), acc1 = f2(ps[2], ps[3]);
              auto body = [&](auto use_poly) { exp_body(use_poly, std::false_type{}, SL2, NM, acc0, acc1, rs); };
              if (!F32 && full)
                body(std::true_type{});
              else
                body(std::false_type{});
              ps[0] = f2_lo(acc0);
              ps[1] = f2_hi(acc0);
              ps[2] = f2_lo(acc1);
              ps[3] = f2_hi(acc1);
              }
              if (row_id == 0 && h == 0) trace_ev(p, t + j, 22 + X);
              if (PI_TRACE && p.trace != nullptr) spec_bits |= (spec_done ? 1u : 0u) << h;
              if (PI_TRACE && row_id == 0 && h == 1 && p.trace != nullptr && blockIdx.x == 0 &&
                  t + j < (uint32_t)TRACE_TILES)
                p.trace[(t + j) * 32 + 17 + 2 * X] = spec_bits;
              if constexpr (!F32) {
                // pair units: P_h at 32h (over S columns already read); single units: warpgroup
                // B's P goes over its own S columns (P1_SINGLE), never over warpgroup A's
                const uint32_t p_col = u.has_b ? 32u * h : (h ? C::P1_SINGLE : 0u);
                tmem_st32(region + p_col, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
              } else {
                tmem_st32(region + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
                tmem_st32(region + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
              }
            }
            if (u.has_b && h == 0) {
              // pair units: load S half 1 (same N = 128 chain, already complete) before releasing
              // P half 0
              if (row_id == 0) trace_ev(p, t + j, 16 + 2 * X);
              if (warp_any) {
                load_s(region + 64u);
                tmem_wait_ld();
                tmem_wait_st();
                reg_fence(r);
              }
            } else if (warp_any) {
              tmem_wait_st();
            }
            tc_fence_before();
            mbar_arrive(&bar[(h == 0 ? B_PHALF0 : B_PFULL0) + b]);
            if (row_id == 0) trace_ev(p, t + j, (h == 0 ? 8 : 9) + 4 * X);
          }
          if (valid) {
            l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
            lr += (F32 || !PI_P_ROUNDED_SUM) ? (ps[0] + ps[1]) + (ps[2] + ps[3]) : (rs[0] + rs[1]) + (rs[2] + rs[3]);
          }
        }
      }
      // ---------------- epilogue: O / l -> out (or partial), lse
      mbar_wait(&bar[B_OFULL0 + X], ix & 1);
      tc_fence_after();
      if (warp == C::ROLE && lane == 0) trace_unit(p, ix, 9);
      const int slot = (row.out >> 4) - 1;
      const int head = u.head0 + (u.has_b ? X : 0) + (row.out & 15);
      PI_CHECK(!valid || (slot < p.n_partial_slots && head < p.hq_count), 6);
      // pair units: out = O_X / l.  Single units: the two warpgroups hold (m, l) of key halves
      // 0..63 / 64..127 of every tile with partial accumulators O_0 / O_1; merge them (reading
      // R10: M = max, w = 2^(m - M), L = sum w l) and let warpgroup X write output columns
      // [X D/2, (X+1) D/2).
      float sc0 = 0.f, sc1 = 0.f, lse_v = 0.f;
      int c4_begin = 0, c4_end = D / 32;
      if constexpr ((UK & 2) && !F32) {
        if (sl) {
          if (wk.row_count <= kSliceFast) {
            // <= 8 rows (one request, or a few packed ones): ONE barrier.  Every warp stores its
            // quarter's raw partials O_0 / O_1 (column half X) and its own (m, l, l_rounded) in the
            // row's padding; then each thread merges the eight partials of one row and 4 columns
            // (reading R10, fixed order k = 0..7) and stores.
            float* pb = reinterpret_cast<float*>(smem + C::OFF_OBUF);   // [8 partials][kSliceFast rows][OBUF_STRIDE]
            constexpr int HC = D / 64;
            uint32_t o0[HC][32], o1[HC][32];
#pragma unroll
            for (int c = 0; c < HC; ++c) {
              tmem_ld32(tmem + lane_base + C::TM_O0 + (X * HC + c) * 32, o0[c]);
              tmem_ld32(tmem + lane_base + C::TM_O1 + (X * HC + c) * 32, o1[c]);
            }
            tmem_wait_ld();
            if (valid) {
              float* d0 = pb + (wq * kSliceFast + lane) * C::OBUF_STRIDE;         // partial k = wq (key half 0)
              float* d1 = pb + ((4 + wq) * kSliceFast + lane) * C::OBUF_STRIDE;   // partial k = 4 + wq (key half 1)
#pragma unroll
              for (int c = 0; c < HC; ++c) {
                reg_fence(o0[c]);
                reg_fence(o1[c]);
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                  const int col = (X * HC + c) * 32 + 4 * v;
                  *reinterpret_cast<float4*>(d0 + col) =
                      make_float4(__uint_as_float(o0[c][4 * v]), __uint_as_float(o0[c][4 * v + 1]),
                                  __uint_as_float(o0[c][4 * v + 2]), __uint_as_float(o0[c][4 * v + 3]));
                  *reinterpret_cast<float4*>(d1 + col) =
                      make_float4(__uint_as_float(o1[c][4 * v]), __uint_as_float(o1[c][4 * v + 1]),
                                  __uint_as_float(o1[c][4 * v + 2]), __uint_as_float(o1[c][4 * v + 3]));
                }
              }
              // this warp's softmax state is partial k = 4 X + wq
              float* ds = pb + ((4 * X + wq) * kSliceFast + lane) * C::OBUF_STRIDE + D;
              ds[0] = m_ref;
              ds[1] = l;
              ds[2] = lr;
            }
            named_bar_sync(1, 256);
            if (warp == C::ROLE && lane == 0) trace_unit(p, ix, 12);
            constexpr int V4 = D / 4;
            static_assert(256 / V4 >= kSliceFast, "one pass of the merge covers every row");
            const int tid = threadIdx.x - 32 * C::ROLE;
            const int rr = tid / V4, c = (tid % V4) * 4;
            if (rr < wk.row_count) {
              float mq[8], lq[8], rq[8], Mx = NEG_INF;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float* st = pb + (k * kSliceFast + rr) * C::OBUF_STRIDE + D;
                mq[k] = st[0];
                lq[k] = st[1];
                rq[k] = st[2];
                if (lq[k] > 0.f) Mx = fmaxf(Mx, mq[k]);
              }
              float L = 0.f, LR = 0.f, wq8[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                wq8[k] = lq[k] > 0.f ? ex2(mq[k] - Mx) : 0.f;
                L += lq[k] * wq8[k];
                LR += rq[k] * wq8[k];
              }
              const float inv = LR > 0.f ? 1.0f / LR : 0.f;
              float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float wk_ = wq8[k] * inv;
                const float4 a = *reinterpret_cast<const float4*>(pb + (k * kSliceFast + rr) * C::OBUF_STRIDE + c);
                f.x = fmaf(a.x, wk_, f.x);
                f.y = fmaf(a.y, wk_, f.y);
                f.z = fmaf(a.z, wk_, f.z);
                f.w = fmaf(a.w, wk_, f.w);
              }
              const pi_row rw = p.rows[wk.row_begin + rr];
              const int rslot = (rw.out >> 4) - 1;
              const int rhead = u.head0 + (rw.out & 15);
              if (rslot < 0) {
                if (!p.out_f32) {
                  uint8_t* dst = p.out + ((int64_t)rw.q_token * p.out_row_stride + (int64_t)rhead * D + c) * 2;
                  *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(f.x, f.y), pack_bf16(f.z, f.w));
                } else {
                  uint8_t* dst = p.out + ((int64_t)rw.q_token * p.out_row_stride + (int64_t)rhead * D + c) * 4;
                  *reinterpret_cast<float4*>(dst) = f;
                }
              } else {
                *reinterpret_cast<float4*>(p.partial_o + ((int64_t)rslot * p.hq_count + rhead) * D + c) = f;
              }
              if (c == 0) {
                const float lv = L > 0.f ? (Mx + __log2f(L)) * 0.69314718055994530942f : NEG_INF;
                if (rslot < 0) {
                  if (p.lse) p.lse[(int64_t)rhead * p.total_q + rw.q_token] = lv;
                } else {
                  p.partial_lse[(int64_t)rslot * p.hq_count + rhead] = lv;
                }
              }
            }
          } else {
            // lane-sliced unit: merge the row's eight partials (key half X' x lane quarter q, reading
            // R10), scale this quarter's O_0 / O_1 into the smem partial of quarter wq, then sum the
            // four quarters in a fixed order (bitwise reproducible) and store.
            float4* xch = reinterpret_cast<float4*>(smem + C::OFF_XCH);
            xch[X * 128 + row_id] = make_float4(m_ref, l, lr, 0.f);
            named_bar_sync(1, 256);
            float M = NEG_INF, mq[8], lq[8], rq[8];
  #pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float4 o = xch[(k >> 2) * 128 + (k & 3) * 32 + lane];
              mq[k] = o.x;
              lq[k] = o.y;
              rq[k] = o.z;
              if (o.y > 0.f) M = fmaxf(M, o.x);
            }
            float L = 0.f, LR = 0.f, w0 = 0.f, w1 = 0.f;
  #pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float wk_ = lq[k] > 0.f ? ex2(mq[k] - M) : 0.f;
              L += lq[k] * wk_;
              LR += rq[k] * wk_;
              if (k == wq) w0 = wk_;
              if (k == 4 + wq) w1 = wk_;
            }
            const float inv = LR > 0.f ? 1.0f / LR : 0.f;
            lse_v = L > 0.f ? (M + __log2f(L)) * 0.69314718055994530942f : NEG_INF;
            if (warp == C::ROLE && lane == 0) trace_unit(p, ix, 12);
            // every thread has read XCH (aliased by the partial buffer below)
            named_bar_sync(1, 256);
            if (warp == C::ROLE && lane == 0) trace_unit(p, ix, 13);
            // quarter sum in a fixed order, (p0 + p2) + (p1 + p3): quarters 2, 3 store their weighted
            // partial of column half X into buffer (q & 1), then quarters 0, 1 add theirs in place,
            // then every thread adds the two buffers and stores
            float* ob = reinterpret_cast<float*>(smem + C::OFF_OBUF);
            // this warp's weighted partial of column half X (both 32-column chunks), all TMEM loads
            // issued before the first wait
            constexpr int HC = D / 64;   // 32-column chunks per column half
            uint32_t o0[HC][32], o1[HC][32];
  #pragma unroll
            for (int c = 0; c < HC; ++c) {
              tmem_ld32(tmem + lane_base + C::TM_O0 + (X * HC + c) * 32, o0[c]);
              tmem_ld32(tmem + lane_base + C::TM_O1 + (X * HC + c) * 32, o1[c]);
            }
            tmem_wait_ld();
  #pragma unroll
            for (int c = 0; c < HC; ++c) {
              reg_fence(o0[c]);
              reg_fence(o1[c]);
  #pragma unroll
              for (int i = 0; i < 32; ++i)
                o0[c][i] = __float_as_uint(fmaf(__uint_as_float(o0[c][i]), w0 * inv, __uint_as_float(o1[c][i]) * (w1 * inv)));
            }
  #pragma unroll
            for (int stage = 0; stage < 2; ++stage) {
              if ((wq >> 1) == 1 - stage && valid) {
  #pragma unroll
                for (int c = 0; c < HC; ++c) {
                  float* dst = ob + ((wq & 1) * kSliceRows + lane) * C::OBUF_STRIDE + (X * HC + c) * 32;
  #pragma unroll
                  for (int v = 0; v < 8; ++v) {
                    float4 f = make_float4(__uint_as_float(o0[c][4 * v]), __uint_as_float(o0[c][4 * v + 1]),
                                           __uint_as_float(o0[c][4 * v + 2]), __uint_as_float(o0[c][4 * v + 3]));
                    if (stage == 1) {
                      const float4 g = reinterpret_cast<const float4*>(dst)[v];
                      f.x += g.x;
                      f.y += g.y;
                      f.z += g.z;
                      f.w += g.w;
                    }
                    reinterpret_cast<float4*>(dst)[v] = f;
                  }
                }
              }
              named_bar_sync(1, 256);
              if (warp == C::ROLE && lane == 0) trace_unit(p, ix, 14 + stage);
            }
            {
              constexpr int V4 = D / 4;
              const int tid = threadIdx.x - 32 * C::ROLE;   // 0..255: 256 / V4 rows per pass
              const int c = (tid % V4) * 4;
              for (int rr = tid / V4; rr < wk.row_count; rr += 256 / V4) {
                const float4 a0 = *reinterpret_cast<const float4*>(ob + rr * C::OBUF_STRIDE + c);
                const float4 a1 = *reinterpret_cast<const float4*>(ob + (kSliceRows + rr) * C::OBUF_STRIDE + c);
                float4 f;
                f.x = a0.x + a1.x;
                f.y = a0.y + a1.y;
                f.z = a0.z + a1.z;
                f.w = a0.w + a1.w;
                const pi_row rw = p.rows[wk.row_begin + rr];
                const int rslot = (rw.out >> 4) - 1;
                const int rhead = u.head0 + (rw.out & 15);
                if (rslot < 0) {
                  if (!p.out_f32) {
                    uint8_t* dst = p.out + ((int64_t)rw.q_token * p.out_row_stride + (int64_t)rhead * D + c) * 2;
                    *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(f.x, f.y), pack_bf16(f.z, f.w));
                  } else {
                    uint8_t* dst = p.out + ((int64_t)rw.q_token * p.out_row_stride + (int64_t)rhead * D + c) * 4;
                    *reinterpret_cast<float4*>(dst) = f;
                  }
                } else {
                  *reinterpret_cast<float4*>(p.partial_o + ((int64_t)rslot * p.hq_count + rhead) * D + c) = f;
                }
              }
            }
            if (valid && X == 0 && wq == 0) {
              if (slot < 0) {
                if (p.lse) p.lse[(int64_t)head * p.total_q + row.q_token] = lse_v;
              } else {
                p.partial_lse[(int64_t)slot * p.hq_count + head] = lse_v;
              }
            }
          }
          c4_end = 0;   // nothing left for the generic store path below
        }
      }
      if (sl) {
      } else if (u.has_b) {
        sc0 = lr > 0.f ? 1.0f / lr : 0.f;
        lse_v = l > 0.f ? (m_ref + __log2f(l)) * 0.69314718055994530942f : NEG_INF;
      } else {
        float4* xch = reinterpret_cast<float4*>(smem + C::OFF_XCH);
        xch[X * 128 + row_id] = make_float4(m_ref, l, lr, 0.f);
        named_bar_sync(1, 256);
        const float4 o = xch[(1 - X) * 128 + row_id];
        const float mA = X ? o.x : m_ref, lA = X ? o.y : l, rA = X ? o.z : lr;
        const float mB = X ? m_ref : o.x, lB = X ? l : o.y, rB = X ? lr : o.z;
        const float M = fmaxf(lA > 0.f ? mA : NEG_INF, lB > 0.f ? mB : NEG_INF);
        const float wA = lA > 0.f ? ex2(mA - M) : 0.f, wB = lB > 0.f ? ex2(mB - M) : 0.f;
        const float L = lA * wA + lB * wB, LR = rA * wA + rB * wB;
        const float inv = LR > 0.f ? 1.0f / LR : 0.f;
        sc0 = wA * inv;
        sc1 = wB * inv;
        lse_v = L > 0.f ? (M + __log2f(L)) * 0.69314718055994530942f : NEG_INF;
        c4_begin = X * (D / 64);
        c4_end = c4_begin + D / 64;
      }
      const uint32_t o0_tm = u.has_b ? o_tm : tmem + lane_base + C::TM_O0;
      const uint32_t o1_tm = tmem + lane_base + C::TM_O1;
      if (warp_any) {
#pragma unroll
        for (int c4 = 0; c4 < D / 32; ++c4) {
          if (c4 < c4_begin || c4 >= c4_end) continue;
          uint32_t o32[32];
          tmem_ld32(o0_tm + c4 * 32, o32);
          tmem_wait_ld();
          reg_fence(o32);
          if (!u.has_b) {
            uint32_t o1[32];
            tmem_ld32(o1_tm + c4 * 32, o1);
            tmem_wait_ld();
            reg_fence(o1);
#pragma unroll
            for (int i = 0; i < 32; ++i)
              o32[i] = __float_as_uint(fmaf(__uint_as_float(o32[i]), sc0, __uint_as_float(o1[i]) * sc1));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) o32[i] = __float_as_uint(__uint_as_float(o32[i]) * sc0);
          }
          if (valid) {
            if (slot < 0) {
              const int oes = (F32 || p.out_f32) ? 4 : 2;
              uint8_t* dst = p.out + ((int64_t)row.q_token * p.out_row_stride + (int64_t)head * D + c4 * 32) * oes;
              if (!F32 && !p.out_f32) {
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                  uint32_t pk[4];
#pragma unroll
                  for (int e = 0; e < 4; ++e)
                    pk[e] = pack_bf16(__uint_as_float(o32[v * 8 + 2 * e]), __uint_as_float(o32[v * 8 + 2 * e + 1]));
                  reinterpret_cast<uint4*>(dst)[v] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
              } else {
#pragma unroll
                for (int v = 0; v < 8; ++v)
                  reinterpret_cast<float4*>(dst)[v] =
                      make_float4(__uint_as_float(o32[4 * v]), __uint_as_float(o32[4 * v + 1]),
                                  __uint_as_float(o32[4 * v + 2]), __uint_as_float(o32[4 * v + 3]));
              }
            } else {
              float* dst = p.partial_o + ((int64_t)slot * p.hq_count + head) * D + c4 * 32;
#pragma unroll
              for (int v = 0; v < 8; ++v)
                reinterpret_cast<float4*>(dst)[v] =
                    make_float4(__uint_as_float(o32[4 * v]), __uint_as_float(o32[4 * v + 1]),
                                __uint_as_float(o32[4 * v + 2]), __uint_as_float(o32[4 * v + 3]));
            }
          }
        }
      }
      if (valid && !sl && (u.has_b || X == 0)) {
        if (slot < 0) {
          if (p.lse) p.lse[(int64_t)head * p.total_q + row.q_token] = lse_v;
        } else {
          p.partial_lse[(int64_t)slot * p.hq_count + head] = lse_v;
        }
      }
      if (warp == C::ROLE && lane == 0) trace_unit(p, ix, 10);
      tc_fence_before();
      if (!u.has_b) named_bar_sync(1, 256);   // both warpgroups are done with O_0, O_1 and xch
      mbar_arrive(&bar[B_OFREE0 + X]);
      if (warp == C::ROLE && lane == 0) trace_unit(p, ix, 11);
      if ((UK & 2) && PI_MERGE_WARP && !u.has_b && p.merge_ctr != nullptr) {
        // in-kernel merge: hand this unit's partials (both column halves + lse, stored above) to the
        // merge warp (ring of 4; the mbarrier arrive releases the stores at CTA scope)
        const uint32_t e = epi & 3;
        mbar_wait(&bar[B_EFREE0 + e], ((epi >> 2) & 1) ^ 1);
        mbar_arrive(&bar[B_EFULL0 + e]);
        ++epi;
      }
      if (u.has_b) {
        cntA += n;
        cntB += n;
      } else {
        cntA += (n + 1) >> 1;
        cntB += n >> 1;
        cnt1A += (n + 1) >> 1;
        cnt1B += n >> 1;
      }
      if (u.has_b) pvh += n;   // PVH completes for pair units only
      t += n;
      ++ix;
      w = wn;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PI_TRACE && threadIdx.x == 0) trace_cta(p, 1, globaltimer());
  if (threadIdx.x == 0) {
    // self-resetting scheduler: this CTA's producer made its last counter access before the
    // barrier above; the CTA that exits last returns both counters to zero for the next launch
    // on the stream (stream order makes the plain stores visible to it)
    __threadfence();
    if (atomicAdd(&p.sched[1], 1u) == gridDim.x - 1) {
      p.sched[0] = 0u;
      p.sched[1] = 0u;
    }
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

unsigned long long* g_debug_trace = nullptr;

template <int D, bool F32, int UK>
static pi_status launch_kernel(const AttnParams& p, const CUtensorMap& tmK, const CUtensorMap& tmV,
                               const CUtensorMap& tmQ, const CUtensorMap& tmQB, int grid, cudaStream_t stream,
                               bool pdl = false) {
  using C = AttnCfg<D, F32, UK>;
  if constexpr (F32 && UK != 2) {
    return fail(PI_EUNSUP, "fp32 operands run single-tile units only");
  } else {
    static std::atomic<int> smem_opt_in[kMaxDevices];   // per template instance and device
    pi_status s = set_max_dynamic_smem(reinterpret_cast<const void*>(packed_attention_kernel<D, F32, UK>),
                                       smem_opt_in, C::SMEM);
    if (s != PI_OK) return s;
    if (pdl) {
      // programmatic dependent launch: this grid's CTAs may start on SMs the previous launch on the
      // stream frees once every CTA of it has run out of units (griddepcontrol.launch_dependents);
      // the two launches write disjoint rows / partials
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)grid);
      cfg.blockDim = dim3(C::THREADS);
      cfg.dynamicSmemBytes = C::SMEM;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cuda_check(cudaLaunchKernelEx(&cfg, packed_attention_kernel<D, F32, UK>, p, tmK, tmV, tmQ, tmQB),
                        "packed_attention_kernel launch (PDL)");
    }
    packed_attention_kernel<D, F32, UK><<<grid, C::THREADS, C::SMEM, stream>>>(p, tmK, tmV, tmQ, tmQB);
    return cuda_check(cudaGetLastError(), "packed_attention_kernel launch");
  }
}

// mode: bit 0 = prefill work items, bit 1 = decode work items (both = one fused launch)
struct PagedSrc {   // packinfer_attention_decode_paged: the paged cache instead of k/v_buf
  const int32_t* block_table;
  int32_t max_blocks, page, num_blocks, hkv_total, hkv_begin;
};

template <int D, bool F32>
static pi_status launch(const pi_device_plan* dp, int mode, bool out_f32, const void* q, int64_t q_row_stride,
                        const void* k_buf, const void* v_buf, int32_t hkv_count, int32_t r, float scale,
                        void* out, int64_t out_row_stride, float* lse, float* partial_o, float* partial_lse,
                        uint32_t* merge_ctr, cudaStream_t stream, const PagedSrc* paged = nullptr,
                        bool pdl = false, int sched_pair = 0, bool pdl_wait = false) {
  using C = AttnCfg<D, F32>;   // tile geometry only (independent of the unit kinds)
  AttnParams p{};
  p.work_p = dp->prefill_work;
  p.work_d = dp->decode_work;
  p.n_work_p = (mode & 1) ? dp->n_prefill_work : 0;
  p.n_work_d = (mode & 2) ? dp->n_decode_work : 0;
  if (p.n_work_p + p.n_work_d == 0) return PI_OK;
  p.rows = dp->rows;
  p.spans = dp->spans;
  // fp32 operands keep one tile per unit: their P fills the whole 128-column S region
  p.tiles_per_unit = F32 ? 1 : 2;
  p.units_p = hkv_count * ((r + p.tiles_per_unit - 1) / p.tiles_per_unit);
  p.units_d = hkv_count;
  p.total_p = p.n_work_p * p.units_p;
  p.r = r;
  p.q = static_cast<const uint8_t*>(q);
  p.q_row_stride = q_row_stride;
  p.out = static_cast<uint8_t*>(out);
  p.out_row_stride = out_row_stride;
  p.lse = lse;
  p.total_q = dp->total_q;
  p.hq_count = hkv_count * r;
  p.partial_o = partial_o;
  p.partial_lse = partial_lse;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.v_buf = static_cast<const uint8_t*>(v_buf);
  p.out_f32 = out_f32 ? 1 : 0;
  p.buffer_tokens = dp->buffer_tokens;
  p.trace = g_debug_trace;
  p.sched = dp->sched ? dp->sched + 2 * sched_pair : nullptr;
  p.pdl_wait = pdl_wait ? 1 : 0;
  pdl = pdl || pdl_wait;
  p.n_partial_slots = dp->n_partial_slots;
  p.merges = dp->merges;
  p.slot_merge = dp->slot_merge;
  // fp32 operands: warp 3 stages V^T, so the entry point merges with a separate launch instead
  p.merge_ctr = (!F32 && dp->n_merges > 0 && (mode & 2)) ? merge_ctr : nullptr;

  CUtensorMap tmK, tmV;
  const CUtensorMapDataType dt = F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const uint64_t dims[3] = {(uint64_t)D, (uint64_t)dp->buffer_tokens, (uint64_t)hkv_count};
  const uint64_t strides[2] = {(uint64_t)C::ROW_BYTES, (uint64_t)dp->buffer_tokens * C::ROW_BYTES};
  const uint32_t box[3] = {(uint32_t)C::ATOM_ELEMS, 128u, 1u};
  pi_status s;
  if (paged == nullptr) {
    s = encode_tmap_3d(&tmK, dt, k_buf, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (s != PI_OK) return s;
    s = encode_tmap_3d(&tmV, dt, v_buf, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (s != PI_OK) return s;
  } else {
    // paged cache [blocks * page slots, hkv_total, d]: box (atom, 1 head, 128 slots) lands in smem
    // exactly like a buffer tile (128 rows of 128 B, SWIZZLE_128B)
    const uint64_t pdims[3] = {(uint64_t)D, (uint64_t)paged->hkv_total, (uint64_t)paged->num_blocks * paged->page};
    const uint64_t pstrides[2] = {(uint64_t)C::ROW_BYTES, (uint64_t)paged->hkv_total * C::ROW_BYTES};
    const uint32_t pbox[3] = {(uint32_t)C::ATOM_ELEMS, 1u, 128u};
    s = encode_tmap_3d(&tmK, dt, k_buf, pdims, pstrides, pbox, CU_TENSOR_MAP_SWIZZLE_128B);
    if (s != PI_OK) return s;
    s = encode_tmap_3d(&tmV, dt, v_buf, pdims, pstrides, pbox, CU_TENSOR_MAP_SWIZZLE_128B);
    if (s != PI_OK) return s;
    p.block_table = paged->block_table;
    p.max_blocks = paged->max_blocks;
    p.page = paged->page;
    p.kv_head0 = paged->hkv_begin;
  }
  // Q as a 2D (row = token * q_heads_stride + head, d) tensor for tile::gather4 (box {atom, 1})
  CUtensorMap tmQ;
  p.q_heads_stride = (int32_t)(q_row_stride / D);
  const uint64_t qdims[3] = {(uint64_t)D, (uint64_t)dp->total_q * (uint64_t)p.q_heads_stride, 1};
  const uint64_t qstrides[2] = {(uint64_t)C::ROW_BYTES, (uint64_t)dp->total_q * p.q_heads_stride * C::ROW_BYTES};
  const uint32_t qbox[3] = {(uint32_t)C::ATOM_ELEMS, 1u, 1u};
  s = encode_tmap_2d(&tmQ, dt, q, qdims, qstrides, qbox, CU_TENSOR_MAP_SWIZZLE_128B);
  if (s != PI_OK) return s;
  // the same Q as (d, head, token) boxes of 128 tokens for tiles whose rows are consecutive tokens
  CUtensorMap tmQB;
  const uint64_t bdims[3] = {(uint64_t)D, (uint64_t)p.q_heads_stride, (uint64_t)dp->total_q};
  const uint64_t bstrides[2] = {(uint64_t)C::ROW_BYTES, (uint64_t)q_row_stride * C::ES};
  const uint32_t bbox[3] = {(uint32_t)C::ATOM_ELEMS, 1u, 128u};
  s = encode_tmap_3d(&tmQB, dt, q, bdims, bstrides, bbox, CU_TENSOR_MAP_SWIZZLE_128B);
  if (s != PI_OK) return s;

  const int64_t total = (int64_t)p.total_p + (int64_t)p.n_work_d * p.units_d;
  const int grid = (int)std::min<int64_t>(total, num_sms());
  if (p.sched == nullptr) return fail(PI_EINVAL, "device plan has no scheduler counter (packinfer_plan_upload)");
  // no reset here: packinfer_plan_upload zeroes the counters and every launch leaves them at zero
  // (the last CTA to exit resets them), so a launch is one kernel and no memset node
  // kernel instance by the unit kinds present (see get_unit): a prefill-only launch with even r
  // has pair units only, a decode-only launch (or fp32 operands) single-tile units only
  const bool pairs_only = !F32 && p.n_work_d == 0 && (r % 2) == 0;
  const bool singles_only = F32 || p.n_work_p == 0 || r == 1;
  if (pairs_only) return launch_kernel<D, F32, 1>(p, tmK, tmV, tmQ, tmQB, grid, stream, pdl);
  if (singles_only) return launch_kernel<D, F32, 2>(p, tmK, tmV, tmQ, tmQB, grid, stream, pdl);
  return launch_kernel<D, F32, 3>(p, tmK, tmV, tmQ, tmQB, grid, stream, pdl);
}

static pi_status attention_entry(int mode, const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                 const void* k_buf, const void* v_buf, int32_t hkv_count, int32_t gqa_ratio,
                                 int32_t head_dim, float softmax_scale, pi_dtype dt, void* out,
                                 int64_t out_row_stride, float* lse, float* partial_o, float* partial_lse,
                                 pi_stream_t stream, uint32_t* merge_ctr = nullptr, bool want_merge = false,
                                 const PagedSrc* paged = nullptr) {
  if (!dp) return fail(PI_EINVAL, "device plan is NULL");
  const bool decode = (mode & 2) && dp->n_decode_work > 0;
  const int32_t n_work = ((mode & 1) ? dp->n_prefill_work : 0) + ((mode & 2) ? dp->n_decode_work : 0);
  if (n_work == 0) return ok();
  if (!q || !k_buf || !v_buf || !out) return fail(PI_EINVAL, "q, k_buf, v_buf and out must be non-NULL");
  if (hkv_count < 1 || gqa_ratio < 1 || gqa_ratio > 16) return fail(PI_EINVAL, "bad hkv_count / gqa_ratio");
  if (decode && gqa_ratio != dp->gqa_ratio)
    return fail(PI_EINVAL, "gqa_ratio differs from the plan's (decode rows are planned per GQA head)");
  if (head_dim != 64 && head_dim != 128) return fail(PI_EUNSUP, "head_dim must be 64 or 128");
  if (dt != PI_BF16 && dt != PI_FP32 && dt != PI_BF16_OUT_F32)
    return fail(PI_EUNSUP, "dtype must be PI_BF16, PI_FP32 or PI_BF16_OUT_F32");
  const bool out_f32 = dt == PI_BF16_OUT_F32;
  if (out_f32) dt = PI_BF16;
  if (dt == PI_FP32 && head_dim != 64) return fail(PI_EUNSUP, "PI_FP32 supports head_dim 64 only");
  if (q_row_stride % head_dim) return fail(PI_EINVAL, "q_row_stride must be a multiple of head_dim");
  if (q_row_stride < (int64_t)hkv_count * gqa_ratio * head_dim ||
      out_row_stride < (int64_t)hkv_count * gqa_ratio * head_dim)
    return fail(PI_EINVAL, "row stride smaller than the local heads");
  if (dp->n_partial_slots > 0 && decode && (!partial_o || !partial_lse))
    return fail(PI_EINVAL, "plan has split rows: partial_o / partial_lse required");
  if (want_merge && decode && dp->n_merges > 0 && (!merge_ctr || !dp->slot_merge))
    return fail(PI_EINVAL, "in-kernel merge needs merge_counters and a plan with a slot->merge table");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(k_buf) |
       reinterpret_cast<uintptr_t>(v_buf)) % 16)
    return fail(PI_EINVAL, "q/out/k_buf/v_buf must be 16-byte aligned");
  pi_status s = require_sm100();
  if (s != PI_OK) return s;
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)head_dim);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (PI_FUSED_PDL && mode == 3 && dt == PI_BF16 && paged == nullptr && dp->n_prefill_work > 0 &&
      dp->n_decode_work > 0) {
    // one call over prefill + decode items: the prefill items on the pair-unit kernel instance,
    // then the decode items on the single-tile instance as a programmatic dependent launch that
    // fills the SMs the prefill launch releases at its tail (its own scheduler counters).  One
    // persistent mixed-instance launch (PI_FUSED_PDL=0) carries both unit kinds' code and register
    // budget: prefill units run 14 % slower there (profiles/r04q).
    for (int part = 1; part <= 2 && s == PI_OK; ++part) {
      if (head_dim == 128)
        s = launch<128, false>(dp, part, out_f32, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, scale, out,
                               out_row_stride, lse, partial_o, partial_lse, merge_ctr, st, nullptr, part == 2, part - 1,
                               PI_STEP_PDL && part == 1);
      else
        s = launch<64, false>(dp, part, out_f32, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, scale, out,
                              out_row_stride, lse, partial_o, partial_lse, merge_ctr, st, nullptr, part == 2, part - 1,
                              PI_STEP_PDL && part == 1);
    }
    return s == PI_OK ? ok() : s;
  }
  if (dt == PI_BF16 && head_dim == 128)
    s = launch<128, false>(dp, mode, out_f32, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, scale, out,
                           out_row_stride, lse, partial_o, partial_lse, merge_ctr, st, paged, false, 0, PI_STEP_PDL);
  else if (dt == PI_BF16 && head_dim == 64)
    s = launch<64, false>(dp, mode, out_f32, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, scale, out,
                          out_row_stride, lse, partial_o, partial_lse, merge_ctr, st, paged);
  else
    s = launch<64, true>(dp, mode, false, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, scale, out,
                         out_row_stride, lse, partial_o, partial_lse, merge_ctr, st, paged);
  return s == PI_OK ? ok() : s;
}

}  // namespace pi

extern "C" {

// Debug hook (not part of the ABI header): device buffer of >= 64*16 uint64 that the next attention
// launches fill with CTA 0's clock64 timeline; NULL disables.
PI_API void packinfer_debug_trace(void* dev_buf) { pi::g_debug_trace = static_cast<unsigned long long*>(dev_buf); }

pi_status packinfer_attention_prefill(const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                      const void* k_buf, const void* v_buf, int32_t hkv_count, int32_t gqa_ratio,
                                      int32_t head_dim, float softmax_scale, pi_dtype dt, void* out,
                                      int64_t out_row_stride, float* lse, float* partial_o, float* partial_lse,
                                      pi_stream_t stream) {
  return pi::attention_entry(1, dp, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, head_dim,
                             softmax_scale, dt, out, out_row_stride, lse, partial_o, partial_lse, stream);
}

pi_status packinfer_attention_decode(const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                     const void* k_buf, const void* v_buf, int32_t hkv_count, int32_t gqa_ratio,
                                     int32_t head_dim, float softmax_scale, pi_dtype dt, void* out,
                                     int64_t out_row_stride, float* lse, float* partial_o, float* partial_lse,
                                     pi_stream_t stream) {
  return pi::attention_entry(2, dp, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, head_dim,
                             softmax_scale, dt, out, out_row_stride, lse, partial_o, partial_lse, stream);
}

pi_status packinfer_attention(const pi_device_plan* dp, const void* q, int64_t q_row_stride, const void* k_buf,
                              const void* v_buf, int32_t hkv_count, int32_t gqa_ratio, int32_t head_dim,
                              float softmax_scale, pi_dtype dt, void* out, int64_t out_row_stride, float* lse,
                              float* partial_o, float* partial_lse, pi_stream_t stream) {
  return pi::attention_entry(3, dp, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, head_dim, softmax_scale,
                             dt, out, out_row_stride, lse, partial_o, partial_lse, stream);
}

pi_status packinfer_attention_decode_paged(const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                          const void* k_paged, const void* v_paged, const int32_t* block_table,
                                          int32_t max_blocks, int32_t page_size, int32_t num_blocks, int32_t hkv_total,
                                          int32_t hkv_begin, int32_t hkv_count, int32_t gqa_ratio, int32_t head_dim,
                                          float softmax_scale, pi_dtype dt, void* out, int64_t out_row_stride,
                                          float* lse, float* partial_o, float* partial_lse, pi_stream_t stream) {
  using namespace pi;
  if (!dp) return fail(PI_EINVAL, "device plan is NULL");
  if (dp->n_prefill_work > 0) return fail(PI_EINVAL, "paged decode needs a decode-only plan (PI_PLAN_PAGED)");
  if (!block_table || max_blocks < 1 || num_blocks < 1) return fail(PI_EINVAL, "bad block table / num_blocks");
  if (page_size < 128 || page_size % 128) return fail(PI_EINVAL, "page_size must be a multiple of 128");
  if (hkv_begin < 0 || hkv_count < 1 || hkv_begin + hkv_count > hkv_total) return fail(PI_EINVAL, "bad KV head range");
  if (dt == PI_FP32) return fail(PI_EUNSUP, "paged decode supports bf16 operands only");
  const PagedSrc src{block_table, max_blocks, page_size, num_blocks, hkv_total, hkv_begin};
  return attention_entry(2, dp, q, q_row_stride, k_paged, v_paged, hkv_count, gqa_ratio, head_dim, softmax_scale, dt,
                         out, out_row_stride, lse, partial_o, partial_lse, stream, nullptr, false, &src);
}

pi_status packinfer_attention_merge(const pi_device_plan* dp, const void* q, int64_t q_row_stride, const void* k_buf,
                                    const void* v_buf, int32_t hkv_count, int32_t gqa_ratio, int32_t head_dim,
                                    float softmax_scale, pi_dtype dt, void* out, int64_t out_row_stride, float* lse,
                                    float* partial_o, float* partial_lse, uint32_t* merge_counters,
                                    pi_stream_t stream) {
  pi_status s = pi::attention_entry(3, dp, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, head_dim,
                                    softmax_scale, dt, out, out_row_stride, lse, partial_o, partial_lse, stream,
                                    merge_counters, true);
  // fp32 operands (the toy config): warp 3 stages V^T there, so the merge is a separate launch
  if (s == PI_OK && dt == PI_FP32 && dp->n_merges > 0)
    s = packinfer_merge(dp, partial_o, partial_lse, hkv_count * gqa_ratio, head_dim, dt, out, out_row_stride, lse,
                        stream);
  return s;
}

}  // extern "C"
