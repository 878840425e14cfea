/*
 * packinfer.h — C ABI of the B200-native PackInfer hot path (arXiv 2602.06072).
 *
 * The interface follows the paper's statement of the problem (Alg. 1 KwIn/KwOut, PAPER.md
 * P:205-206): inputs are the batch R (per-request lengths, prefix lineage), the group
 * capacity C and the paged KV cache M_paged; outputs are the groups {S_g}, the contiguous
 * buffers {B_g} and the offset tables {O_g}, plus the packed attention over the "union of
 * valid query-key regions" and the lossless merge of split requests.
 * It is exported as a FlashAttention-style drop-in: varlen Q/O, fp32 LSE.
 *
 * Conventions (every entry point):
 *   - returns pi_status; never throws; never allocates device memory; never synchronises a
 *     stream (device work is enqueued on the caller's stream, like cuBLAS).
 *   - the caller owns every buffer; pointers marked "device" must be device memory of the
 *     current CUDA device, "host" pointers host memory.
 *   - invalid arguments return PI_EINVAL with no side effects (details: packinfer_last_error);
 *     asynchronous device faults surface at the caller's next synchronisation.
 *   - an empty batch (n = 0) is valid: planning returns zero counts, device calls are no-ops.
 *   - thread-safe across distinct plans/streams; the library keeps no global mutable state
 *     beyond a thread-local error string and cached CUDA function attributes.
 *   - plans are reproducible: identical inputs give byte-identical host tables.
 *
 * Element layouts (all row-major, innermost last):
 *   q, out        [total_q, q_row_stride] elements; the local Q heads of token t start at
 *                 q + t*q_row_stride, head h at + h*head_dim (varlen, caller order: request i
 *                 owns rows q_off[i] .. q_off[i]+q_len[i]-1, q_off = exclusive cumsum of q_len)
 *   lse           fp32 [hq_count, total_q]   (natural log; hq_count = hkv_count * gqa_ratio)
 *   k/v_paged     [num_blocks, page_size, hkv_total, head_dim]          (D6)
 *   block_table   int32 [n + n_prefix, max_blocks]: row i < n maps request i's logical tokens
 *                 [0, kv_len[i]) (a shared prefix's physical blocks first); row n + p maps
 *                 prefix p's tokens [0, prefix_len[p]).
 *   k/v_buf       [hkv_count, buffer_tokens, head_dim]  group-contiguous buffers B_g laid end
 *                 to end (base_g = sum of earlier group capacities)       (Alg. 1 Part 2).
 *                 Element type = the cache's (bf16 or fp32): every cell is a bitwise copy of
 *                 the paged cache (no conversion, the full bf16 range is preserved).
 *   partial_o     fp32 [n_partial_slots, hq_count, head_dim]; partial_lse fp32
 *                 [n_partial_slots, hq_count] — partial results of split rows (reading R10).
 */
#ifndef PACKINFER_H_
#define PACKINFER_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PI_API __attribute__((visibility("default")))
#else
#define PI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* pi_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  PI_OK = 0,
  PI_EINVAL = -1, /* invalid argument (see packinfer_last_error)                         */
  PI_ENOSPC = -2, /* caller buffer too small; required sizes were written back          */
  PI_ECUDA = -3,  /* a CUDA runtime/driver call failed (launch or tensor-map encode)     */
  PI_EUNSUP = -4, /* unsupported dtype / head_dim / device (needs sm_100a)              */
  PI_EREGROUP = -5 /* decode headroom exhausted: regroup (re-plan + relayout)      */
} pi_status;

typedef enum {
  PI_BF16 = 0,         /* bf16 operands, bf16 out/in-place results (tcgen05 kind::f16)          */
  PI_FP32 = 1,         /* fp32 operands and output (tcgen05 kind::tf32; head_dim 64)            */
  PI_BF16_OUT_F32 = 2  /* bf16 operands, fp32 output: isolates kernel arithmetic from output
                          rounding (reading R13); for attention/merge only                      */
} pi_dtype;

/* Static string for a status code. */
PI_API const char* packinfer_strerror(pi_status s);
/* Thread-local detail of the last failing call on this thread ("" if none). */
PI_API const char* packinfer_last_error(void);
/* Library version string. */
PI_API const char* packinfer_version(void);

/* ------------------------------------------------------------------------------------------
 * Planner configuration (Alg. 1 inputs; defaults from Table tab:hyperparams).
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  int32_t capacity;     /* C, max prefix-deduplicated tokens per group (Eq. 2); default
                           8192.  Requests with kv_len > C are split into pieces of C
                           tokens (reading R5).  Must be >= 1.                         */
  int32_t num_groups;   /* initial G override; 0 => max(1, ceil(L_dedup / C)) (Alg.1 l.1,
                           P:212; reading R2)                                                */
  int64_t mem_cap;      /* M_max in tokens incl. headroom (Eq. 2 second term); 0 disables it;
                           else must be >= capacity + headroom                              */
  int32_t headroom;     /* delta: tokens reserved after every suffix; >= 0        */
  int32_t tile_q;       /* rows per packed work tile; must be 128 (tcgen05 M=128)            */
  int32_t tile_k;       /* keys per K tile; must be 128 (P:159 T in {128,256})               */
  int32_t decode_chunk; /* max keys per decode work item (multiple of tile_k; e.g. 1024)      */
  int32_t gqa_ratio;    /* r = Hq / Hkv in [1, 16]: decode rows are (request, GQA head)       */
  int32_t flags;        /* PI_PLAN_* bits (default PI_PLAN_DPACK).  (Occupies the struct's former tail
                           padding: sizeof(pi_config) is unchanged.)                           */
} pi_config;

/* Ablation (NEXT-4; Fig. "breakdown" P:480-489): every request's query rows start
 * their own 128-row tiles (no packing of short requests into shared tiles) - the
 * "unpacked compute" baseline.  Groups, layout and results are unchanged; only tile count and
 * tile efficiency change.                                                                     */
#define PI_PLAN_NO_QPACK 1
/* Packed decode items (on in packinfer_default_config): consecutive short decode suffixes of one
 * group share one decode work item - the decode analogue of packed prefill tiles - whose
 * key span is their hull (<= decode_chunk keys, <= tile_q rows); each row sees only its own
 * suffix [lo, hi), so every key is still read once.  With rows <= 32 lane-sliced in the kernel
 * this amortises the per-unit epilogue over several requests (configs[3] decode kernel -7 %,
 * configs[2] -2 %, profiles/r03b).  flags = 0 plans one item per suffix.                      */
#define PI_PLAN_DPACK 2
/* Ablation (NEXT-4, Fig. "breakdown" P:480-489: "packed I/O" off): a decode-only plan whose work
 * items cover each request's LOGICAL tokens, read straight from the paged cache by
 * packinfer_attention_decode_paged - no consolidation and no prefix co-location.  Groups, offsets
 * and the copy plan are still computed (unused).  q_len must be 1 for every request.           */
#define PI_PLAN_PAGED 4
/* Scheduling hint: order prefill work items by exact cost (LPT) instead of 32-key-tile cost buckets
 * that keep emission order (L2 locality).  For launches with few units per SM - e.g. one or two KV
 * heads per rank under KV-head sharding - balance matters more than locality (configs[1] at one
 * KV head: kernel 0.267 -> 0.24 ms; at 8 KV heads it is ~3 % slower).                      */
#define PI_PLAN_LPT_EXACT 8

/* Fill *cfg with the defaults: C=8192, G auto, no M_max, delta=0, 128/128 tiles,
 * decode_chunk=1024, gqa_ratio=1, flags = PI_PLAN_DPACK. */
PI_API void packinfer_default_config(pi_config* cfg);

/* ---- plan tables (host, written by packinfer_plan; compared bit-exactly with the oracle) -- */
typedef struct { int32_t request, piece, kv_begin, kv_len, group; } pi_piece;
/* O_g entry (Alg. 1 l.12): (Delta_prefix, L_P, Delta_suffix, L_Q), group-local.     */
typedef struct { int32_t d_prefix, l_prefix, d_suffix, l_suffix; } pi_offset;
/* Group S_g: global buffer base, L(S_g) (dedup tokens), member count, capacity incl. delta. */
typedef struct { int64_t base; int32_t load, members, cap, reserved; } pi_group;
/* Copy(M_paged[src] -> B_g): src_kind 0 = request block table row src_id, 1 = prefix src_id;
 * logical tokens [src_begin, src_begin+len) -> buffer tokens [dst, dst+len).                */
typedef struct { int32_t src_kind, src_id, src_begin, len; int64_t dst; } pi_copy;

/* ---- packed execution domain (implementation-side; checked by the coverage invariant) ---- */
/* A work item: <= tile_q query rows attending over span_count key spans (buffer tokens).
 * Every span but the last is fully visible to every row; in the last span row r sees keys
 * [rows[r].lo, rows[r].hi).  Items are LPT-sorted by n_ktiles (descending).               */
typedef struct {
  int32_t kind;       /* 0 = prefill (rows are tokens, one Q head per launch unit)
                         1 = decode  (rows are (request, GQA head), one KV head per unit)   */
  int32_t group;      /* group of the last span                                             */
  int32_t row_begin, row_count;
  int32_t span_begin, span_count;
  int32_t n_ktiles;   /* cost: sum over spans of ceil(len / tile_k)                         */
  int32_t reserved;
} pi_work;
/* A query row: token index into q/out, visible interval [lo, hi) in the last span, and
 * out = ((slot + 1) << 4) | h_sub, slot = -1 for a direct write, h_sub = GQA sub-head
 * (decode rows; 0 for prefill rows).                                                       */
typedef struct { int32_t q_token, lo, hi, out; } pi_row;
typedef struct { int32_t begin, len; } pi_span;
/* A row segment: `count` consecutive rows [row_begin, row_begin + count) of the row table, row j
 * of the segment being
 *   PI_SEG_PREFILL: {q_token + j, lo, hi + j, out}   (consecutive query positions of one piece:
 *                   the causal own-suffix gains one key per row)
 *   PI_SEG_DECODE:  {q_token, lo, hi, out | j}       (GQA sub-head j of one decode request)
 * The planner emits segments (O(requests + work items) host work); packinfer_plan_upload expands
 * them into the device row table and packinfer_plan_rows into a host one.                  */
typedef struct { int32_t row_begin, count, q_token, lo, hi, out, kind, reserved; } pi_rowseg;
#define PI_SEG_PREFILL 0
#define PI_SEG_DECODE 1
/* Merge entry: output token q_token combines partial slots [slot_begin, slot_begin+count). */
typedef struct { int32_t q_token, slot_begin, slot_count, reserved; } pi_merge;

typedef struct {
  /* all pointers point into the caller's host arena (packinfer_plan) */
  pi_piece* pieces;    int32_t n_pieces;
  pi_offset* offsets;  /* indexed like pieces */
  pi_group* groups;    int32_t n_groups;   int32_t g0;
  pi_copy* copies;     int32_t n_copies;
  int64_t* copy_prefix;                    /* [n_copies+1] cumsum of cells per copy: len (+ headroom
                                              after a suffix); copy_prefix[n_copies] == buffer_tokens */
  pi_work* prefill_work; int32_t n_prefill_work;
  pi_work* decode_work;  int32_t n_decode_work;
  pi_rowseg* segs;     int32_t n_segs;   /* row segments (host); the row table itself is
                                              expanded on the device (packinfer_plan_upload)   */
  int32_t n_rows;                          /* rows of the expanded table                      */
  pi_span* spans;      int32_t n_spans;
  pi_merge* merges;    int32_t n_merges;   int32_t n_partial_slots;
  int32_t* slot_merge;                     /* [n_partial_slots] merge entry of each slot   */
  int64_t buffer_tokens;                   /* sum of group capacities                    */
  int64_t copy_tokens;                     /* Eq. 5 volume = sum of loads                */
  int32_t n_requests, n_prefix, total_q, gqa_ratio;
  int64_t eta_num, eta_den;                /* literal Eq. 1 with T = tile_k       */
  int64_t valid_cells, tile_cells;         /* prefill tile efficiency (reading R-eta)     */
  int32_t discrepancy;                     /* Eq. 3                               */
  int32_t reserved;
  int32_t* append_pos;   /* [n] buffer token where request i's next decode token goes (headroom,
                            P:306-309), -1 if none (not a decode request / headroom exhausted) */
  int64_t drift;         /* Eq. 4 dL = max_g L(S_g) - min_g L(S_g) including appended tokens    */
  int64_t appended_total;
  void* arena;  size_t arena_bytes;        /* the host arena holding every table          */
  size_t rows_offset;                      /* byte offset of the row table in the DEVICE arena */
  size_t sched_offset;                     /* byte offset of the attention launches' dynamic
                                              scheduler counter in the DEVICE arena            */
  size_t device_arena_bytes;               /* device arena size: host tables + row table +
                                              scheduler counter                               */
} pi_plan;

/* Alg. 1 Parts 1-2 plus the packed execution domain.
 *   n, kv_len[n] (>= 1), q_len[n] (1 <= q_len <= kv_len; the last q_len positions are the
 *   queries; q_len == 1 rows take the decode path), prefix_id[n] (-1 = none, else
 *   < n_prefix; may be NULL), prefix_len[n_prefix] (1 <= prefix_len[p] <= kv_len - q_len of
 *   every member).  All host pointers.
 *   host_arena/arena_bytes: caller host memory (pinned memory makes the upload async).
 *   If arena_bytes is too small returns PI_ENOSPC and sets out->arena_bytes to the size
 *   needed (two-call sizing; NULL/0 is allowed for the first call).                        */
PI_API pi_status packinfer_plan(int32_t n, const int32_t* kv_len, const int32_t* q_len,
                         const int32_t* prefix_id, int32_t n_prefix, const int32_t* prefix_len,
                         const pi_config* cfg, void* host_arena, size_t arena_bytes,
                         pi_plan* out);

/* Decode loop without re-consolidation.  Same inputs as packinfer_plan
 * (the lengths of the last consolidation) plus appended[n] (host): the number of decode tokens
 * request i has appended into its suffix headroom since then (packinfer_append_kv).  Groups,
 * offsets and the copy plan are those of packinfer_plan on the same inputs (bit-identical); the
 * execution domain covers kv_len[i] + appended[i] keys.  appended[i] > 0 requires q_len[i] == 1;
 * appended[i] > headroom returns PI_EREGROUP (the caller must regroup: re-plan + relayout).  */
PI_API pi_status packinfer_plan_step(int32_t n, const int32_t* kv_len, const int32_t* q_len,
                                     const int32_t* prefix_id, int32_t n_prefix,
                                     const int32_t* prefix_len, const int32_t* appended,
                                     const pi_config* cfg, void* host_arena, size_t arena_bytes,
                                     pi_plan* out);

/* Eq. 4: 1 iff steps * drift >= capacity / 2 (inclusive, exact integer test). */
PI_API int32_t packinfer_should_regroup(int32_t steps, int64_t drift, int32_t capacity);

/* Expands the plan's row segments into rows[0 .. plan->n_rows) (host memory, caller-owned,
 * cap >= n_rows else PI_ENOSPC): the same table packinfer_plan_upload builds on the device.   */
PI_API pi_status packinfer_plan_rows(const pi_plan* plan, pi_row* rows, int32_t cap);

/* Device view of a plan: the same tables in device memory. */
typedef struct {
  const pi_copy* copies;  const int64_t* copy_prefix; int32_t n_copies; int64_t copy_tokens;
  const pi_work* prefill_work; int32_t n_prefill_work;
  const pi_work* decode_work;  int32_t n_decode_work;
  const pi_row* rows;  const pi_span* spans;
  const pi_merge* merges; int32_t n_merges; int32_t n_partial_slots;
  int64_t buffer_tokens;
  int32_t n_requests, total_q, gqa_ratio, tile_k;
  const int32_t* append_pos;                 /* [n_requests] (see pi_plan)                      */
  const int32_t* slot_merge;                 /* [n_partial_slots] (see pi_plan); NULL disables
                                                packinfer_attention_merge                        */
  uint32_t* sched;                           /* [4] two (unit counter, exits) pairs of the
                                                attention launches (the second for the decode half
                                                of a prefill + decode call): zeroed by
                                                packinfer_plan_upload, left at zero by every
                                                completed launch (the last CTA resets them), so
                                                one attention call per device plan at a time     */
} pi_device_plan;

/* Enqueue one host->device copy of plan->arena (arena_bytes) into dev_arena (device, >=
 * plan->device_arena_bytes, 256-byte aligned) and one small kernel that expands the row
 * segments into the row table at dev_arena + rows_offset (and zeroes the scheduler counters at
 * dev_arena + sched_offset), both on `stream`; fill *out with device pointers into dev_arena. */
PI_API pi_status packinfer_plan_upload(const pi_plan* plan, void* dev_arena, size_t dev_bytes,
                                pi_stream_t stream, pi_device_plan* out);

/* ------------------------------------------------------------------------------------------
 * Contiguous memory consolidation (Alg. 1 Copy lines P:244/P:250; §3.2):
 * gather every copy-plan entry from the paged cache into k_buf/v_buf for KV heads
 * [hkv_begin, hkv_begin + hkv_count).  Bitwise copy of K and V; headroom cells
 * are zero-filled.  The cells written are those of the device plan's copy list (copy_prefix
 * [n_copies] of them; a batch plan covers all buffer_tokens).  A caller may pass a device plan
 * whose copies / copy_prefix are a subsequence of the batch's (group sharding of one batch,
 * SURVEY 8(e)): destinations stay in batch coordinates, k_buf/v_buf keep buffer_tokens rows.
 * ---------------------------------------------------------------------------------------- */
PI_API pi_status packinfer_relayout_kv(const pi_device_plan* dp, const void* k_paged,
                                const void* v_paged, const int32_t* block_table,
                                int32_t max_blocks, int32_t page_size, int32_t hkv_total,
                                int32_t hkv_begin, int32_t hkv_count, int32_t head_dim,
                                pi_dtype dt, void* k_buf, void* v_buf, pi_stream_t stream);

/* Append one decode token per request into its headroom slot (plan->append_pos):
 * k_new / v_new [n_requests, hkv_total, head_dim] (host layout of one paged token row; rows of
 * requests without a slot are ignored), heads [hkv_begin, hkv_begin + hkv_count) -> k_buf / v_buf
 * (V stored as in packinfer_relayout_kv).  Follow with packinfer_plan_step(appended + 1).      */
PI_API pi_status packinfer_append_kv(const pi_device_plan* dp, const void* k_new, const void* v_new,
                                     int32_t hkv_total, int32_t hkv_begin, int32_t hkv_count,
                                     int32_t head_dim, pi_dtype dt, void* k_buf, void* v_buf,
                                     pi_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * Packed attention ("union of valid query-key regions"; P:172 one launch for every
 * group): ONE persistent launch over all prefill (resp. decode) work items x local heads.
 * S = scale * Q K^T and O += P V run on tcgen05 (TMEM accumulators, TMA-fed K/V), softmax is
 * online with fp32 statistics; bf16 Q/K/V, fp32 accumulation, P rounded to bf16 for P.V
 * (reading R13; PI_FP32 uses kind::tf32).  q/out: local heads [0, hkv_count*gqa_ratio) of each token
 * (strides in elements); rows with a single result write out/lse directly, split rows write
 * (o, lse) to partial slots for packinfer_merge.  head_dim in {64, 128}.
 * lse may be NULL.  softmax_scale <= 0 selects 1/sqrt(head_dim).
 * ---------------------------------------------------------------------------------------- */
PI_API pi_status packinfer_attention_prefill(const pi_device_plan* dp, const void* q,
                                      int64_t q_row_stride, const void* k_buf,
                                      const void* v_buf, int32_t hkv_count, int32_t gqa_ratio,
                                      int32_t head_dim, float softmax_scale, pi_dtype dt,
                                      void* out, int64_t out_row_stride, float* lse,
                                      float* partial_o, float* partial_lse, pi_stream_t stream);

PI_API pi_status packinfer_attention_decode(const pi_device_plan* dp, const void* q,
                                     int64_t q_row_stride, const void* k_buf,
                                     const void* v_buf, int32_t hkv_count, int32_t gqa_ratio,
                                     int32_t head_dim, float softmax_scale, pi_dtype dt,
                                     void* out, int64_t out_row_stride, float* lse,
                                     float* partial_o, float* partial_lse, pi_stream_t stream);

/* Fused form (NEXT-3; BASELINE.json north star "one packed attention kernel launch
 * per layer ... covering both prefill and decode"): ONE call over the prefill AND the decode
 * work items of the plan.  For bf16 operands with both kinds present it is two persistent
 * launches of the kernel's specialised instances - prefill units, then decode units as a
 * programmatic dependent launch whose CTAs fill the SMs the prefill launch frees at its tail;
 * otherwise (and when built with -DPI_FUSED_PDL=0) one persistent launch of the mixed instance
 * (prefill units first, the cheaper decode units fill the tail).  Arguments, layouts and errors
 * as above; q/out hold every request's rows (q_len = 1 for decode requests) in the caller's
 * varlen order.  Results are bitwise those of packinfer_attention_prefill followed by
 * packinfer_attention_decode.                                                                   */
PI_API pi_status packinfer_attention(const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                     const void* k_buf, const void* v_buf, int32_t hkv_count,
                                     int32_t gqa_ratio, int32_t head_dim, float softmax_scale,
                                     pi_dtype dt, void* out, int64_t out_row_stride, float* lse,
                                     float* partial_o, float* partial_lse, pi_stream_t stream);

/* Packed decode straight from the paged KV cache (NEXT-4 ablation; plans made with PI_PLAN_PAGED):
 * the same kernel as packinfer_attention_decode, but each 128-key tile is one TMA box of the
 * paged cache k/v_paged [num_blocks, page_size, hkv_total, head_dim] at the block the request's
 * block_table row maps (page_size a multiple of 128).  KV heads [hkv_begin, hkv_begin+hkv_count);
 * q/out/partials as in packinfer_attention_decode.  PI_BF16 / PI_BF16_OUT_F32, head_dim 64/128. */
PI_API pi_status packinfer_attention_decode_paged(const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                                  const void* k_paged, const void* v_paged,
                                                  const int32_t* block_table, int32_t max_blocks,
                                                  int32_t page_size, int32_t num_blocks, int32_t hkv_total,
                                                  int32_t hkv_begin, int32_t hkv_count, int32_t gqa_ratio,
                                                  int32_t head_dim, float softmax_scale, pi_dtype dt, void* out,
                                                  int64_t out_row_stride, float* lse, float* partial_o,
                                                  float* partial_lse, pi_stream_t stream);

/* Fully fused form (NEXT-3; "reducing ... kernel launch overhead"): as
 * packinfer_attention, and the LSE merge of split rows happens inside the same launch - the CTA
 * that writes the LAST partial of a (split row, head) merges it (last-arriver epilogue: partials
 * fenced, then one atomic per (row, head) on merge_counters), with packinfer_merge's arithmetic in
 * the same order (outputs bitwise equal to packinfer_attention + packinfer_merge).
 * merge_counters: device uint32 [n_merges * hkv_count * gqa_ratio], all ZERO on entry (e.g. one
 * cudaMemset at allocation); the kernel leaves them zero when it completes.  partial_o /
 * partial_lse are still written (the merge reads them back).                                  */
PI_API pi_status packinfer_attention_merge(const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                           const void* k_buf, const void* v_buf, int32_t hkv_count,
                                           int32_t gqa_ratio, int32_t head_dim, float softmax_scale,
                                           pi_dtype dt, void* out, int64_t out_row_stride, float* lse,
                                           float* partial_o, float* partial_lse, uint32_t* merge_counters,
                                           pi_stream_t stream);

/* ------------------------------------------------------------------------------------------
 * Lossless LSE merge of split rows (reading R10):
 *   M = max_b lse_b; w_b = exp(lse_b - M); o = sum w_b o_b / sum w_b; lse = M + ln sum w_b,
 * empty partials (lse = -inf) carry zero weight.  Writes out (dt) and lse for every merge
 * entry and every local head.
 * ---------------------------------------------------------------------------------------- */
PI_API pi_status packinfer_merge(const pi_device_plan* dp, const float* partial_o,
                          const float* partial_lse, int32_t hq_count, int32_t head_dim,
                          pi_dtype dt, void* out, int64_t out_row_stride, float* lse,
                          pi_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* PACKINFER_H_ */
