// Contiguous memory consolidation (PackInfer §3.2; Alg. 1 Copy lines P:244/P:250).
//
// Gathers every copy-plan entry from the paged KV cache [num_blocks, page, Hkv, d] into the
// group-contiguous buffers [hkv_count, buffer_tokens, d]: K and V are copied bitwise (R-layout).
// One warp per RL_TPW consecutive buffer
// tokens (one 32-ary search for their copy entry): per token it reads the hkv_count*d contiguous
// elements of all local heads of one paged slot (coalesced) and scatters them into the per-head
// buffers.  Cells in a suffix's headroom (delta) are
// written with zeros so every buffer cell is finite (the attention kernels read whole 128-key
// tiles; masked keys meet P = 0, which must not multiply NaN garbage).
// HBM-bound: algorithmic bytes = 2 (K,V) x copied tokens x hkv_count x d x elem (read + write).
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.h"
#include "packinfer.h"

namespace pi {

struct RelayoutParams {
  const pi_copy* copies;
  const int64_t* ext_prefix;  // [n_copies + 1] cumsum of buffer cells per copy (len + headroom)
  int32_t n_copies;
  int64_t total;              // buffer_tokens: grid size (an upper bound of the cells to write)
  int32_t n_requests;
  const uint8_t* kp;
  const uint8_t* vp;
  const int32_t* bt;
  int32_t max_blocks;
  int32_t page;
  int64_t token_bytes;        // hkv_total * d * es  (one paged slot, all heads)
  int64_t head_off_bytes;     // hkv_begin * d * es
  int32_t chunks;             // hkv_count * d * es / 16
  int32_t head_chunks;        // d * es / 16
  int64_t buf_head_bytes;     // buffer_tokens * d * es
  uint8_t* kb;
  uint8_t* vb;
  int32_t tpw;                // buffer tokens per warp: 1, or 128 / chunks when a token is < 128 chunks
};

#ifndef PI_RL_TPW
#define PI_RL_TPW 1
#endif
#ifndef PI_RL_MULTI
#define PI_RL_MULTI 1   // several tokens per warp when a token has < 128 chunks of 16 B (few local KV heads)
#endif
constexpr int RL_TPW = PI_RL_TPW;   // consecutive buffer tokens per warp (one copy-entry search)
constexpr int RL_U = 4;             // 16-byte chunks per lane in flight per tensor
#ifndef PI_RLM_U
#define PI_RLM_U 4
#endif
constexpr int RLM_U = PI_RLM_U;     // the same for the several-tokens-per-warp path

// Largest c with ext_prefix[c] <= g (ext_prefix strictly increasing, ext_prefix[0] = 0 <= g):
// 32-ary warp search, each round narrows [lo, hi] ~32x with one coalesced probe per lane, so the
// dependent-load chain is log32(n_copies) deep instead of log2.
__device__ __forceinline__ int find_copy(const int64_t* __restrict__ ext_prefix, int n, int64_t g, int lane) {
  int lo = 0, hi = n - 1;
  while (hi > lo) {
    const int64_t span = hi - lo;
    const int c = lo + (int)((span * (lane + 1) + 31) / 32);   // lane 31 probes hi
    const bool le = __ldg(&ext_prefix[c]) <= g;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    const int k = __popc(m);                                   // probes are monotone: a prefix is true
    const int c_prev = k > 0 ? lo + (int)((span * k + 31) / 32) : lo;
    const int c_next = k < 32 ? lo + (int)((span * (k + 1) + 31) / 32) - 1 : hi;
    lo = c_prev;
    hi = c_next;
  }
  return lo;
}

// Few local KV heads (KV-head sharding: 1-4 heads per rank) make a token only 16-64 chunks of
// 16 B, so one token per warp leaves most lanes idle behind a chain of dependent loads (copy-entry
// search, copy entry, block table, data).  Then a warp takes p.tpw = 128 / chunks consecutive
// tokens and each lane 4 (token, chunk) pairs of them: every warp moves 2 x 2 KB per chain.
__device__ __forceinline__ void relayout_multi(const RelayoutParams& p, int64_t g0, int lane) {
  const int64_t total = __ldg(&p.ext_prefix[p.n_copies]);
  const int c0 = find_copy(p.ext_prefix, p.n_copies, g0, lane);
  const int64_t row_bytes = (int64_t)p.head_chunks * 16;
  uint4 kv[RLM_U], vv[RLM_U];
  int64_t dsts[RLM_U];
  bool live[RLM_U];
#pragma unroll
  for (int u = 0; u < RLM_U; ++u) {
    const int f = u * 32 + lane;
    const int64_t g = g0 + f / p.chunks;
    const int i = f % p.chunks;
    live[u] = f < p.tpw * p.chunks && g < total;
    kv[u] = vv[u] = make_uint4(0, 0, 0, 0);
    dsts[u] = 0;
    if (live[u]) {
      int c = c0;
      while (c + 1 < p.n_copies && g >= __ldg(&p.ext_prefix[c + 1])) ++c;   // a copy ends inside the warp
      const pi_copy cp = p.copies[c];
      const int64_t off = g - __ldg(&p.ext_prefix[c]);
      const int h = i / p.head_chunks, cc = i % p.head_chunks;
      dsts[u] = h * p.buf_head_bytes + (cp.dst + off) * row_bytes + (int64_t)cc * 16;
      if (off < cp.len) {   // else headroom: zeros
        const int row = cp.src_kind == 0 ? cp.src_id : p.n_requests + cp.src_id;
        const int64_t j = cp.src_begin + off;
        const int blk = __ldg(&p.bt[(int64_t)row * p.max_blocks + j / p.page]);
        const int64_t src = ((int64_t)blk * p.page + j % p.page) * p.token_bytes + p.head_off_bytes;
        kv[u] = __ldg(reinterpret_cast<const uint4*>(p.kp + src) + i);
        vv[u] = __ldg(reinterpret_cast<const uint4*>(p.vp + src) + i);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < RLM_U; ++u) {
    if (live[u]) {
      *reinterpret_cast<uint4*>(p.kb + dsts[u]) = kv[u];
      *reinterpret_cast<uint4*>(p.vb + dsts[u]) = vv[u];
    }
  }
}

__global__ void __launch_bounds__(256) relayout_kernel(const RelayoutParams p) {
  const int lane = threadIdx.x & 31;
  if (p.tpw > 1) {
    const int64_t g0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * p.tpw;
    if (g0 >= __ldg(&p.ext_prefix[p.n_copies])) return;
    relayout_multi(p, g0, lane);
    return;
  }
  const int64_t g0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * RL_TPW;
  // cells to write = the copy list's own cell count (== buffer_tokens for a batch plan; a rank's
  // share under group sharding, shard.RankPlan, is smaller: the grid covers buffer_tokens)
  const int64_t total = __ldg(&p.ext_prefix[p.n_copies]);
  if (g0 >= total) return;
  int c = find_copy(p.ext_prefix, p.n_copies, g0, lane);
  int64_t next = c + 1 < p.n_copies ? __ldg(&p.ext_prefix[c + 1]) : INT64_MAX;
  const int64_t row_bytes = (int64_t)p.head_chunks * 16;
  const int64_t g_end = min(g0 + RL_TPW, total);
  for (int64_t g = g0; g < g_end; ++g) {
    while (g >= next) {   // next copy entry (copies are long: rarely taken)
      ++c;
      next = c + 1 < p.n_copies ? __ldg(&p.ext_prefix[c + 1]) : INT64_MAX;
    }
    const pi_copy cp = p.copies[c];
    const int64_t off = g - __ldg(&p.ext_prefix[c]);
    const int64_t dst = cp.dst + off;
    if (off < cp.len) {
      const int row = cp.src_kind == 0 ? cp.src_id : p.n_requests + cp.src_id;
      const int64_t j = cp.src_begin + off;
      const int blk = __ldg(&p.bt[(int64_t)row * p.max_blocks + j / p.page]);
      const int64_t src = ((int64_t)blk * p.page + j % p.page) * p.token_bytes + p.head_off_bytes;
      for (int base = 0; base < p.chunks; base += 32 * RL_U) {
        uint4 kv[RL_U], vv[RL_U];
#pragma unroll
        for (int u = 0; u < RL_U; ++u) {
          const int i = base + u * 32 + lane;
          if (i < p.chunks) {
            kv[u] = __ldg(reinterpret_cast<const uint4*>(p.kp + src) + i);
            vv[u] = __ldg(reinterpret_cast<const uint4*>(p.vp + src) + i);
          }
        }
#pragma unroll
        for (int u = 0; u < RL_U; ++u) {
          const int i = base + u * 32 + lane;
          if (i < p.chunks) {
            const int h = i / p.head_chunks, cc = i % p.head_chunks;
            const int64_t d = h * p.buf_head_bytes + dst * row_bytes + (int64_t)cc * 16;
            *reinterpret_cast<uint4*>(p.kb + d) = kv[u];
            *reinterpret_cast<uint4*>(p.vb + d) = vv[u];
          }
        }
      }
    } else {
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (int i = lane; i < p.chunks; i += 32) {
        const int h = i / p.head_chunks, cc = i % p.head_chunks;
        const int64_t d = h * p.buf_head_bytes + dst * row_bytes + (int64_t)cc * 16;
        *reinterpret_cast<uint4*>(p.kb + d) = z;
        *reinterpret_cast<uint4*>(p.vb + d) = z;
      }
    }
  }
}

// One warp per request: copy its new token's hkv_count*d K and V elements into the headroom slot
// append_pos[i] of every local head ("allows multiple decoding iterations to proceed
// without triggering re-alignment").
__global__ void __launch_bounds__(256) append_kernel(const int32_t* __restrict__ append_pos, int32_t n,
                                                      const uint8_t* kn, const uint8_t* vn, int64_t token_bytes,
                                                      int64_t head_off_bytes, int32_t chunks, int32_t head_chunks,
                                                      int64_t buf_head_bytes, uint8_t* kb, uint8_t* vb) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int32_t dst = append_pos[i];
  if (dst < 0) return;
  const int64_t row_bytes = (int64_t)head_chunks * 16;
  const uint8_t* ks = kn + i * token_bytes + head_off_bytes;
  const uint8_t* vs = vn + i * token_bytes + head_off_bytes;
  for (int c = lane; c < chunks; c += 32) {
    const int h = c / head_chunks, cc = c % head_chunks;
    const int64_t d = h * buf_head_bytes + (int64_t)dst * row_bytes + (int64_t)cc * 16;
    const uint4 kv = reinterpret_cast<const uint4*>(ks)[c];
    const uint4 vv = reinterpret_cast<const uint4*>(vs)[c];
    *reinterpret_cast<uint4*>(kb + d) = kv;
    *reinterpret_cast<uint4*>(vb + d) = vv;
  }
}

}  // namespace pi

extern "C" pi_status packinfer_append_kv(const pi_device_plan* dp, const void* k_new, const void* v_new,
                                         int32_t hkv_total, int32_t hkv_begin, int32_t hkv_count,
                                         int32_t head_dim, pi_dtype dt, void* k_buf, void* v_buf,
                                         pi_stream_t stream) {
  using namespace pi;
  if (!dp) return fail(PI_EINVAL, "device plan is NULL");
  if (dp->n_requests == 0 || dp->buffer_tokens == 0) return ok();
  if (!k_new || !v_new || !k_buf || !v_buf || !dp->append_pos) return fail(PI_EINVAL, "NULL pointer argument");
  if (hkv_total < 1 || hkv_begin < 0 || hkv_count < 1 || hkv_begin + hkv_count > hkv_total)
    return fail(PI_EINVAL, "KV head range out of bounds");
  if (dt != PI_BF16 && dt != PI_FP32) return fail(PI_EUNSUP, "dtype must be PI_BF16 or PI_FP32");
  const int es = dt == PI_BF16 ? 2 : 4;
  if ((head_dim * es) % 16) return fail(PI_EINVAL, "head_dim * element size must be a multiple of 16 bytes");
  if ((reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new) |
       reinterpret_cast<uintptr_t>(k_buf) | reinterpret_cast<uintptr_t>(v_buf)) % 16)
    return fail(PI_EINVAL, "tensors must be 16-byte aligned");
  const int32_t head_chunks = head_dim * es / 16;
  const unsigned blocks = (unsigned)((dp->n_requests + 7) / 8);
  append_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      dp->append_pos, dp->n_requests, static_cast<const uint8_t*>(k_new), static_cast<const uint8_t*>(v_new),
      (int64_t)hkv_total * head_dim * es, (int64_t)hkv_begin * head_dim * es, hkv_count * head_chunks, head_chunks,
      dp->buffer_tokens * head_dim * es, static_cast<uint8_t*>(k_buf), static_cast<uint8_t*>(v_buf));
  pi_status s = cuda_check(cudaGetLastError(), "append_kernel launch");
  return s == PI_OK ? ok() : s;
}

extern "C" pi_status packinfer_relayout_kv(const pi_device_plan* dp, const void* k_paged, const void* v_paged,
                                           const int32_t* block_table, int32_t max_blocks, int32_t page_size,
                                           int32_t hkv_total, int32_t hkv_begin, int32_t hkv_count,
                                           int32_t head_dim, pi_dtype dt, void* k_buf, void* v_buf,
                                           pi_stream_t stream) {
  using namespace pi;
  if (!dp) return fail(PI_EINVAL, "device plan is NULL");
  if (dp->buffer_tokens == 0) return ok();
  if (!k_paged || !v_paged || !block_table || !k_buf || !v_buf) return fail(PI_EINVAL, "NULL pointer argument");
  if (max_blocks < 1 || page_size < 1) return fail(PI_EINVAL, "max_blocks and page_size must be >= 1");
  if (hkv_total < 1 || hkv_begin < 0 || hkv_count < 1 || hkv_begin + hkv_count > hkv_total)
    return fail(PI_EINVAL, "KV head range out of bounds");
  if (dt != PI_BF16 && dt != PI_FP32) return fail(PI_EUNSUP, "dtype must be PI_BF16 or PI_FP32");
  const int es = dt == PI_BF16 ? 2 : 4;
  if ((head_dim * es) % 16) return fail(PI_EINVAL, "head_dim * element size must be a multiple of 16 bytes");
  if ((reinterpret_cast<uintptr_t>(k_paged) | reinterpret_cast<uintptr_t>(v_paged) |
       reinterpret_cast<uintptr_t>(k_buf) | reinterpret_cast<uintptr_t>(v_buf)) % 16)
    return fail(PI_EINVAL, "tensors must be 16-byte aligned");
  RelayoutParams p{};
  p.copies = dp->copies;
  p.ext_prefix = dp->copy_prefix;
  p.n_copies = dp->n_copies;
  p.total = dp->buffer_tokens;
  p.n_requests = dp->n_requests;
  p.kp = static_cast<const uint8_t*>(k_paged);
  p.vp = static_cast<const uint8_t*>(v_paged);
  p.bt = block_table;
  p.max_blocks = max_blocks;
  p.page = page_size;
  p.token_bytes = (int64_t)hkv_total * head_dim * es;
  p.head_off_bytes = (int64_t)hkv_begin * head_dim * es;
  p.head_chunks = head_dim * es / 16;
  p.chunks = hkv_count * p.head_chunks;
  p.buf_head_bytes = dp->buffer_tokens * head_dim * es;
  p.kb = static_cast<uint8_t*>(k_buf);
  p.vb = static_cast<uint8_t*>(v_buf);
  p.tpw = (PI_RL_MULTI && p.chunks < 32 * RLM_U) ? (32 * RLM_U) / p.chunks : 1;
  const int64_t per_warp = p.tpw > 1 ? p.tpw : RL_TPW;
  const int64_t blocks = (p.total + 8 * per_warp - 1) / (8 * per_warp);
  if (blocks > 0x7fffffff) return fail(PI_EINVAL, "buffer too large");
  relayout_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  pi_status s = cuda_check(cudaGetLastError(), "relayout_kernel launch");
  return s == PI_OK ? ok() : s;
}
