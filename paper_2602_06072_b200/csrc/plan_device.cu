// Plan upload: one H2D copy of the host tables + the device-side expansion of the row segments
// into the row table the attention kernel reads (include/packinfer.h, pi_rowseg).  Host planning
// stays O(requests + work items); the O(query rows) table is built here, off the host's critical
// path (cfg5: 289k rows).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "common.h"
#include "device_common.h"
#include "packinfer.h"

namespace pi {

// One CTA per segment (<= 128 rows each, r <= 16 for decode segments): thread j writes row j.
// CTA 0 also zeroes the attention launches' scheduler counters (pi_device_plan.sched).
__global__ void __launch_bounds__(128) expand_rows_kernel(const pi_rowseg* __restrict__ segs, pi_row* __restrict__ rows,
                                                          uint32_t* __restrict__ sched) {
  if (blockIdx.x == 0 && threadIdx.x < 4) sched[threadIdx.x] = 0u;   // two (counter, exits) pairs
  const pi_rowseg g = segs[blockIdx.x];
  for (int j = threadIdx.x; j < g.count; j += blockDim.x) {
    const bool pre = g.kind == PI_SEG_PREFILL;
    int4 v;
    v.x = pre ? g.q_token + j : g.q_token;
    v.y = g.lo;
    v.z = pre ? g.hi + j : g.hi;
    v.w = pre ? g.out : (g.out | j);
    reinterpret_cast<int4*>(rows)[g.row_begin + j] = v;
  }
}

}  // namespace pi

extern "C" pi_status packinfer_plan_upload(const pi_plan* p, void* dev_arena, size_t dev_bytes, pi_stream_t stream,
                                           pi_device_plan* out) {
  if (!p || !out) return pi::fail(PI_EINVAL, "plan and out must be non-NULL");
  if (!p->arena) return pi::fail(PI_EINVAL, "plan has no host arena (planning failed?)");
  if (!dev_arena || dev_bytes < p->device_arena_bytes)
    return pi::fail(PI_ENOSPC, "device arena too small: need " + std::to_string(p->device_arena_bytes));
  if (reinterpret_cast<uintptr_t>(dev_arena) % 256) return pi::fail(PI_EINVAL, "device arena must be 256-byte aligned");
  if (p->n_rows > 0 && (!p->segs || p->n_segs < 1)) return pi::fail(PI_EINVAL, "plan has rows but no segments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dev_arena, p->arena, p->arena_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return pi::fail(PI_ECUDA, std::string("plan upload: ") + cudaGetErrorString(e));
  const char* H = static_cast<const char*>(p->arena);
  char* D = static_cast<char*>(dev_arena);
  auto dev = [&](const void* h) -> const void* {
    return h ? static_cast<const void*>(D + (static_cast<const char*>(h) - H)) : nullptr;
  };
  pi_row* rows = reinterpret_cast<pi_row*>(D + p->rows_offset);
  uint32_t* sched = reinterpret_cast<uint32_t*>(D + p->sched_offset);
  if (p->n_segs > 0) {
    pi::expand_rows_kernel<<<p->n_segs, 128, 0, st>>>(static_cast<const pi_rowseg*>(dev(p->segs)), rows, sched);
    pi_status s = pi::cuda_check(cudaGetLastError(), "expand_rows_kernel launch");
    if (s != PI_OK) return s;
  } else {
    e = cudaMemsetAsync(sched, 0, 4 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return pi::fail(PI_ECUDA, std::string("plan upload: ") + cudaGetErrorString(e));
  }
  std::memset(out, 0, sizeof(*out));
  out->copies = static_cast<const pi_copy*>(dev(p->copies));
  out->copy_prefix = static_cast<const int64_t*>(dev(p->copy_prefix));
  out->n_copies = p->n_copies;
  out->copy_tokens = p->copy_tokens;
  out->prefill_work = static_cast<const pi_work*>(dev(p->prefill_work));
  out->n_prefill_work = p->n_prefill_work;
  out->decode_work = static_cast<const pi_work*>(dev(p->decode_work));
  out->n_decode_work = p->n_decode_work;
  out->rows = rows;
  out->spans = static_cast<const pi_span*>(dev(p->spans));
  out->merges = static_cast<const pi_merge*>(dev(p->merges));
  out->n_merges = p->n_merges;
  out->n_partial_slots = p->n_partial_slots;
  out->append_pos = static_cast<const int32_t*>(dev(p->append_pos));
  out->slot_merge = static_cast<const int32_t*>(dev(p->slot_merge));
  out->sched = sched;
  out->buffer_tokens = p->buffer_tokens;
  out->n_requests = p->n_requests;
  out->total_q = p->total_q;
  out->gqa_ratio = p->gqa_ratio;
  out->tile_k = 128;
  return pi::ok();
}
