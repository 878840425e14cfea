// Lossless LSE merge of split rows (PackInfer §1, "merged in a lossless manner consistent
// with FlashAttention semantics"; equations per reading R10):
//   M = max_b lse_b,  w_b = exp(lse_b - M),  o = sum_b w_b o_b / sum_b w_b,  lse = M + ln sum_b w_b
// One warp per (merge entry, local head); lanes own d/32 channels, so every partial row is read
// as contiguous 128-byte segments.  HBM-bound and tiny next to the KV stream it follows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "device_common.h"
#include "packinfer.h"

#ifndef PI_CHECKS
#define PI_CHECKS 0   // debug build: bounds checks on the merge table (see attention.cu)
#endif

namespace pi {

template <int D, bool F32>
__global__ void __launch_bounds__(256) merge_kernel(const pi_merge* __restrict__ merges, int32_t n_merges,
                                                    const float* __restrict__ po, const float* __restrict__ pl,
                                                    int32_t hq, uint8_t* out, int64_t out_row_stride, float* lse,
                                                    int32_t total_q, int32_t n_slots) {
  // launched as a programmatic dependent of the attention launch that wrote the partials
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= (int64_t)n_merges * hq) return;
  const int m = (int)(gw / hq), h = (int)(gw % hq);
  const pi_merge mg = merges[m];
#if PI_CHECKS
  if (!(mg.slot_begin >= 0 && mg.slot_count >= 1 && mg.slot_begin + mg.slot_count <= n_slots && mg.q_token >= 0 &&
        mg.q_token < total_q)) {
    printf("packinfer device check 7 failed: merge %d\n", m);
    __trap();
  }
#endif
  float M = -INFINITY;
  for (int b = lane; b < mg.slot_count; b += 32) M = fmaxf(M, __ldcg(&pl[(int64_t)(mg.slot_begin + b) * hq + h]));
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  constexpr int V = D / 32;
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;
  float W = 0.f;
  if (M != -INFINITY) {
    // slots in batches of MB: every load of a batch is in flight at once (the partials were
    // written during the attention launch and mostly evicted from L2 by its KV stream, so each
    // batch is one HBM round trip), then the batch is accumulated in slot order - the same
    // arithmetic in the same order as the in-kernel merge (packinfer_attention_merge), bitwise
    constexpr int MB = 4;
    for (int b0 = 0; b0 < mg.slot_count; b0 += MB) {
      float lw[MB], x[MB][V];
#pragma unroll
      for (int q = 0; q < MB; ++q) {
        if (b0 + q < mg.slot_count) {
          const int64_t sl = mg.slot_begin + b0 + q;
          lw[q] = __ldcg(&pl[sl * hq + h]);
          const float* src = po + (sl * hq + h) * D;
#pragma unroll
          for (int i = 0; i < V; ++i) x[q][i] = __ldcg(src + lane + 32 * i);
        }
      }
#pragma unroll
      for (int q = 0; q < MB; ++q) {
        if (b0 + q < mg.slot_count) {
          const float w = expf(lw[q] - M);
          W += w;
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] += w * x[q][i];
        }
      }
    }
  }
  const float inv = W > 0.f ? 1.f / W : 0.f;
  uint8_t* dst = out + ((int64_t)mg.q_token * out_row_stride + (int64_t)h * D) * (F32 ? 4 : 2);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if constexpr (F32)
      reinterpret_cast<float*>(dst)[lane + 32 * i] = acc[i] * inv;
    else
      reinterpret_cast<__nv_bfloat16*>(dst)[lane + 32 * i] = __float2bfloat16_rn(acc[i] * inv);
  }
  if (lse && lane == 0) lse[(int64_t)h * total_q + mg.q_token] = W > 0.f ? M + logf(W) : -INFINITY;
}

}  // namespace pi

extern "C" pi_status packinfer_merge(const pi_device_plan* dp, const float* partial_o, const float* partial_lse,
                                     int32_t hq_count, int32_t head_dim, pi_dtype dt, void* out,
                                     int64_t out_row_stride, float* lse, pi_stream_t stream) {
  using namespace pi;
  if (!dp) return fail(PI_EINVAL, "device plan is NULL");
  if (dp->n_merges == 0) return ok();
  if (!partial_o || !partial_lse || !out) return fail(PI_EINVAL, "NULL pointer argument");
  if (hq_count < 1) return fail(PI_EINVAL, "hq_count must be >= 1");
  if (out_row_stride < (int64_t)hq_count * head_dim) return fail(PI_EINVAL, "out_row_stride too small");
  const int64_t warps = (int64_t)dp->n_merges * hq_count;
  const unsigned blocks = (unsigned)((warps + 7) / 8);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dt == PI_BF16_OUT_F32) dt = PI_FP32;  // output element type is what the merge writes
  uint8_t* o = static_cast<uint8_t*>(out);
  if (dt == PI_BF16 && head_dim == 128) {
    // programmatic dependent launch: the merge's launch and CTA start overlap the attention
    // launch's tail; griddepcontrol.wait in the kernel orders its reads after it
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, merge_kernel<128, false>, dp->merges, dp->n_merges, partial_o,
                                       partial_lse, hq_count, o, out_row_stride, lse, dp->total_q,
                                       dp->n_partial_slots);
    if (e != cudaSuccess) return cuda_check(e, "merge_kernel launch (PDL)");
  }
  else if (dt == PI_BF16 && head_dim == 64)
    merge_kernel<64, false><<<blocks, 256, 0, st>>>(dp->merges, dp->n_merges, partial_o, partial_lse, hq_count, o,
                                                    out_row_stride, lse, dp->total_q, dp->n_partial_slots);
  else if (dt == PI_FP32 && head_dim == 64)
    merge_kernel<64, true><<<blocks, 256, 0, st>>>(dp->merges, dp->n_merges, partial_o, partial_lse, hq_count, o,
                                                   out_row_stride, lse, dp->total_q, dp->n_partial_slots);
  else if (dt == PI_FP32 && head_dim == 128)
    merge_kernel<128, true><<<blocks, 256, 0, st>>>(dp->merges, dp->n_merges, partial_o, partial_lse, hq_count, o,
                                                    out_row_stride, lse, dp->total_q, dp->n_partial_slots);
  else
    return fail(PI_EUNSUP, "head_dim must be 64 or 128; dtype PI_BF16 or PI_FP32");
  pi_status s = cuda_check(cudaGetLastError(), "merge_kernel launch");
  return s == PI_OK ? ok() : s;
}
