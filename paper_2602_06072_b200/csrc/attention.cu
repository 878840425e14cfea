// Packed attention over the union of valid query-key regions (PackInfer §3.1): ONE
// persistent launch per call covers every work item of every group (reading R18).
//
// Work unit = (work item, head).  A work item holds <= 128 query rows (prefill: tokens of one or
// more packed requests; decode: (request, GQA sub-head) rows) and a list of key spans in
// the group-contiguous KV buffers (Alg. 1 Part 2).  Every span but the last is visible to every
// row; in the last span row r sees keys [lo_r, hi_r) (causal own-suffix / decode chunk).
//
// Per CTA (one per SM, 256 threads, warp-specialised):
//   warp 0  : TMA producer — K and V tiles (128 keys x head_dim, SWIZZLE_128B) into a 2-stage ring
//   warp 1  : TMEM allocator + single-thread tcgen05.mma issuer:
//               S_t = Q K_t^T  -> TMEM S[t%2]      (M=128, N=128, K=head_dim)
//               O  += P_t V_t  -> TMEM O           (M=128, N=head_dim, K=128; V MN-major)
//   warp 2  : Q gather — rows addressed through the plan's row table (cp.async, manual 128B swizzle)
//   warps 4-7: softmax / correction / epilogue; thread i owns row i (= TMEM lane i), so the row max
//             and sum need no cross-thread reduction.  Online softmax in the exp2 domain with a lazy
//             rescale (O is rescaled in TMEM only when the running max grows by > 2^8).
// bf16 operands run tcgen05 kind::f16, fp32 operands kind::tf32; accumulation is fp32 (R13).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "device_common.h"
#include "packinfer.h"
#include "sm100.cuh"

namespace pi {

using namespace sm100;

struct AttnParams {
  const pi_work* work;
  const pi_row* rows;
  const pi_span* spans;
  int32_t n_work;
  int32_t units;      // launch units per item: local Q heads (prefill) or local KV heads (decode)
  int32_t is_decode;
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
};

template <int D, bool F32>
struct AttnCfg {
  static constexpr int ES = F32 ? 4 : 2;
  static constexpr int ROW_BYTES = D * ES;            // one Q/K/V row
  static constexpr int ATOMS = ROW_BYTES / 128;       // 128-byte swizzle atoms per row
  static constexpr int ATOM_ELEMS = 128 / ES;
  static constexpr int ATOM_BYTES = 128 * 128;        // one atom column of 128 rows
  static constexpr int TILE_BYTES = 128 * ROW_BYTES;  // 128 rows
  static constexpr int P_ROW_BYTES = 128 * ES;        // 128 keys of P
  static constexpr int P_BYTES = 128 * P_ROW_BYTES;
  static constexpr int NS = 2;                        // K/V pipeline stages
  static constexpr int QK_STEPS = ROW_BYTES / 32;     // MMAs per S tile (32 bytes of K each)
  static constexpr int PV_STEPS = P_ROW_BYTES / 32;   // MMAs per O update
  static constexpr int KEYS_PER_PV_STEP = 32 / ES;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + TILE_BYTES;
  static constexpr int OFF_V = OFF_K + NS * TILE_BYTES;
  static constexpr int OFF_P = OFF_V + NS * TILE_BYTES;
  static constexpr int OFF_BAR = OFF_P + P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;   // + barriers + alignment slack
  static constexpr uint32_t FMT = F32 ? 2u : 1u;
  static constexpr uint32_t IDESC_QK = idesc_make(FMT, 128, 128, 0, 0);
  // bf16: V is the MN-major B operand straight from TMA.  fp32 (kind::tf32): MN-major tf32 needs the
  // 32B-atom swizzle, so warp 3 stages V^T (K-major, SWIZZLE_128B) instead.
  static constexpr uint32_t IDESC_PV = idesc_make(FMT, 128, D, 0, F32 ? 0 : 1);
  static constexpr int VT_ATOM_BYTES = D * 128;       // fp32 V^T: D rows x 32 keys
  static constexpr uint32_t TM_S0 = 0, TM_S1 = 128, TM_O = 256;
  static_assert(SMEM <= 232448, "shared memory budget");
};

enum BarId {
  B_QFULL = 0, B_QFREE, B_KFULL0, B_KFULL1, B_KFREE0, B_KFREE1, B_VFULL0, B_VFULL1, B_VFREE0, B_VFREE1,
  B_SFULL0, B_SFULL1, B_SFREE0, B_SFREE1, B_PFULL, B_PDONE, B_OFREE, B_COUNT
};

// Makes the compiler treat r[] as produced after the preceding tcgen05.wait::ld.
template <int N>
__device__ __forceinline__ void reg_fence(uint32_t (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}

template <int D, bool F32>
__global__ void __launch_bounds__(256, 1)
    packed_attention_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmK,
                            const __grid_constant__ CUtensorMap tmV) {
  using C = AttnCfg<D, F32>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_BAR + 8 * B_COUNT);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar[B_QFULL], 32);
    mbar_init(&bar[B_QFREE], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar[B_KFULL0 + s], 1);
      mbar_init(&bar[B_KFREE0 + s], 1);
      mbar_init(&bar[B_VFULL0 + s], F32 ? 32 : 1);
      mbar_init(&bar[B_VFREE0 + s], 1);
      mbar_init(&bar[B_SFULL0 + s], 1);
      mbar_init(&bar[B_SFREE0 + s], 128);
    }
    mbar_init(&bar[B_PFULL], 128);
    mbar_init(&bar[B_PDONE], 1);
    mbar_init(&bar[B_OFREE], 128);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = p.n_work * p.units;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t t = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        const pi_work wk = p.work[w / p.units];
        const int u = w % p.units;
        const int kvh = p.is_decode ? u : u / p.r;
        for (int s = 0; s < wk.span_count; ++s) {
          const pi_span sp = p.spans[wk.span_begin + s];
          for (int k0 = sp.begin; k0 < sp.begin + sp.len; k0 += 128, ++t) {
            const int st = t % C::NS;
            const uint32_t ph = (t / C::NS) & 1;
            mbar_wait(&bar[B_KFREE0 + st], ph ^ 1);
            mbar_arrive_expect_tx(&bar[B_KFULL0 + st], C::TILE_BYTES);
#pragma unroll
            for (int a = 0; a < C::ATOMS; ++a)
              tma_load_3d(smem + C::OFF_K + st * C::TILE_BYTES + a * C::ATOM_BYTES, &tmK, &bar[B_KFULL0 + st],
                          a * C::ATOM_ELEMS, k0, kvh);
            if constexpr (!F32) {
              mbar_wait(&bar[B_VFREE0 + st], ph ^ 1);
              mbar_arrive_expect_tx(&bar[B_VFULL0 + st], C::TILE_BYTES);
#pragma unroll
              for (int a = 0; a < C::ATOMS; ++a)
                tma_load_3d(smem + C::OFF_V + st * C::TILE_BYTES + a * C::ATOM_BYTES, &tmV, &bar[B_VFULL0 + st],
                            a * C::ATOM_ELEMS, k0, kvh);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t t = 0, item = 0;
      const uint32_t q_addr = sbase + C::OFF_Q;
      const uint32_t p_addr = sbase + C::OFF_P;
      auto issue_pv = [&](uint32_t tt, bool first) {
        const int st = tt % C::NS;
        mbar_wait(&bar[B_PFULL], tt & 1);
        mbar_wait(&bar[B_VFULL0 + st], (tt / C::NS) & 1);
        if (first) mbar_wait(&bar[B_OFREE], (item & 1) ^ 1);
        tc_fence_after();
        const uint32_t v_addr = sbase + C::OFF_V + st * C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < C::PV_STEPS; ++kk) {
          const uint64_t ad = sdesc_sw128(p_addr + (kk >> 2) * C::ATOM_BYTES + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = F32 ? sdesc_sw128(v_addr + (kk >> 2) * C::VT_ATOM_BYTES + (kk & 3) * 32, 16, 1024)
                                  : sdesc_sw128(v_addr + kk * C::KEYS_PER_PV_STEP * 128, C::ATOM_BYTES, 1024);
          mma_ss<F32>(tmem + C::TM_O, ad, bd, C::IDESC_PV, (first && kk == 0) ? 0u : 1u);
        }
        mma_commit(&bar[B_VFREE0 + st]);
        mma_commit(&bar[B_PDONE]);
      };
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        const pi_work wk = p.work[w / p.units];
        const int n = wk.n_ktiles;
        mbar_wait(&bar[B_QFULL], item & 1);
        tc_fence_after();
        for (int j = 0; j < n; ++j) {
          const uint32_t tt = t + j;
          const int st = tt % C::NS;
          const int sb = tt & 1;
          mbar_wait(&bar[B_KFULL0 + st], (tt / C::NS) & 1);
          mbar_wait(&bar[B_SFREE0 + sb], ((tt >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_addr = sbase + C::OFF_K + st * C::TILE_BYTES;
          const uint32_t d_tmem = tmem + (sb ? C::TM_S1 : C::TM_S0);
#pragma unroll
          for (int kk = 0; kk < C::QK_STEPS; ++kk) {
            const uint32_t off = (kk >> 2) * C::ATOM_BYTES + (kk & 3) * 32;
            mma_ss<F32>(d_tmem, sdesc_sw128(q_addr + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024),
                        C::IDESC_QK, kk > 0 ? 1u : 0u);
          }
          mma_commit(&bar[B_KFREE0 + st]);
          mma_commit(&bar[B_SFULL0 + sb]);
          if (j == n - 1) mma_commit(&bar[B_QFREE]);
          if (j > 0) issue_pv(tt - 1, j == 1);
        }
        issue_pv(t + n - 1, n == 1);
        t += n;
        ++item;
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ------------------------------------------------------------------ Q gather
    constexpr int CH = C::ROW_BYTES / 16;  // 16-byte chunks per row
    uint32_t item = 0;
    const uint32_t q_addr = sbase + C::OFF_Q;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      const pi_work wk = p.work[w / p.units];
      const int u = w % p.units;
      mbar_wait(&bar[B_QFREE], (item & 1) ^ 1);
      const int n_chunks = wk.row_count * CH;
      for (int idx = lane; idx < n_chunks; idx += 32) {
        const int rr = idx / CH, c = idx % CH;
        const pi_row row = p.rows[wk.row_begin + rr];
        const int h = p.is_decode ? (u * p.r + (row.out & 15)) : u;
        const uint8_t* src = p.q + ((int64_t)row.q_token * p.q_row_stride + (int64_t)h * D) * C::ES + c * 16;
        const uint32_t dst = q_addr + (c >> 3) * C::ATOM_BYTES + rr * 128 + (((c & 7) ^ (rr & 7)) << 4);
        cp_async_16(dst, src);
      }
      cp_async_wait_all();
      fence_proxy_async_smem();
      mbar_arrive(&bar[B_QFULL]);
      ++item;
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------------ fp32 only: V^T staging
    if constexpr (F32) {
      uint32_t t = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        const pi_work wk = p.work[w / p.units];
        const int u = w % p.units;
        const int kvh = p.is_decode ? u : u / p.r;
        const float* vsrc = reinterpret_cast<const float*>(p.v_buf) + (int64_t)kvh * p.buffer_tokens * D;
        for (int s = 0; s < wk.span_count; ++s) {
          const pi_span sp = p.spans[wk.span_begin + s];
          for (int k0 = sp.begin; k0 < sp.begin + sp.len; k0 += 128, ++t) {
            const int st = t % C::NS;
            mbar_wait(&bar[B_VFREE0 + st], ((t / C::NS) & 1) ^ 1);
            uint8_t* vt = smem + C::OFF_V + st * C::TILE_BYTES;
            for (int idx = lane; idx < 128 * (D / 4); idx += 32) {
              const int key = idx / (D / 4), c4 = idx % (D / 4);
              float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
              if (k0 + key < p.buffer_tokens) v = *reinterpret_cast<const float4*>(vsrc + (int64_t)(k0 + key) * D + c4 * 4);
              const float ve[4] = {v.x, v.y, v.z, v.w};
              const int a = key >> 5, jj = (key & 31) >> 2, wb = (key & 3) * 4;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int dch = c4 * 4 + e;
                *reinterpret_cast<float*>(vt + a * C::VT_ATOM_BYTES + dch * 128 + ((jj ^ (dch & 7)) << 4) + wb) = ve[e];
              }
            }
            fence_proxy_async_smem();
            mbar_arrive(&bar[B_VFULL0 + st]);
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ softmax / epilogue
    const int row_id = threadIdx.x - 128;  // == TMEM lane
    const int wq = row_id >> 5;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t p_gen_base = C::OFF_P;  // generic offset
    uint32_t t = 0, item = 0;
    const float NEG_INF = -INFINITY;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      const pi_work wk = p.work[w / p.units];
      const int u = w % p.units;
      const bool valid = row_id < wk.row_count;
      const bool warp_any = wq * 32 < wk.row_count;
      pi_row row = {0, 0, 0, 0};
      if (valid) row = p.rows[wk.row_begin + row_id];
      float m_ref = NEG_INF, l = 0.f, lr = 0.f;
      uint32_t j = 0;
      for (int s = 0; s < wk.span_count; ++s) {
        const pi_span sp = p.spans[wk.span_begin + s];
        const bool last = (s == wk.span_count - 1);
        const int se = sp.begin + sp.len;
        for (int k0 = sp.begin; k0 < se; k0 += 128, ++j) {
          const uint32_t tt = t + j;
          const int sb = tt & 1;
          mbar_wait(&bar[B_SFULL0 + sb], (tt >> 1) & 1);
          tc_fence_after();
          uint32_t sr[128];
          if (warp_any) {
            const uint32_t sa = tmem + lane_base + (sb ? C::TM_S1 : C::TM_S0);
            tmem_ld32(sa + 0, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
            tmem_ld32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
            tmem_ld32(sa + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[64]));
            tmem_ld32(sa + 96, *reinterpret_cast<uint32_t(*)[32]>(&sr[96]));
            tmem_wait_ld();
            reg_fence(sr);
          }
          tc_fence_before();
          mbar_arrive(&bar[B_SFREE0 + sb]);

          // visible key columns of this row in this tile: [c_lo, c_hi)
          int c_lo = 0, c_hi = 0;
          if (valid) {
            int lo_k = k0, hi_k = min(k0 + 128, se);
            if (last) {
              lo_k = max(lo_k, row.lo);
              hi_k = min(hi_k, row.hi);
            }
            c_lo = lo_k - k0;
            c_hi = hi_k - k0;
          }
          float mx = NEG_INF;
          if (c_lo == 0 && c_hi == 128) {
#pragma unroll
            for (int c = 0; c < 128; ++c) {
              const float x = __uint_as_float(sr[c]) * p.scale_log2;
              sr[c] = __float_as_uint(x);
              mx = fmaxf(mx, x);
            }
          } else {
#pragma unroll
            for (int c = 0; c < 128; ++c) {
              const float x = (c >= c_lo && c < c_hi) ? __uint_as_float(sr[c]) * p.scale_log2 : NEG_INF;
              sr[c] = __float_as_uint(x);
              mx = fmaxf(mx, x);
            }
          }
          const float m_new = fmaxf(m_ref, mx);
          const bool need = valid && (m_ref != NEG_INF) && (m_new > m_ref + 8.0f);
          if (warp_any && __any_sync(0xffffffffu, need)) {
            // rescale O (TMEM) once the previous P.V has landed
            mbar_wait(&bar[B_PDONE], (tt & 1) ^ 1);
            tc_fence_after();
            const float alpha = need ? ex2(m_ref - m_new) : 1.0f;
#pragma unroll
            for (int c4 = 0; c4 < D / 32; ++c4) {
              uint32_t o32[32];
              const uint32_t oa = tmem + lane_base + C::TM_O + c4 * 32;
              tmem_ld32(oa, o32);
              tmem_wait_ld();
              reg_fence(o32);
#pragma unroll
              for (int i = 0; i < 32; ++i) o32[i] = __float_as_uint(__uint_as_float(o32[i]) * alpha);
              tmem_st32(oa, o32);
            }
            tmem_wait_st();
            if (need) {
              l *= alpha;
              lr *= alpha;
              m_ref = m_new;
            }
          }
          if (m_ref == NEG_INF) m_ref = m_new;

          // P = exp2(x - m_ref) -> bf16 (tf32) into the swizzled K-major P tile
          mbar_wait(&bar[B_PDONE], (tt & 1) ^ 1);  // previous P.V finished reading P
          if (valid) {
            const bool live = (m_ref != NEG_INF);
            float psum = 0.f, prsum = 0.f;
            uint8_t* prow = smem + p_gen_base + row_id * 128;
            if constexpr (!F32) {
#pragma unroll
              for (int cc = 0; cc < 16; ++cc) {  // 8 keys per 16-byte chunk
                uint32_t pk[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float a = live ? ex2(__uint_as_float(sr[cc * 8 + 2 * e]) - m_ref) : 0.f;
                  const float b = live ? ex2(__uint_as_float(sr[cc * 8 + 2 * e + 1]) - m_ref) : 0.f;
                  pk[e] = pack_bf16(a, b);
                  psum += a + b;
                  // O is normalised with the P the tensor core actually multiplies (bf16-rounded);
                  // the LSE keeps the exact fp32 sum
                  prsum += __uint_as_float(pk[e] << 16) + __uint_as_float(pk[e] & 0xffff0000u);
                }
                uint4* dst = reinterpret_cast<uint4*>(prow + (cc >> 3) * C::ATOM_BYTES +
                                                      (((cc & 7) ^ (row_id & 7)) << 4));
                *dst = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              }
            } else {
#pragma unroll
              for (int cc = 0; cc < 32; ++cc) {  // 4 keys per chunk
                float pv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  pv[e] = live ? ex2(__uint_as_float(sr[cc * 4 + e]) - m_ref) : 0.f;
                  psum += pv[e];
                  prsum += pv[e];
                }
                uint4* dst = reinterpret_cast<uint4*>(prow + (cc >> 3) * C::ATOM_BYTES +
                                                      (((cc & 7) ^ (row_id & 7)) << 4));
                *dst = make_uint4(__float_as_uint(pv[0]), __float_as_uint(pv[1]), __float_as_uint(pv[2]),
                                  __float_as_uint(pv[3]));
              }
            }
            l += psum;
            lr += prsum;
          }
          fence_proxy_async_smem();
          tc_fence_before();
          mbar_arrive(&bar[B_PFULL]);
        }
      }
      // ---------------- epilogue: O / l -> out (or partial), lse
      const uint32_t tlast = t + j - 1;
      mbar_wait(&bar[B_PDONE], tlast & 1);
      tc_fence_after();
      const float inv_l = lr > 0.f ? 1.0f / lr : 0.f;
      const float lse_v = l > 0.f ? (m_ref + __log2f(l)) * 0.69314718055994530942f : NEG_INF;
      const int slot = (row.out >> 4) - 1;
      const int hsub = row.out & 15;
      const int head = p.is_decode ? (u * p.r + hsub) : u;
      if (warp_any) {
#pragma unroll
        for (int c4 = 0; c4 < D / 32; ++c4) {
          uint32_t o32[32];
          tmem_ld32(tmem + lane_base + C::TM_O + c4 * 32, o32);
          tmem_wait_ld();
          reg_fence(o32);
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
                    pk[e] = pack_bf16(__uint_as_float(o32[v * 8 + 2 * e]) * inv_l,
                                      __uint_as_float(o32[v * 8 + 2 * e + 1]) * inv_l);
                  reinterpret_cast<uint4*>(dst)[v] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
              } else {
#pragma unroll
                for (int v = 0; v < 8; ++v)
                  reinterpret_cast<float4*>(dst)[v] =
                      make_float4(__uint_as_float(o32[4 * v]) * inv_l, __uint_as_float(o32[4 * v + 1]) * inv_l,
                                  __uint_as_float(o32[4 * v + 2]) * inv_l, __uint_as_float(o32[4 * v + 3]) * inv_l);
              }
            } else {
              float* dst = p.partial_o + ((int64_t)slot * p.hq_count + head) * D + c4 * 32;
#pragma unroll
              for (int v = 0; v < 8; ++v)
                reinterpret_cast<float4*>(dst)[v] =
                    make_float4(__uint_as_float(o32[4 * v]) * inv_l, __uint_as_float(o32[4 * v + 1]) * inv_l,
                                __uint_as_float(o32[4 * v + 2]) * inv_l, __uint_as_float(o32[4 * v + 3]) * inv_l);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bar[B_OFREE]);
      if (valid) {
        if (slot < 0) {
          if (p.lse) p.lse[(int64_t)head * p.total_q + row.q_token] = lse_v;
        } else {
          p.partial_lse[(int64_t)slot * p.hq_count + head] = lse_v;
        }
      }
      t += j;
      ++item;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D, bool F32>
static pi_status launch(const pi_device_plan* dp, bool decode, bool out_f32, const void* q, int64_t q_row_stride,
                        const void* k_buf, const void* v_buf, int32_t hkv_count, int32_t r, float scale,
                        void* out, int64_t out_row_stride, float* lse, float* partial_o, float* partial_lse,
                        cudaStream_t stream) {
  using C = AttnCfg<D, F32>;
  const int32_t n_work = decode ? dp->n_decode_work : dp->n_prefill_work;
  if (n_work == 0) return PI_OK;
  AttnParams p{};
  p.work = decode ? dp->decode_work : dp->prefill_work;
  p.rows = dp->rows;
  p.spans = dp->spans;
  p.n_work = n_work;
  p.units = decode ? hkv_count : hkv_count * r;
  p.is_decode = decode ? 1 : 0;
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

  CUtensorMap tmK, tmV;
  const CUtensorMapDataType dt = F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const uint64_t dims[3] = {(uint64_t)D, (uint64_t)dp->buffer_tokens, (uint64_t)hkv_count};
  const uint64_t strides[2] = {(uint64_t)C::ROW_BYTES, (uint64_t)dp->buffer_tokens * C::ROW_BYTES};
  const uint32_t box[3] = {(uint32_t)C::ATOM_ELEMS, 128u, 1u};
  pi_status s = encode_tmap_3d(&tmK, dt, k_buf, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  if (s != PI_OK) return s;
  s = encode_tmap_3d(&tmV, dt, v_buf, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  if (s != PI_OK) return s;

  static bool attr_set = false;  // per template instance
  if (!attr_set) {
    s = cuda_check(cudaFuncSetAttribute(packed_attention_kernel<D, F32>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM),
                   "cudaFuncSetAttribute");
    if (s != PI_OK) return s;
    attr_set = true;
  }
  const int64_t total = (int64_t)n_work * p.units;
  const int grid = (int)std::min<int64_t>(total, num_sms());
  packed_attention_kernel<D, F32><<<grid, 256, C::SMEM, stream>>>(p, tmK, tmV);
  return cuda_check(cudaGetLastError(), "packed_attention_kernel launch");
}

static pi_status attention_entry(bool decode, const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                 const void* k_buf, const void* v_buf, int32_t hkv_count, int32_t gqa_ratio,
                                 int32_t head_dim, float softmax_scale, pi_dtype dt, void* out,
                                 int64_t out_row_stride, float* lse, float* partial_o, float* partial_lse,
                                 pi_stream_t stream) {
  if (!dp) return fail(PI_EINVAL, "device plan is NULL");
  const int32_t n_work = decode ? dp->n_decode_work : dp->n_prefill_work;
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
  if (q_row_stride < (int64_t)hkv_count * gqa_ratio * head_dim || out_row_stride < (int64_t)hkv_count * gqa_ratio * head_dim)
    return fail(PI_EINVAL, "row stride smaller than the local heads");
  if (dp->n_partial_slots > 0 && decode && (!partial_o || !partial_lse))
    return fail(PI_EINVAL, "plan has split rows: partial_o / partial_lse required");
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(k_buf) |
       reinterpret_cast<uintptr_t>(v_buf)) % 16)
    return fail(PI_EINVAL, "q/out/k_buf/v_buf must be 16-byte aligned");
  pi_status s = require_sm100();
  if (s != PI_OK) return s;
  const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)head_dim);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dt == PI_BF16 && head_dim == 128)
    s = launch<128, false>(dp, decode, out_f32, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, scale, out,
                           out_row_stride, lse, partial_o, partial_lse, st);
  else if (dt == PI_BF16 && head_dim == 64)
    s = launch<64, false>(dp, decode, out_f32, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, scale, out,
                          out_row_stride, lse, partial_o, partial_lse, st);
  else
    s = launch<64, true>(dp, decode, false, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, scale, out,
                         out_row_stride, lse, partial_o, partial_lse, st);
  return s == PI_OK ? ok() : s;
}

}  // namespace pi

extern "C" {

pi_status packinfer_attention_prefill(const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                      const void* k_buf, const void* v_buf, int32_t hkv_count, int32_t gqa_ratio,
                                      int32_t head_dim, float softmax_scale, pi_dtype dt, void* out,
                                      int64_t out_row_stride, float* lse, float* partial_o, float* partial_lse,
                                      pi_stream_t stream) {
  return pi::attention_entry(false, dp, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, head_dim,
                             softmax_scale, dt, out, out_row_stride, lse, partial_o, partial_lse, stream);
}

pi_status packinfer_attention_decode(const pi_device_plan* dp, const void* q, int64_t q_row_stride,
                                     const void* k_buf, const void* v_buf, int32_t hkv_count, int32_t gqa_ratio,
                                     int32_t head_dim, float softmax_scale, pi_dtype dt, void* out,
                                     int64_t out_row_stride, float* lse, float* partial_o, float* partial_lse,
                                     pi_stream_t stream) {
  return pi::attention_entry(true, dp, q, q_row_stride, k_buf, v_buf, hkv_count, gqa_ratio, head_dim,
                             softmax_scale, dt, out, out_row_stride, lse, partial_o, partial_lse, stream);
}

}  // extern "C"
