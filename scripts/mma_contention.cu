// Microbenchmark: tcgen05.mma throughput (M128 N128 K16, SS and TS) while other warps stress
// (a) TMEM reads (tcgen05.ld 32x32b.x32 in a loop) or (b) shared-memory reads (ld.shared.v4).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2602_06072_b200/csrc scripts/mma_contention.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace pi::sm100;

__device__ volatile int g_stop;

template <bool TS, int STRESS>  // STRESS: 0 none, 1 TMEM ld, 2 smem ld, 3 TMEM st
__global__ void __launch_bounds__(384, 1) bench(int iters, unsigned long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32) {
    const uint32_t sb = smem_u32(smem);
    const uint64_t da = sdesc_sw128(sb, 16, 1024);
    const uint64_t db = sdesc_sw128(sb + 32768, 16, 1024);
    const uint32_t idesc = idesc_make(1, 128, 128, 0, 0);
    for (int i = 0; i < 16; ++i) mma_ss<false>(tmem + 256, da, db, idesc, 1);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS)
        mma_ts<false>(tmem + 256, tmem + 0, db + ((i & 3) * 2), idesc, 1);
      else
        mma_ss<false>(tmem + 256, da + ((i & 3) * 2), db + ((i & 3) * 2), idesc, 1);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
    done = 1;
  } else if (warp >= 4 && STRESS != 0) {
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    float acc = 0.f;
    int it = 0;
    while (!done) {
      if (STRESS == 1) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + 128 + ((it & 1) * 32), r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
      } else if (STRESS == 2) {
        const uint4* s4 = reinterpret_cast<const uint4*>(smem + 65536);
        uint4 v = s4[(threadIdx.x + it * 384) & 4095];
        acc += __uint_as_float(v.x ^ v.y ^ v.z ^ v.w);
      } else {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = it + i;
        tmem_st32(tmem + lane_base + 128 + ((it & 1) * 32), r);
        tmem_wait_st();
      }
      ++it;
    }
    if (acc == 12345.f) sink[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Pattern test: 8 TS MMAs (A = P in TMEM cols [a0, a0+64), D = O cols 256..) then 8 SS MMAs writing
// D = S cols [s0, s0+128).  conflict: s0 == a0 region (the FA4-style P/S aliasing).
template <int MODE>  // 0: S writes cols 128.. (no overlap), 1: S writes cols 0.. (overlaps P), 2: two regions alternating
__global__ void __launch_bounds__(128, 1) pattern(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t sb = smem_u32(smem);
    const uint64_t da = sdesc_sw128(sb, 16, 1024);
    const uint64_t db = sdesc_sw128(sb + 32768, 16, 1024);
    const uint32_t id_s = idesc_make(1, 128, 128, 0, 0);
    const uint32_t id_pv = idesc_make(1, 128, 128, 0, 1);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t preg = (MODE == 2 && (i & 1)) ? 128 : 0;
      for (int kk = 0; kk < 8; ++kk) mma_ts<false>(tmem + 256 + (i & 1) * 128, tmem + preg + kk * 8, db + kk * 2, id_pv, 1);
      const uint32_t sreg = MODE == 0 ? 128 : (MODE == 1 ? 0 : preg);
      for (int kk = 0; kk < 8; ++kk) mma_ss<false>(tmem + sreg, da + kk * 2, db + kk * 2, id_s, kk > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int MODE>
void run_pattern(int sms, const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 96 * 1024;
  cudaFuncSetAttribute(pattern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 1024;
  pattern<MODE><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("pattern %-40s: %.1f cycles/MMA  err=%s\n", name, avg / (iters * 16), cudaGetErrorString(e));
  cudaFree(d);
}

template <bool TS, int STRESS>
void run(int sms, const char* name) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, sms * 8);
  cudaMalloc(&sink, 4);
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(bench<TS, STRESS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 8192;
  bench<TS, STRESS><<<sms, 384, smem>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("%s %-22s: %.1f cycles/MMA  err=%s\n", TS ? "TS" : "SS", name, avg / iters, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<false, 0>(sms, "alone");
  run<false, 1>(sms, "+8 warps tcgen05.ld");
  run<false, 2>(sms, "+8 warps ld.shared");
  run<false, 3>(sms, "+8 warps tcgen05.st");
  run<true, 0>(sms, "alone");
  run<true, 1>(sms, "+8 warps tcgen05.ld");
  run<true, 2>(sms, "+8 warps ld.shared");
  run<true, 3>(sms, "+8 warps tcgen05.st");
  run_pattern<0>(sms, "PV(A=P@0) then S->@128 (no overlap)");
  run_pattern<1>(sms, "PV(A=P@0) then S->@0 (WAR on P)");
  run_pattern<2>(sms, "alternating regions (WAR every other)");
  return 0;
}
