// Microbenchmark: cycles per tcgen05.mma (cta_group::1, kind::f16, M=128, K=16) for SS and TS
// operand modes and N in {64, 128, 256}, one CTA per SM, back-to-back issue by one thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2602_06072_b200/csrc scripts/mma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace pi::sm100;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
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
    const uint32_t idesc = idesc_make(1, 128, N, 0, 0);
    // warm-up
    for (int i = 0; i < 16; ++i) mma_ss<false>(tmem, da, db, idesc, 1);
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
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int N, bool TS>
void run(int sms) {
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 96 * 1024;
  cudaFuncSetAttribute(bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  bench<N, TS><<<sms, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  printf("%s N=%3d: %.1f cycles/MMA (M128xN%dxK16; nominal %.0f)  err=%s\n", TS ? "TS" : "SS", N, avg / iters, N,
         128.0 * N / 256.0, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false>(sms);
  run<128, false>(sms);
  run<256, false>(sms);
  run<128, true>(sms);
  run<256, true>(sms);
  run<128, false>(1);
  run<128, true>(1);
  return 0;
}
