// Microbenchmark: tcgen05.ld / tcgen05.st throughput (bytes/cycle/SM) for 4 and 8 warps,
// x32 (32 columns) per instruction, waiting after every 1, 2 or 4 loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2602_06072_b200/csrc scripts/tmem_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace pi::sm100;

template <int WARPS, int BATCH, bool STORE>
__global__ void __launch_bounds__(512, 1) bench(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  float acc = 0.f;
  long long t0 = clock64();
  if (warp < WARPS) {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) & 3) * 128;
    for (int it = 0; it < iters; ++it) {
      if (STORE) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = it + i;
#pragma unroll
        for (int b = 0; b < BATCH; ++b) tmem_st32(base + b * 32, r);
        tmem_wait_st();
      } else {
        uint32_t r[BATCH][32];
#pragma unroll
        for (int b = 0; b < BATCH; ++b) tmem_ld32(base + b * 32, r[b]);
        tmem_wait_ld();
        // consume without a dependent arithmetic chain (a serial FADD chain over the 32 values
        // would take ~4 cycles per value and hide the load rate)
#pragma unroll
        for (int b = 0; b < BATCH; ++b)
#pragma unroll
          for (int i = 0; i < 32; ++i) asm volatile("" ::"r"(r[b][i]));
        acc += __uint_as_float(r[0][0]);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 1.2345f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int WARPS, int BATCH, bool STORE>
void run(int sms) {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, sms * 8);
  cudaMalloc(&sink, 4);
  const int iters = 2048;
  bench<WARPS, BATCH, STORE><<<sms, 512>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double bytes = (double)WARPS * iters * BATCH * 32 * 32 * 4;
  printf("%s warps=%d batch=%d: %.1f B/cycle/SM, %.1f cycles per x32 per warp  err=%s\n", STORE ? "st" : "ld",
         WARPS, BATCH, bytes / avg, avg / (iters * BATCH), cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 1, false>(sms);
  run<4, 2, false>(sms);
  run<4, 4, false>(sms);
  run<8, 1, false>(sms);
  run<8, 2, false>(sms);
  run<16, 1, false>(sms);
  run<16, 2, false>(sms);
  run<4, 1, true>(sms);
  run<4, 2, true>(sms);
  run<8, 2, true>(sms);
  return 0;
}
