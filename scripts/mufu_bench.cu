// Microbenchmark: MUFU exp2 throughput per SM for ex2.approx.ftz.f32 (1 result per lane) vs
// ex2.approx.f16x2 (2 results per lane), plus the cvt.rn.f16x2.f32 pack and HADD2 / FADD2 rates,
// 4 warps per SMSP, independent chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/mufu_bench.cu -o scripts/mufu_bench
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(int iters, float* sink, unsigned long long* cyc) {
  uint32_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(-0.001f * (threadIdx.x + i));
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__uint_as_float(v[i])));
        v[i] = __float_as_uint(y);
      } else if (MODE == 1) {
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(v[i]));
        v[i] = y;
      } else if (MODE == 2) {
        uint32_t y;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(__uint_as_float(v[i])), "f"(1.0f));
        v[i] = y;
      } else if (MODE == 3) {
        uint32_t y;
        asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(y) : "r"(v[i]), "r"(v[(i + 1) & 7]));
        v[i] = y;
      } else if (MODE == 4) {
        uint32_t y;
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(v[i]));
        v[i] = y;
      } else if (MODE == 5) {
        // packed fp32x2 FMA on (v[i], v[i^1]) pairs
        uint64_t a = ((uint64_t)v[i ^ 1] << 32) | v[i], y;
        asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(y) : "l"(a));
        v[i] = (uint32_t)y;
        v[i ^ 1] = (uint32_t)(y >> 32);
      } else {
        float y;
        asm volatile("fma.rn.f32 %0, %1, %1, %1;" : "=f"(y) : "f"(__uint_as_float(v[i])));
        v[i] = __float_as_uint(y);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __uint_as_float(v[i]);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int sms, int threads, double per_op) {
  float* sink;
  unsigned long long* cyc;
  cudaMalloc(&sink, sms * 512 * 4);
  cudaMalloc(&cyc, sms * 8);
  const int iters = 2048;
  bench<MODE><<<sms, threads>>>(iters, sink, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double ops = (double)iters * 8 * threads;  // lane-instructions per SM
  printf("%-28s threads=%3d: %.2f lane-instr/clk/SM = %.2f results/clk/SM  err=%s\n", name, threads, ops / avg,
         ops * per_op / avg, cudaGetErrorString(e));
  cudaFree(sink);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int th : {128, 256, 512}) {
    run<0>("ex2.approx.ftz.f32", sms, th, 1);
    run<1>("ex2.approx.f16x2", sms, th, 2);
    run<4>("ex2.approx.ftz.bf16x2", sms, th, 2);
    run<2>("cvt.rn.f16x2.f32", sms, th, 1);
    run<3>("add.rn.f16x2", sms, th, 2);
    run<5>("fma.rn.f32x2", sms, th, 2);
    run<6>("fma.rn.f32", sms, th, 1);
  }
  return 0;
}
