#include "device_common.h"

#include <atomic>
#include <mutex>

namespace pi {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn g_encode = nullptr;
std::once_flag g_encode_once;
}  // namespace

static pi_status encode_tmap(int rank, CUtensorMap* map, CUtensorMapDataType dtype, const void* base,
                             const uint64_t dims[3], const uint64_t strides_bytes[2], const uint32_t box[3],
                             CUtensorMapSwizzle swizzle) {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeFn>(fn);
  });
  if (!g_encode) return fail(PI_ECUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t gd[3] = {dims[0], dims[1], dims[2]};
  cuuint64_t gs[2] = {strides_bytes[0], strides_bytes[1]};
  cuuint32_t bd[3] = {box[0], box[1], box[2]};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(map, dtype, rank, const_cast<void*>(base), gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(PI_ECUDA, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
  return PI_OK;
}

pi_status encode_tmap_3d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base,
                         const uint64_t dims[3], const uint64_t strides_bytes[2], const uint32_t box[3],
                         CUtensorMapSwizzle swizzle) {
  return encode_tmap(3, map, dtype, base, dims, strides_bytes, box, swizzle);
}

pi_status encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base,
                         const uint64_t dims[3], const uint64_t strides_bytes[2], const uint32_t box[3],
                         CUtensorMapSwizzle swizzle) {
  return encode_tmap(2, map, dtype, base, dims, strides_bytes, box, swizzle);
}

// Per-device caches are atomics: concurrent first calls on several host threads may both query
// the (idempotent) attribute, never read a torn value.
int num_sms() {
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int v = cache[dev].load(std::memory_order_acquire);
  if (!v) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    v = n > 0 ? n : 148;
    cache[dev].store(v, std::memory_order_release);
  }
  return v;
}

pi_status require_sm100() {
  static std::atomic<int> cache[kMaxDevices];  // 0 unknown, 1 ok, 2 bad
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(PI_ECUDA, "no CUDA device");
  if (dev < 0 || dev >= kMaxDevices) return fail(PI_EUNSUP, "device ordinal beyond the library's table");
  int v = cache[dev].load(std::memory_order_acquire);
  if (!v) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    v = (major == 10 && minor == 0) ? 1 : 2;
    cache[dev].store(v, std::memory_order_release);
  }
  if (v != 1) return fail(PI_EUNSUP, "libpackinfer is built for sm_100a (B200) only");
  return PI_OK;
}

pi_status set_max_dynamic_smem(const void* func, std::atomic<int>* done, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(PI_ECUDA, "no CUDA device");
  if (dev < 0 || dev >= kMaxDevices) return fail(PI_EUNSUP, "device ordinal beyond the library's table");
  if (done[dev].load(std::memory_order_acquire)) return PI_OK;
  pi_status s = cuda_check(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                           "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
  if (s == PI_OK) done[dev].store(1, std::memory_order_release);
  return s;
}

}  // namespace pi
