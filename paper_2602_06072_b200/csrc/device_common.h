// Host helpers shared by the CUDA translation units: TMA tensor-map encoding through the driver
// entry point (no -lcuda link dependency) and cached device properties.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <string>

#include "common.h"
#include "packinfer.h"

namespace pi {

// Encodes a rank-3 tiled tensor map (innermost first).  Returns PI_OK or PI_ECUDA/PI_EUNSUP.
pi_status encode_tmap_3d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base,
                         const uint64_t dims[3], const uint64_t strides_bytes[2],
                         const uint32_t box[3], CUtensorMapSwizzle swizzle);

// Rank-2 variant (dims[2] / strides[1] / box[2] ignored).
pi_status encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base,
                         const uint64_t dims[3], const uint64_t strides_bytes[2],
                         const uint32_t box[3], CUtensorMapSwizzle swizzle);

constexpr int kMaxDevices = 64;

// Number of SMs of the current device (cached per device).
int num_sms();

// Fails with PI_EUNSUP unless the current device is compute capability 10.0 (sm_100a).
pi_status require_sm100();

inline pi_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PI_OK;
  return fail(PI_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Opts `func` into `bytes` of dynamic shared memory on the CURRENT device, once per device
// (done[kMaxDevices]: one flag per device ordinal, owned by the caller's kernel instance).
pi_status set_max_dynamic_smem(const void* func, std::atomic<int>* done, int bytes);

}  // namespace pi
