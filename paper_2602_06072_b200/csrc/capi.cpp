// C ABI entry points that need no device code: status strings, config defaults, planning and
// plan upload.  Device entry points live next to their kernels (relayout.cu, attention.cu,
// merge.cu).
#include <cstring>
#include <string>

#include <cuda_runtime.h>

#include "common.h"
#include "packinfer.h"

namespace pi {
namespace {
thread_local std::string g_last_error;
}
pi_status fail(pi_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
pi_status ok() {
  g_last_error.clear();
  return PI_OK;
}
}  // namespace pi

extern "C" {

const char* packinfer_strerror(pi_status s) {
  switch (s) {
    case PI_OK: return "ok";
    case PI_EINVAL: return "invalid argument";
    case PI_ENOSPC: return "buffer too small";
    case PI_ECUDA: return "CUDA error";
    case PI_EUNSUP: return "unsupported";
    case PI_EREGROUP: return "headroom exhausted: regroup";
  }
  return "unknown status";
}

const char* packinfer_last_error(void) { return pi::g_last_error.c_str(); }

const char* packinfer_version(void) { return "packinfer-b200 0.1 (sm_100a)"; }

void packinfer_default_config(pi_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->capacity = 8192;
  cfg->num_groups = 0;
  cfg->mem_cap = 0;
  cfg->headroom = 0;
  cfg->tile_q = 128;
  cfg->tile_k = 128;
  cfg->decode_chunk = 1024;
  cfg->gqa_ratio = 1;
  cfg->flags = PI_PLAN_DPACK;   // packed decode items (measured faster since lane slicing covers <= 32 rows)
}

pi_status packinfer_plan(int32_t n, const int32_t* kv_len, const int32_t* q_len,
                         const int32_t* prefix_id, int32_t n_prefix, const int32_t* prefix_len,
                         const pi_config* cfg, void* host_arena, size_t arena_bytes,
                         pi_plan* out) {
  pi_status s = pi::plan_impl(n, kv_len, q_len, prefix_id, n_prefix, prefix_len, nullptr, cfg,
                              host_arena, arena_bytes, out);
  if (s == PI_OK) pi::ok();
  return s;
}

pi_status packinfer_plan_step(int32_t n, const int32_t* kv_len, const int32_t* q_len,
                              const int32_t* prefix_id, int32_t n_prefix, const int32_t* prefix_len,
                              const int32_t* appended, const pi_config* cfg, void* host_arena,
                              size_t arena_bytes, pi_plan* out) {
  pi_status s = pi::plan_impl(n, kv_len, q_len, prefix_id, n_prefix, prefix_len, appended, cfg,
                              host_arena, arena_bytes, out);
  if (s == PI_OK) pi::ok();
  return s;
}

int32_t packinfer_should_regroup(int32_t steps, int64_t drift, int32_t capacity) {
  // Eq. 4: t * dL >= C / 2, exact in integers (2 t dL >= C)
  return (2 * (int64_t)steps * drift >= (int64_t)capacity) ? 1 : 0;
}

}  // extern "C"
