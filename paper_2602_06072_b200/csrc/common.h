// Shared host-side helpers of libpackinfer (error reporting).  Not device code.
#pragma once

#include <string>

#include "packinfer.h"

namespace pi {

// Records `msg` as this thread's last error and returns `s`.
pi_status fail(pi_status s, const std::string& msg);
// Clears the thread's last error; returns PI_OK.
pi_status ok();

pi_status plan_impl(int32_t n, const int32_t* kv_len, const int32_t* q_len,
                    const int32_t* prefix_id, int32_t n_prefix, const int32_t* prefix_len,
                    const int32_t* appended, const pi_config* cfg, void* arena, size_t arena_bytes,
                    pi_plan* out);

}  // namespace pi
