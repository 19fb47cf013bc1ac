// Shared helpers for libsagann: status / last-error plumbing (no exceptions cross the ABI).
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/sagann.h"

namespace sg {

void set_error(const char* fmt, ...);
// Count of device kernels launched by this library (sg_launch_count()).
void count_launch(int n = 1);

// Return `code` after recording a formatted message (thread-local, sg_last_error()).
#define SG_FAIL(code, ...)      \
  do {                          \
    ::sg::set_error(__VA_ARGS__); \
    return (code);              \
  } while (0)

#define SG_REQUIRE(cond, code, ...) \
  do {                              \
    if (!(cond)) SG_FAIL(code, __VA_ARGS__); \
  } while (0)

#ifdef __CUDACC__
// ReLU with numpy's np.maximum(x, 0) semantics (tensor.py:207): NaN propagates (fmaxf
// would map NaN to 0 and hide it from the strict non-finite check).
__device__ __forceinline__ float relu_np(float v) { return (v >= 0.f || v != v) ? v : 0.f; }
#endif

}  // namespace sg
