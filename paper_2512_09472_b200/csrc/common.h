// Shared helpers for the warmserve native library (C-ABI in include/warmserve.h).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/warmserve.h"

namespace ws {

// Thread-local last-error text, surfaced through ws_last_error().
void set_error(const std::string& msg);
const char* last_error();

// Status codes are stable: the Python mirror maps them to ClusterError with the
// reference's message substrings (cluster.py:253-386, test_cluster.py:137-342).
#define WS_FAIL(code, ...)                                   \
  do {                                                       \
    char _buf[512];                                          \
    snprintf(_buf, sizeof(_buf), __VA_ARGS__);               \
    ::ws::set_error(_buf);                                   \
    return (code);                                           \
  } while (0)

#define WS_CUDA(expr)                                                          \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      WS_FAIL(WS_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
              __FILE__, __LINE__);                                             \
    }                                                                          \
  } while (0)

constexpr int kNumSMs = 148;

// Count of kernel launches issued by this library (ws_kernel_launches()).
void count_launch(int n = 1);

}  // namespace ws
