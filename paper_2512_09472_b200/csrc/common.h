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

// Shapes outside the tcgen05 tilings run a legacy kernel; every such launch
// is counted (ws_fallback_counts) and the first of each kind logged to stderr.
enum FallbackKind {
  kFallbackGemmMma = 0,   // GEMM on the mma.sync kernel (M >= 16, no tcgen05 tiling)
  kFallbackGemv = 1,      // GEMM on the CUDA-core GEMV (M < 16, no skinny tcgen05 tiling)
  kFallbackAttnMma = 2,   // prefill attention on the mma.sync kernel (head_dim / GQA outside attn_tc)
  kFallbackKinds = 3
};
void count_fallback(FallbackKind k, const char* what);

}  // namespace ws
