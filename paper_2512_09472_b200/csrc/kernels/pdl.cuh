// Programmatic dependent launch (PDL) for the prefill/decode kernel chain.
//
// Every model kernel is launched with programmatic stream serialization and
// (1) triggers its dependents as soon as it starts (all of its CTAs are then
// resident, so an early-launched dependent can never starve it), and
// (2) waits for its predecessor grid — completion plus memory visibility —
// before touching any global data. The dependent's launch latency and its
// prologue (barrier init, TMEM allocation, tensor-map prefetch) overlap the
// predecessor's tail instead of sitting in the kernel boundary.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "pdl_flag.h"

namespace ws {

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// WS_PDL=0 launches the chain with plain stream ordering (A/B measurement).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("WS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// The PDL attribute for one launch: off once after pdl_break_next().
inline bool pdl_for_launch() {
  if (t_pdl_break) {
    t_pdl_break = false;
    return false;
  }
  return pdl_enabled();
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_for_launch() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace ws
