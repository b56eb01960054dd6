#include "driver.h"

#include <cuda_runtime.h>
#include <atomic>
#include <cstdio>
#include <mutex>
#include <string>

#include "common.h"

namespace ws {

namespace {
thread_local std::string g_err;
Driver g_drv;
bool g_ok = false;
std::once_flag g_once;
std::string g_load_err;

template <typename F>
bool load(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) {
    g_load_err = std::string("driver entry point ") + name + " unavailable: " +
                 cudaGetErrorString(e);
    return false;
  }
  *fn = reinterpret_cast<F>(p);
  return true;
}
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }

static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static std::atomic<int64_t> g_fallbacks[kFallbackKinds];
static std::atomic<bool> g_fallback_logged[kFallbackKinds];
void count_fallback(FallbackKind k, const char* what) {
  g_fallbacks[k].fetch_add(1, std::memory_order_relaxed);
  if (!g_fallback_logged[k].exchange(true))  // first occurrence per kind goes to stderr
    fprintf(stderr, "[warmserve] fallback (counted in ws_fallback_counts[%d]): %s\n", (int)k, what);
}
const char* last_error() { return g_err.c_str(); }

const Driver* driver() {
  std::call_once(g_once, [] {
    g_ok = load("cuMemCreate", &g_drv.cuMemCreate) && load("cuMemRelease", &g_drv.cuMemRelease) &&
           load("cuMemAddressReserve", &g_drv.cuMemAddressReserve) &&
           load("cuMemAddressFree", &g_drv.cuMemAddressFree) && load("cuMemMap", &g_drv.cuMemMap) &&
           load("cuMemUnmap", &g_drv.cuMemUnmap) && load("cuMemSetAccess", &g_drv.cuMemSetAccess) &&
           load("cuMemGetAllocationGranularity", &g_drv.cuMemGetAllocationGranularity) &&
           load("cuTensorMapEncodeTiled", &g_drv.cuTensorMapEncodeTiled) &&
           load("cuGetErrorString", &g_drv.cuGetErrorString) &&
           load("cuMemExportToShareableHandle", &g_drv.cuMemExportToShareableHandle) &&
           load("cuMemImportFromShareableHandle", &g_drv.cuMemImportFromShareableHandle);
  });
  if (!g_ok) {
    set_error(g_load_err);
    return nullptr;
  }
  return &g_drv;
}

}  // namespace ws

extern "C" const char* ws_last_error(void) { return ws::last_error(); }
extern "C" int ws_kernel_launches(int64_t* out) {
  *out = ws::g_launches.load();
  return WS_OK;
}

extern "C" int ws_fallback_counts(int64_t* out, int32_t n) {
  for (int32_t i = 0; i < n && i < ws::kFallbackKinds; ++i) out[i] = ws::g_fallbacks[i].load();
  return WS_OK;
}

extern "C" int ws_version(int* major, int* minor) {
  *major = 0;
  *minor = 1;
  return WS_OK;
}
