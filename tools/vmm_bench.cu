// Micro-benchmark of the CUDA VMM driver calls behind the page pool on this
// B200: cuMemCreate, cuMemMap (first mapping / second alias mapping),
// cuMemSetAccess (per page vs one call per 64-page chunk), cuMemUnmap.
// Gives the measured per-page map cost mu that replaces the reference's
// calibrated 0.0390625 ms (config.py:38). Build: nvcc -O2 -o vmm_bench
// vmm_bench.cu -lcuda
#include <cuda.h>

#include <chrono>
#include <cstdio>
#include <vector>

#define CK(x)                                                            \
  do {                                                                   \
    CUresult r = (x);                                                    \
    if (r != CUDA_SUCCESS) {                                             \
      const char* s;                                                     \
      cuGetErrorString(r, &s);                                           \
      printf("%s failed: %s\n", #x, s);                                  \
      return 1;                                                          \
    }                                                                    \
  } while (0)

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 2048;
  const size_t page = 2u << 20;
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  std::vector<CUmemGenericAllocationHandle> h(n);
  double t0 = now_us();
  for (int i = 0; i < n; ++i) CK(cuMemCreate(&h[i], page, &prop, 0));
  double t_create = now_us() - t0;
  CUdeviceptr win, slot, slot2;
  CK(cuMemAddressReserve(&win, n * page, page, 0, 0));
  CK(cuMemAddressReserve(&slot, n * page, page, 0, 0));
  CK(cuMemAddressReserve(&slot2, n * page, page, 0, 0));
  t0 = now_us();
  for (int i = 0; i < n; ++i) CK(cuMemMap(win + i * page, page, 0, h[i], 0));
  double t_map1 = now_us() - t0;
  t0 = now_us();
  CK(cuMemSetAccess(win, n * page, &acc, 1));
  double t_acc_range = now_us() - t0;
  // alias mappings (what a prewarm slot does), access per 64-page chunk
  t0 = now_us();
  for (int i = 0; i < n; ++i) CK(cuMemMap(slot + i * page, page, 0, h[i], 0));
  double t_map2 = now_us() - t0;
  t0 = now_us();
  for (int c = 0; c < n; c += 64) CK(cuMemSetAccess(slot + c * page, 64 * page, &acc, 1));
  double t_acc_chunk = now_us() - t0;
  // alias mappings with per-page access
  t0 = now_us();
  for (int i = 0; i < n; ++i) {
    CK(cuMemMap(slot2 + i * page, page, 0, h[i], 0));
    CK(cuMemSetAccess(slot2 + i * page, page, &acc, 1));
  }
  double t_map_acc_page = now_us() - t0;
  t0 = now_us();
  for (int i = 0; i < n; ++i) CK(cuMemUnmap(slot + i * page, page));
  double t_unmap_page = now_us() - t0;
  t0 = now_us();
  CK(cuMemUnmap(slot2, n * page));
  double t_unmap_range = now_us() - t0;
  printf("{\"pages\": %d, \"create_us_per_page\": %.2f, \"map_first_us_per_page\": %.2f, "
         "\"setaccess_whole_range_us\": %.1f, \"map_alias_us_per_page\": %.2f, "
         "\"setaccess_per64_us_per_page\": %.2f, \"map_plus_setaccess_per_page_us\": %.2f, "
         "\"unmap_us_per_page\": %.2f, \"unmap_range_us_per_page\": %.2f}\n",
         n, t_create / n, t_map1 / n, t_acc_range, t_map2 / n, t_acc_chunk / n, t_map_acc_page / n,
         t_unmap_page / n, t_unmap_range / n);
  return 0;
}
