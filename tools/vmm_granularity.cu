// How do cuMemCreate / cuMemMap / cuMemSetAccess costs scale with the
// physical handle size? (2 MiB pages vs larger handles) — B200 measurement.
#include <cuda.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s: %s\n", #x, s); return 1; } } while (0)
static double us() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  CK(cuInit(0)); CUdevice d; CK(cuDeviceGet(&d, 0)); CUcontext c; CK(cuDevicePrimaryCtxRetain(&c, d)); CK(cuCtxSetCurrent(c));
  CUmemAllocationProp p{}; p.type = CU_MEM_ALLOCATION_TYPE_PINNED; p.location.type = CU_MEM_LOCATION_TYPE_DEVICE; p.location.id = 0;
  CUmemAccessDesc a{}; a.location = p.location; a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  const size_t total = 4ull << 30;  // 4 GiB per configuration
  for (size_t hs : {2ull << 20, 8ull << 20, 32ull << 20, 128ull << 20, 512ull << 20}) {
    int n = total / hs; std::vector<CUmemGenericAllocationHandle> h(n);
    double t0 = us(); for (int i = 0; i < n; ++i) CK(cuMemCreate(&h[i], hs, &p, 0)); double tc = us() - t0;
    CUdeviceptr va; CK(cuMemAddressReserve(&va, total, hs, 0, 0));
    t0 = us(); for (int i = 0; i < n; ++i) CK(cuMemMap(va + i * hs, hs, 0, h[i], 0)); double tm = us() - t0;
    t0 = us(); CK(cuMemSetAccess(va, total, &a, 1)); double ta = us() - t0;
    // second alias VA (what a slot mapping costs when the page is already in the window)
    CUdeviceptr vb; CK(cuMemAddressReserve(&vb, total, hs, 0, 0));
    t0 = us(); for (int i = 0; i < n; ++i) CK(cuMemMap(vb + i * hs, hs, 0, h[i], 0)); CK(cuMemSetAccess(vb, total, &a, 1)); double tb = us() - t0;
    t0 = us(); CK(cuMemUnmap(vb, total)); double tu = us() - t0;
    double per2m = (double)(2ull << 20) / hs;
    printf("{\"handle_mib\": %zu, \"create_us_per_2mib\": %.2f, \"map_us_per_2mib\": %.2f, \"setaccess_us_per_2mib\": %.2f, \"alias_map_access_us_per_2mib\": %.2f, \"unmap_us_per_2mib\": %.2f}\n",
           hs >> 20, tc / n * per2m, tm / n * per2m, ta / n * per2m, tb / n * per2m, tu / n * per2m);
    CK(cuMemUnmap(va, total)); CK(cuMemAddressFree(va, total)); CK(cuMemAddressFree(vb, total));
    for (auto x : h) CK(cuMemRelease(x));
  }
  return 0;
}
