// Do CUDA VMM driver calls serialise against in-flight kernels on this B200?
// (SURVEY.md §7 hard parts: the async-unmap contract of engine.py:615-632
// only holds if cuMemUnmap / cuMemMap / cuMemSetAccess on unrelated ranges
// neither wait for running kernels nor slow them down.)
//
// A spin kernel (all SMs, ~T ms) runs on a stream; while it runs the host
// unmaps, remaps and re-grants access to N pages of an unrelated slot VA.
// Reported: each call's wall time (a call that waits for the kernel takes ~T),
// whether the calls returned before the kernel finished, and the kernel's
// device time with and without the concurrent VMM traffic.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o vmm_overlap vmm_overlap.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

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

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void spin(long long cycles, int* flag) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(flag, 1);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 64;               // pages touched while the kernel runs
  const long long cycles = argc > 2 ? atoll(argv[2]) : 200000000LL;  // ~100 ms at ~1.9 GHz
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
  std::vector<CUmemGenericAllocationHandle> h(n);
  for (int i = 0; i < n; ++i) CK(cuMemCreate(&h[i], page, &prop, 0));
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, n * page, page, 0, 0));
  CUmemAccessDesc acc{};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (int i = 0; i < n; ++i) CK(cuMemMap(va + i * page, page, 0, h[i], 0));
  CK(cuMemSetAccess(va, n * page, &acc, 1));

  int* flag;
  cudaMalloc(&flag, sizeof(int));
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

  double first_unmap_ms = 0;
  auto vmm_idle = [&](double* u, double* m, double* a) {  // the same calls with the GPU idle
    cudaDeviceSynchronize();
    double t = now_ms();
    for (int i = 0; i < n; ++i) cuMemUnmap(va + i * page, page);
    *u = now_ms() - t;
    t = now_ms();
    for (int i = 0; i < n; ++i) cuMemMap(va + i * page, page, 0, h[i], 0);
    *m = now_ms() - t;
    t = now_ms();
    cuMemSetAccess(va, n * page, &acc, 1);
    *a = now_ms() - t;
  };
  auto run_kernel = [&](bool with_vmm, double* unmap_ms, double* map_ms, double* access_ms, int* done_before) {
    cudaMemset(flag, 0, sizeof(int));
    cudaDeviceSynchronize();
    cudaEventRecord(e0, st);
    spin<<<sms * 2, 128, 0, st>>>(cycles, flag);
    cudaEventRecord(e1, st);
    if (with_vmm) {
      double t = now_ms();
      cuMemUnmap(va, page);
      first_unmap_ms = now_ms() - t;
      for (int i = 1; i < n; ++i) cuMemUnmap(va + i * page, page);
      *unmap_ms = now_ms() - t;
      t = now_ms();
      for (int i = 0; i < n; ++i) cuMemMap(va + i * page, page, 0, h[i], 0);
      *map_ms = now_ms() - t;
      t = now_ms();
      cuMemSetAccess(va, n * page, &acc, 1);
      *access_ms = now_ms() - t;
      int f = 0;
      cudaMemcpy(&f, flag, sizeof(int), cudaMemcpyDeviceToHost);  // default stream: does not wait for `st`
      *done_before = f;  // 0: every VMM call above returned while the kernel was still running
    }
    cudaStreamSynchronize(st);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return (double)ms;
  };
  double u = 0, m = 0, a = 0;
  int done = -1;
  run_kernel(false, &u, &m, &a, &done);  // warm-up
  const double base = run_kernel(false, &u, &m, &a, &done);
  double iu = 0, im = 0, ia = 0;
  vmm_idle(&iu, &im, &ia);
  vmm_idle(&iu, &im, &ia);
  const double with = run_kernel(true, &u, &m, &a, &done);
  printf("{\"pages\": %d, \"kernel_ms_alone\": %.3f, \"kernel_ms_with_vmm\": %.3f, "
         "\"busy\": {\"first_unmap_ms\": %.3f, \"unmap_ms\": %.3f, \"map_ms\": %.3f, \"setaccess_ms\": %.3f}, "
         "\"idle\": {\"unmap_ms\": %.3f, \"map_ms\": %.3f, \"setaccess_ms\": %.3f}, "
         "\"kernel_finished_before_vmm_calls_returned\": %d}\n",
         n, base, with, first_unmap_ms, u, m, a, iu, im, ia, done);
  return 0;
}
