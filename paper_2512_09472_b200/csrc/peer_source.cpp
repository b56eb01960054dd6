// Peer-HBM weight source: a universal worker
// that holds a model's slot exports the physical handles behind it
// (ws_pool_export_slot, POSIX fds); another worker's process imports them and
// maps them into its own VA, granting its device access. The layer streamer
// then copies layers k..L from that VA — a device-to-device copy the copy
// engine runs over NVLink 5 / NVSwitch when the exporter is another GPU
// (the reference's k = 1 regime at >= 750 GB/s, cluster.py:145-166), or
// within HBM when it is the same GPU. No host staging: the source is device
// memory of the peer, mapped P2P.
#include <unistd.h>

#include <vector>

#include "common.h"
#include "driver.h"

struct ws_peer_map {
  int dev = -1;
  CUdeviceptr va = 0;
  size_t bytes = 0;
  std::vector<CUmemGenericAllocationHandle> handles;
  std::vector<size_t> sizes;
};

namespace {
void release(const ws::Driver* d, ws_peer_map* m) {
  size_t off = 0;
  for (size_t i = 0; i < m->handles.size(); ++i) {
    if (i < m->sizes.size() && m->va) d->cuMemUnmap(m->va + off, m->sizes[i]);
    if (i < m->sizes.size()) off += m->sizes[i];
    d->cuMemRelease(m->handles[i]);
  }
  if (m->va) d->cuMemAddressFree(m->va, m->bytes);
  delete m;
}
}  // namespace

extern "C" {

int ws_device_can_access_peer(int32_t device, int32_t peer_device, int32_t* out) {
  int v = 0;
  WS_CUDA(cudaDeviceCanAccessPeer(&v, device, peer_device));
  *out = v;
  return WS_OK;
}

int ws_peer_map_import(int32_t device, const int32_t* fds, const int64_t* sizes, int64_t n, void** va_out,
                       ws_peer_map** out) {
  const ws::Driver* d = ws::driver();
  if (!d) return WS_ERR_NO_DEVICE;
  if (n < 1) WS_FAIL(WS_ERR_INVALID, "nothing to import");
  WS_CUDA(cudaSetDevice(device));
  ws_peer_map* m = new ws_peer_map();
  m->dev = device;
  for (int64_t i = 0; i < n; ++i) m->bytes += (size_t)sizes[i];
  auto fail = [&](const char* what, CUresult r) {
    const char* s = "?";
    d->cuGetErrorString(r, &s);
    ws::set_error(std::string(what) + " failed: " + s);
    release(d, m);
    return WS_ERR_CUDA;
  };
  CUresult r = d->cuMemAddressReserve(&m->va, m->bytes, (size_t)sizes[0], 0, 0);
  if (r != CUDA_SUCCESS) {
    m->va = 0;
    return fail("cuMemAddressReserve", r);
  }
  size_t off = 0;
  for (int64_t i = 0; i < n; ++i) {
    CUmemGenericAllocationHandle h;
    r = d->cuMemImportFromShareableHandle(&h, reinterpret_cast<void*>((intptr_t)fds[i]),
                                          CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) return fail("cuMemImportFromShareableHandle", r);
    m->handles.push_back(h);
    r = d->cuMemMap(m->va + off, (size_t)sizes[i], 0, h, 0);
    if (r != CUDA_SUCCESS) return fail("cuMemMap(peer handle)", r);
    m->sizes.push_back((size_t)sizes[i]);
    off += (size_t)sizes[i];
  }
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READ;
  r = d->cuMemSetAccess(m->va, m->bytes, &acc, 1);
  if (r != CUDA_SUCCESS) return fail("cuMemSetAccess(peer mapping; needs P2P between the devices)", r);
  *va_out = reinterpret_cast<void*>(m->va);
  *out = m;
  return WS_OK;
}

int ws_peer_map_release(ws_peer_map* m) {
  if (!m) return WS_OK;
  const ws::Driver* d = ws::driver();
  if (!d) return WS_ERR_NO_DEVICE;
  cudaSetDevice(m->dev);
  cudaDeviceSynchronize();
  release(d, m);
  return WS_OK;
}

}  // extern "C"
