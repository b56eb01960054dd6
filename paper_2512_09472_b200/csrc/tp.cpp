// Tensor-parallel communicator for the large-model config (BASELINE config 4):
// NCCL over NVLink/NVSwitch, created once at prewarm time (the paper's
// pre-established communication group) and used only on the
// TP boundary — the row-parallel O / down projections (allreduce) and the
// vocab-parallel lm_head (allgather).
//
// NCCL is resolved with dlopen("libnccl.so.2") at first use, so the library
// has no link-time NCCL dependency and shares the NCCL torch already loaded.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "common.h"
#include "tp.h"

namespace {

// Minimal NCCL ABI (stable across NCCL 2.x).
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
enum { ncclSum = 0 };
enum { ncclFloat32 = 7, ncclBfloat16 = 9 };

struct Nccl {
  ncclResult_t (*getUniqueId)(ncclUniqueId*);
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);
  const char* (*getErrorString)(ncclResult_t);
};

Nccl g_nccl;
bool g_ok = false;
std::once_flag g_once;
std::string g_err;

const Nccl* nccl() {
  std::call_once(g_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      g_err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    g_nccl.getUniqueId = reinterpret_cast<decltype(g_nccl.getUniqueId)>(sym("ncclGetUniqueId"));
    g_nccl.commInitRank = reinterpret_cast<decltype(g_nccl.commInitRank)>(sym("ncclCommInitRank"));
    g_nccl.commDestroy = reinterpret_cast<decltype(g_nccl.commDestroy)>(sym("ncclCommDestroy"));
    g_nccl.allReduce = reinterpret_cast<decltype(g_nccl.allReduce)>(sym("ncclAllReduce"));
    g_nccl.allGather = reinterpret_cast<decltype(g_nccl.allGather)>(sym("ncclAllGather"));
    g_nccl.getErrorString = reinterpret_cast<decltype(g_nccl.getErrorString)>(sym("ncclGetErrorString"));
    g_ok = g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.commDestroy && g_nccl.allReduce &&
           g_nccl.allGather && g_nccl.getErrorString;
    if (!g_ok) g_err = "libnccl.so.2 lacks a required symbol";
  });
  if (!g_ok) {
    ws::set_error(g_err);
    return nullptr;
  }
  return &g_nccl;
}

}  // namespace

struct ws_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
  ws_peer* peer = nullptr;  // peer-memory allreduce (csrc/peer.cu); null = ncclAllReduce
  int64_t peer_max = 0;
};

namespace ws {

int comm_allreduce_f32(ws_comm* c, float* buf, int64_t count, cudaStream_t st) {
  if (c->peer && count <= c->peer_max) return ws_peer_allreduce_f32(c->peer, buf, count, st);
  if (!c->comm) WS_FAIL(WS_ERR_INVALID, "allreduce of %lld floats above the peer buffer", (long long)count);
  const Nccl* n = nccl();
  if (!n) return WS_ERR_INVALID;
  ncclResult_t r = n->allReduce(buf, buf, (size_t)count, ncclFloat32, ncclSum, c->comm, st);
  if (r != ncclSuccess) WS_FAIL(WS_ERR_CUDA, "ncclAllReduce: %s", n->getErrorString(r));
  return WS_OK;
}

int comm_allreduce_bf16(ws_comm* c, void* buf, int64_t count, cudaStream_t st) {
  if (!c->comm) WS_FAIL(WS_ERR_INVALID, "bf16 allreduce needs the NCCL communicator");
  const Nccl* n = nccl();
  if (!n) return WS_ERR_INVALID;
  ncclResult_t r = n->allReduce(buf, buf, (size_t)count, ncclBfloat16, ncclSum, c->comm, st);
  if (r != ncclSuccess) WS_FAIL(WS_ERR_CUDA, "ncclAllReduce(bf16): %s", n->getErrorString(r));
  return WS_OK;
}

bool comm_has_nccl(const ws_comm* c) { return c->comm != nullptr; }

ws_peer* comm_peer(const ws_comm* c, int64_t count) { return c->peer && count <= c->peer_max ? c->peer : nullptr; }

int comm_allgather_f32(ws_comm* c, const float* send, float* recv, int64_t count, cudaStream_t st) {
  if (c->peer && count <= c->peer_max) return ws_peer_allgather_f32(c->peer, send, recv, count, st);
  if (!c->comm) WS_FAIL(WS_ERR_INVALID, "allgather of %lld floats above the peer buffer", (long long)count);
  const Nccl* n = nccl();
  if (!n) return WS_ERR_INVALID;
  ncclResult_t r = n->allGather(send, recv, (size_t)count, ncclFloat32, c->comm, st);
  if (r != ncclSuccess) WS_FAIL(WS_ERR_CUDA, "ncclAllGather: %s", n->getErrorString(r));
  return WS_OK;
}

int comm_rank(const ws_comm* c) { return c->rank; }
int comm_size(const ws_comm* c) { return c->nranks; }

}  // namespace ws

extern "C" {

int ws_comm_set_peer(ws_comm* comm, ws_peer* peer, int64_t max_count) {
  if (!comm) WS_FAIL(WS_ERR_INVALID, "null communicator");
  comm->peer = peer;
  comm->peer_max = peer ? max_count : 0;
  return WS_OK;
}

int ws_comm_create_peer(int32_t rank, int32_t nranks, int32_t device, ws_peer* peer, int64_t max_count,
                        ws_comm** out) {
  if (!peer || !out || rank < 0 || nranks < 1 || rank >= nranks) WS_FAIL(WS_ERR_INVALID, "bad communicator arguments");
  ws_comm* c = new ws_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  c->peer = peer;
  c->peer_max = max_count;
  *out = c;
  return WS_OK;
}

int ws_nccl_unique_id(uint8_t* out, int32_t n) {
  if (n < 128) WS_FAIL(WS_ERR_INVALID, "unique id buffer needs 128 bytes");
  const Nccl* nc = nccl();
  if (!nc) return WS_ERR_INVALID;
  ncclUniqueId id;
  ncclResult_t r = nc->getUniqueId(&id);
  if (r != ncclSuccess) WS_FAIL(WS_ERR_CUDA, "ncclGetUniqueId: %s", nc->getErrorString(r));
  memcpy(out, id.internal, 128);
  return WS_OK;
}

int ws_comm_create(const uint8_t* id, int32_t rank, int32_t nranks, int32_t device, ws_comm** out) {
  if (!id || rank < 0 || nranks < 1 || rank >= nranks) WS_FAIL(WS_ERR_INVALID, "bad communicator arguments");
  const Nccl* nc = nccl();
  if (!nc) return WS_ERR_INVALID;
  WS_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  ws_comm* c = new ws_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  ncclResult_t r = nc->commInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    WS_FAIL(WS_ERR_CUDA, "ncclCommInitRank: %s", nc->getErrorString(r));
  }
  *out = c;
  return WS_OK;
}

int ws_comm_destroy(ws_comm* c) {
  if (!c) return WS_OK;
  if (c->comm && nccl()) nccl()->commDestroy(c->comm);
  delete c;
  return WS_OK;
}

}  // extern "C"
