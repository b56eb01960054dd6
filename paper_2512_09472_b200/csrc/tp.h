// Internal TP collective helpers (the C-ABI lives in include/warmserve.h).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/warmserve.h"

namespace ws {
int comm_allreduce_f32(ws_comm* c, float* buf, int64_t count, cudaStream_t st);
int comm_allreduce_bf16(ws_comm* c, void* buf, int64_t count, cudaStream_t st);
bool comm_has_nccl(const ws_comm* c);
int comm_allgather_f32(ws_comm* c, const float* send, float* recv, int64_t count, cudaStream_t st);
// the communicator's peer-memory allreduce if one is attached and covers
// `count` floats, else null (NCCL path)
ws_peer* comm_peer(const ws_comm* c, int64_t count);
int comm_rank(const ws_comm* c);
int comm_size(const ws_comm* c);
}  // namespace ws
