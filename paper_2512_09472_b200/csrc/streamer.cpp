// Layer streamer: the copy half of a cold activation. Copies layers k..L of a
// prewarmed slot from pinned host memory (PCIe Gen5) or a peer GPU's HBM
// (NVLink 5, cudaMemcpyDefault resolves peer addresses) on a DMA copy engine,
// recording one event per layer so the compute stream waits layer by layer —
// the physical form of catch-up streaming (cluster.py:169-182,
// engine.py:513-538). No SM cycles are spent on the copy.
#include <vector>

#include "common.h"
#include "kernels/ops.cuh"
#include "kernels/pdl_flag.h"

struct ws_streamer {
  std::vector<cudaEvent_t> done;    // per range, timing-enabled: the range is usable
  std::vector<cudaEvent_t> copied;  // packed mode: the range's packed bytes are in staging
  cudaEvent_t start = nullptr;
  int32_t started = 0;
};

extern "C" {

int ws_streamer_create(int32_t max_ranges, ws_streamer** out) {
  if (max_ranges < 1) WS_FAIL(WS_ERR_INVALID, "streamer needs at least one range");
  ws_streamer* s = new ws_streamer();
  s->done.resize(max_ranges, nullptr);
  if (cudaEventCreate(&s->start) != cudaSuccess) {
    delete s;
    WS_FAIL(WS_ERR_CUDA, "cudaEventCreate failed");
  }
  for (auto& e : s->done)
    if (cudaEventCreate(&e) != cudaSuccess) {
      ws_streamer_destroy(s);
      WS_FAIL(WS_ERR_CUDA, "cudaEventCreate failed");
    }
  *out = s;
  return WS_OK;
}

int ws_streamer_destroy(ws_streamer* s) {
  if (!s) return WS_OK;
  if (s->start) cudaEventDestroy(s->start);
  for (auto e : s->done)
    if (e) cudaEventDestroy(e);
  for (auto e : s->copied)
    if (e) cudaEventDestroy(e);
  delete s;
  return WS_OK;
}

int ws_streamer_start(ws_streamer* s, void* dst_base, const void* src_base, const int64_t* ranges,
                      int32_t n, void* copy_stream) {
  if (!s) WS_FAIL(WS_ERR_INVALID, "null streamer");
  if (n < 0 || n > (int32_t)s->done.size()) WS_FAIL(WS_ERR_INVALID, "too many ranges");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(copy_stream);
  WS_CUDA(cudaEventRecord(s->start, st));
  for (int32_t i = 0; i < n; ++i) {
    const int64_t dst_off = ranges[3 * i], src_off = ranges[3 * i + 1], bytes = ranges[3 * i + 2];
    if (bytes > 0)
      WS_CUDA(cudaMemcpyAsync(static_cast<char*>(dst_base) + dst_off,
                              static_cast<const char*>(src_base) + src_off, (size_t)bytes,
                              cudaMemcpyDefault, st));
    WS_CUDA(cudaEventRecord(s->done[i], st));
  }
  s->started = n;
  return WS_OK;
}

int ws_streamer_start_packed(ws_streamer* s, void* dst_base, const void* packed_base, const int64_t* desc,
                             int32_t n, void* staging, int64_t staging_bytes, void* copy_stream,
                             void* unpack_stream) {
  if (!s) WS_FAIL(WS_ERR_INVALID, "null streamer");
  if (n < 0 || n > (int32_t)s->done.size()) WS_FAIL(WS_ERR_INVALID, "too many ranges");
  if (!staging || ((uintptr_t)staging & 255)) WS_FAIL(WS_ERR_INVALID, "staging must be 256-byte aligned");
  const int64_t half = staging_bytes / 2 / 256 * 256;  // two alternating slots
  if (s->copied.size() < s->done.size()) {
    s->copied.resize(s->done.size(), nullptr);
    for (auto& e : s->copied)
      if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
        WS_FAIL(WS_ERR_CUDA, "cudaEventCreate failed");
  }
  for (int32_t i = 0; i < n; ++i) {
    const int64_t* d = desc + 6 * i;
    if (d[5] > half) WS_FAIL(WS_ERR_INVALID, "packed range %d (%lld B) exceeds the staging slot (%lld B)", i,
                             (long long)d[5], (long long)half);
    if (d[3] != -1 && (d[3] < 0 || d[3] > 240)) WS_FAIL(WS_ERR_INVALID, "exponent base out of range");
  }
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(copy_stream);
  cudaStream_t us = reinterpret_cast<cudaStream_t>(unpack_stream);
  WS_CUDA(cudaEventRecord(s->start, cs));
  for (int32_t i = 0; i < n; ++i) {
    // desc[i] = {dst_offset, packed_offset, n_values, e_base (-1: Huffman), n_escapes, packed_bytes}
    const int64_t* d = desc + 6 * i;
    char* slot = static_cast<char*>(staging) + (i & 1) * half;
    if (i >= 2) WS_CUDA(cudaStreamWaitEvent(cs, s->done[i - 2], 0));  // slot free once range i-2 unpacked
    WS_CUDA(cudaMemcpyAsync(slot, static_cast<const char*>(packed_base) + d[1], (size_t)d[5], cudaMemcpyDefault, cs));
    WS_CUDA(cudaEventRecord(s->copied[i], cs));
    WS_CUDA(cudaStreamWaitEvent(us, s->copied[i], 0));
    if (d[3] < 0)
      ws::launch_unpack_huff(static_cast<char*>(dst_base) + d[0], slot, d[2], us);
    else
      ws::launch_unpack_bf16(static_cast<char*>(dst_base) + d[0], slot, d[2], (int)d[3], d[4], us);
    WS_CUDA(cudaEventRecord(s->done[i], us));
  }
  WS_CUDA(cudaGetLastError());
  s->started = n;
  return WS_OK;
}

int ws_streamer_wait(ws_streamer* s, int32_t i, void* stream) {
  if (!s) WS_FAIL(WS_ERR_INVALID, "null streamer");
  if (i < 0 || i >= s->started) return WS_OK;
  WS_CUDA(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), s->done[i], 0));
  ws::pdl_break_next();  // the kernel behind this wait launches without PDL (pdl_flag.h)
  return WS_OK;
}

int ws_streamer_progress(ws_streamer* s, int32_t* done_out) {
  if (!s) WS_FAIL(WS_ERR_INVALID, "null streamer");
  int32_t d = 0;
  while (d < s->started) {  // ranges complete in order (one copy stream)
    cudaError_t e = cudaEventQuery(s->done[d]);
    if (e == cudaErrorNotReady) break;
    if (e != cudaSuccess) WS_FAIL(WS_ERR_CUDA, "cudaEventQuery: %s", cudaGetErrorString(e));
    ++d;
  }
  *done_out = d;
  return WS_OK;
}

int ws_streamer_sync(ws_streamer* s, int32_t i) {
  if (!s) WS_FAIL(WS_ERR_INVALID, "null streamer");
  if (i < 0 || i >= s->started) return WS_OK;
  WS_CUDA(cudaEventSynchronize(s->done[i]));
  return WS_OK;
}

int ws_streamer_times(ws_streamer* s, float* ms_out, int32_t n) {
  if (!s) WS_FAIL(WS_ERR_INVALID, "null streamer");
  for (int32_t i = 0; i < n && i < s->started; ++i) {
    WS_CUDA(cudaEventSynchronize(s->done[i]));
    WS_CUDA(cudaEventElapsedTime(&ms_out[i], s->start, s->done[i]));
  }
  return WS_OK;
}

}  // extern "C"
