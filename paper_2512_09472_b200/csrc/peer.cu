// Allreduce (sum, fp32) over peer memory for the TP row-parallel partials
// — the NVSwitch replacement for ncclAllReduce on
// the O / down outputs. Below 1 MiB one-shot (one kernel, every rank reads
// all peers: latency-bound decode messages); from 1 MiB two-shot (reduce
// this rank's 1/W chunk, then gather the reduced chunks: 2(W-1)/W of the
// bytes per rank instead of W-1, for prefill partials).
//
// Every rank owns one IPC-exported buffer: a flag row (one epoch word per
// source rank) and two data slots. A call copies the rank's partial into slot
// (epoch & 1) of its own buffer, then one kernel
//   1. block 0 publishes `epoch` into every peer's flag row (system-scope
//      release after a system fence),
//   2. every CTA waits until all peers' words in its own flag row reached
//      `epoch` (system-scope acquire),
//   3. sums the W slots in rank order over peer loads (NVLink reads on a
//      multi-GPU node), grid-stride with 16 B accesses.
// The sum order is the same on every rank, so all ranks hold bit-identical
// results. Two slots make a reused buffer safe: a rank can only run one
// epoch ahead of the slowest peer (it needs that peer's flag for the next
// epoch, which the peer writes only after finishing its previous reduce), so
// slot (epoch & 1) is never overwritten while a peer still reads it.
// The grid never exceeds the resident CTA count (the waits would otherwise
// starve block 0). One rank: allreduce is the identity and returns at once.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.h"
#include "kernels/ops.cuh"
#include "kernels/pdl.cuh"

using bf16_t = __nv_bfloat16;

namespace {

constexpr int kMaxPeers = 8;
// Fused GEMM + allreduce: per 128-row x 256-column block of the row-parallel
// output, a "partial stored" flag (written by the GEMM epilogue) and a
// "block reduced" flag (written by its owner rank's reduce), per rank.
constexpr int kMaxBlocks = 8192;
constexpr int64_t kRowFlagBytes = 4096;  // epoch flag rows of the unfused kernels
constexpr int64_t kFlagBytes = kRowFlagBytes + 2 * kMaxBlocks * 4;  // + tile flags; data slots follow

int64_t slot_bytes(int64_t max_count) { return (max_count * 4 + 255) / 256 * 256; }

struct PeerArgs {
  const float* data[kMaxPeers];  // slot (epoch & 1) of every rank's buffer
  float* res[kMaxPeers];         // two-shot: reduced-chunk region (epoch & 1) of every rank
  uint32_t* flags[kMaxPeers];    // every rank's flag row: [0, 64) phase A (data ready), [64, 128) phase B
  int rank, world;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Publish `epoch` to every peer's flag word (row offset `phase`), then wait
// for every peer's word in this rank's own row. Block 0 signals; every CTA waits.
__device__ __forceinline__ void peer_barrier(const PeerArgs& a, int phase, uint32_t epoch) {
  if (blockIdx.x == 0 && threadIdx.x < a.world && (int)threadIdx.x != a.rank) {
    __threadfence_system();
    st_release_sys(a.flags[threadIdx.x] + phase + a.rank, epoch);
  }
  if (threadIdx.x == 0) {
    const uint32_t* mine = a.flags[a.rank] + phase;
    for (int p = 0; p < a.world; ++p) {
      if (p == a.rank) continue;
      while ((int32_t)(ld_acquire_sys(mine + p) - epoch) < 0) __nanosleep(128);
    }
  }
  __syncthreads();
}

// MODE 0: out = sum, 1: out += sum, 2: allgather (out[r * n + i] = slot_r[i])
template <int MODE>
__global__ void __launch_bounds__(256, 4) peer_allreduce_kernel(const __grid_constant__ PeerArgs a, float* out,
                                                             int64_t n, uint32_t epoch) {
  peer_barrier(a, 0, epoch);
  const int64_t n4 = n / 4, stride = (int64_t)gridDim.x * blockDim.x;
  if constexpr (MODE == 2) {
    for (int p = 0; p < a.world; ++p) {
      float* dst = out + (int64_t)p * n;
      const bool vec = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
      for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (vec ? n4 : 0); i += stride)
        reinterpret_cast<float4*>(dst)[i] = __ldcv(reinterpret_cast<const float4*>(a.data[p]) + i);
      for (int64_t i = (vec ? n4 * 4 : 0) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = __ldcv(a.data[p] + i);
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 s = __ldcv(reinterpret_cast<const float4*>(a.data[0]) + i);
    for (int p = 1; p < a.world; ++p) {
      const float4 v = __ldcv(reinterpret_cast<const float4*>(a.data[p]) + i);
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    if constexpr (MODE == 1) {  // out += sum (the residual add of a row-parallel projection)
      const float4 o = reinterpret_cast<const float4*>(out)[i];
      s = make_float4(o.x + s.x, o.y + s.y, o.z + s.z, o.w + s.w);
    }
    reinterpret_cast<float4*>(out)[i] = s;
  }
  for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float s = __ldcv(a.data[0] + i);
    for (int p = 1; p < a.world; ++p) s += __ldcv(a.data[p] + i);
    out[i] = MODE == 1 ? out[i] + s : s;
  }
}

// Two-shot (large messages: every rank reads 2(W-1)/W of the data over the
// links instead of (W-1)x). Phase 1: rank r sums chunk r of every rank's
// slot (rank order) into its own res region. Phase 2 (next kernel, so all of
// phase 1 is complete before the signal): gather every rank's reduced chunk.
__global__ void __launch_bounds__(256, 4) peer_reduce_chunk_kernel(const __grid_constant__ PeerArgs a, int64_t n,
                                                                int64_t chunk, uint32_t epoch) {
  peer_barrier(a, 0, epoch);
  const int64_t lo = (int64_t)a.rank * chunk, hi = min(n, lo + chunk);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float* dst = a.res[a.rank];
  for (int64_t i = lo / 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi / 4; i += stride) {
    float4 s = __ldcv(reinterpret_cast<const float4*>(a.data[0]) + i);
    for (int p = 1; p < a.world; ++p) {
      const float4 v = __ldcv(reinterpret_cast<const float4*>(a.data[p]) + i);
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    reinterpret_cast<float4*>(dst)[i] = s;
  }
  for (int64_t i = max(lo, hi / 4 * 4) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += stride) {
    float s = __ldcv(a.data[0] + i);
    for (int p = 1; p < a.world; ++p) s += __ldcv(a.data[p] + i);
    dst[i] = s;
  }
}

template <bool ACC>
__global__ void __launch_bounds__(256, 4) peer_gather_chunks_kernel(const __grid_constant__ PeerArgs a, float* out,
                                                                 int64_t n, int64_t chunk, uint32_t epoch) {
  peer_barrier(a, 64, epoch);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += stride) {
    const float4 v = __ldcv(reinterpret_cast<const float4*>(a.res[(i * 4) / chunk]) + i);
    float4 o = v;
    if constexpr (ACC) {
      const float4 x = reinterpret_cast<const float4*>(out)[i];
      o = make_float4(x.x + v.x, x.y + v.y, x.z + v.z, x.w + v.w);
    }
    reinterpret_cast<float4*>(out)[i] = o;
  }
  for (int64_t i = n / 4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = __ldcv(a.res[i / chunk] + i);
    out[i] = ACC ? out[i] + v : v;
  }
}

// ---- fused row-parallel GEMM + allreduce (prefill-sized TP partials) ----
// Block b = 128 rows x 256 columns of the [M, N] output: tile b / 2 of the
// CTA-pair GEMM (m-block tile % mb, n-block tile / mb), rows (b & 1) * 128.
// Phase 1: rank r owns blocks b % W == r; as soon as every rank's GEMM has
// published block b, the owner sums the W bf16 partials in rank order (fp32)
// into its own reduced region (bf16) and publishes it. Phase 2: every rank
// takes every block from its owner once published: x += reduced. Each CTA
// walks its blocks in tile order, so both phases trail the GEMM's waves tile
// by tile over the links instead of waiting for the whole partial; every
// element is reduced once, in rank order: all ranks hold the same bits.
struct TileArgs {
  const bf16_t* part[kMaxPeers];  // every rank's partial slot (bf16 [M, N])
  bf16_t* red[kMaxPeers];         // every rank's reduced region (bf16 [M, N], owner blocks only)
  const uint32_t* done[kMaxPeers];  // every rank's "partial stored" flags
  uint32_t* reduced[kMaxPeers];     // every rank's "block reduced" flags
  int rank, world, M, N, mb;        // mb: 256-row m-blocks
};

__device__ __forceinline__ void wait_flag(const uint32_t* f, uint32_t epoch) {
  while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) __nanosleep(64);
}

__global__ void __launch_bounds__(256, 4) peer_tile_reduce_kernel(const __grid_constant__ TileArgs a, float* x,
                                                               uint32_t epoch) {
  // no griddepcontrol.wait: launched as the GEMM's programmatic dependent, it
  // runs beside the GEMM and synchronises on the per-block flags (a flag is
  // only published after the GEMM passed its own wait, i.e. after every
  // earlier kernel of the stream completed)
  const int nb = a.N / 256, blocks = a.mb * 2 * nb;
  auto rows_of = [&](int b, int& r0, int& c0) {
    const int tile = b >> 1;
    r0 = (tile % a.mb) * 256 + (b & 1) * 128;
    c0 = (tile / a.mb) * 256;
  };
  // phase 1: owned blocks
  for (int b = a.rank + (int)blockIdx.x * a.world; b < blocks; b += (int)gridDim.x * a.world) {
    if (threadIdx.x < a.world) wait_flag(a.done[threadIdx.x] + b, epoch);
    __syncthreads();
    int r0, c0;
    rows_of(b, r0, c0);
    const int rows = min(128, a.M - r0);
    // 128 x 256 bf16 = 4096 16-byte vectors; thread: 16 of them
    for (int v = threadIdx.x; v < rows * 32; v += 256) {
      const int64_t off = (int64_t)(r0 + v / 32) * a.N + c0 + (v % 32) * 8;
      float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int p = 0; p < a.world; ++p) {
        const uint4 u = __ldcv(reinterpret_cast<const uint4*>(a.part[p] + off));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          s[2 * k] += __uint_as_float(w[k] << 16);
          s[2 * k + 1] += __uint_as_float(w[k] & 0xffff0000u);
        }
      }
      uint4 o;
      uint32_t* ow = &o.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 h = __floats2bfloat162_rn(s[2 * k], s[2 * k + 1]);
        ow[k] = *reinterpret_cast<uint32_t*>(&h);
      }
      *reinterpret_cast<uint4*>(a.red[a.rank] + off) = o;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) st_release_sys(a.reduced[a.rank] + b, epoch);
  }
  // phase 2: every block, from its owner
  for (int b = (int)blockIdx.x; b < blocks; b += (int)gridDim.x) {
    const int owner = b % a.world;
    if (threadIdx.x == 0) wait_flag(a.reduced[owner] + b, epoch);
    __syncthreads();
    int r0, c0;
    rows_of(b, r0, c0);
    const int rows = min(128, a.M - r0);
    for (int v = threadIdx.x; v < rows * 32; v += 256) {
      const int64_t off = (int64_t)(r0 + v / 32) * a.N + c0 + (v % 32) * 8;
      const uint4 u = __ldcv(reinterpret_cast<const uint4*>(a.red[owner] + off));
      float4* xp = reinterpret_cast<float4*>(x + off);
      float4 x0 = xp[0], x1 = xp[1];
      x0.x += __uint_as_float(u.x << 16);
      x0.y += __uint_as_float(u.x & 0xffff0000u);
      x0.z += __uint_as_float(u.y << 16);
      x0.w += __uint_as_float(u.y & 0xffff0000u);
      x1.x += __uint_as_float(u.z << 16);
      x1.y += __uint_as_float(u.z & 0xffff0000u);
      x1.z += __uint_as_float(u.w << 16);
      x1.w += __uint_as_float(u.w & 0xffff0000u);
      xp[0] = x0;
      xp[1] = x1;
    }
    __syncthreads();  // the next block's wait is issued after every thread left this one
  }
}

}  // namespace

struct ws_peer {
  int rank = 0, world = 1, device = 0;
  int64_t max_count = 0;
  uint32_t epoch = 0;
  std::vector<char*> bufs;  // every rank's buffer base (own + IPC-opened)
};

extern "C" {

int ws_peer_buffer_bytes(int64_t max_count, int64_t* out) {
  if (max_count < 1 || !out) WS_FAIL(WS_ERR_INVALID, "bad peer buffer size");
  *out = kFlagBytes + 4 * slot_bytes(max_count);  // 2 data slots + 2 reduced-chunk regions
  return WS_OK;
}

int ws_peer_buffer_alloc(int64_t max_count, void** ptr, uint8_t* handle, int32_t handle_bytes) {
  if (!ptr || !handle || handle_bytes < (int32_t)sizeof(cudaIpcMemHandle_t))
    WS_FAIL(WS_ERR_INVALID, "peer buffer: need a %d-byte handle", (int)sizeof(cudaIpcMemHandle_t));
  int64_t bytes = 0;
  if (int e = ws_peer_buffer_bytes(max_count, &bytes)) return e;
  void* p = nullptr;
  WS_CUDA(cudaMalloc(&p, (size_t)bytes));
  WS_CUDA(cudaMemset(p, 0, kFlagBytes));
  cudaIpcMemHandle_t h;
  WS_CUDA(cudaIpcGetMemHandle(&h, p));
  memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return WS_OK;
}

int ws_peer_buffer_free(void* ptr) {
  if (ptr) WS_CUDA(cudaFree(ptr));
  return WS_OK;
}

int ws_peer_buffer_open(const uint8_t* handle, void** ptr) {
  if (!handle || !ptr) WS_FAIL(WS_ERR_INVALID, "bad peer handle");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  WS_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return WS_OK;
}

int ws_peer_buffer_close(void* ptr) {
  if (ptr) WS_CUDA(cudaIpcCloseMemHandle(ptr));
  return WS_OK;
}

int ws_peer_create(int32_t rank, int32_t world, void* const* bufs, int64_t max_count, ws_peer** out) {
  if (!out || !bufs || world < 1 || world > kMaxPeers || rank < 0 || rank >= world || max_count < 1)
    WS_FAIL(WS_ERR_INVALID, "bad peer group (rank %d of %d, at most %d)", rank, world, kMaxPeers);
  auto* p = new ws_peer;
  p->rank = rank;
  p->world = world;
  p->max_count = max_count;
  cudaGetDevice(&p->device);
  for (int r = 0; r < world; ++r) p->bufs.push_back(static_cast<char*>(bufs[r]));
  *out = p;
  return WS_OK;
}

int ws_peer_destroy(ws_peer* p) {
  delete p;
  return WS_OK;
}

// One epoch: out = (ACC ? out : 0) + sum of every rank's slot (epoch & 1);
// the caller's partial must already sit in its own slot.
// Messages of at least this many bytes (per rank) take the two-shot path.
constexpr int64_t kTwoShotBytes = 1 << 20;

static int run_epoch(ws_peer* p, float* out, int64_t count, int mode, cudaStream_t st) {
  const uint32_t epoch = ++p->epoch;
  const int64_t sb = slot_bytes(p->max_count);
  const int64_t slot = kFlagBytes + (int64_t)(epoch & 1) * sb, res = kFlagBytes + (2 + (int64_t)(epoch & 1)) * sb;
  PeerArgs a{};
  a.rank = p->rank;
  a.world = p->world;
  for (int r = 0; r < p->world; ++r) {
    a.data[r] = reinterpret_cast<const float*>(p->bufs[r] + slot);
    a.res[r] = reinterpret_cast<float*>(p->bufs[r] + res);
    a.flags[r] = reinterpret_cast<uint32_t*>(p->bufs[r]);
  }
  if (mode != 2 && p->world > 1 && count * 4 >= kTwoShotBytes) {
    const int64_t chunk = ((count + p->world - 1) / p->world + 3) / 4 * 4;  // float4-aligned chunks
    const int grid1 = (int)std::max<int64_t>(1, std::min<int64_t>(4 * ws::kNumSMs, (chunk / 4 + 255) / 256));
    const int grid2 = (int)std::max<int64_t>(1, std::min<int64_t>(4 * ws::kNumSMs, (count / 4 + 255) / 256));
    ws::count_launch(2);
    peer_reduce_chunk_kernel<<<grid1, 256, 0, st>>>(a, count, chunk, epoch);
    if (mode == 1)
      peer_gather_chunks_kernel<true><<<grid2, 256, 0, st>>>(a, out, count, chunk, epoch);
    else
      peer_gather_chunks_kernel<false><<<grid2, 256, 0, st>>>(a, out, count, chunk, epoch);
    WS_CUDA(cudaGetLastError());
    return WS_OK;
  }
  // up to 4 CTAs of 256 threads per SM: all resident (no smem, the next
  // kernel waits for this grid), more peer loads in flight than one per SM
  const int64_t want = (count / 4 + 255) / 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * ws::kNumSMs, want));
  ws::count_launch();
  if (mode == 1)
    peer_allreduce_kernel<1><<<grid, 256, 0, st>>>(a, out, count, epoch);
  else if (mode == 2)
    peer_allreduce_kernel<2><<<grid, 256, 0, st>>>(a, out, count, epoch);
  else
    peer_allreduce_kernel<0><<<grid, 256, 0, st>>>(a, out, count, epoch);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

static bool bad_args(const ws_peer* p, const float* buf, int64_t count) {
  return !p || !buf || count < 0 || count > p->max_count || reinterpret_cast<uintptr_t>(buf) % 16;
}

int ws_peer_allreduce_f32(ws_peer* p, float* buf, int64_t count, void* stream) {
  if (bad_args(p, buf, count))
    WS_FAIL(WS_ERR_INVALID, "bad peer allreduce (count <= max_count, 16-byte aligned buffer)");
  if (count == 0 || p->world == 1) return WS_OK;  // one rank: the sum is the input
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* slot = nullptr;
  if (int e = ws_peer_next_slot(p, &slot)) return e;
  WS_CUDA(cudaMemcpyAsync(slot, buf, (size_t)count * 4, cudaMemcpyDeviceToDevice, st));
  return run_epoch(p, buf, count, 0, st);
}

int ws_peer_allgather_f32(ws_peer* p, const float* send, float* recv, int64_t count, void* stream) {
  if (bad_args(p, send, count) || !recv)
    WS_FAIL(WS_ERR_INVALID, "bad peer allgather (count <= max_count, 16-byte aligned send buffer)");
  if (count == 0) return WS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* slot = nullptr;
  if (int e = ws_peer_next_slot(p, &slot)) return e;
  WS_CUDA(cudaMemcpyAsync(slot, send, (size_t)count * 4, cudaMemcpyDeviceToDevice, st));
  return run_epoch(p, recv, count, 2, st);
}

int ws_peer_next_slot(ws_peer* p, float** slot) {
  if (!p || !slot) WS_FAIL(WS_ERR_INVALID, "bad peer slot query");
  const uint32_t next = p->epoch + 1;
  *slot = reinterpret_cast<float*>(p->bufs[p->rank] + kFlagBytes + (int64_t)(next & 1) * slot_bytes(p->max_count));
  return WS_OK;
}

int ws_peer_gemm_reduce_add(ws_peer* p, const void* A, const void* W, int32_t M, int32_t N, int32_t K, float* x,
                            void* stream) {
  if (!p || !A || !W || !x || M < 1 || N < 1 || K < 1 || (int64_t)M * N > p->max_count ||
      reinterpret_cast<uintptr_t>(x) % 16)
    WS_FAIL(WS_ERR_INVALID, "bad fused GEMM + allreduce (M x N <= max_count, 16-byte aligned x)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bf16_t* a = static_cast<const bf16_t*>(A);
  const bf16_t* w = static_cast<const bf16_t*>(W);
  const int mb = (M + 255) / 256;
  const bool fused = p->world > 1 && ws::gemm_tc_pair_enabled(M) && N % 256 == 0 && K % 64 == 0 &&
                     mb * 2 * (N / 256) <= kMaxBlocks;
  if (!fused) {  // unfused: fp32 partial into the slot, then one reduce-add kernel
    float* slot = nullptr;
    if (int e = ws_peer_next_slot(p, &slot)) return e;
    ws::launch_gemm(a, w, M, N, K, ws::Epi::kStoreF32, slot, nullptr, st);
    if (p->world == 1) {
      ws::launch_add_f32(x, slot, (int64_t)M * N, st);
      return WS_OK;
    }
    return run_epoch(p, x, (int64_t)M * N, 1, st);
  }
  const uint32_t epoch = ++p->epoch;
  const int64_t sb = slot_bytes(p->max_count);
  const int64_t slot = kFlagBytes + (int64_t)(epoch & 1) * sb, res = kFlagBytes + (2 + (int64_t)(epoch & 1)) * sb;
  TileArgs t{};
  t.rank = p->rank;
  t.world = p->world;
  t.M = M;
  t.N = N;
  t.mb = mb;
  for (int r = 0; r < p->world; ++r) {
    t.part[r] = reinterpret_cast<const bf16_t*>(p->bufs[r] + slot);
    t.red[r] = reinterpret_cast<bf16_t*>(p->bufs[r] + res);
    t.done[r] = reinterpret_cast<const uint32_t*>(p->bufs[r] + kRowFlagBytes);
    t.reduced[r] = reinterpret_cast<uint32_t*>(p->bufs[r] + kRowFlagBytes + kMaxBlocks * 4);
  }
  ws::TcEpilogue e;
  e.mode = ws::Epi::kStoreBf16;
  e.C = p->bufs[p->rank] + slot;
  e.tile_flags = reinterpret_cast<uint32_t*>(p->bufs[p->rank] + kRowFlagBytes);
  e.tile_epoch = epoch;
  if (!ws::launch_gemm_tc_epi(a, w, M, N, K, e, st)) WS_FAIL(WS_ERR_CUDA, "fused row-parallel GEMM declined");
  ws::count_launch();
  ws::launch_pdl(peer_tile_reduce_kernel, dim3(ws::kNumSMs), dim3(256), 0, st, t, x, epoch);
  WS_CUDA(cudaGetLastError());
  return WS_OK;
}

int ws_peer_reduce_add_f32(ws_peer* p, float* x, int64_t count, void* stream) {
  if (bad_args(p, x, count))
    WS_FAIL(WS_ERR_INVALID, "bad peer reduce-add (count <= max_count, 16-byte aligned buffer)");
  if (count == 0) return WS_OK;
  return run_epoch(p, x, count, 1, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
