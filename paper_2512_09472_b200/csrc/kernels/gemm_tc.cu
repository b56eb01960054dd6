// tcgen05 / TMEM / TMA GEMM for sm_100a — the prefill projections
// (QKV, O, gate/up, down) and large-M lm_head rows.
//
//   C[M,N] = A[M,K] . B[N,K]^T   (both operands K-major bf16, fp32 accumulate)
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer (one elected lane): A 128x64 + B 256x64 tiles,
//               SWIZZLE_128B, 4-stage smem ring guarded by full/empty mbarriers
//   warp 1      MMA issuer (one lane): tcgen05.mma.cta_group::1.kind::f16
//               M=128 N=256 K=16 x4 per stage, accumulator in TMEM,
//               tcgen05.commit frees the smem stage / publishes the tile
//   warp 2      TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4-7   epilogue: tcgen05.ld 32x32b.x32 -> registers -> bf16 (+bias)
//               or fp32 (+= residual) -> global; runs on accumulator b while
//               the MMA warp fills accumulator b^1 (double-buffered TMEM)
// Tile order: m fastest, so the 16 CTAs sharing a 256-row weight block run
// together and the weight tile is read from HBM once (L2 reuse).
#include <cuda.h>

#include <map>
#include <mutex>

#include "../common.h"
#include "../driver.h"
#include "device.cuh"
#include "ops.cuh"
#include "pdl.cuh"

namespace ws {

bool kv_window_tmap(const KvGeom& kv, int hd, CUtensorMap* out);  // attn_tc.cu
namespace {

using namespace dev;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, THREADS = 256;
constexpr int A_BYTES = BM * BK * 2;          // 16 KiB
constexpr int B_BYTES = BN * BK * 2;          // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 512;

// Instruction descriptor (kind::f16): D=F32 (bit 4), A=BF16 (bits 7-9 = 1),
// B=BF16 (bits 10-12 = 1), both K-major, N>>3 at bits 17-22, M>>4 at 24-28.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

// Shared-memory matrix descriptor for a K-major SWIZZLE_128B tile: rows of
// 128 B, 8-row core groups 1024 B apart (SBO), LBO unused (=1), version 1,
// layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n" ::"r"(dst),
      "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accum));
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}

#define TMEM_LD32(taddr, v)                                                                        \
  asm volatile(                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"             \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),       \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),   \
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),             \
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),             \
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])              \
      : "r"(taddr))

// 32 consecutive accumulator columns of one row -> bf16, 4 x 16 B stores
__device__ __forceinline__ void store_bf16x32(bf16* dst, const float* f) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    d[j] = make_uint4(pack_bf16x2(f[8 * j], f[8 * j + 1]), pack_bf16x2(f[8 * j + 2], f[8 * j + 3]),
                      pack_bf16x2(f[8 * j + 4], f[8 * j + 5]), pack_bf16x2(f[8 * j + 6], f[8 * j + 7]));
}

template <int MODE>
__device__ __forceinline__ void epilogue_tile(const TcEpilogue& ep, uint32_t tacc, int row, int n0, int N,
                                              int head_dim) {
  if constexpr (MODE == (int)Epi::kSwiGLU) {
    // tile columns [0,128) = gate block, [128,256) = matching up block
    bf16* out = static_cast<bf16*>(ep.C) + (int64_t)row * (N / 2) + n0 / 2;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t g[32], u[32];
      TMEM_LD32(tacc + c * 32, g);
      TMEM_LD32(tacc + 128 + c * 32, u);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (row < 0) continue;
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = __uint_as_float(g[j]);
        f[j] = silu(x) * __uint_as_float(u[j]);
      }
      store_bf16x32(out + c * 32, f);
    }
  } else if constexpr (MODE == (int)Epi::kRopeKV) {
    // tile = BN/head_dim whole heads; rotate_half pairs (i, i + hd/2) sit in
    // chunks (c, c + hd/64) of the same row, so one thread rotates its row.
    const KvGeom& kv = ep.kv;
    const int pos = row < 0 ? 0 : (ep.pos_arr ? ep.pos_arr[row] : ep.pos0 + row);
    const int seq = row < 0 ? 0 : (ep.seq_arr ? ep.seq_arr[row] : ep.seq0);
    const int half_chunks = head_dim / 64, per_head = head_dim / 32;
    const float2* cs = ep.rope + (int64_t)pos * (head_dim / 2);
    bf16* page = nullptr;
    if (row >= 0) {
      const int32_t pg = kv.block_tables[(int64_t)seq * kv.max_blocks + pos / kv.tpb];
      page = reinterpret_cast<bf16*>(kv.window + (int64_t)pg * kv.page_size) + (int64_t)(pos % kv.tpb) * head_dim;
    }
#pragma unroll 1
    for (int hl = 0; hl < BN / head_dim; ++hl) {
      const int hs = (n0 + hl * head_dim) / head_dim;  // head slot in [0, H + 2KV)
      const bool is_v = hs >= ep.heads + kv.kv_heads;
      const bool is_k = !is_v && hs >= ep.heads;
#pragma unroll 1
      for (int c = 0; c < half_chunks; ++c) {
        uint32_t a[32], b[32];
        const int ca = hl * per_head + c, cb = ca + half_chunks;
        TMEM_LD32(tacc + ca * 32, a);
        TMEM_LD32(tacc + cb * 32, b);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (row < 0) continue;
        float fa[32], fb[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          fa[j] = __uint_as_float(a[j]);
          fb[j] = __uint_as_float(b[j]);
        }
        if (ep.bias) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            fa[j] += bf2f(ep.bias[n0 + ca * 32 + j]);
            fb[j] += bf2f(ep.bias[n0 + cb * 32 + j]);
          }
        }
        if (!is_v) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float2 t = cs[c * 32 + j];
            const float x = fa[j], y = fb[j];
            fa[j] = x * t.x - y * t.y;
            fb[j] = y * t.x + x * t.y;
          }
        }
        if (!is_k && !is_v) {
          bf16* q = static_cast<bf16*>(ep.C) + (int64_t)row * N + n0;
          store_bf16x32(q + ca * 32, fa);
          store_bf16x32(q + cb * 32, fb);
        } else {
          const int kvh = is_v ? hs - ep.heads - kv.kv_heads : hs - ep.heads;
          bf16* dst = page + kv.plane(ep.layer, is_v ? 1 : 0, kvh);
          store_bf16x32(dst + c * 32, fa);
          store_bf16x32(dst + c * 32 + head_dim / 2, fb);
        }
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      TMEM_LD32(tacc + c * 32, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (row < 0) continue;
      const int col = n0 + c * 32;
      if constexpr (MODE == (int)Epi::kAddF32 || MODE == (int)Epi::kStoreF32) {
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(ep.C) + (int64_t)row * N + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 o = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                 __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
          if constexpr (MODE == (int)Epi::kAddF32) {
            const float4 r = dst[j];
            o.x += r.x;
            o.y += r.y;
            o.z += r.z;
            o.w += r.w;
          }
          dst[j] = o;
        }
      } else {
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        if constexpr (MODE == (int)Epi::kBiasBf16) {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] += bf2f(ep.bias[col + j]);
        }
        store_bf16x32(static_cast<bf16*>(ep.C) + (int64_t)row * N + col, f);
      }
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   int M, int N, int K, const __grid_constant__ TcEpilogue ep) {
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023) & ~1023u;  // SWIZZLE_128B atoms need 1024 B alignment
  const uint32_t bars = base + STAGES * STAGE_BYTES;
  // barrier layout: full[STAGES], empty[STAGES], tfull[2], tempty[2], then the TMEM slot
  auto full = [&](int s) { return bars + 8 * s; };
  auto empty = [&](int s) { return bars + 8 * (STAGES + s); };
  auto tfull = [&](int b) { return bars + 8 * (2 * STAGES + b); };
  auto tempty = [&](int b) { return bars + 8 * (2 * STAGES + 2 + b); };
  const uint32_t tmem_slot = bars + 8 * (2 * STAGES + 4);
  uint32_t* tmem_slot_ptr =
      reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_blocks = (M + BM - 1) / BM, n_blocks = N / BN, k_blocks = K / BK;
  const int tiles = m_blocks * n_blocks;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_b) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  pdl_wait();  // everything above is prologue; global data from here on

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m0 = (t % m_blocks) * BM, n0 = (t / m_blocks) * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(empty(stage), phase ^ 1);
          const uint32_t sa = base + stage * STAGE_BYTES;
          mbar_expect_tx(full(stage), STAGE_BYTES);
          tma_load(sa, &map_a, full(stage), kb * BK, m0);
          tma_load(sa + A_BYTES, &map_b, full(stage), kb * BK, n0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        mbar_wait(tempty(acc), acc_phase ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(full(stage), phase);
          tc_fence_after();
          const uint32_t sa = base + stage * STAGE_BYTES;
          const uint64_t da = smem_desc(sa), db = smem_desc(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // +32 B per K=16 step inside the 128 B swizzle row
            tc_mma(d, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), (kb | k) != 0);
          tc_commit(empty(stage));  // smem stage free once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(tfull(acc));  // accumulator complete
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    __syncwarp();  // reconverge before the CTA-wide (aligned) barrier below
  } else if (warp >= 4) {
    // ===== epilogue: TMEM lanes 32*q .. 32*q+31 belong to warp q = warp % 4 =====
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m0 = (t % m_blocks) * BM, n0 = (t / m_blocks) * BN;
      mbar_wait(tfull(acc), acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      epilogue_tile<MODE>(ep, tmem + ((uint32_t)(q * 32) << 16) + acc * BN, row < M ? row : -1, n0, N,
                          ep.kv.head_dim);
      tc_fence_before();
      mbar_arrive(tempty(acc));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
}

// ---------------------------------------------------------------------------
// CTA-pair version (tcgen05.mma.cta_group::2): a 2-CTA cluster computes a
// 256x256 tile; each CTA stages its 128 rows of A and 128 of the 256 B rows
// (half the smem operand traffic per SM of the 1-CTA 128x256 tile), the leader
// CTA issues M=256 MMAs reading both CTAs' smem, and each CTA's TMEM holds its
// 128 rows x 256 columns, drained by its own epilogue warps (same epilogues).
constexpr int P_BM = 128, P_BN = 256, P_BNH = 128, P_STAGES = 6;
constexpr int P_A_BYTES = P_BM * BK * 2, P_B_BYTES = P_BNH * BK * 2;
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;
constexpr int P_STG_BYTES = 4 * 2 * 4096;  // epilogue staging: 2 x (32 rows x 128 B) per epilogue warp
constexpr int P_SMEM_BYTES = P_STAGES * P_STAGE_BYTES + P_STG_BYTES + 1024 + 256;
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(P_BN >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// ---- coalesced epilogue: TMEM -> registers -> swizzled smem box -> TMA ----
// The tcgen05.ld 32x32b shape gives each thread one accumulator row, so direct
// global stores from registers touch 32 lines per warp instruction (one per
// row). Instead each epilogue warp writes its 32 rows x 128 B into a
// SWIZZLE_128B staging box (16-byte chunk j of row r at chunk j ^ (r & 7):
// conflict-free) and one lane issues a TMA store — or a TMA reduce-add for the
// fp32 residual, so x += acc is a single coalesced async op per 32x32 box.
// Two boxes per warp alternate; a box is rewritten only after the TMA engine
// has read it (bulk wait_group.read 1).
__device__ __forceinline__ void stage_f32(uint32_t buf, int lane, const uint32_t* v) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(buf + lane * 128 + ((j ^ (lane & 7)) << 4)),
                 "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                 : "memory");
}
// 32 bf16 values = chunks [4 * half, 4 * half + 4) of this lane's 128 B row
__device__ __forceinline__ void stage_bf16(uint32_t buf, int lane, int half, const float* f) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(buf + lane * 128 + (((half * 4 + j) ^ (lane & 7)) << 4)),
                 "r"(pack_bf16x2(f[8 * j], f[8 * j + 1])), "r"(pack_bf16x2(f[8 * j + 2], f[8 * j + 3])),
                 "r"(pack_bf16x2(f[8 * j + 4], f[8 * j + 5])), "r"(pack_bf16x2(f[8 * j + 6], f[8 * j + 7]))
                 : "memory");
}

struct Stager {
  uint32_t base;  // this warp's two 4 KB boxes
  int lane, b = 0;
  __device__ uint32_t acquire() {  // a box the TMA engine has finished reading
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
    __syncwarp();
    return base + b * 4096;
  }
  // make the generic-proxy smem writes visible to TMA, then store/reduce the box at (x, y)
  template <bool ADD>
  __device__ void issue(const CUtensorMap* map, int x, int y) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    const uint32_t src = base + b * 4096;
    if (lane == 0) {
      if constexpr (ADD)
        asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map),
                     "r"(x), "r"(y), "r"(src)
                     : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map),
                     "r"(x), "r"(y), "r"(src)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    b ^= 1;
  }
  __device__ void drain() {  // all issued TMA stores complete (global writes done)
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    __syncwarp();
  }
};

// One 128-row x 256-column accumulator (this warp: rows row0..row0+31) through
// the staging boxes.
template <int MODE>
__device__ __forceinline__ void epilogue_tile_tma(const TcEpilogue& ep, const CUtensorMap* map_c, Stager& st,
                                                  uint32_t tacc, int row0, int n0) {
  const int lane = st.lane;
  if constexpr (MODE == (int)Epi::kAddF32 || MODE == (int)Epi::kStoreF32) {
#pragma unroll 1
    for (int c = 0; c < 8; ++c) {
      uint32_t v[32];
      TMEM_LD32(tacc + c * 32, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      stage_f32(st.acquire(), lane, v);
      st.issue<MODE == (int)Epi::kAddF32>(map_c, n0 + c * 32, row0);
    }
  } else if constexpr (MODE == (int)Epi::kSwiGLU) {
    // tile columns [0,128) = gate block, [128,256) = matching up block -> 128 output columns
#pragma unroll 1
    for (int c = 0; c < 4; c += 2) {
      const uint32_t buf = st.acquire();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t g[32], u[32];
        TMEM_LD32(tacc + (c + h) * 32, g);
        TMEM_LD32(tacc + 128 + (c + h) * 32, u);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = __uint_as_float(g[j]);
          f[j] = silu(x) * __uint_as_float(u[j]);
        }
        stage_bf16(buf, lane, h, f);
      }
      st.issue<false>(map_c, n0 / 2 + c * 32, row0);
    }
  } else {  // kStoreBf16 / kBiasBf16: 64 columns per box
#pragma unroll 1
    for (int c = 0; c < 8; c += 2) {
      const uint32_t buf = st.acquire();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t v[32];
        TMEM_LD32(tacc + (c + h) * 32, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
        if constexpr (MODE == (int)Epi::kBiasBf16) {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] += bf2f(ep.bias[n0 + (c + h) * 32 + j]);
        }
        stage_bf16(buf, lane, h, f);
      }
      st.issue<false>(map_c, n0 + c * 32, row0);
    }
  }
}

// QKV + RoPE + paged KV append through the staging boxes (CTA-pair kernel,
// ep.kv_tma): this warp's 32 rows x one head (128 columns) are rotated in
// registers and staged as two 64-column SWIZZLE_128B boxes; q heads leave by
// TMA into the qkv buffer (map_c), k / v heads as two 16-token boxes each
// into the page window (map_kv: rows of head_dim bf16, 64 x 16 boxes) at the
// pages the block table names. A 16-token group that is not fully inside the
// prompt is stored row by row instead. Replaces 32-line-per-instruction
// direct stores (the QKV GEMM ran 25% slower with this epilogue than plain).
__device__ __forceinline__ void epilogue_rope_tma(const TcEpilogue& ep, const CUtensorMap* map_c,
                                                  const CUtensorMap* map_kv, uint32_t stg_base, int lane,
                                                  uint32_t tacc, int row0, int n0, int M) {
  constexpr int HD = 128;
  const KvGeom& kv = ep.kv;
  const int row = row0 + lane;
  const bool valid = row < M;
  const int pos = ep.pos0 + (valid ? row : row0);
  const float2* cs = ep.rope + (int64_t)pos * (HD / 2);
  // pages of the warp's two 16-token groups (rows row0.., row0 + 16..)
  const int32_t* bt = kv.block_tables + (int64_t)ep.seq0 * kv.max_blocks;
  const int rows_pp = (int)(kv.page_size / (HD * 2));
  const int p0 = ep.pos0 + row0;
  const bool g_full0 = row0 + 15 < M, g_full1 = row0 + 31 < M;
  const int32_t pg0 = g_full0 ? bt[p0 / kv.tpb] : 0, pg1 = g_full1 ? bt[(p0 + 16) / kv.tpb] : 0;
  bf16* page = nullptr;
  if (valid) {
    const int32_t pg = bt[pos / kv.tpb];
    page = reinterpret_cast<bf16*>(kv.window + (int64_t)pg * kv.page_size) + (int64_t)(pos % kv.tpb) * HD;
  }
  const bool my_group_tma = (lane < 16) ? g_full0 : g_full1;
#pragma unroll 1
  for (int hl = 0; hl < BN / HD; ++hl) {
    const int hs = (n0 + hl * HD) / HD;  // head slot in [0, H + 2KV)
    const bool is_v = hs >= ep.heads + kv.kv_heads;
    const bool is_k = !is_v && hs >= ep.heads;
    // both boxes free: every earlier TMA store has read its smem
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {  // c: columns [32c, 32c+32) and their rotate_half partners +64
      uint32_t a[32], b[32];
      const int ca = hl * 4 + c, cb = ca + 2;
      TMEM_LD32(tacc + ca * 32, a);
      TMEM_LD32(tacc + cb * 32, b);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      float fa[32], fb[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        fa[j] = __uint_as_float(a[j]);
        fb[j] = __uint_as_float(b[j]);
      }
      if (ep.bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          fa[j] += bf2f(ep.bias[n0 + ca * 32 + j]);
          fb[j] += bf2f(ep.bias[n0 + cb * 32 + j]);
        }
      }
      if (!is_v) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 t = cs[c * 32 + j];
          const float x = fa[j], y = fb[j];
          fa[j] = x * t.x - y * t.y;
          fb[j] = y * t.x + x * t.y;
        }
      }
      if ((is_k || is_v) && valid && !my_group_tma) {  // a partial 16-token group: row stores
        const int kvh = is_v ? hs - ep.heads - kv.kv_heads : hs - ep.heads;
        bf16* dst = page + kv.plane(ep.layer, is_v ? 1 : 0, kvh);
        store_bf16x32(dst + c * 32, fa);
        store_bf16x32(dst + c * 32 + HD / 2, fb);
      }
      stage_bf16(stg_base, lane, c, fa);         // box 0: head columns [0, 64)
      stage_bf16(stg_base + 4096, lane, c, fb);  // box 1: head columns [64, 128)
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      if (!is_k && !is_v) {
#pragma unroll
        for (int bx = 0; bx < 2; ++bx)
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map_c),
                       "r"(n0 + hl * HD + bx * 64), "r"(row0), "r"(stg_base + bx * 4096)
                       : "memory");
      } else {
        const int kvh = is_v ? hs - ep.heads - kv.kv_heads : hs - ep.heads;
        const int plane_rows = (int)(kv.plane(ep.layer, is_v ? 1 : 0, kvh) / HD);
        const int y0 = pg0 * rows_pp + plane_rows + p0 % kv.tpb;
        const int y1 = pg1 * rows_pp + plane_rows + (p0 + 16) % kv.tpb;
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
          if (g_full0)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map_kv),
                         "r"(bx * 64), "r"(y0), "r"(stg_base + bx * 4096)
                         : "memory");
          if (g_full1)
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map_kv),
                         "r"(bx * 64), "r"(y1), "r"(stg_base + bx * 4096 + 2048)
                         : "memory");
        }
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
}

// Work schedule of the pair kernel: tiles go round-robin to the pairs (m
// fastest), so all pairs run the same k-range of neighbouring tiles at the
// same time and each weight block is read from HBM once (L2 reuse).
// Residual GEMMs (x += A.B^T) with a partial last wave and a long K (the down
// projection: 128 tiles on 74 pairs) cut only the tiles of that last wave
// into `slices` k-slices dealt round-robin after the full waves: 54 tiles x 4
// slices run as 3 rounds of quarter tiles instead of one round of whole tiles
// on 54 of the 74 pairs. Slices of a tile reduce-add into x in slice order
// (slice q waits on the tile's flag for slice q-1, which ran one round
// earlier): one summation order, deterministic. (Stream-K ranges and slicing
// every tile were measured slower: they lose the lock-step L2 reuse of the
// full waves.)
struct TailSched {
  int dp_tiles;     // tiles [0, dp_tiles) whole; the rest sliced
  int slices;       // 1 = no tail slicing
  uint32_t* flags;  // [tail tile][2 ranks]: epoch * 16 + slices landed
  uint32_t epoch;
};

struct TileIter {
  int t, step, dp, tail, units, slices, KB;
  int u;
  __device__ TileIter(int pair, int n_pairs, int tiles, const TailSched& s, int kb)
      : t(pair), step(n_pairs), dp(s.dp_tiles), tail(tiles - s.dp_tiles), units((tiles - s.dp_tiles) * s.slices),
        slices(s.slices), KB(kb), u(-1) {}
  // tile, slice q, k-blocks [kb0, kb1)
  __device__ bool next(int& tile, int& q, int& kb0, int& kb1) {
    if (t < dp) {
      tile = t;
      q = 0;
      kb0 = 0;
      kb1 = KB;
      t += step;
      return true;
    }
    u = u < 0 ? t - dp : u + step;  // first tail unit continues the round-robin
    if (u >= units) return false;
    tile = dp + u % tail;
    q = u / tail;
    kb0 = q * KB / slices;
    kb1 = (q + 1) * KB / slices;
    return true;
  }
};

// WS_GEMM_TRACE build: per-CTA globaltimer trace [cta][0 start, 1-3 tile
// accumulators ready, 4-6 tile epilogues issued, 7 end] (tools/gemm_trace.py)
__device__ long long g_gemm_trace[148][8];
#ifdef WS_GEMM_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, int M,
                    int N, int K, const __grid_constant__ TcEpilogue ep,
                    const __grid_constant__ CUtensorMap map_c, const __grid_constant__ TailSched sched,
                    const __grid_constant__ CUtensorMap map_kv) {
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023) & ~1023u;
  const uint32_t stg = base + P_STAGES * P_STAGE_BYTES;  // 1024-aligned staging boxes
  const uint32_t bars = stg + P_STG_BYTES;
  auto full = [&](int s) { return bars + 8 * s; };
  auto empty = [&](int s) { return bars + 8 * (P_STAGES + s); };
  auto tfull = [&](int b) { return bars + 8 * (2 * P_STAGES + b); };
  auto tempty = [&](int b) { return bars + 8 * (2 * P_STAGES + 2 + b); };
  const uint32_t tmem_slot = bars + 8 * (2 * P_STAGES + 4);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - raw));
  const uint32_t peer_mask = 0xFEFFFFFFu;  // same offset in the leader (rank 0) CTA

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int m_blocks = (M + 255) / 256, n_blocks = N / P_BN, k_blocks = K / BK;
  const int tiles = m_blocks * n_blocks;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_b) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_c) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 1);
      mbar_init(tempty(b), 256);  // both CTAs' epilogue threads
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  auto load_a = [&](uint32_t sa, uint32_t bar, int kb, int m0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
        "[%1, {%3, %4}], [%2];\n" ::"r"(sa),
        "l"(&map_a), "r"(bar), "r"(kb * BK), "r"(m0)
        : "memory");
  };
  auto load_b = [&](uint32_t sa, uint32_t bar, int kb, int n0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
        "[%1, {%3, %4}], [%2];\n" ::"r"(sa + P_A_BYTES),
        "l"(&map_b), "r"(bar), "r"(kb * BK), "r"(n0)
        : "memory");
  };
  // The weight operand (B) is immutable: the producer fills the first ring
  // stages with B tiles before the PDL wait, so they stream in under the tail
  // of the previous kernel; A (the previous kernel's output) follows the wait.
  int tile, sq, kb0, kb1;
  int pre = 0, pre_m0 = 0, pre_kb0 = 0;
  if (warp == 0 && lane == 0) {
    TileIter it(pair, n_pairs, tiles, sched, k_blocks);
    if (it.next(tile, sq, kb0, kb1)) {
      pre = min(P_STAGES, kb1 - kb0);
      pre_m0 = (tile % m_blocks) * 256 + rank * P_BM;
      pre_kb0 = kb0;
      const int n0 = (tile / m_blocks) * P_BN + rank * P_BNH;
      for (int s = 0; s < pre; ++s) {
        if (rank == 0) mbar_expect_tx(full(s), 2 * P_STAGE_BYTES);  // both CTAs' bytes
        load_b(base + s * P_STAGE_BYTES, full(s) & peer_mask, kb0 + s, n0);
      }
    }
  }
  pdl_wait();  // global data produced by earlier kernels from here on

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < pre; ++s) load_a(base + s * P_STAGE_BYTES, full(s) & peer_mask, pre_kb0 + s, pre_m0);
      int stage = pre % P_STAGES;
      uint32_t phase = pre == P_STAGES ? 1 : 0;
      int skip = pre;  // k-blocks of the first unit already issued
      TileIter it(pair, n_pairs, tiles, sched, k_blocks);
      while (it.next(tile, sq, kb0, kb1)) {
        const int m0 = (tile % m_blocks) * 256 + rank * P_BM, n0 = (tile / m_blocks) * P_BN + rank * P_BNH;
        for (int kb = kb0 + skip; kb < kb1; ++kb) {
          mbar_wait(empty(stage), phase ^ 1);
          const uint32_t sa = base + stage * P_STAGE_BYTES;
          if (rank == 0) mbar_expect_tx(full(stage), 2 * P_STAGE_BYTES);  // both CTAs' bytes
          const uint32_t bar = full(stage) & peer_mask;
          load_a(sa, bar, kb, m0);
          load_b(sa, bar, kb, n0);
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        skip = 0;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      TileIter it(pair, n_pairs, tiles, sched, k_blocks);
      while (it.next(tile, sq, kb0, kb1)) {
        mbar_wait(tempty(acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * P_BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(full(stage), phase);
          tc_fence_after();
          const uint32_t sa = base + stage * P_STAGE_BYTES;
          const uint64_t da = smem_desc(sa), db = smem_desc(sa + P_A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(kIdesc2),
                "r"((uint32_t)(kb != kb0 || k != 0)));
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                  empty(stage)),
              "h"((uint16_t)3)
              : "memory");
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                tfull(acc)),
            "h"((uint16_t)3)
            : "memory");
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int r_in = q * 32 + lane;  // this thread's row inside the CTA's 128
    const bool tr = kTrace && r_in == 0;
    Stager st{stg + (uint32_t)q * 8192, lane};
    if (tr) g_gemm_trace[blockIdx.x][0] = gtimer();
    int acc = 0, seg = 0;
    uint32_t acc_phase = 0;
    TileIter it(pair, n_pairs, tiles, sched, k_blocks);
    while (it.next(tile, sq, kb0, kb1)) {
      const int m0 = (tile % m_blocks) * 256 + rank * P_BM, n0 = (tile / m_blocks) * P_BN;
      mbar_wait(tfull(acc), acc_phase);
      tc_fence_after();
      if (tr && seg < 3) g_gemm_trace[blockIdx.x][1 + seg] = gtimer();
      const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + acc * P_BN;
      const bool sliced = MODE == (int)Epi::kAddF32 && tile >= sched.dp_tiles && sched.slices > 1;
      uint32_t* flag = sched.flags + (tile - sched.dp_tiles) * 2 + rank;  // this CTA's 128 rows of the tile
      if (sliced && sq > 0) {  // slice sq reduce-adds after slice sq-1 of this tile has landed
        if (r_in == 0) {
          uint32_t v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flag) : "memory");
          } while (v != sched.epoch * 16 + sq);
        }
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
      }
      if constexpr (MODE == (int)Epi::kRopeKV) {
        if (ep.kv_tma) {
          epilogue_rope_tma(ep, &map_c, &map_kv, st.base, lane, tacc, m0 + q * 32, n0, M);
        } else {
          const int row = m0 + r_in;
          epilogue_tile<MODE>(ep, tacc, row < M ? row : -1, n0, N, ep.kv.head_dim);
        }
      } else {
        epilogue_tile_tma<MODE>(ep, &map_c, st, tacc, m0 + q * 32, n0);
      }
      tc_fence_before();
      // release this accumulator to the leader's MMA thread (remote arrive)
      asm volatile(
          "{\n.reg .b32 remAddr32;\nmapa.shared::cluster.u32 remAddr32, %0, 0;\n"
          "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [remAddr32];\n}\n" ::"r"(tempty(acc))
          : "memory");
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      if (ep.tile_flags != nullptr) {  // publish: these 128 rows x 256 columns are in C
        st.drain();
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        __threadfence_system();
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (r_in == 0)
          asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(ep.tile_flags + 2 * tile + rank),
                       "r"(ep.tile_epoch)
                       : "memory");
      }
      if (sliced && sq + 1 < sched.slices) {  // publish: slice sq of these 128 rows is in x
        st.drain();
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        __threadfence();
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (r_in == 0)
          asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(flag), "r"(sched.epoch * 16 + sq + 1)
                       : "memory");
      }
      if (tr && seg < 3) g_gemm_trace[blockIdx.x][4 + seg] = gtimer();
      ++seg;
    }
    st.drain();  // staging smem must outlive the TMA reads
  }
  if (kTrace && threadIdx.x == 128) g_gemm_trace[blockIdx.x][7] = gtimer();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
}

bool make_map(CUtensorMap* map, const void* ptr, int rows, int K, int box_rows) {
  const Driver* d = driver();
  if (!d) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return d->cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Epilogue store map: row-major [rows, cols] of `elem` bytes, 32-row boxes of
// 128 B (32 fp32 or 64 bf16), SWIZZLE_128B to match the staging layout.
bool make_out_map(CUtensorMap* map, const void* ptr, int rows, int cols, int elem) {
  const Driver* d = driver();
  if (!d || ((uintptr_t)ptr & 15) || (cols * elem) % 16) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * elem};
  cuuint32_t box[2] = {(cuuint32_t)(128 / elem), 32};
  cuuint32_t estr[2] = {1, 1};
  return d->cuTensorMapEncodeTiled(map, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                   2, const_cast<void*>(ptr), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool gemm_tc_supported(int M, int N, int K) { return M >= 16 && N % BN == 0 && K % BK == 0; }

bool gemm_tc_epilogue_supported(const TcEpilogue& e, int N, int head_dim) {
  if (e.mode == Epi::kRopeKV) return (head_dim == 64 || head_dim == 128) && N % BN == 0;
  return true;
}

template <int MODE>
void launch_mode(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, const TcEpilogue& e,
                 cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr = true;
  }
  const int tiles = ((M + BM - 1) / BM) * (N / BN);
  const int grid = tiles < kNumSMs ? tiles : kNumSMs;
  count_launch();
  launch_pdl(gemm_tc_kernel<MODE>, dim3(grid), dim3(THREADS), SMEM_BYTES, st, ma, mb, M, N, K, e);
}

// Tail slicing for residual GEMMs (see TailSched): the slice count with the
// shortest tail, only when every slice keeps >= 48 k-blocks (long enough to
// hide the slice's reduce-add epilogue behind the next slice's mainloop).
TailSched tail_schedule(int mode, int tiles, int& n_pairs, int k_blocks, cudaStream_t st) {
  TailSched p{};
  p.dp_tiles = tiles;
  p.slices = 1;
  static const bool on = !(getenv("WS_TAIL_SLICES") && getenv("WS_TAIL_SLICES")[0] == '0');
  if (!on || mode != (int)Epi::kAddF32) return p;
  int dp, best_s = 1;
  if (tiles < kNumSMs / 2) {
    // Less than one wave (O / down below ~1k prompt rows: 16 x 256-column
    // tiles per 256 rows): k-slice every tile so the pairs cover the GPU;
    // the slices reduce-add in k order. Llama-3-8B at 256 rows: O on 16
    // pairs of 74 read 33.5 MB in 26 us, down 117 MB in 70 us.
    dp = 0;
    best_s = std::min(8, (kNumSMs / 2) / tiles);
    while (best_s > 1 && k_blocks / best_s < 16) --best_s;
  } else {
    if (tiles <= n_pairs || tiles % n_pairs == 0) return p;
    dp = tiles / n_pairs * n_pairs;
    const int tail = tiles - dp;
    double best = 1.0;  // tail time in whole-tile units without slicing
    for (int s = 2; s <= 4 && k_blocks / s >= 48; ++s) {
      const double t = (double)((tail * s + n_pairs - 1) / n_pairs) / s;
      if (t < best - 0.01) {
        best = t;
        best_s = s;
      }
    }
  }
  if (best_s == 1 || tiles - dp > 4096) return p;
  // one flag array per (device, stream): launches on a stream are ordered, so
  // they can share it; concurrent streams must not (a waiter compares for equality)
  struct Flags {
    uint32_t* f = nullptr;
    uint32_t epoch = 0;
  };
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, Flags> all;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  Flags& fl = all[{dev, st}];
  if (!fl.f) {
    if (cudaMalloc(&fl.f, 2 * 4096 * sizeof(uint32_t)) != cudaSuccess) return p;
    cudaMemsetAsync(fl.f, 0, 2 * 4096 * sizeof(uint32_t), st);
  }
  if (++fl.epoch >= (1u << 27)) {  // a flag left by an earlier launch is below epoch * 16
    cudaMemsetAsync(fl.f, 0, 2 * 4096 * sizeof(uint32_t), st);
    fl.epoch = 1;
  }
  p.dp_tiles = dp;
  p.slices = best_s;
  p.flags = fl.f;
  p.epoch = fl.epoch;
  if (dp == 0) n_pairs = std::min(tiles * best_s, kNumSMs / 2);
  return p;
}

template <int MODE>
bool launch_mode2(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K, const TcEpilogue& e,
                  cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc2_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM_BYTES);
    attr = true;
  }
  const int tiles = ((M + 255) / 256) * (N / P_BN);
  int n_pairs = tiles < kNumSMs / 2 ? tiles : kNumSMs / 2;  // raised by tail_schedule when it k-slices
  CUtensorMap mc = ma;  // RoPE mode stores directly; the map is unused there
  if constexpr (MODE == (int)Epi::kAddF32 || MODE == (int)Epi::kStoreF32) {
    if (!make_out_map(&mc, e.C, M, N, 4)) return false;
  } else if constexpr (MODE == (int)Epi::kSwiGLU) {
    if (!make_out_map(&mc, e.C, M, N / 2, 2)) return false;
  } else if constexpr (MODE != (int)Epi::kRopeKV) {
    if (!make_out_map(&mc, e.C, M, N, 2)) return false;
  }
  CUtensorMap mkv = mc;
  TcEpilogue ee = e;
  if constexpr (MODE == (int)Epi::kRopeKV) {
    // TMA stores of the rotated rows: one sequence (prefill), 16-token runs
    // per block starting at a run boundary, head_dim 128, the window mappable
    static const bool on = !(getenv("WS_ROPE_TMA") && getenv("WS_ROPE_TMA")[0] == '0');
    ee.kv_tma = on && e.kv.head_dim == 128 && !e.seq_arr && !e.pos_arr && e.kv.tpb % 16 == 0 && e.pos0 % 16 == 0 &&
                make_out_map(&mc, e.C, M, N, 2) && kv_window_tmap(e.kv, 128, &mkv);
  }
  const TailSched sched = tail_schedule(MODE, tiles, n_pairs, K / BK, st);
  count_launch();
  launch_pdl(gemm_tc2_kernel<MODE>, dim3(2 * n_pairs), dim3(THREADS), P_SMEM_BYTES, st, ma, mb, M, N, K, ee, mc, sched,
             mkv);
  return true;
}

int g_pair_mode = -1;  // -1: unset (env WS_GEMM_PAIR, default on), 0 off, 1 on

bool use_pair(int M) {
  if (g_pair_mode < 0) {
    const char* v = getenv("WS_GEMM_PAIR");
    g_pair_mode = (v && v[0] == '0') ? 0 : 1;
  }
  // From 129 rows (the skinny kernel serves <= 128): one 256-row pair tile
  // streams the weights once where two 128-row tiles of the 1-CTA kernel
  // stream them twice (192-token prefill 8.6 -> see DESIGN §5).
  static const int min_m = getenv("WS_PAIR_MIN_M") ? atoi(getenv("WS_PAIR_MIN_M")) : 129;
  return g_pair_mode == 1 && M >= min_m;
}

bool gemm_tc_pair_enabled(int M) { return use_pair(M); }

bool launch_gemm_tc_epi(const bf16* A, const bf16* B, int M, int N, int K, const TcEpilogue& e,
                        cudaStream_t st) {
  if (!gemm_tc_supported(M, N, K) || !gemm_tc_epilogue_supported(e, N, e.kv.head_dim)) return false;
  if (e.tile_flags && !use_pair(M)) return false;  // only the pair kernel publishes its blocks
  CUtensorMap ma, mb;
  if (use_pair(M)) {
    if (!make_map(&ma, A, M, K, P_BM) || !make_map(&mb, B, N, K, P_BNH)) return false;
    switch (e.mode) {
      case Epi::kStoreBf16: return launch_mode2<0>(ma, mb, M, N, K, e, st);
      case Epi::kBiasBf16: return launch_mode2<1>(ma, mb, M, N, K, e, st);
      case Epi::kAddF32: return launch_mode2<2>(ma, mb, M, N, K, e, st);
      case Epi::kStoreF32: return launch_mode2<3>(ma, mb, M, N, K, e, st);
      case Epi::kSwiGLU: return launch_mode2<4>(ma, mb, M, N, K, e, st);
      case Epi::kRopeKV: return launch_mode2<5>(ma, mb, M, N, K, e, st);
    }
    return false;
  }
  if (!make_map(&ma, A, M, K, BM) || !make_map(&mb, B, N, K, BN)) return false;
  switch (e.mode) {
    case Epi::kStoreBf16: launch_mode<0>(ma, mb, M, N, K, e, st); break;
    case Epi::kBiasBf16: launch_mode<1>(ma, mb, M, N, K, e, st); break;
    case Epi::kAddF32: launch_mode<2>(ma, mb, M, N, K, e, st); break;
    case Epi::kStoreF32: launch_mode<3>(ma, mb, M, N, K, e, st); break;
    case Epi::kSwiGLU: launch_mode<4>(ma, mb, M, N, K, e, st); break;
    case Epi::kRopeKV: launch_mode<5>(ma, mb, M, N, K, e, st); break;
  }
  return true;
}

bool launch_gemm_tc(const bf16* A, const bf16* B, int M, int N, int K, Epi epi, void* C, const bf16* bias,
                    cudaStream_t st) {
  if (epi == Epi::kSwiGLU || epi == Epi::kRopeKV) return false;
  TcEpilogue e;
  e.mode = epi;
  e.C = C;
  e.bias = bias;
  return launch_gemm_tc_epi(A, B, M, N, K, e, st);
}

}  // namespace ws

extern "C" int ws_gemm_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, ws::g_gemm_trace, sizeof(ws::g_gemm_trace)) == cudaSuccess ? 0 : 6;
}
