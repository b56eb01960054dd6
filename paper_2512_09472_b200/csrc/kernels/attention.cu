// Paged attention over the pool's page window (block = one 2 MiB page).
//
// Prefill: FlashAttention-2 style causal GQA — one CTA per (64-query tile,
// q head), 4 warps x 16 query rows, K/V tiles of 64 keys gathered page by page
// with cp.async (double-buffered), S = QK^T and O += PV on mma.sync, online
// softmax in fp32 registers (exp2 with the log2e-folded scale).
// Decode: split-K over the context, one CTA per (split, kv head, sequence),
// the GQA group on the M side of mma.sync, then a combine kernel.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "../common.h"
#include "device.cuh"
#include "ops.cuh"
#include "pdl.cuh"

namespace ws {

bool kv_window_tmap(const KvGeom& kv, int hd, CUtensorMap* out);  // attn_tc.cu

namespace {

using namespace dev;

constexpr int kQTile = 64, kKTile = 64, kWarps = 4;

template <int HD>
struct PrefillSmem {
  static constexpr int kStride = HD + 8;  // padded rows: conflict-free ldmatrix
  static constexpr int kQ = kQTile * kStride;
  static constexpr int kKV = kKTile * kStride;
  static constexpr int kBytes = (kQ + 4 * kKV) * 2;  // Q + double-buffered K,V
};

template <int HD>
__global__ void __launch_bounds__(kWarps * 32) attn_prefill_kernel(const bf16* __restrict__ qkv,
                                                                   bf16* __restrict__ out, KvGeom kv,
                                                                   int layer, int seq, int rows,
                                                                   int pos0, int heads,
                                                                   float scale_log2) {
  pdl_trigger();
  pdl_wait();
  using S = PrefillSmem<HD>;
  constexpr int ST = S::kStride;
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  extern __shared__ __align__(128) uint8_t smem_raw[];
  bf16* sQ = reinterpret_cast<bf16*>(smem_raw);
  bf16* sK = sQ + S::kQ;        // [2][kKTile][ST]
  bf16* sV = sK + 2 * S::kKV;   // [2][kKTile][ST]

  const int n_qt = (rows + kQTile - 1) / kQTile;
  const int qt = n_qt - 1 - blockIdx.x;  // heaviest (latest) query tiles first
  const int h = blockIdx.y;
  const int kvh = h / (heads / kv.kv_heads);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q_row0 = qt * kQTile;
  const int ldq = (heads + 2 * kv.kv_heads) * HD;
  const int n_keys = pos0 + min(rows, q_row0 + kQTile);  // keys visible to this tile
  const int n_kt = (n_keys + kKTile - 1) / kKTile;
  const int32_t* bt = kv.block_tables + (int64_t)seq * kv.max_blocks;
  const int64_t k_plane = kv.plane(layer, 0, kvh), v_plane = kv.plane(layer, 1, kvh);

  // Q tile -> smem
  for (int i = tid; i < kQTile * CH; i += kWarps * 32) {
    const int r = i / CH, c = i % CH;
    const int gr = q_row0 + r;
    const bf16* src = qkv + (int64_t)(gr < rows ? gr : 0) * ldq + h * HD + c * 8;
    cp_async16(sQ + r * ST + c * 8, src, gr < rows);
  }
  auto load_kv = [&](int buf, int kt) {
    for (int i = tid; i < kKTile * CH; i += kWarps * 32) {
      const int r = i / CH, c = i % CH;
      const int key = kt * kKTile + r;
      const bool ok = key < n_keys;
      const int kk = ok ? key : 0;
      const int32_t page = bt[kk / kv.tpb];
      const bf16* base = reinterpret_cast<const bf16*>(kv.window + (int64_t)page * kv.page_size) +
                         (int64_t)(kk % kv.tpb) * HD + c * 8;
      cp_async16(sK + buf * S::kKV + r * ST + c * 8, base + k_plane, ok);
      cp_async16(sV + buf * S::kKV + r * ST + c * 8, base + v_plane, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[j][e] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];
  const int my_row0 = q_row0 + warp * 16 + (lane >> 2);  // rows my_row0 and my_row0 + 8
  const int qpos0 = pos0 + my_row0, qpos1 = qpos0 + 8;

  for (int kt = 0; kt < n_kt; ++kt) {
    if (kt + 1 < n_kt) load_kv((kt + 1) & 1, kt + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldmatrix_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3],
                    sQ + (warp * 16 + (lane & 15)) * ST + kk * 16 + (lane >> 4) * 8);
    }
    const bf16* tK = sK + (kt & 1) * S::kKV;
    const bf16* tV = sV + (kt & 1) * S::kKV;
    // S = Q K^T for 16 rows x 64 keys
    float s[kKTile / 8][4];
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int j = 0; j < kKTile / 16; ++j) {
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4(b0, b1, b2, b3,
                    tK + (j * 16 + (lane & 7) + ((lane >> 4) << 3)) * ST + kk * 16 +
                        ((lane >> 3) & 1) * 8);
        uint32_t bl[2] = {b0, b1}, bh[2] = {b2, b3};
        mma_bf16_16816(s[2 * j], qf[kk], bl);
        mma_bf16_16816(s[2 * j + 1], qf[kk], bh);
      }
    }
    // causal + bounds mask, online softmax (base 2)
    const int key_base = kt * kKTile + (lane & 3) * 2;
    float mx[2] = {m_run[0], m_run[1]};
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = key_base + j * 8 + (e & 1);
        const int qp = (e >> 1) ? qpos1 : qpos0;
        float v = s[j][e] * scale_log2;
        if (key > qp || key >= n_keys) v = -INFINITY;
        s[j][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], lsum[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float base = mx[r] == -INFINITY ? 0.f : mx[r];
      corr[r] = exp2f(m_run[r] - base);
      m_run[r] = mx[r];
      mx[r] = base;
    }
    uint32_t pf[kKTile / 16][4];
#pragma unroll
    for (int j = 0; j < kKTile / 8; ++j) {
      const float p0 = exp2f(s[j][0] - mx[0]), p1 = exp2f(s[j][1] - mx[0]);
      const float p2 = exp2f(s[j][2] - mx[1]), p3 = exp2f(s[j][3] - mx[1]);
      lsum[0] += p0 + p1;
      lsum[1] += p2 + p3;
      pf[j / 2][(j & 1) * 2 + 0] = pack_bf16x2(p0, p1);
      pf[j / 2][(j & 1) * 2 + 1] = pack_bf16x2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_run[r] = l_run[r] * corr[r] + lsum[r];
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      o[j][0] *= corr[0];
      o[j][1] *= corr[0];
      o[j][2] *= corr[1];
      o[j][3] *= corr[1];
    }
    // O += P V ; P as A fragments: a0/a1 from n8 tile 2t (rows lo/hi), a2/a3 from tile 2t+1
#pragma unroll
    for (int t = 0; t < kKTile / 16; ++t) {
      uint32_t a[4] = {pf[t][0], pf[t][1], pf[t][2], pf[t][3]};
#pragma unroll
      for (int d = 0; d < HD / 16; ++d) {
        uint32_t b0, b1, b2, b3;
        ldmatrix_x4_trans(b0, b1, b2, b3,
                          tV + (t * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * ST + d * 16 +
                              (lane >> 4) * 8);
        uint32_t bl[2] = {b0, b1}, bh[2] = {b2, b3};
        mma_bf16_16816(o[2 * d], a, bl);
        mma_bf16_16816(o[2 * d + 1], a, bh);
      }
    }
    __syncthreads();
  }
  // normalise (quad-reduce the row sums) and store bf16
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
  }
  const float inv0 = l_run[0] > 0 ? 1.f / l_run[0] : 0.f;
  const float inv1 = l_run[1] > 0 ? 1.f / l_run[1] : 0.f;
  const int ldo = heads * HD;
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) {
    const int col = h * HD + j * 8 + (lane & 3) * 2;
    if (my_row0 < rows)
      *reinterpret_cast<uint32_t*>(out + (int64_t)my_row0 * ldo + col) =
          pack_bf16x2(o[j][0] * inv0, o[j][1] * inv0);
    if (my_row0 + 8 < rows)
      *reinterpret_cast<uint32_t*>(out + (int64_t)(my_row0 + 8) * ldo + col) =
          pack_bf16x2(o[j][2] * inv1, o[j][3] * inv1);
  }
}

// ---------------------------------------------------------------- decode
__device__ __forceinline__ void cluster_arrive_wait() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t local, int cta) {
  uint32_t remote;
  float v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local), "r"(cta));
  asm volatile("ld.shared::cluster.f32 %0, [%1];\n" : "=f"(v) : "r"(remote) : "memory");
  return v;
}

// HBM-bound: every K/V byte of the context is read once per step. Work unit =
// (key split, kv head, sequence); the CTA's 4 warps take interleaved 16-key
// tiles of the split, each with its own 3-stage cp.async ring, so one SM keeps
// ~100 KB of K/V in flight. The GQA group (G <= 16 q heads sharing the kv
// head) is the M=16 side of mma.sync: S = Q K^T (16 x 16 keys), O += P V,
// online softmax in registers. The warps' states merge in smem into one
// unnormalised partial (m, l, O) per split; a combine kernel merges the splits.
#ifndef WS_DEC_STAGES
#define WS_DEC_STAGES 3
#endif
constexpr int kDecWarps = 4, kDecKeys = 16, kDecStages = WS_DEC_STAGES;
// K/V TMA tiles' L2 policy: 0 default, 1 evict_first, 2 evict_last. A step
// reads each K/V tile once; as evict_first they stop displacing what the
// step reuses. Graphed decode, ctx 1024, same box, 0 -> 1 (-> 2): B = 1 / 16
// / 64 3.22 / 3.68 / 5.45 -> 3.22 / 3.61 / 5.30-5.35 (3.22 / 3.68 / 5.45) ms
// (tools/ab_kvpol.sh).
#ifndef WS_DEC_KVPOL
#define WS_DEC_KVPOL 1
#endif
constexpr int kDecKvPolicy = WS_DEC_KVPOL;
// Split the context only until there is one CTA per SM: more, shorter CTAs
// measured slower (B = 16 / 64 at ~4 / ~7 CTAs per SM: 4.32 -> 4.84 / 5.84 ->
// 6.80 ms per step: prologue and merge per CTA); a single sequence still gets
// 64-key splits.
constexpr int kDecTargetCtas = kNumSMs;

template <int HD, bool TMA>
struct DecodeSmem {
  static constexpr int kStride = TMA ? HD : HD + 8;  // cp.async: padded rows (conflict-free ldmatrix)
  static constexpr int kTile = kDecKeys * kStride;    // elements
  static constexpr int kWarp = kDecStages * 2 * kTile;  // K and V per stage
  static constexpr int kRing = kDecWarps * kWarp * 2;   // bytes
  static constexpr int kBar = kRing;                    // TMA: [warp][stage] full barriers
  static constexpr int kMerge = (kDecWarps * 16 + 16) * (HD + 2) * 4;  // warp merge + cluster partial
  static constexpr int kUsed = TMA ? kRing + kDecWarps * kDecStages * 8 + 1024 : kRing;  // + 1 KB alignment
  static constexpr int kBytes = kUsed > kMerge ? kUsed : kMerge;
};

__device__ __forceinline__ void dec_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nDEC_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DEC_DONE;\nbra DEC_WAIT;\nDEC_DONE:\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// partial layout per (seq, q head, part): o[HD] (unnormalised), m, l
//
// TMA (sm_100a): when a block holds whole 16-token runs (tpb % 16 == 0) a
// tile's K (and V) is 16 consecutive rows of the page window's 2D tensor map
// (rows of HD bf16, 64 x 16 boxes, 128B swizzle, shared with attn_tc): lane 0
// of the warp issues HD/64 box loads per operand on the stage's mbarrier
// (expect_tx), the warp waits on its parity — 2*HD/64 instructions per tile
// instead of 2*16*HD/8 16-byte cp.async, and the swizzled rows need no padding
// for conflict-free ldmatrix. Other geometries (70B: 6 tokens per block) keep
// the cp.async row gather.
template <int HD, bool TMA>
__global__ void __launch_bounds__(kDecWarps * 32) attn_decode_kernel(
    const bf16* __restrict__ qkv, KvGeom kv, int layer, const int32_t* __restrict__ seqs,
    const int32_t* __restrict__ pos, int heads, float scale_log2, float* __restrict__ part,
    int n_splits, int split_keys, bf16* __restrict__ out, int in_cluster,
    const __grid_constant__ CUtensorMap kvmap, const __grid_constant__ L2Pf pf) {
  pdl_trigger();
  if (threadIdx.x == 32)  // a later kernel's weights into L2 while this latency-bound one runs
    l2_prefetch(pf, blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z),
                gridDim.x * gridDim.y * gridDim.z);
  using S = DecodeSmem<HD, TMA>;
  constexpr int ST = S::kStride, CH = HD / 8;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* sbase = smem_raw;
  if constexpr (TMA) {  // SWIZZLE_128B destinations need 1 KB alignment
    const uint32_t raw = smem_u32(smem_raw);
    sbase = smem_raw + (((raw + 1023) & ~1023u) - raw);
  }
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  bf16* sw = reinterpret_cast<bf16*>(sbase) + warp * S::kWarp;
  const uint32_t bar0 = smem_u32(sbase + S::kBar) + warp * kDecStages * 8;
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < kDecWarps * kDecStages; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(sbase + S::kBar) + 8 * i));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  pdl_wait();
  const int G = heads / kv.kv_heads;
  const int len = pos[b] + 1;  // the new token's K/V is already appended
  const int k_lo = split * split_keys, k_hi = min(len, k_lo + split_keys);
  const int n_tiles = k_hi > k_lo ? (k_hi - k_lo + kDecKeys - 1) / kDecKeys : 0;
  const int my_n = n_tiles > warp ? (n_tiles - warp + kDecWarps - 1) / kDecWarps : 0;
  const int32_t* bt = kv.block_tables + (int64_t)seqs[b] * kv.max_blocks;
  const int64_t k_plane = kv.plane(layer, 0, kvh), v_plane = kv.plane(layer, 1, kvh);

  // tpb a multiple of the 16-key tile (every model but the 70B): a tile is one
  // contiguous 4 KB run of K (and of V) inside one page. Each lane holds the
  // page of one of the warp's next 32 tiles (a coalesced block-table read per
  // 32 tiles, issued 32 tiles ahead), so no tile load waits on a block-table
  // lookup or a division by tpb.
  const bool aligned = TMA || kv.tpb % kDecKeys == 0;
  auto page_of = [&](int j) -> int32_t {
    return j < my_n ? bt[(k_lo + (warp + j * kDecWarps) * kDecKeys) / kv.tpb] : 0;
  };
  int32_t pg_cur = 0, pg_nxt = 0;
  if (aligned) {
    pg_cur = page_of(lane);
    pg_nxt = page_of(32 + lane);
  }
  // byte offset of element (row, col) in a K or V tile
  auto toff = [](int row, int col) -> int {
    if constexpr (TMA)
      return (col >> 6) * (kDecKeys * 128) + row * 128 + ((((col >> 3) & 7) ^ (row & 7)) << 4);
    else
      return (row * ST + col) * 2;
  };
  const int rows_pp = (int)(kv.page_size / (HD * 2));
  auto load = [&](int stage, int j) {
    bf16* tk = sw + stage * 2 * S::kTile;
    bf16* tv = tk + S::kTile;
    const int t = warp + j * kDecWarps;
    if (aligned) {
      if ((j & 31) == 0 && j > 0) {
        pg_cur = pg_nxt;
        pg_nxt = page_of(j + 32 + lane);
      }
      const int32_t page = __shfl_sync(0xffffffffu, pg_cur, j & 31);
      const int key0 = k_lo + t * kDecKeys, rows = k_hi - key0;
      if constexpr (TMA) {
        // rows past k_hi in the tile's page hold finite data (the pool is
        // zeroed at creation and only ever holds bf16 weights / KV): their
        // scores are masked, so P = 0 and they add nothing
        if (lane == 0) {
          const int y = page * rows_pp + (key0 % kv.tpb);
          const uint32_t bar = bar0 + stage * 8, dk = smem_u32(tk), dv = smem_u32(tv);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // ldmatrix reads before the refill
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                       "r"(2 * kDecKeys * HD * 2)
                       : "memory");
#pragma unroll
          for (int hh = 0; hh < HD / 64; ++hh) {
            if constexpr (kDecKvPolicy != 0) {  // K/V tiles with an L2 cache policy (A/B build knob)
              uint64_t pol;
              if constexpr (kDecKvPolicy == 1)
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
              else
                asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
                  "[%1, {%3, %4}], [%2], %5;\n" ::"r"(dk + hh * kDecKeys * 128),
                  "l"(&kvmap), "r"(bar), "r"(hh * 64), "r"(y + (int)(k_plane / HD)), "l"(pol)
                  : "memory");
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
                  "[%1, {%3, %4}], [%2], %5;\n" ::"r"(dv + hh * kDecKeys * 128),
                  "l"(&kvmap), "r"(bar), "r"(hh * 64), "r"(y + (int)(v_plane / HD)), "l"(pol)
                  : "memory");
            } else {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                ::"r"(dk + hh * kDecKeys * 128), "l"(&kvmap), "r"(bar), "r"(hh * 64), "r"(y + (int)(k_plane / HD))
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
                ::"r"(dv + hh * kDecKeys * 128), "l"(&kvmap), "r"(bar), "r"(hh * 64), "r"(y + (int)(v_plane / HD))
                : "memory");
            }
          }
        }
        (void)rows;
        return;
      } else {
        const bf16* tile = reinterpret_cast<const bf16*>(kv.window + (int64_t)page * kv.page_size) +
                           (int64_t)(key0 % kv.tpb) * HD;
#pragma unroll
        for (int i = lane; i < kDecKeys * CH; i += 32) {
          const int r = i / CH, c = i % CH;
          cp_async16(tk + r * ST + c * 8, tile + k_plane + i * 8, r < rows);
          cp_async16(tv + r * ST + c * 8, tile + v_plane + i * 8, r < rows);
        }
        return;
      }
    }
#pragma unroll
    for (int i = lane; i < kDecKeys * CH; i += 32) {
      const int r = i / CH, c = i % CH;
      const int key = k_lo + t * kDecKeys + r;
      const bool ok = key < k_hi;
      const int kk = ok ? key : k_lo;
      const int32_t page = bt[kk / kv.tpb];
      const bf16* base = reinterpret_cast<const bf16*>(kv.window + (int64_t)page * kv.page_size) +
                         (int64_t)(kk % kv.tpb) * HD + c * 8;
      cp_async16(tk + r * ST + c * 8, base + k_plane, ok);
      cp_async16(tv + r * ST + c * 8, base + v_plane, ok);
    }
  };
#pragma unroll
  for (int s = 0; s < kDecStages - 1; ++s) {
    if (s < my_n) load(s, s);
    if constexpr (!TMA) cp_async_commit();
  }

  // Q as the A operand: rows = the group's q heads (rows >= G are zero)
  const int g0 = lane >> 2, g1 = g0 + 8;
  const int ldq = (heads + 2 * kv.kv_heads) * HD;
  const bf16* q0 = qkv + (int64_t)b * ldq + (int64_t)(kvh * G + g0) * HD;
  const bf16* q1 = qkv + (int64_t)b * ldq + (int64_t)(kvh * G + g1) * HD;
  uint32_t qf[HD / 16][4];
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const int c = kk * 16 + (lane & 3) * 2;
    qf[kk][0] = g0 < G ? *reinterpret_cast<const uint32_t*>(q0 + c) : 0u;
    qf[kk][1] = g1 < G ? *reinterpret_cast<const uint32_t*>(q1 + c) : 0u;
    qf[kk][2] = g0 < G ? *reinterpret_cast<const uint32_t*>(q0 + c + 8) : 0u;
    qf[kk][3] = g1 < G ? *reinterpret_cast<const uint32_t*>(q1 + c + 8) : 0u;
  }

  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[j][e] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};

  for (int it = 0; it < my_n; ++it) {
    const int nx = it + kDecStages - 1;
    if (nx < my_n) load(nx % kDecStages, nx);
    if constexpr (TMA) {
      dec_mbar_wait(bar0 + (it % kDecStages) * 8, (it / kDecStages) & 1);
    } else {
      cp_async_commit();
      cp_async_wait<kDecStages - 1>();
      __syncwarp();
    }
    const uint8_t* tk = reinterpret_cast<const uint8_t*>(sw + (it % kDecStages) * 2 * S::kTile);
    const uint8_t* tv = tk + S::kTile * 2;
    float s[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4(b0, b1, b2, b3, tk + toff((lane & 7) + ((lane >> 4) << 3), kk * 16 + ((lane >> 3) & 1) * 8));
      uint32_t bl[2] = {b0, b1}, bh[2] = {b2, b3};
      mma_bf16_16816(s[0], qf[kk], bl);
      mma_bf16_16816(s[1], qf[kk], bh);
    }
    const int key_base = k_lo + (warp + it * kDecWarps) * kDecKeys + (lane & 3) * 2;
    float mx[2] = {m_run[0], m_run[1]};
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[j][e] * scale_log2;
        if (key_base + j * 8 + (e & 1) >= k_hi) v = -INFINITY;
        s[j][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float base = mx[r] == -INFINITY ? 0.f : mx[r];
      corr[r] = exp2f(m_run[r] - base);
      m_run[r] = mx[r];
      mx[r] = base;
    }
    uint32_t a[4];
    float lsum[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float p0 = exp2f(s[j][0] - mx[0]), p1 = exp2f(s[j][1] - mx[0]);
      const float p2 = exp2f(s[j][2] - mx[1]), p3 = exp2f(s[j][3] - mx[1]);
      lsum[0] += p0 + p1;
      lsum[1] += p2 + p3;
      a[2 * j] = pack_bf16x2(p0, p1);
      a[2 * j + 1] = pack_bf16x2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_run[r] = l_run[r] * corr[r] + lsum[r];
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      o[j][0] *= corr[0];
      o[j][1] *= corr[0];
      o[j][2] *= corr[1];
      o[j][3] *= corr[1];
    }
#pragma unroll
    for (int d = 0; d < HD / 16; ++d) {
      uint32_t b0, b1, b2, b3;
      ldmatrix_x4_trans(b0, b1, b2, b3, tv + toff((lane & 7) + ((lane >> 3) & 1) * 8, d * 16 + (lane >> 4) * 8));
      uint32_t bl[2] = {b0, b1}, bh[2] = {b2, b3};
      mma_bf16_16816(o[2 * d], a, bl);
      mma_bf16_16816(o[2 * d + 1], a, bh);
    }
    __syncwarp();  // every lane is done with this stage before it is refilled
  }
  if constexpr (!TMA) cp_async_wait<0>();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 1);
    l_run[r] += __shfl_xor_sync(0xffffffffu, l_run[r], 2);
  }
  // merge the 4 warps' states in smem (the K/V rings are free now), one part per split
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem_raw);  // [warp][16 rows][HD + 2]
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    float* row = red + ((int64_t)warp * 16 + (r ? g1 : g0)) * (HD + 2);
#pragma unroll
    for (int j = 0; j < HD / 8; ++j)
      *reinterpret_cast<float2*>(row + j * 8 + (lane & 3) * 2) = make_float2(o[j][2 * r], o[j][2 * r + 1]);
    if ((lane & 3) == 0) {
      row[HD] = my_n > 0 ? m_run[r] : -INFINITY;
      row[HD + 1] = l_run[r];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * HD; idx += kDecWarps * 32) {
    const int g = idx / HD, d = idx % HD;
    float mw[kDecWarps], mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) {
      mw[w] = red[((int64_t)w * 16 + g) * (HD + 2) + HD];
      mx = fmaxf(mx, mw[w]);
    }
    float acc = 0.f, l = 0.f;
#pragma unroll
    for (int w = 0; w < kDecWarps; ++w) {
      if (mw[w] == -INFINITY) continue;
      const float f = exp2f(mw[w] - mx);
      const float* row = red + ((int64_t)w * 16 + g) * (HD + 2);
      acc += f * row[d];
      l += f * row[HD + 1];
    }
    if (n_splits == 1) {  // the whole context in this CTA: final output, no combine pass
      out[(int64_t)b * heads * HD + (kvh * G + g) * HD + d] = f2bf(l > 0.f ? acc / l : 0.f);
      continue;
    }
    // cluster: this CTA's partial stays in its shared memory; otherwise global scratch
    float* dst = in_cluster ? red + kDecWarps * 16 * (HD + 2) + g * (HD + 2)
                            : part + (((int64_t)b * heads + kvh * G + g) * n_splits + split) * (HD + 2);
    dst[d] = acc;
    if (d == 0) {
      dst[HD] = mx;
      dst[HD + 1] = l;
    }
  }
  if (!in_cluster) return;
  // The splits of one (kv head, sequence) form a thread-block cluster: after
  // the cluster barrier every CTA merges a slice of the G x HD outputs from
  // all splits' partials over distributed shared memory — no scratch round
  // trip through L2 and no combine launch.
  cluster_arrive_wait();
  const uint32_t cp = smem_u32(red + kDecWarps * 16 * (HD + 2));
  for (int idx = split * kDecWarps * 32 + threadIdx.x; idx < G * HD; idx += n_splits * kDecWarps * 32) {
    const int g = idx / HD, d = idx % HD;
    const uint32_t row = cp + 4u * (uint32_t)(g * (HD + 2));
    float mx = -INFINITY;
    for (int c = 0; c < n_splits; ++c) mx = fmaxf(mx, ld_dsmem_f32(row + 4u * HD, c));
    float acc = 0.f, l = 0.f;
    for (int c = 0; c < n_splits; ++c) {
      const float m = ld_dsmem_f32(row + 4u * HD, c);
      if (m == -INFINITY) continue;
      const float f = exp2f(m - mx);
      acc += f * ld_dsmem_f32(row + 4u * d, c);
      l += f * ld_dsmem_f32(row + 4u * (HD + 1), c);
    }
    out[(int64_t)b * heads * HD + (kvh * G + g) * HD + d] = f2bf(l > 0.f ? acc / l : 0.f);
  }
  cluster_arrive_wait();  // no CTA leaves while its partial may still be read
}

// out[b, h] = sum_p w_p o_p / sum_p w_p l_p with w_p = 2^(m_p - max m). Warp 0
// computes the weights of all parts, then every thread owns one dim.
constexpr int kMaxSplits = 256;
template <int HD>
__global__ void __launch_bounds__(HD) attn_combine_kernel(const float* __restrict__ part,
                                                          bf16* __restrict__ out, int heads,
                                                          int n_parts) {
  pdl_trigger();
  pdl_wait();
  const int h = blockIdx.x, b = blockIdx.y, d = threadIdx.x;
  const float* p = part + ((int64_t)b * heads + h) * n_parts * (HD + 2);
  __shared__ float sw[kMaxSplits];
  __shared__ float s_inv;
  if (d < 32) {
    float mx = -INFINITY;
    for (int s = d; s < n_parts; s += 32) mx = fmaxf(mx, p[s * (HD + 2) + HD]);
    mx = warp_max(mx);
    float den = 0.f;
    for (int s = d; s < n_parts; s += 32) {
      const float m = p[s * (HD + 2) + HD];
      const float w = m == -INFINITY ? 0.f : exp2f(m - mx);
      sw[s] = w;
      den += w * p[s * (HD + 2) + HD + 1];
    }
    den = warp_sum(den);
    if (d == 0) s_inv = den > 0 ? 1.f / den : 0.f;
  }
  __syncthreads();
  float num = 0.f;
#pragma unroll 8
  for (int s = 0; s < n_parts; ++s) num += sw[s] * p[s * (HD + 2) + d];
  out[(int64_t)b * heads * HD + h * HD + d] = f2bf(num * s_inv);
}

template <int HD>
void prefill_impl(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows,
                  int pos0, int heads, float scale, cudaStream_t st) {
  const int smem = PrefillSmem<HD>::kBytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_prefill_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((rows + kQTile - 1) / kQTile, heads);
  count_launch();
  launch_pdl(attn_prefill_kernel<HD>, dim3(grid), dim3(kWarps * 32), smem, st, qkv, out, kv, layer, seq, rows, pos0,
                                                           heads, scale * 1.4426950408889634f);
}

// Largest split cluster the decode kernel may use: 16 when the non-portable
// size schedules at this shared-memory footprint, else the portable 8;
// WS_DEC_CLUSTER=0 disables clusters (scratch + combine kernel, A/B).
template <typename K>
int decode_cluster_limit(K kernel, int smem) {
  const bool non_portable = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                            cudaSuccess;
  if (!non_portable) cudaGetLastError();
  if (const char* e = std::getenv("WS_DEC_CLUSTER")) return std::min(std::atoi(e), non_portable ? 16 : 8);
  // 8 (portable) by default since the L2 evict_first streams: graphed decode,
  // ctx 1024, same box, 16 -> 8: B = 1 / 4 / 16 3.207 / 3.321 / 3.593 ->
  // 3.189 / 3.315 / 3.597 ms (profiles/r2h_ab_dec_cluster.txt)
  if (!non_portable || !std::getenv("WS_DEC_CLUSTER16")) return 8;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(16, 1, 1);
  cfg.blockDim = dim3(kDecWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  return n > 0 ? 16 : 8;
}

// launch_pdl plus an optional (cluster, 1, 1) cluster shape
template <typename... KArgs, typename... Args>
void launch_decode(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, int cluster, cudaStream_t st,
                   Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_for_launch()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n++].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int HD, bool TMA>
void decode_launch(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, const int32_t* seqs,
                   const int32_t* ctx, int n_seqs, int heads, int max_ctx, float scale, float* scratch,
                   const CUtensorMap& map, cudaStream_t st, const L2Pf& pf) {
  using S = DecodeSmem<HD, TMA>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_kernel<HD, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes);
    attr = true;
  }
  static int max_cluster = -1;
  if (max_cluster < 0) max_cluster = decode_cluster_limit(attn_decode_kernel<HD, TMA>, S::kBytes);
  // enough (split, kv head, seq) units to fill the SMs; >= 64 keys per split
  const int units = n_seqs * kv.kv_heads;
  int n_splits = std::max(1, std::min({(kDecTargetCtas + units - 1) / units, (max_ctx + 63) / 64, kMaxSplits}));
  // up to twice the cluster limit: fold into one cluster's worth of longer
  // splits rather than add a combine launch (WS_DEC_SPLIT_CAP=0: A/B)
  static const bool cap = !(std::getenv("WS_DEC_SPLIT_CAP") && std::getenv("WS_DEC_SPLIT_CAP")[0] == '0');
  if (cap && n_splits > max_cluster && n_splits <= 2 * max_cluster) n_splits = max_cluster;
  const int split_keys = ((max_ctx + n_splits - 1) / n_splits + kDecKeys - 1) / kDecKeys * kDecKeys;
  n_splits = (max_ctx + split_keys - 1) / split_keys;
  // few splits (small batches): one cluster per (kv head, sequence) merges
  // them in distributed shared memory; many (one long context): scratch + combine
  const int in_cluster = n_splits > 1 && n_splits <= max_cluster;
  dim3 grid(n_splits, kv.kv_heads, n_seqs);
  count_launch();
  launch_decode(attn_decode_kernel<HD, TMA>, grid, dim3(kDecWarps * 32), S::kBytes, in_cluster ? n_splits : 0, st,
                qkv, kv, layer, seqs, ctx, heads, scale * 1.4426950408889634f, scratch, n_splits, split_keys, out,
                in_cluster, map, pf);
  if (n_splits > 1 && !in_cluster) {
    count_launch();
    launch_pdl(attn_combine_kernel<HD>, dim3(heads, n_seqs), dim3(HD), 0, st, scratch, out, heads, n_splits);
  }
}

template <int HD>
void decode_impl(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, const int32_t* seqs,
                 const int32_t* ctx, int n_seqs, int heads, int max_ctx, float scale, float* scratch,
                 cudaStream_t st, const L2Pf& pf) {
  // TMA tiles need whole 16-token runs per block and the window addressable
  // as HD-wide rows; WS_DEC_TMA=0 forces the cp.async gather (A/B)
  static const bool tma_env = !(std::getenv("WS_DEC_TMA") && std::getenv("WS_DEC_TMA")[0] == '0');
  CUtensorMap map{};
  if constexpr (HD % 64 == 0) {
    if (tma_env && kv.tpb % kDecKeys == 0 && kv_window_tmap(kv, HD, &map)) {
      decode_launch<HD, true>(qkv, out, kv, layer, seqs, ctx, n_seqs, heads, max_ctx, scale, scratch, map, st, pf);
      return;
    }
  }
  decode_launch<HD, false>(qkv, out, kv, layer, seqs, ctx, n_seqs, heads, max_ctx, scale, scratch, map, st, pf);
}

}  // namespace

void launch_attn_prefill(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, int seq, int rows,
                         int pos0, int heads, float scale, cudaStream_t st) {
  switch (kv.head_dim) {
    case 64: prefill_impl<64>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st); break;
    case 96: prefill_impl<96>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st); break;
    case 128: prefill_impl<128>(qkv, out, kv, layer, seq, rows, pos0, heads, scale, st); break;
    default: break;
  }
}

void launch_attn_decode(const bf16* qkv, bf16* out, const KvGeom& kv, int layer, const int32_t* seqs,
                        const int32_t* ctx, int n_seqs, int heads, int max_ctx, float scale,
                        float* scratch, cudaStream_t st, const L2Pf& pf) {
  switch (kv.head_dim) {
    case 64: decode_impl<64>(qkv, out, kv, layer, seqs, ctx, n_seqs, heads, max_ctx, scale, scratch, st, pf); break;
    case 96: decode_impl<96>(qkv, out, kv, layer, seqs, ctx, n_seqs, heads, max_ctx, scale, scratch, st, pf); break;
    case 128: decode_impl<128>(qkv, out, kv, layer, seqs, ctx, n_seqs, heads, max_ctx, scale, scratch, st, pf); break;
    default: break;
  }
}

int decode_scratch_floats(int n_seqs, int heads, int kv_heads, int head_dim) {
  // one part per split, n_splits <= ceil(target / (n_seqs * kv_heads))
  return (head_dim + 2) * (kDecTargetCtas * (heads / kv_heads) + n_seqs * heads);
}

}  // namespace ws
