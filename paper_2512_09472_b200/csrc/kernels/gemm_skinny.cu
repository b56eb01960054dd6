// Decode-shaped tcgen05 GEMM: C[M,N] = A[M,K] . W[N,K]^T for M <= 128.
//
// Decode rows are few, so the GEMM is a weight stream (HBM bound): the kernel
// swaps the operands — 128 weight rows are the MMA's M side, the M activation
// rows (padded to Mp, a multiple of 16) its N side — so one
// tcgen05.mma.cta_group::1 M=128 N=Mp K=16 consumes a whole 128x16 weight
// slice however small the batch is.
//
// Persistent stream-K: one CTA per SM; the (unit, k-block) iteration space —
// unit = one 128-row weight block (a 256-row gate|up group for SwiGLU) — is
// cut into equal contiguous ranges, so every SM streams the same number of
// weight bytes through one uninterrupted TMA ring, with no wave quantization
// whatever N and K are. A CTA's range is a list of segments (one per unit it
// touches); only its first and last segment can cover part of a unit.
//
//   warp 0 lane 0  TMA producer: sub x (W block(s) 128x64 + A Mp x64) per stage (SW128)
//   warp 1 lane 0  MMA issuer; double-buffered TMEM accumulators [128][NB*Mp]
//   warp 2         TMEM allocation
//   warps 4-7      epilogue: TMEM lane i = weight row i, columns = batch rows
//
// A segment covering a whole unit is stored directly. Partial segments write
// fp32 partials to a per-(CTA, first|last) slot and skinny_fixup_kernel sums
// each split unit's contributors in k order — deterministic — and applies the
// epilogue: bf16, +bias, fp32 store, fp32 residual add, or SwiGLU over the
// gate block (TMEM columns [0,Mp)) and the matching up block (columns
// [Mp,2Mp)) of the interleaved Wgu.
#include <cuda.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "../common.h"
#include "../driver.h"
#include "device.cuh"
#include "ops.cuh"
#include "pdl.cuh"
#include "tcgen05.cuh"

namespace ws {
namespace {

using namespace dev;

constexpr int kRows = 128, kBox = 64, kThreads = 256;
constexpr int kW_BYTES = kRows * kBox * 2;  // 16 KiB weight box (128 rows x 128 B, SW128)
constexpr int kSmemBudget = 216 * 1024;     // TMA ring, one CTA per SM
constexpr int kMaxSmem = 227 * 1024;        // opt-in dynamic shared memory per CTA

// An iteration covers sub (1, 2 or 4) boxes of 64 k-columns: the producer
// fetches sub x 128 contiguous bytes of every weight row per issue.
struct SkinnyArgs {
  int M, N, K, Mp, stages, stage_bytes, total_iters, sub, kbs;
  float* partial;      // [grid][2][NB*128][Mp]
  int csplit;          // >= 2: cluster split-K (see launch_gemm_skinny); 0: stream-K
  int evict_first;     // weight tiles loaded with an L2 evict_first policy (WS_SK_EVF, A/B)
  int splitj;          // SwiGLU, whole units only: a stage holds the gate OR the up rows of a
                       // k-block (kbs counts 2 iterations per k-block), so a stage spans twice
                       // the k-columns of each weight row (WS_SK_SPLITJ, A/B)
};

// Residual producer of a folded RMSNorm (norm_role 1): x_new is final (one
// writer per element); store it, the next projection's A = bf16(x_new * g),
// and the warp's sum of squares over its 32 consecutive columns (a fixed
// shuffle tree: deterministic). Called by all 32 lanes of a warp.
__device__ __forceinline__ void norm_produce(const TcEpilogue& ep, int N, int b, int col, float x_new, float* dst) {
  *dst = x_new;
  ep.norm_out[(int64_t)b * N + col] = f2bf(x_new * bf2f(ep.norm_g[col]));
  const float sq = warp_sum(x_new * x_new);
  if ((threadIdx.x & 31) == 0) ep.row_ss[(int64_t)b * (N / 32) + col / 32] = sq;
}

// Consumer of a folded RMSNorm (norm_role 2): rsqrt(mean(x^2) + eps) of batch
// row b from the producer's partials; one thread per row, every load issued
// before the (fixed-order) adds.
__device__ __forceinline__ float norm_row_scale(const TcEpilogue& ep, int b) {
  const int n = ep.norm_d / 32;
  const float* p = ep.row_ss + (int64_t)b * n;
  float a = 0.f;
  int k = 0;
  for (; k + 16 <= n; k += 16) {
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcg(reinterpret_cast<const float4*>(p + k) + j);
#pragma unroll
    for (int j = 0; j < 4; ++j) a += (v[j].x + v[j].y) + (v[j].z + v[j].w);
  }
  for (; k < n; ++k) a += __ldcg(p + k);
  return rsqrtf(a / (float)ep.norm_d + ep.norm_eps);
}

template <int MODE>
__device__ __forceinline__ void store_out(const TcEpilogue& ep, const SkinnyArgs& a, int row, const float* v,
                                          int c0) {
  // v[j]: batch row c0 + j of output column `row`
  if (row >= (MODE == (int)Epi::kSwiGLU ? a.N / 2 : a.N)) return;  // ragged last unit
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int b = c0 + j;
    if (b >= a.M) break;
    float x = v[j];
    if constexpr (MODE == (int)Epi::kAddF32) {
      float* dst = static_cast<float*>(ep.C) + (int64_t)b * a.N + row;
      if (ep.norm_role == 1) {
        norm_produce(ep, a.N, b, row, *dst + x, dst);
      } else {
        // exactly one add per element (whole unit or reduced sum): deterministic,
        // and a fire-and-forget reduction instead of a load-add-store chain
        atomicAdd(dst, x);
      }
    } else if constexpr (MODE == (int)Epi::kStoreF32) {
      static_cast<float*>(ep.C)[(int64_t)b * a.N + row] = x;
    } else if constexpr (MODE == (int)Epi::kSwiGLU) {
      static_cast<bf16*>(ep.C)[(int64_t)b * (a.N / 2) + row] = f2bf(x);
    } else {
      if constexpr (MODE == (int)Epi::kBiasBf16) x += bf2f(ep.bias[row]);
      static_cast<bf16*>(ep.C)[(int64_t)b * a.N + row] = f2bf(x);
    }
  }
}

// CTA whose iteration range [it_begin(c), it_begin(c+1)) contains `it`
__device__ __forceinline__ int cta_of(int64_t it, int G, int total) { return (int)(((it + 1) * G - 1) / total); }
__device__ __forceinline__ int it_begin(int c, int G, int total) { return (int)((int64_t)c * total / G); }

// Epilogue of one (unit, weight row i, 4 batch rows) after the split-K sum:
// folded-norm row scales, SwiGLU, then store / add / norm-produce.
template <int MODE>
__device__ __forceinline__ void fixup_store(const SkinnyArgs& args, const TcEpilogue& ep, int unit, int i, int q4,
                                            const float4* sum, const float* row_scale) {
  constexpr int NB = MODE == (int)Epi::kSwiGLU ? 2 : 1;
  float v[4] = {sum[0].x, sum[0].y, sum[0].z, sum[0].w};
  float u[4] = {sum[NB - 1].x, sum[NB - 1].y, sum[NB - 1].z, sum[NB - 1].w};
  if (ep.norm_role == 2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float sc = q4 * 4 + k < args.M ? row_scale[q4 * 4 + k] : 0.f;
      v[k] *= sc;
      u[k] *= sc;
    }
  }
  if constexpr (NB == 2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = silu(v[k]) * u[k];
  }
  const int row = unit * kRows + i;
  if (row >= (MODE == (int)Epi::kSwiGLU ? args.N / 2 : args.N)) return;  // ragged last unit
  if constexpr (MODE == (int)Epi::kAddF32) {
    // every load before any store: one L2 round trip for the 4 batch rows
    // (and the norm weight), not one per row behind the previous row's stores
    float* x = static_cast<float*>(ep.C) + row;
    float old[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) old[k] = q4 * 4 + k < args.M ? x[(int64_t)(q4 * 4 + k) * args.N] : 0.f;
    const float g = ep.norm_role == 1 ? bf2f(ep.norm_g[row]) : 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int b = q4 * 4 + k;
      if (b >= args.M) break;
      const float x_new = old[k] + v[k];
      x[(int64_t)b * args.N] = x_new;
      if (ep.norm_role == 1) {  // folded RMSNorm producer (see norm_produce)
        ep.norm_out[(int64_t)b * args.N + row] = f2bf(x_new * g);
        const float sq = warp_sum(x_new * x_new);
        if ((threadIdx.x & 31) == 0) ep.row_ss[(int64_t)b * (args.N / 32) + row / 32] = sq;
      }
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int b = q4 * 4 + k;
    if (b >= args.M) break;
    if constexpr (MODE == (int)Epi::kAddF32) {
    } else if constexpr (MODE == (int)Epi::kStoreF32) {
      static_cast<float*>(ep.C)[(int64_t)b * args.N + row] = v[k];
    } else if constexpr (MODE == (int)Epi::kSwiGLU) {
      static_cast<bf16*>(ep.C)[(int64_t)b * (args.N / 2) + row] = f2bf(v[k]);
    } else {
      float x = v[k];
      if constexpr (MODE == (int)Epi::kBiasBf16) x += bf2f(ep.bias[row]);
      static_cast<bf16*>(ep.C)[(int64_t)b * args.N + row] = f2bf(x);
    }
  }
}

// RoPE + paged KV append of one rotate-half pair (columns col_a, col_b = col_a
// + hd/2 of a head) for 4 batch rows, after the split-K sums va / vb.
__device__ __forceinline__ void rope_store(const SkinnyArgs& args, const TcEpilogue& ep, int col_a, int q4,
                                           float* va, float* vb, const float* row_scale) {
  const KvGeom& kv = ep.kv;
  const int hd = kv.head_dim, half = hd / 2, col_b = col_a + half, dd = col_a % half;
  if (ep.norm_role == 2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float sc = q4 * 4 + k < args.M ? row_scale[q4 * 4 + k] : 0.f;
      va[k] *= sc;
      vb[k] *= sc;
    }
  }
  const float bias_a = ep.bias ? bf2f(ep.bias[col_a]) : 0.f, bias_b = ep.bias ? bf2f(ep.bias[col_b]) : 0.f;
  const int hs = col_a / hd;  // head slot in [0, H + 2KV)
  const bool is_v = hs >= ep.heads + kv.kv_heads, is_k = !is_v && hs >= ep.heads;
  // loads of all 4 batch rows first (positions, then the rotations and pages
  // they index), stores after: two L2 round trips, not two per row
  int pos[4], page[4];
  float2 cs[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int b = q4 * 4 + k;
    pos[k] = b < args.M ? (ep.pos_arr ? ep.pos_arr[b] : ep.pos0 + b) : 0;
    page[k] = b < args.M && (is_k || is_v) ? (ep.seq_arr ? ep.seq_arr[b] : ep.seq0) : 0;  // seq for now
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool ok = q4 * 4 + k < args.M;
    cs[k] = ok && !is_v ? ep.rope[(int64_t)pos[k] * half + dd] : make_float2(1.f, 0.f);
    page[k] = ok && (is_k || is_v) ? kv.block_tables[(int64_t)page[k] * kv.max_blocks + pos[k] / kv.tpb] : 0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int b = q4 * 4 + k;
    if (b >= args.M) break;
    float x = va[k] + bias_a, y = vb[k] + bias_b;
    if (!is_v) {
      const float rx = x * cs[k].x - y * cs[k].y, ry = y * cs[k].x + x * cs[k].y;
      x = rx;
      y = ry;
    }
    if (!is_k && !is_v) {
      bf16* q = static_cast<bf16*>(ep.C) + (int64_t)b * args.N;
      q[col_a] = f2bf(x);
      q[col_b] = f2bf(y);
    } else {
      const int kvh = is_v ? hs - ep.heads - kv.kv_heads : hs - ep.heads;
      bf16* dst = reinterpret_cast<bf16*>(kv.window + (int64_t)page[k] * kv.page_size) +
                  kv.plane(ep.layer, is_v ? 1 : 0, kvh) + (int64_t)(pos[k] % kv.tpb) * hd;
      dst[dd] = f2bf(x);
      dst[dd + half] = f2bf(y);
    }
  }
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ float4 ld_dsmem_v4(uint32_t local, int cta) {
  uint32_t remote;
  float4 v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local), "r"(cta));
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote)
               : "memory");
  return v;
}

// Shared-memory slot of (row, quad) in a cluster split's fp32 partial
// [NB*128][Mp]: quads XOR-swizzled by the row, so the 32 rows a warp touches
// at one logical quad spread over all bank groups (unswizzled, a row stride
// of 128 B or more put every lane of a 16 B access in the same banks:
// 32-way conflicts on both the epilogue's stores and the reduce's remote loads).
__device__ __forceinline__ uint32_t part_off(int row, int q4, int Mp) {
  const int quads = Mp >> 2, group = quads & -quads;  // XOR inside aligned power-of-two groups of quads
  return (uint32_t)((row * Mp + ((q4 ^ (row & (group - 1))) << 2)) << 2);
}

__device__ __forceinline__ void st_dsmem_v4(uint32_t local, int cta, float4 v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(local), "r"(cta));
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(remote), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// Push form of the cluster split (<= 16 batch rows): block b of a unit's 128
// rows (RoPE: rotate-half pair block b) is reduced by cluster rank b mod S.
// Every CTA stores its partial rows straight into their owner's push region
// ([source rank][owner-local row][NB][Mp], part_off swizzle) with remote
// shared-memory stores, so after one cluster barrier each owner sums S local
// copies — no DSMEM round trip per load and no second barrier (the pull form
// spent ~1.6 us reducing and ~0.8 us in the closing barrier of an O GEMM
// whose weights took 3.4 us to stream).
__host__ __device__ constexpr int push_rows_per_owner(bool rope, int S) {
  return rope ? (2 + S - 1) / S * 64 : (kRows / 32 + S - 1) / S * 32;
}
template <int MODE>
__device__ __forceinline__ void push_slot(const TcEpilogue& ep, int i, int S, int& owner, int& local) {
  if constexpr (MODE == (int)Epi::kRopeKV) {
    const int hd = ep.kv.head_dim, half = hd / 2;
    const int j = (i / hd) * half + (i % hd) % half, side = (i % hd) >= half ? 1 : 0, blk = j / 32;
    owner = blk % S;
    local = (blk / S) * 64 + (j % 32) * 2 + side;
  } else {
    const int b = i / 32;
    owner = b % S;
    local = (b / S) * 32 + (i % 32);
  }
}

// Cluster split-K reduction: the S CTAs of a cluster computed k-slices of one
// unit and left their fp32 partials [NB][128][Mp] at shared address `part` in
// their own shared memory (part_off layout). All 8 warps of each CTA (t =
// 0..255) sum, in k (= cluster rank) order over distributed shared memory,
// the 32-row blocks b of the unit with b mod S == rank (rotate-half pair
// blocks for RoPE) and apply the epilogue — the fix-up pass without a launch
// or a global round trip. An item is (block, 4 batch rows), lanes = 32
// consecutive rows (the folded-norm producer's warp sums need that); a thread
// issues the remote loads of UC items before any add, so one DSMEM round trip
// covers UC x S loads (serial per-item round trips made the 64-row reduce
// longer than the GEMM).
template <int MODE, bool kWide>
__device__ __forceinline__ void cluster_reduce(const SkinnyArgs& args, const TcEpilogue& ep, int unit, int rank,
                                               uint32_t part, const float* push_ptr, const float* row_scale, int t) {
  constexpr int NB = MODE == (int)Epi::kSwiGLU ? 2 : 1;
  constexpr int kMaxS = 4, kWarps = kThreads / 32;
  constexpr int UC = MODE == (int)Epi::kRopeKV || NB == 2 ? 2 : 4;  // items per batch (~64 registers of loads)
  const int S = args.csplit, Mp = args.Mp, quads = Mp / 4;
  const int warp = t >> 5, lane = t & 31;
  constexpr int kBlocks = MODE == (int)Epi::kRopeKV ? 2 : kRows / 32;
  const int nblk = (kBlocks - rank + S - 1) / S;  // blocks rank, rank + S, ...
  const int n_items = nblk * quads;
  auto add4 = [](float4& a, const float4& b) {
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  };
  if constexpr (!kWide) {
    // <= 16 batch rows (at most 2 items per epilogue warp): the 4 epilogue
    // warps, one DSMEM load at a time. A separate kernel instantiation: with
    // the batched form below compiled into the same kernel, the decode step
    // at B = 1 measured 3.34 -> 3.41 ms even where that code never ran.
    if (t < 128) return;
    const int ew = warp - 4;
    const int rpo = push_rows_per_owner(MODE == (int)Epi::kRopeKV, S);
    auto at = [&](int c, int local, int jb, int q4) -> float4 {
      return *reinterpret_cast<const float4*>(reinterpret_cast<const uint8_t*>(push_ptr) +
                                              part_off((c * rpo + local) * NB + jb, q4, Mp));
    };
    int w = 0;
    for (int blk = rank; blk < kBlocks; blk += S)
      for (int q4 = 0; q4 < quads; ++q4, ++w) {
        if ((w & 3) != ew) continue;
        if constexpr (MODE == (int)Epi::kRopeKV) {
          const int hd = ep.kv.head_dim, half = hd / 2;
          const int j = blk * 32 + lane;
          const int ia = (j / half) * hd + j % half;
          const int la = (blk / S) * 64 + lane * 2;
          float4 sa = make_float4(0.f, 0.f, 0.f, 0.f), sb = sa;
          for (int c = 0; c < S; ++c) {
            add4(sa, at(c, la, 0, q4));
            add4(sb, at(c, la + 1, 0, q4));
          }
          float va[4] = {sa.x, sa.y, sa.z, sa.w}, vb[4] = {sb.x, sb.y, sb.z, sb.w};
          rope_store(args, ep, unit * kRows + ia, q4, va, vb, row_scale);
        } else {
          const int i = blk * 32 + lane, li = (blk / S) * 32 + lane;
          float4 sum[NB];
#pragma unroll
          for (int jb = 0; jb < NB; ++jb) sum[jb] = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int c = 0; c < S; ++c)
#pragma unroll
            for (int jb = 0; jb < NB; ++jb) add4(sum[jb], at(c, li, jb, q4));
          fixup_store<MODE>(args, ep, unit, i, q4, sum, row_scale);
        }
      }
    return;
  } else {
  for (int w0 = warp; w0 < n_items; w0 += UC * kWarps) {
    if constexpr (MODE == (int)Epi::kRopeKV) {
      // pairs j in [0, 64): columns (unit*128 + (j / half) * hd + j % half, + half)
      const int hd = ep.kv.head_dim, half = hd / 2;
      float4 pa[UC][kMaxS], pb[UC][kMaxS];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int w = w0 + u * kWarps;
        if (w >= n_items) break;
        const int j = (rank + (w / quads) * S) * 32 + lane, q4 = w % quads;
        const int ia = (j / half) * hd + j % half, ib = ia + half;
#pragma unroll
        for (int c = 0; c < kMaxS; ++c)
          if (c < S) {
            pa[u][c] = ld_dsmem_v4(part + part_off(ia, q4, Mp), c);
            pb[u][c] = ld_dsmem_v4(part + part_off(ib, q4, Mp), c);
          }
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int w = w0 + u * kWarps;
        if (w >= n_items) break;
        const int j = (rank + (w / quads) * S) * 32 + lane, q4 = w % quads;
        const int ia = (j / half) * hd + j % half;
        float4 sa = pa[u][0], sb = pb[u][0];
#pragma unroll
        for (int c = 1; c < kMaxS; ++c)
          if (c < S) {
            add4(sa, pa[u][c]);
            add4(sb, pb[u][c]);
          }
        float va[4] = {sa.x, sa.y, sa.z, sa.w}, vb[4] = {sb.x, sb.y, sb.z, sb.w};
        rope_store(args, ep, unit * kRows + ia, q4, va, vb, row_scale);
      }
    } else {
      float4 p[UC][kMaxS][NB];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int w = w0 + u * kWarps;
        if (w >= n_items) break;
        const int i = (rank + (w / quads) * S) * 32 + lane, q4 = w % quads;
#pragma unroll
        for (int c = 0; c < kMaxS; ++c)
          if (c < S)
#pragma unroll
            for (int jb = 0; jb < NB; ++jb) p[u][c][jb] = ld_dsmem_v4(part + part_off(jb * kRows + i, q4, Mp), c);
      }
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int w = w0 + u * kWarps;
        if (w >= n_items) break;
        const int i = (rank + (w / quads) * S) * 32 + lane, q4 = w % quads;
        float4 sum[NB];
#pragma unroll
        for (int jb = 0; jb < NB; ++jb) sum[jb] = p[u][0][jb];
#pragma unroll
        for (int c = 1; c < kMaxS; ++c)
          if (c < S)
#pragma unroll
            for (int jb = 0; jb < NB; ++jb) add4(sum[jb], p[u][c][jb]);
        fixup_store<MODE>(args, ep, unit, i, q4, sum, row_scale);
      }
    }
  }
}  // kWide
}

// WS_SKINNY_TRACE build: per-CTA globaltimer timeline of the last launch
// [cta][0 entry, 1 setup done, 2 producer past the PDL wait, 3 first stage
// landed (MMA), 4 last MMA committed, 5 first accumulator ready (epilogue),
// 6 epilogue done, 7 past the first cluster barrier, 8 reduce done, 9 exit]
// (tools/skinny_trace.py).
__device__ long long g_skinny_trace[148][10];
#ifdef WS_SKINNY_TRACE
constexpr bool kSkTrace = true;
#else
constexpr bool kSkTrace = false;
#endif
__device__ __forceinline__ void sk_mark(int ev) {
  if constexpr (kSkTrace) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 148) g_skinny_trace[blockIdx.x][ev] = t;
  }
}

template <int MODE, bool kWide = false>  // kWide: cluster reduce for > 16 batch rows
__global__ void __launch_bounds__(kThreads, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_a,
                       const __grid_constant__ SkinnyArgs args, const __grid_constant__ TcEpilogue ep) {
  constexpr int NB = MODE == (int)Epi::kSwiGLU ? 2 : 1;
  if (threadIdx.x == 0) sk_mark(0);
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023) & ~1023u;
  const int S = args.stages;
  const uint32_t bars = base + S * args.stage_bytes;
  auto full = [&](int s) { return bars + 8 * s; };
  auto empty = [&](int s) { return bars + 8 * (S + s); };
  auto tfull = [&](int b) { return bars + 8 * (2 * S + b); };
  auto tempty = [&](int b) { return bars + 8 * (2 * S + 2 + b); };
  const uint32_t tmem_slot = bars + 8 * (2 * S + 4);
  const uint32_t push_base = bars + 1024;  // push-form cluster split region (launcher sizes it)
  volatile uint32_t* tmem_slot_ptr = reinterpret_cast<volatile uint32_t*>(smem_raw + (tmem_slot - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Mp = args.Mp, G = gridDim.x, total = args.total_iters;
  const int kbs = args.kbs, sub = args.sub, kBK = kBox * sub;
  const int SJ = (NB == 2 && args.splitj) ? 2 : 1;  // iterations per k-block
  const uint32_t a_off = (SJ == 2 ? 1 : NB) * sub * kW_BYTES, a_box = args.Mp * kBox * 2;
  // stream-K: equal contiguous ranges of the (unit, k-block) space; cluster
  // split: CTA rank s of cluster u takes k-slice s of unit u
  const int cs = args.csplit;
  const int it0 = cs > 1 ? (blockIdx.x / cs) * kbs + (blockIdx.x % cs) * kbs / cs : it_begin(blockIdx.x, G, total);
  const int it1 = cs > 1 ? (blockIdx.x / cs) * kbs + (blockIdx.x % cs + 1) * kbs / cs
                         : it_begin(blockIdx.x + 1, G, total);
  const uint32_t acc_cols = NB * Mp;
  uint32_t tmem_cols = 32;
  while (tmem_cols < 2 * acc_cols) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_w) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&map_a) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(full(s), 1);
      tc::mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(tfull(b), 1);
      tc::mbar_init(tempty(b), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tmem_slot),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (threadIdx.x == 0) sk_mark(1);
  const uint32_t tmem = *tmem_slot_ptr;
  // Weights are immutable: the producer fills the first ring stages with W
  // tiles before waiting for the previous kernel (PDL), so a short GEMM's
  // weight stream overlaps the tail of the kernel before it; activations
  // (the previous kernel's output) are loaded after the wait. Every other
  // thread waits up front.
  const int pre = (warp == 0 && lane == 0) ? min(S, it1 - it0) : 0;
  const uint64_t wpol = args.evict_first ? tc::policy_evict_first() : 0;
  // weight boxes of iteration it into the stage at sa: both row blocks of the
  // unit (SJ = 1) or only row block j = it % 2 (SJ = 2)
  auto load_w = [&](uint32_t sa, uint32_t bar, int it) {
    const int unit = it / kbs, r = it % kbs, kb = r / SJ;
    for (int jj = 0; jj < (SJ == 2 ? 1 : NB); ++jj) {
      const int j = SJ == 2 ? r % 2 : jj;
      for (int h = 0; h < sub; ++h) {
        const uint32_t dst = sa + (jj * sub + h) * kW_BYTES;
        if (args.evict_first)
          tc::tma_load_2d_hint(dst, &map_w, bar, kb * kBK + h * kBox, (unit * NB + j) * kRows, wpol);
        else
          tc::tma_load_2d(dst, &map_w, bar, kb * kBK + h * kBox, (unit * NB + j) * kRows);
      }
    }
  };
  if (warp == 0 && lane == 0) {
    for (int k = 0; k < pre; ++k) {
      const int it = it0 + k;
      const uint32_t sa = base + k * args.stage_bytes;
      tc::mbar_expect_tx(full(k), args.stage_bytes);
      load_w(sa, full(k), it);
    }
  }
  if (warp == 3 && lane == 0 && ep.l2pf_at == 0) l2_prefetch(ep.l2pf, blockIdx.x, gridDim.x);
  pdl_wait();  // global data produced by earlier kernels from here on
  if (threadIdx.x == 0) sk_mark(2);

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      for (int k = 0; k < pre; ++k)
        for (int h = 0; h < sub; ++h)
          tc::tma_load_2d(base + k * args.stage_bytes + a_off + h * a_box, &map_a, full(k),
                          ((it0 + k) % kbs / SJ) * kBK + h * kBox, 0);
      int stage = pre == S ? 0 : pre;
      uint32_t phase = pre == S ? 1 : 0;
      for (int it = it0 + pre; it < it1; ++it) {
        const int kb = it % kbs / SJ;
        tc::mbar_wait(empty(stage), phase ^ 1);
        const uint32_t sa = base + stage * args.stage_bytes;
        tc::mbar_expect_tx(full(stage), args.stage_bytes);
        load_w(sa, full(stage), it);
        for (int h = 0; h < sub; ++h)
          tc::tma_load_2d(sa + a_off + h * a_box, &map_a, full(stage), kb * kBK + h * kBox, 0);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (ep.l2pf_at == 1) l2_prefetch(ep.l2pf, blockIdx.x, gridDim.x);
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer: one accumulator per segment =====
      const uint32_t idesc = tc::idesc_bf16(kRows, Mp);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int it = it0; it < it1;) {
        const int seg_end = min(it1, (it / kbs + 1) * kbs);
        tc::mbar_wait(tempty(acc), acc_phase ^ 1);
        tc::fence_after();
        const uint32_t d = tmem + acc * acc_cols;
        for (int i = it; i < seg_end; ++i) {
          tc::mbar_wait(full(stage), phase);
          tc::fence_after();
          if (i == it0) sk_mark(3);
          const uint32_t sa = base + stage * args.stage_bytes;
          // SJ = 2: segments are whole units, so iterations 0 / 1 open the gate / up accumulators
          const uint32_t acc_on = SJ == 2 ? (uint32_t)(i - it >= 2) : (uint32_t)(i > it);
          for (int h = 0; h < sub; ++h) {
            const uint64_t db = tc::sdesc_sw128(sa + a_off + h * a_box);
#pragma unroll
            for (int jj = 0; jj < (SJ == 2 ? 1 : NB); ++jj) {
              const int j = SJ == 2 ? (i % kbs) % 2 : jj;
              const uint64_t da = tc::sdesc_sw128(sa + (jj * sub + h) * kW_BYTES);
#pragma unroll
              for (int k = 0; k < kBox / 16; ++k)  // +32 B per K=16 step inside the 128 B swizzle row
                tc::mma_f16(d + j * Mp, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), idesc, acc_on | h | k);
            }
          }
          tc::commit(empty(stage));
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc::commit(tfull(acc));
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
        it = seg_end;
      }
      sk_mark(4);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ===== epilogue: thread i <-> TMEM lane i <-> weight row i of the unit's block(s) =====
    const int i = threadIdx.x - 128;
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const int64_t slot_floats = (int64_t)NB * kRows * Mp;
    float* s_row = reinterpret_cast<float*>(smem_raw + (bars + 8 * (2 * S + 6) - raw));  // [128] row scales
    if (ep.norm_role == 2) {
      if (i < args.M) {
        const float sc = norm_row_scale(ep, i);
        s_row[i] = sc;
        if (blockIdx.x == 0) ep.row_scale[i] = sc;  // for the fix-up kernels
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the 4 epilogue warps
    }
    int acc = 0, seg = 0;
    uint32_t acc_phase = 0;
    const int rank = cs > 1 ? (int)(blockIdx.x % cs) : 0;
    const int rpo = push_rows_per_owner(MODE == (int)Epi::kRopeKV, cs > 1 ? cs : 1);
    int p_owner = 0, p_local = 0;
    if (cs > 1 && !kWide) push_slot<MODE>(ep, i, cs, p_owner, p_local);
    for (int it = it0; it < it1; ++seg) {
      const int unit = it / kbs;
      const int seg_end = min(it1, (unit + 1) * kbs);
      // RoPE + KV append needs both halves of a head: always via the fix-up
      const bool whole = MODE != (int)Epi::kRopeKV && it % kbs == 0 && seg_end == (unit + 1) * kbs;
      const int out_row = unit * kRows + i;  // output column (SwiGLU: act column)
      tc::mbar_wait(tfull(acc), acc_phase);
      tc::fence_after();
      if (i == 0 && seg == 0) sk_mark(5);
      const uint32_t tacc = trow + acc * acc_cols;
      // cluster split: the partial stays in this CTA's shared memory (the TMA
      // ring, idle once the unit's last stage was consumed) for cluster_reduce
      float* mine = cs > 1 ? reinterpret_cast<float*>(smem_raw + (base - raw))
                           : args.partial + ((int64_t)blockIdx.x * 2 + (seg == 0 ? 0 : 1)) * slot_floats;
      for (int c = 0; c < Mp; c += 16) {
        uint32_t v[NB][16];
#pragma unroll
        for (int j = 0; j < NB; ++j) WS_TMEM_LD16(tacc + j * Mp + c, v[j]);
        tc::wait_ld();
        if (whole) {
          float f[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const float sc = ep.norm_role == 2 ? (c + q < args.M ? s_row[c + q] : 0.f) : 1.f;
            f[q] = __uint_as_float(v[0][q]) * sc;
            if constexpr (NB == 2) f[q] = silu(f[q]) * (__uint_as_float(v[NB - 1][q]) * sc);
          }
          store_out<MODE>(ep, args, out_row, f, c);
        } else {
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            float4* dst = reinterpret_cast<float4*>(mine + ((int64_t)j * kRows + i) * Mp + c);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 o = make_float4(__uint_as_float(v[j][4 * q]), __uint_as_float(v[j][4 * q + 1]),
                                           __uint_as_float(v[j][4 * q + 2]), __uint_as_float(v[j][4 * q + 3]));
              if (cs > 1 && !kWide) {  // push into the owner's region (remote shared-memory store)
                st_dsmem_v4(push_base + part_off((rank * rpo + p_local) * NB + j, c / 4 + q, Mp), p_owner, o);
              } else if (cs > 1) {  // own swizzled shared-memory slot (part_off), pulled by cluster_reduce
                *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(mine) + part_off(j * kRows + i, c / 4 + q, Mp)) = o;
              } else {
                __stcg(dst + q, o);
              }
            }
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(tempty(acc));  // accumulator drained: the MMA may reuse it
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
      it = seg_end;
    }
  }
  if (threadIdx.x == 128) sk_mark(6);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tmem_cols));
  if (cs > 1) {
    cluster_sync();  // every k-slice's partial is in its owner's (push) / its own (pull) shared memory
    if (threadIdx.x == 0) sk_mark(7);
    {  // every warp: the producer / MMA / allocator warps are idle by now
      const float* s_row = reinterpret_cast<const float*>(smem_raw + (bars + 8 * (2 * S + 6) - raw));
      const float* push_ptr = reinterpret_cast<const float*>(smem_raw + (push_base - raw));
      cluster_reduce<MODE, kWide>(args, ep, blockIdx.x / cs, blockIdx.x % cs, base, push_ptr, s_row, threadIdx.x);
    }
    if (threadIdx.x == 128) sk_mark(8);
    // pull form: no CTA leaves while its partial may still be read; the push
    // form's remote stores all landed before the barrier above
    if constexpr (kWide) cluster_sync();
  }
  if (threadIdx.x == 0) sk_mark(9);
}

// Split-K fix-up for the units no single CTA covered: out = epilogue(sum of
// the contributors' partials in k order). Deterministic, and spread over the
// whole GPU instead of one CTA per unit at the tail of the GEMM. Thread =
// (unit, weight row i, 4 batch rows); rows fastest so the output stores of a
// warp are coalesced. Launched with PDL right behind the GEMM.
template <int MODE>
__device__ __forceinline__ void fixup_columns(const SkinnyArgs& args, const TcEpilogue& ep, int G, int unit, int i,
                                              int q4) {
  constexpr int NB = MODE == (int)Epi::kSwiGLU ? 2 : 1;
  const int Mp = args.Mp, kbs = args.kbs, total = args.total_iters;
  const int c_first = cta_of((int64_t)unit * kbs, G, total);
  const int c_last = cta_of((int64_t)(unit + 1) * kbs - 1, G, total);
  if (c_first == c_last) return;  // whole unit: stored by the GEMM
  const int64_t slot_floats = (int64_t)NB * kRows * Mp;
  float4 sum[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) sum[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  // contributors in k order, 8 at a time: their loads are all in flight
  // before the (ordered) adds, so the tail costs one L2 round trip, not one per contributor
  for (int c0 = c_first; c0 <= c_last; c0 += 8) {
    float4 p[8][NB];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int cc = c0 + k;
      const int slot = cc <= c_last && unit == it_begin(cc, G, total) / kbs ? 0 : 1;
      const float* src = args.partial + ((int64_t)(cc <= c_last ? cc : c_last) * 2 + slot) * slot_floats;
#pragma unroll
      for (int j = 0; j < NB; ++j)
        p[k][j] = cc <= c_last ? __ldcg(reinterpret_cast<const float4*>(src + ((int64_t)j * kRows + i) * Mp) + q4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        sum[j].x += p[k][j].x;
        sum[j].y += p[k][j].y;
        sum[j].z += p[k][j].z;
        sum[j].w += p[k][j].w;
      }
  }
  fixup_store<MODE>(args, ep, unit, i, q4, sum, ep.row_scale);
}
template <int MODE>
__global__ void __launch_bounds__(256) skinny_fixup_kernel(const __grid_constant__ SkinnyArgs args,
                                                           const __grid_constant__ TcEpilogue ep, int G) {
  pdl_trigger();
  pdl_wait();
  const int kbs = args.kbs, total = args.total_iters;
  const int q4 = blockIdx.y;  // batch rows 4*q4 .. 4*q4+3
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int unit = x / kRows, i = x % kRows;
  if (unit < total / kbs) fixup_columns<MODE>(args, ep, G, unit, i, q4);
}


// RoPE + paged KV append fix-up (decode QKV): thread = (unit, 4 batch rows,
// pair j < 64) owns columns (d, d + hd/2) of one head, sums both over the
// unit's contributors in k order, adds the bias, rotates q/k heads, writes q
// to the qkv buffer and k/v into the sequence's KV page (layout of KvGeom).
__global__ void __launch_bounds__(256) skinny_rope_fixup_kernel(const __grid_constant__ SkinnyArgs args,
                                                                const __grid_constant__ TcEpilogue ep, int G) {
  pdl_trigger();
  pdl_wait();
  const KvGeom& kv = ep.kv;
  const int Mp = args.Mp, kbs = args.kbs, total = args.total_iters;
  const int quads = Mp / 4, hd = kv.head_dim, half = hd / 2;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int unit = (int)(t / (64 * quads));
  if (unit >= total / kbs) return;
  const int rem = (int)(t % (64 * quads));
  const int q4 = rem / 64, j = rem % 64;
  const int dd = j % half;
  const int col_a = unit * kRows + (j / half) * hd + dd, col_b = col_a + half;
  const int c_first = cta_of((int64_t)unit * kbs, G, total);
  const int c_last = cta_of((int64_t)(unit + 1) * kbs - 1, G, total);
  const int64_t slot_floats = (int64_t)kRows * Mp;
  float4 sa = make_float4(0.f, 0.f, 0.f, 0.f), sb = sa;
  for (int c0 = c_first; c0 <= c_last; c0 += 8) {  // loads of 8 contributors in flight, k-ordered adds
    float4 pa[8], pb[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int cc = c0 + k <= c_last ? c0 + k : c_last;
      const int slot = unit == it_begin(cc, G, total) / kbs ? 0 : 1;
      const float* src = args.partial + ((int64_t)cc * 2 + slot) * slot_floats;
      const bool ok = c0 + k <= c_last;
      pa[k] = ok ? __ldcg(reinterpret_cast<const float4*>(src + (int64_t)(col_a - unit * kRows) * Mp) + q4)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
      pb[k] = ok ? __ldcg(reinterpret_cast<const float4*>(src + (int64_t)(col_b - unit * kRows) * Mp) + q4)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      sa.x += pa[k].x; sa.y += pa[k].y; sa.z += pa[k].z; sa.w += pa[k].w;
      sb.x += pb[k].x; sb.y += pb[k].y; sb.z += pb[k].z; sb.w += pb[k].w;
    }
  }
  float va[4] = {sa.x, sa.y, sa.z, sa.w}, vb[4] = {sb.x, sb.y, sb.z, sb.w};
  rope_store(args, ep, col_a, q4, va, vb, ep.row_scale);
}

bool make_map(CUtensorMap* map, const void* ptr, int rows, int K, int box_rows) {
  const Driver* d = driver();
  if (!d) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBox, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return d->cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Partial slots, one set per (device, stream): launches on one
// stream are ordered, so they can share it. Slots: 148 CTAs x 2 x 256 rows x
// 128 columns fp32 = 38.8 MB.
constexpr int64_t kPartialFloats = (int64_t)kNumSMs * 2 * 2 * kRows * 128;
struct Scratch {
  float* partial = nullptr;
};
std::mutex g_mu;
std::map<std::pair<int, cudaStream_t>, Scratch> g_scratch;

bool scratch_for(cudaStream_t st, Scratch* out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_scratch.find({dev, st});
  if (it == g_scratch.end()) {
    Scratch s;
    if (cudaMalloc(&s.partial, kPartialFloats * sizeof(float)) != cudaSuccess) return false;
    it = g_scratch.emplace(std::make_pair(dev, st), s).first;
  }
  *out = it->second;
  return true;
}

int g_skinny_mode = -1;  // env WS_SKINNY=0 disables (A/B against the GEMV / 128-row tiles)

// Clusters of S skinny CTAs (one per SM at this shared-memory footprint) the
// GPU can hold at once; cached per (S, smem).
int max_clusters(int S, int smem) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({S, smem});
  if (it != cache.end()) return it->second;
  // the largest opt-in size: never lower the attribute below a footprint
  // launch_mode<0> already set (its cache only raises it)
  cudaFuncSetAttribute(gemm_skinny_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(S * 64);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, gemm_skinny_kernel<0>, &cfg);
  if (e != cudaSuccess) n = 0;
  cudaGetLastError();  // a failed query only disables the cluster split
  cache[{S, smem}] = n;
  return n;
}

template <int MODE>
void launch_mode(const CUtensorMap& mw, const CUtensorMap& ma, const SkinnyArgs& a, int grid, int smem,
                 const TcEpilogue& e, cudaStream_t st) {
  // the opt-in shared-memory size only ever rises (a lower value set later
  // would make an earlier, larger configuration fail to launch)
  const bool wide = a.csplit > 1 && a.Mp > 16;
  auto kern = wide ? gemm_skinny_kernel<MODE, true> : gemm_skinny_kernel<MODE, false>;
  static int attr[2] = {0, 0};
  if (smem > attr[wide]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr[wide] = smem;
  }
  count_launch();
  if (a.csplit > 1) {  // cluster split-K: the reduction runs inside the GEMM, no fix-up launch
    static bool np[2] = {false, false};
    if (!np[wide]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaGetLastError();
      np[wide] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = a.csplit;
    attr[n].val.clusterDim.y = 1;
    attr[n++].val.clusterDim.z = 1;
    if (pdl_for_launch()) {
      attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[n++].val.programmaticStreamSerializationAllowed = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    cudaLaunchKernelEx(&cfg, kern, mw, ma, a, e);
    return;
  }
  launch_pdl(gemm_skinny_kernel<MODE>, dim3(grid), dim3(kThreads), (size_t)smem, st, mw, ma, a, e);
  const int kbs = a.kbs, units = a.total_iters / kbs;
  if constexpr (MODE == (int)Epi::kRopeKV) {
    const int64_t threads = (int64_t)units * 64 * (a.Mp / 4);
    count_launch();
    launch_pdl(skinny_rope_fixup_kernel, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, st, a, e, grid);
    return;
  }
  bool split = false;  // does any CTA boundary fall inside a unit?
  for (int c = 1; c < grid && !split; ++c) split = ((int64_t)c * a.total_iters / grid) % kbs != 0;
  if (split) {
    count_launch();
    launch_pdl(skinny_fixup_kernel<MODE>, dim3((unsigned)((units * kRows + 255) / 256), a.Mp / 4), dim3(256), 0, st,
               a, e, grid);
  }
}

}  // namespace

bool gemm_skinny_enabled() {
  if (g_skinny_mode < 0) {
    const char* v = getenv("WS_SKINNY");
    g_skinny_mode = (v && v[0] == '0') ? 0 : 1;
  }
  return g_skinny_mode == 1;
}

// N need not be a multiple of the 128-row unit for the plain epilogues (a
// vocabulary of 32064 rows: Phi-3's lm_head): the last unit's weight rows past
// N are zero-filled by the TMA bounds and its outputs past N are not stored.
bool gemm_skinny_supported(int M, int N, int K, Epi mode) {
  const bool ragged_ok = mode == Epi::kStoreBf16 || mode == Epi::kBiasBf16 || mode == Epi::kStoreF32 ||
                         mode == Epi::kAddF32;
  return gemm_skinny_enabled() && M >= 1 && M <= 128 && K >= kBox && K % kBox == 0 && N >= 1 &&
         (N % (kRows * (mode == Epi::kSwiGLU ? 2 : 1)) == 0 || ragged_ok);
}

bool launch_gemm_skinny(const bf16* A, const bf16* W, int M, int N, int K, const TcEpilogue& e, cudaStream_t st) {
  if (!gemm_skinny_supported(M, N, K, e.mode)) return false;
  if (e.mode == Epi::kRopeKV && e.kv.head_dim != 64 && e.kv.head_dim != 128) return false;  // heads tile 128 rows
  if (e.norm_role == 1 && e.mode != Epi::kAddF32) return false;
  if (e.norm_role != 0 && N % kRows) return false;  // folded norms work on whole 32-column groups
  if (e.norm_role == 2 && (e.mode == Epi::kAddF32 || e.mode == Epi::kStoreF32)) return false;
  const int NB = e.mode == Epi::kSwiGLU ? 2 : 1;
  // Widest iteration (up to 4 boxes = 512 contiguous bytes of each weight row
  // per TMA issue) that divides K and still leaves a 3-stage ring: the weight
  // stream then reaches HBM as long runs instead of 128 B pieces of 128 rows
  // 8+ KB apart (B = 1 / 16 / 64 decode: 4.20 / 4.50 / 6.07 -> 4.04 / 4.27 /
  // 5.89 ms per step).
  const int mp = (M + 15) / 16 * 16;
  int sub = 4;
  while (sub > 1 && (K % (sub * kBox) || 3 * sub * (NB * kW_BYTES + mp * kBox * 2) > kSmemBudget)) sub /= 2;
  const int units = (N + kRows * NB - 1) / (kRows * NB), kbs = K / (kBox * sub);
  SkinnyArgs a{};
  a.sub = sub;
  a.kbs = kbs;
  a.M = M;
  a.N = N;
  a.K = K;
  a.Mp = (M + 15) / 16 * 16;
  a.stage_bytes = sub * (NB * kW_BYTES + a.Mp * kBox * 2);
  a.stages = std::max(2, std::min(12, kSmemBudget / a.stage_bytes));
  a.total_iters = units * kbs;
  int smem = a.stages * a.stage_bytes + 1024 + 1024;  // align slack + barriers + TMEM slot + [128] row scales
  // one CTA per SM, >= 2 k-blocks each
  int grid = std::max(1, std::min(kNumSMs, a.total_iters / 2));
  // Enough units to occupy most SMs (gate/up: 112): one whole unit per CTA.
  // No unit is split, so no fix-up pass runs, and the ~25% of idle SMs cost
  // less than the fix-up: measured 4-9% faster decode steps (B = 1..64) than
  // stream-K over all 148 SMs. Below ~90 units whole units lose: one SM pulls
  // ~64 GB/s, so 32-48 CTAs cannot stream at HBM rate (down: 57 vs 25 us).
  if (units * 10 >= kNumSMs * 6 && units <= kNumSMs) grid = units;
  // Too few units to fill the SMs (decode O / down: 32, QKV: 48): split each
  // unit's k-range over a thread-block cluster of S CTAs (units x S <= 148,
  // S = 4, 3 or 2) whose fp32 partials are summed in k order over
  // distributed shared memory inside the same kernel — deterministic like
  // the fix-up kernel, without its launch and global round trip.
  // WS_SKINNY_CLUSTER=0: stream-K + fix-up (A/B).
  static const bool cl_on = !(getenv("WS_SKINNY_CLUSTER") && getenv("WS_SKINNY_CLUSTER")[0] == '0');
  a.csplit = 0;
  // Weight tiles stream through L2 as evict_first: each is read once per step,
  // and at the normal priority the stream evicts what the step reuses (the
  // activations, partials, norm rows, K/V). Graphed decode steps, ctx 1024,
  // same box, WS_SK_EVF=0 -> 1: B = 1 / 4 / 16 3.37 / 3.56 / 3.88 -> 3.22-3.32 /
  // 3.35 / 3.68 ms (tools/ab_l2pf2.sh).
  static const int evf = getenv("WS_SK_EVF") ? atoi(getenv("WS_SK_EVF")) : 1;
  a.evict_first = evf;
  a.splitj = 0;
  // Above 32 batch rows the fp32 partials the stream-K fix-up moves through
  // L2 grow with the rows; the cluster form wins where they are large next
  // to the weights and the clusters still cover >= 120 SMs (same-box per-GEMM
  // A/B, us, cluster vs stream-K + fix-up): SwiGLU up to 128 rows (Phi-3
  // gate/up as 64 pairs: 24 vs 36 at 64 rows, 29 vs 46 at 128), other
  // epilogues up to 64 rows in clusters of 4 (Llama-3-8B O / down: 14.6 /
  // 30.9 vs 15.5 / 31.8; decode B = 64 5.77 -> 5.66 ms) but not in pairs
  // (Phi-3 QKV as 72 pairs: 19.3 vs 17.4) nor above 64 rows (Llama down at
  // 128 rows: 39.4 vs 36.2).
  static const int cl_mp = getenv("WS_SKINNY_CLUSTER_MP") ? atoi(getenv("WS_SKINNY_CLUSTER_MP")) : 128;
  const bool swiglu = e.mode == Epi::kSwiGLU;
  if (cl_on && grid != units && a.Mp <= cl_mp)
    for (int S_ = 4; S_ >= 2; --S_)
      // every cluster resident at once (clusters are placed within a GPC: 48
      // clusters of 3 did not fit in one wave and ran the QKV GEMM at half speed)
      if (units * S_ <= kNumSMs && kbs >= 2 * S_ && units <= max_clusters(S_, smem)) {
        if (a.Mp > 32 && (units * S_ < 120 || (!swiglu && (S_ < 4 || a.Mp > 64)))) break;
        a.csplit = S_;
        grid = units * S_;
        break;
      }
  // Split-j SwiGLU stages for whole-unit launches (WS_SK_SPLITJ=1, A/B): a
  // stage carries one 128-row block (gate or up) over twice the k-columns,
  // so every TMA issue fetches twice the contiguous bytes of each weight row
  static const bool sj_env = getenv("WS_SK_SPLITJ") && getenv("WS_SK_SPLITJ")[0] == '1';
  if (sj_env && swiglu && grid == units && a.csplit == 0) {
    int sj_sub = 4;
    while (sj_sub > 1 && (K % (sj_sub * kBox) || 3 * sj_sub * (kW_BYTES + mp * kBox * 2) > kSmemBudget)) sj_sub /= 2;
    a.splitj = 1;
    a.sub = sj_sub;
    a.kbs = 2 * (K / (kBox * sj_sub));
    a.stage_bytes = sj_sub * (kW_BYTES + a.Mp * kBox * 2);
    a.stages = std::max(2, std::min(12, kSmemBudget / a.stage_bytes));
    a.total_iters = units * a.kbs;
    smem = a.stages * a.stage_bytes + 1024 + 1024;
  }
  if (a.csplit > 1 && a.Mp <= 16) {  // push-form cluster split: the owners' receive region after the barriers
    const int push = a.csplit * push_rows_per_owner(e.mode == Epi::kRopeKV, a.csplit) * NB * a.Mp * 4;
    while (a.stages > 2 && a.stages * a.stage_bytes + 2048 + push > kMaxSmem) --a.stages;
    smem = a.stages * a.stage_bytes + 2048 + push;
    if (smem > kMaxSmem) return false;
  }
  static const bool dbg = getenv("WS_SKINNY_DEBUG") != nullptr;
  if (dbg) fprintf(stderr, "[skinny] M=%d N=%d K=%d mode=%d units=%d kbs=%d grid=%d cluster=%d\n", M, N, K, (int)e.mode,
                   units, kbs, grid, a.csplit);
  if (e.mode == Epi::kRopeKV && units > grid) return false;  // <= 2 segments (partial slots) per CTA
  Scratch s;
  if (!scratch_for(st, &s)) return false;
  a.partial = s.partial;
  CUtensorMap mw, ma;
  if (!make_map(&mw, W, N, K, kRows) || !make_map(&ma, A, M, K, a.Mp)) return false;
  switch (e.mode) {
    case Epi::kStoreBf16: launch_mode<0>(mw, ma, a, grid, smem, e, st); break;
    case Epi::kBiasBf16: launch_mode<1>(mw, ma, a, grid, smem, e, st); break;
    case Epi::kAddF32: launch_mode<2>(mw, ma, a, grid, smem, e, st); break;
    case Epi::kStoreF32: launch_mode<3>(mw, ma, a, grid, smem, e, st); break;
    case Epi::kSwiGLU: launch_mode<4>(mw, ma, a, grid, smem, e, st); break;
    case Epi::kRopeKV: launch_mode<5>(mw, ma, a, grid, smem, e, st); break;
  }
  if (dbg) {
    const cudaError_t err = cudaPeekAtLastError();
    if (err != cudaSuccess) fprintf(stderr, "[skinny] launch failed: %s (smem %d)\n", cudaGetErrorString(err), smem);
  }
  return true;
}

}  // namespace ws

extern "C" int ws_skinny_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, ws::g_skinny_trace, sizeof(ws::g_skinny_trace)) == cudaSuccess ? 0 : 6;
}
